"""Independent brute-force LTL/FLTL evaluators used to PIN the oracle.

Shares nothing with oracle/ or the product: formulas are Python tuples,
infinite words are lassos u·x·(y)^ω, and every operator is evaluated by its
textbook fixpoint on the lasso positions (F/G/U least/greatest fixpoints),
not by the expansion used inside the oracle.  FLTL is the literal
"exists k ... forall l < k" definition of P:278-283.
"""
from __future__ import annotations

import itertools
import random

# formula tuples: ("true",) ("ap", name) ("not", f) ("and", f, g) ("or", f, g)
#                 ("imp", f, g) ("X", f) ("F", f) ("G", f) ("U", f, g)


def to_text(f) -> str:
    op = f[0]
    if op == "true":
        return "true"
    if op == "ap":
        return f[1]
    if op == "not":
        return f"!({to_text(f[1])})"
    if op in ("and", "or", "imp", "U"):
        sym = {"and": "&&", "or": "||", "imp": "->", "U": "U"}[op]
        return f"({to_text(f[1])}) {sym} ({to_text(f[2])})"
    return f"{op} ({to_text(f[1])})"


def atoms_in_order(f, out=None):
    if out is None:
        out = []
    if f[0] == "ap":
        if f[1] not in out:
            out.append(f[1])
    else:
        for g in f[1:]:
            if isinstance(g, tuple):
                atoms_in_order(g, out)
    return out


def lasso_eval(f, word, loop, bit):
    """Truth of f at every position of the lasso word[0..L-1] with back-edge to `loop`.
    `bit` maps atom name -> bit index of the letter."""
    L = len(word)
    succ = [i + 1 if i + 1 < L else loop for i in range(L)]

    def ev(g):
        op = g[0]
        if op == "true":
            return [True] * L
        if op == "ap":
            return [bool((word[i] >> bit[g[1]]) & 1) for i in range(L)]
        if op == "not":
            return [not v for v in ev(g[1])]
        if op == "and":
            a, b = ev(g[1]), ev(g[2])
            return [x and y for x, y in zip(a, b)]
        if op == "or":
            a, b = ev(g[1]), ev(g[2])
            return [x or y for x, y in zip(a, b)]
        if op == "imp":
            a, b = ev(g[1]), ev(g[2])
            return [(not x) or y for x, y in zip(a, b)]
        if op == "X":
            a = ev(g[1])
            return [a[succ[i]] for i in range(L)]
        if op == "F":  # least fixpoint of  Z = a | X Z
            a = ev(g[1])
            z = [False] * L
            for _ in range(L + 1):
                z = [a[i] or z[succ[i]] for i in range(L)]
            return z
        if op == "G":  # greatest fixpoint of Z = a & X Z
            a = ev(g[1])
            z = [True] * L
            for _ in range(L + 1):
                z = [a[i] and z[succ[i]] for i in range(L)]
            return z
        if op == "U":  # least fixpoint of Z = b | (a & X Z)
            a, b = ev(g[1]), ev(g[2])
            z = [False] * L
            for _ in range(L + 1):
                z = [b[i] or (a[i] and z[succ[i]]) for i in range(L)]
            return z
        raise ValueError(op)

    return ev(f)


def fltl(f, word, bit) -> bool:
    """[u |=_F f] by the literal definitions of P:269-289 (finite, strong X)."""
    n = len(word)

    def ev(g, i):
        op = g[0]
        if op == "true":
            return True
        if op == "ap":
            return bool((word[i] >> bit[g[1]]) & 1)
        if op == "not":
            return not ev(g[1], i)
        if op == "and":
            return ev(g[1], i) and ev(g[2], i)
        if op == "or":
            return ev(g[1], i) or ev(g[2], i)
        if op == "imp":
            return (not ev(g[1], i)) or ev(g[2], i)
        if op == "X":
            return i + 1 < n and ev(g[1], i + 1)
        if op == "U":
            return any(ev(g[2], k) and all(ev(g[1], l) for l in range(i, k)) for k in range(i, n))
        if op == "F":  # F p == true U p
            return any(ev(g[1], k) for k in range(i, n))
        if op == "G":  # G p == !F !p
            return not any(not ev(g[1], k) for k in range(i, n))
        raise ValueError(op)

    return ev(f, 0)


def ltl4_bruteforce(f, u, n_atoms, bit, max_x=2, max_y=2):
    """LTL4 verdict of Def. 4 with forall-v over all lassos x·y^ω, |x|<=max_x,
    1<=|y|<=max_y.  Returns (verdict, exhaustive_flags)."""
    letters = range(1 << n_atoms)
    sat = vio = False
    for lx in range(max_x + 1):
        for x in itertools.product(letters, repeat=lx):
            for ly in range(1, max_y + 1):
                for y in itertools.product(letters, repeat=ly):
                    w = list(u) + list(x) + list(y)
                    v = lasso_eval(f, w, len(u) + lx, bit)[0]
                    sat |= v
                    vio |= not v
                    if sat and vio:
                        break
                if sat and vio:
                    break
            if sat and vio:
                break
        if sat and vio:
            break
    if not vio:
        return 5
    if not sat:
        return 0
    return 3 if fltl(f, u, bit) else 2


def random_formula(rng: random.Random, atoms, depth):
    if depth == 0 or rng.random() < 0.25:
        return ("ap", rng.choice(atoms)) if rng.random() < 0.9 else ("true",)
    op = rng.choice(["not", "and", "or", "imp", "X", "F", "G", "U", "U"])
    if op in ("not", "X", "F", "G"):
        return (op, random_formula(rng, atoms, depth - 1))
    return (op, random_formula(rng, atoms, depth - 1), random_formula(rng, atoms, depth - 1))
