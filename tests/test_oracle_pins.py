"""Pins of the oracle against what the paper and the mathematics fix.

Each test names the passage it pins.  None of them re-types an oracle formula:
they use the paper's printed values (tests/golden/), closed forms derived by
hand for the workload formulas, brute force over lasso extensions
(tests/ltl_bruteforce.py) and over histogram extensions, and invariants.
"""
import itertools
import os
import random

import numpy as np
import pytest

import oracle
import tracegen
from tests import ltl_bruteforce as bf

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
T, Tc, Tp, Fp, Fc, F = 5, 4, 3, 2, 1, 0
NAME = {"T": T, "Tc": Tc, "Tp": Tp, "Fp": Fp, "Fc": Fc, "F": F}


# ---------------------------------------------------------------- worked example
def _golden_login():
    ev, exp = [], {}
    for line in open(os.path.join(GOLDEN, "login_example.txt")):
        line = line.split("#")[0].strip()
        if not line:
            continue
        parts = line.split()
        if parts[0] in ("Adam", "Jack"):
            ev.append((parts[0], int(parts[1]), int(parts[2]), int(parts[3])))
        else:
            exp[" ".join(parts[:2]) if parts[0] == "node" else parts[0]] = parts[1:] if parts[0] != "node" else parts[2:]
    return ev, exp


def test_worked_example_login_P715():
    ev, exp = _golden_login()
    ids = {"Adam": 1, "Jack": 2}
    users = np.array([ids[e[0]] for e in ev], np.uint32)
    rids = np.array([e[1] for e in ev], np.uint32)
    letters = np.array([e[2] | (e[3] << 1) for e in ev], np.uint8)
    p = oracle.Property(tracegen.LOGIN)
    assert p.atoms == ["login", "unauthorized"]
    m = oracle.Monitor(p)
    m.feed([users, rids], letters)
    r = m.evaluate()
    # five distinct value vectors; B(Adam, T) = 4
    assert r["hist"][2].sum() == 5
    leaves = dict(kv.split("=") for kv in exp["leaves"])
    assert r["hist"][2][T] == int(leaves["T"]) and r["hist"][2][F] == int(leaves["F"])
    assert m.node_verdict([1]) == NAME[exp["node Adam"][0]]   # "4 not<= 3" -> F
    assert m.node_verdict([2]) == NAME[exp["node Jack"][0]]   # reading A4
    assert r["verdict"] == NAME[exp["root"][0]]
    assert m.node_verdict([1, 12]) == T and m.node_verdict([2, 14]) == F


def test_worked_example_online_batch1():
    ev, exp = _golden_login()
    tr = tracegen.worked_example()
    m = oracle.Monitor(oracle.Property(tr.formula))
    out = [m.evaluate()["verdict"]]
    for j in range(tr.n):
        m.feed([k[j:j + 1] for k in tr.keys], tr.letters[j:j + 1])
        out.append(m.evaluate()["verdict"])
    assert out == [NAME[x] for x in exp["online_batch1"]]


def test_toy_trace_slices_P596():
    # u = {px(1),py(2)} {px(1),py(3)} {px(1),py(2)} ; u^<1,2> = u0 u2, u^<1,3> = u1
    p = oracle.Property("forall x : px(x) => forall y : py(y) => G q")
    xs = np.array([1, 1, 1], np.uint32)
    ys = np.array([2, 3, 2], np.uint32)
    # q holds in u0 and u2 only: the <1,2> slice satisfies G q so far, the <1,3> slice violates it
    m = oracle.Monitor(p)
    m.feed([xs, ys], np.array([1, 0, 1], np.uint8))
    r = m.evaluate()
    assert r["hist"][1].sum() == 1 and r["hist"][2].sum() == 2     # P(<1>) = {<1,2>,<1,3>}
    assert m.node_verdict([1, 2]) == Tp and m.node_verdict([1, 3]) == F
    # if u^<1,2> were not the subsequence u0u2 (e.g. u0u1u2) the first leaf would be F
    m2 = oracle.Monitor(p)
    m2.feed([xs, ys], np.array([1, 1, 0], np.uint8))
    m2.evaluate()
    assert m2.node_verdict([1, 2]) == F and m2.node_verdict([1, 3]) == Tp


# ------------------------------------------------------------------- leaf (LTL4)
def _letter(s, atoms):
    return sum(1 << atoms.index(c) for c in s if c != "-")


def test_fig1_probe_words():
    p = oracle.Property(tracegen.FIG1)
    atoms = p.atoms
    assert atoms == ["a", "b", "c"]
    for line in open(os.path.join(GOLDEN, "fig1_probes.txt")):
        line = line.split("#")[0].strip()
        if not line:
            continue
        letters, verdict = line.split()
        assert p.ltl4([_letter(letters, atoms)]) == NAME[verdict], line


def _closed_socket(word):
    # G(receive -> F respond) on a finite slice: never permanently decided (every
    # pending receive can still be answered; any answered prefix can be broken);
    # Tp iff every receive has a respond at the same or a later position.
    last_recv = max([i for i, a in enumerate(word) if a & 1], default=-1)
    last_resp = max([i for i, a in enumerate(word) if a & 2], default=-1)
    return Tp if last_recv <= last_resp else Fp


def _closed_fig1(word):
    # G a || (b U c): b U c is decided at the first position that is not (b & !c)
    a = [(x >> 0) & 1 for x in word]
    b = [(x >> 1) & 1 for x in word]
    c = [(x >> 2) & 1 for x in word]
    until = None
    for i in range(len(word)):
        if c[i]:
            until = True
            break
        if not b[i]:
            until = False
            break
    if until is True:
        return T
    ga_alive = all(a)
    if until is False and not ga_alive:
        return F
    return Tp if ga_alive else Fp


def _closed_files(word):
    # opened U close: T at the first close with opened everywhere before,
    # F at a first position with neither opened nor close, else Fp.
    for x in word:
        if x & 2:
            return T
        if not (x & 1):
            return F
    return Fp


def _closed_F(word):
    return T if any(x & 1 for x in word) else Fp


def _closed_login(word):
    return T if word[0] == 3 else F


@pytest.mark.parametrize("formula,closed,n_atoms,maxlen", [
    (tracegen.SOCKET, _closed_socket, 2, 6),
    (tracegen.FIG1, _closed_fig1, 3, 4),
    (tracegen.FILES, _closed_files, 2, 6),
    ("forall u : user(u) => F authfail", _closed_F, 1, 7),
    (tracegen.LOGIN, _closed_login, 2, 4),
])
def test_leaf_closed_forms_all_words(formula, closed, n_atoms, maxlen):
    p = oracle.Property(formula)
    for L in range(1, maxlen + 1):
        for w in itertools.product(range(1 << n_atoms), repeat=L):
            assert p.ltl4(list(w)) == closed(list(w)), (formula, w)


def test_leaf_traps_are_permanent():
    # T and F are traps -- every extension keeps them
    for formula, na in [(tracegen.FIG1, 3), (tracegen.FILES, 2), (tracegen.LOGIN, 2)]:
        p = oracle.Property(formula)
        for L in range(1, 4):
            for w in itertools.product(range(1 << na), repeat=L):
                v = p.ltl4(list(w))
                if v in (T, F):
                    for ext in itertools.product(range(1 << na), repeat=2):
                        assert p.ltl4(list(w) + list(ext)) == v


def test_leaf_random_formulas_vs_lasso_bruteforce():
    """Def. 4 on random tiny formulas: the oracle's T/F agree with brute force over
    all lasso extensions x·y^ω (|x|,|y| <= 2); Tp/Fp agree with the literal FLTL."""
    rng = random.Random(1411)
    checked = 0
    while checked < 60:
        f = bf.random_formula(rng, ["a", "b"], 3)
        body = bf.to_text(f)
        names = bf.atoms_in_order(f)
        if not names:
            continue
        p = oracle.Property("forall x : k(x) => " + body)
        assert p.atoms == names
        bit = {nm: i for i, nm in enumerate(names)}
        na = len(names)
        for _ in range(4):
            L = rng.randint(1, 3)
            u = [rng.randrange(1 << na) for _ in range(L)]
            assert p.ltl4(u) == bf.ltl4_bruteforce(f, u, na, bit), (body, u)
            assert p.fltl(u) == int(bf.fltl(f, u, bit)), (body, u)
        checked += 1


def test_ltl3_collapse_P1414():
    # LTL3: T iff every extension satisfies, F iff none, else '?'.
    # Collapsing Tp/Fp of the oracle to '?' must give the LTL3 verdict, which the
    # lasso brute force decides without any FLTL.
    rng = random.Random(7)
    for _ in range(40):
        f = bf.random_formula(rng, ["a", "b"], 3)
        names = bf.atoms_in_order(f)
        if not names:
            continue
        p = oracle.Property("forall x : k(x) => " + bf.to_text(f))
        bit = {nm: i for i, nm in enumerate(names)}
        u = [rng.randrange(1 << len(names)) for _ in range(rng.randint(1, 3))]
        v = p.ltl4(u)
        ref = bf.ltl4_bruteforce(f, u, len(names), bit)
        collapse = lambda x: x if x in (T, F) else "?"
        assert collapse(v) == collapse(ref)


# ------------------------------------------------------------- node rule (Def. 6)
def test_table1_crossings_P703():
    """For each E operator and c, children become T one at a time; the node latches
    exactly at the crossing Table 1 prints."""
    rows = {}
    for line in open(os.path.join(GOLDEN, "table1.txt")):
        line = line.split("#")[0].strip()
        if line:
            op, kind, rel, _ = line.split()
            rows[op] = (kind, rel)
    for op, (kind, rel) in rows.items():
        for c in range(0, 4):
            for k in range(0, 7):  # k permanently-true children, plus one Fp child
                h = [0, 0, 1, 0, 0, k]
                v = oracle.rule("E", op, c, 1, h)
                crossed = (k > c) if rel == ">" else (k >= c)
                if kind == "permanent-satisfaction-if":
                    assert (v == T) == crossed, (op, c, k, v)
                    assert v != F
                else:
                    assert (v == F) == crossed, (op, c, k, v)
                    assert v != T


def test_scripted_table1_traces():
    # E_{<=3}: a single parent whose rid-children become T one event at a time;
    # F exactly on the 4th satisfied instance, Tc before.
    p = oracle.Property("forall x : user(x) => exists[<=3] r : rid(r) => (login && unauthorized)")
    m = oracle.Monitor(p)
    seq = []
    for j in range(6):
        m.feed([np.array([7], np.uint32), np.array([100 + j], np.uint32)], np.array([3], np.uint8))
        m.evaluate()
        seq.append(m.node_verdict([7]))
    assert seq == [Tc, Tc, Tc, F, F, F]
    # E_{>=2}: T exactly at the 2nd satisfied instance
    p = oracle.Property("exists[>=2] r : rid(r) => (login && unauthorized)")
    m = oracle.Monitor(p)
    seq = []
    for j, a in enumerate([1, 3, 0, 3, 1]):
        m.feed([np.array([200 + j], np.uint32)], np.array([a], np.uint8))
        seq.append(m.evaluate()["verdict"])
    assert seq == [Fc, Fc, Fc, T, T]


def test_A_eq1_single_violation_P690():
    for n_ok in range(0, 5):
        assert oracle.rule("A", "=", 1, 1, [1, 0, 0, 0, 0, n_ok]) == F
        assert oracle.rule("A", "=", 1, 1, [0, 1, 0, 0, 0, n_ok]) == Fc
    assert oracle.rule("A", "=", 1, 1, [0, 0, 0, 0, 0, 3]) == Tc
    assert oracle.rule("A", "=", 1, 1, [0, 0, 0, 2, 0, 3]) == Tp   # all presumably-true or better
    assert oracle.rule("A", "=", 1, 1, [0, 0, 1, 2, 0, 3]) == Fp


def test_exact_rational_boundary_S324():
    # A_{>=0.5}: 1 of 2 children meets 1 >= 0.5 * 2 exactly
    assert oracle.rule("A", ">=", 1, 2, [0, 0, 1, 0, 0, 1]) == Tc
    assert oracle.rule("A", ">=", 1, 2, [0, 0, 2, 0, 0, 1]) == Fp
    # A_{>=0.95} of 20: 19 Tp children pass, 18 do not (C1 closed form)
    assert oracle.rule("A", ">=", 19, 20, [0, 0, 1, 19, 0, 0]) == Tp
    assert oracle.rule("A", ">=", 19, 20, [0, 0, 2, 18, 0, 0]) == Fp
    # 0.95 * 20 = 19 is exactly representable only as a rational
    p = oracle.Property("forall[>=0.95] s : socket(s) => true")
    assert p.quantifier(0)["num"] == 19 and p.quantifier(0)["den"] == 20


def _grid():
    for op in ["<", "<=", ">", ">=", "="]:
        for c in range(0, 4):
            yield ("E", op, c, 1)
        for num, den in [(0, 1), (1, 4), (1, 3), (1, 2), (2, 3), (1, 1)]:
            yield ("A", op, num, den)


def _S(q, h, t):
    kind, op, num, den = q
    cnt, N = sum(h[t:]), sum(h)
    lhs, rhs = (cnt * den, num * N) if kind == "A" else (cnt, num)
    return {"<": lhs < rhs, "<=": lhs <= rhs, ">": lhs > rhs, ">=": lhs >= rhs, "=": lhs == rhs}[op]


def test_rule_latch_rows_equal_forall_v_bruteforce():
    """Def. 6's forall-v clauses: T iff S({T}) holds for the current
    histogram AND every histogram a continuation can reach; F likewise for
    S(B6-{F}) = 0.  Under reading A2 a continuation keeps permanently-true (h5) and
    permanently-false (h0) children, may move every other child anywhere and may add
    new children of any verdict.  Brute force over up to EXT new children."""
    EXT = 24
    hists = [h for N in range(0, 5) for h in itertools.product(range(5), repeat=6) if sum(h) == N]
    M = 4 + EXT + 1
    for q in _grid():
        # S5[c][N] = S({T}) with c permanently-true children of N ; S1[c][N] = S(B6-{F})
        S5 = np.zeros((M, M), bool)
        for c in range(M):
            for N2 in range(c, M):
                S5[c, N2] = _S(q, [N2 - c, 0, 0, 0, 0, c], 5)
        for h in hists:
            h = list(h)
            N = sum(h)
            top_ok = bot_ok = True
            for N2 in range(N, N + EXT + 1):
                # reachable (h5', N2): h5 <= h5' <= N2 - h0
                if not S5[h[5]:N2 - h[0] + 1, N2].all():
                    top_ok = False
                # reachable count of B6-{F} = N2 - h0' with h0 <= h0' <= N2 - h5
                for c1 in range(h[5], N2 - h[0] + 1):
                    if _S(q, [N2 - c1, 0, 0, 0, 0, c1], 5):  # S on up-set >=1 == count c1
                        bot_ok = False
                        break
                if not bot_ok and not top_ok:
                    break
            v = oracle.rule(q[0], q[1], q[2], q[3], h)
            assert (v == T) == top_ok, (q, h, v)
            assert (v == F) == (bot_ok and not top_ok), (q, h, v)


def test_rule_nonlatched_rows_lattice_order():
    """Rows Tc/Tp/Fp/Fc of Def. 6 with readings A1 and A3: the verdict is the
    highest lattice value whose up-set satisfies the constraint."""
    hists = [h for N in range(0, 6) for h in itertools.product(range(6), repeat=6) if sum(h) == N]
    for q in _grid():
        for h in hists:
            h = list(h)
            v = oracle.rule(q[0], q[1], q[2], q[3], h)
            if v in (T, F):
                continue
            expect = Fc
            for t, val in [(4, Tc), (3, Tp), (2, Fp)]:
                if _S(q, h, t):
                    expect = val
                    break
            assert v == expect, (q, h, v)


def test_empty_root_reading_A9():
    assert oracle.run_offline(tracegen.LOGIN, [np.zeros(0, np.uint32)] * 2,
                              np.zeros(0, np.uint8))["verdict"] == Tc
    assert oracle.run_offline("exists r : rid(r) => login", [np.zeros(0, np.uint32)],
                              np.zeros(0, np.uint8))["verdict"] == Fc


# ------------------------------------------------------------ whole pipeline
def _closed_socket_trace(tr):
    keys, letters = tr.keys[0], tr.letters
    valid = keys != tracegen.ABSENT
    k, a = keys[valid], letters[valid]
    idx = np.arange(k.shape[0])
    socks = np.unique(k)
    tp = 0
    for s in socks:
        sel = k == s
        r = idx[sel][(a[sel] & 1) > 0]
        sp = idx[sel][(a[sel] & 2) > 0]
        last_r = r.max() if r.size else -1
        last_s = sp.max() if sp.size else -1
        tp += int(last_r <= last_s)
    N = socks.shape[0]
    root = (Tc if N == 0 else (Tp if 20 * tp >= 19 * N else Fp))
    return root, tp, N - tp


@pytest.mark.parametrize("seed", range(6))
def test_C1_closed_form(seed):
    tr = tracegen.socket_trace(seed=seed)
    r = oracle.run_offline(tr.formula, tr.keys, tr.letters)
    root, tp, fp = _closed_socket_trace(tr)
    assert r["verdict"] == root
    assert r["hist"][1][Tp] == tp and r["hist"][1][Fp] == fp
    assert r["hist"][1].sum() == tp + fp
    assert r["events_bound"] == int((tr.keys[0] != tracegen.ABSENT).sum())


def test_C1_seeds_cover_both_sides_of_95pct():
    roots = {oracle.run_offline(t.formula, t.keys, t.letters)["verdict"]
             for t in (tracegen.socket_trace(seed=s) for s in range(12))}
    assert roots == {Tp, Fp}


def _closed_login_trace(tr):
    u, r = tr.keys
    a = tr.letters
    valid = (u != tracegen.ABSENT) & (r != tracegen.ABSENT)
    u, r, a = u[valid], r[valid], a[valid]
    # leaf = first event of each (user, rid) decides: T iff login & unauthorized
    order = np.lexsort((np.arange(u.shape[0]), r, u))
    su, sr, sa = u[order], r[order], a[order]
    first = np.r_[True, (su[1:] != su[:-1]) | (sr[1:] != sr[:-1])]
    lu, lv = su[first], (sa[first] == 3)
    users, inv = np.unique(lu, return_inverse=True)
    tcount = np.bincount(inv, weights=lv.astype(np.float64), minlength=users.shape[0])
    user_bad = tcount > 3
    root = F if user_bad.any() else Tc
    return root, int(lv.sum()), int((~lv).sum()), int(user_bad.sum()), int((~user_bad).sum())


@pytest.mark.parametrize("variant", ["random", "clean", "violator"])
def test_C2_closed_form(variant):
    tr = tracegen.login_trace(seed=3, n=60_000, users=500, variant=variant, p_unauth=0.05)
    r = oracle.run_offline(tr.formula, tr.keys, tr.letters)
    root, lt, lf, ub, uok = _closed_login_trace(tr)
    assert r["verdict"] == root
    assert list(r["hist"][2][[T, F]]) == [lt, lf] and r["hist"][2].sum() == lt + lf
    assert list(r["hist"][1][[F, Tc]]) == [ub, uok] and r["hist"][1].sum() == ub + uok
    if variant == "clean":
        assert root == Tc
    if variant == "violator":
        assert root == F


def test_C2_repeated_rids_closed_form():
    tr = tracegen.login_trace(seed=5, n=30_000, users=300, rid_events=3, p_unauth=0.1)
    r = oracle.run_offline(tr.formula, tr.keys, tr.letters)
    root, lt, lf, ub, uok = _closed_login_trace(tr)
    assert r["verdict"] == root and r["hist"][2][T] == lt and r["hist"][1][F] == ub


def test_C4_closed_form():
    tr = tracegen.proxy_trace(seed=1, n=50_000, videos=2000, p_ext_cached=0.01)
    r = oracle.run_offline(tr.formula, tr.keys, tr.letters)
    v, q = tr.keys
    a = tr.letters
    order = np.lexsort((np.arange(v.shape[0]), q, v))
    sv, sq, sa = v[order], q[order], a[order]
    first = np.r_[True, (sv[1:] != sv[:-1]) | (sq[1:] != sq[:-1])]
    lv = sa[first] == 3
    vids, inv = np.unique(sv[first], return_inverse=True)
    bad = np.bincount(inv, weights=lv.astype(np.float64), minlength=vids.shape[0]) > 0
    assert r["hist"][1][F] == bad.sum() and r["hist"][1][Tc] == (~bad).sum()
    assert r["verdict"] == (F if bad.any() else Tc)


@pytest.mark.parametrize("seed,p_heavy", [(0, 0.02), (1, 0.0)])
def test_C6_dropbox_closed_form(seed, p_heavy):
    """C6, A u : user(u) => F small(u): a user's leaf is T once one of
    its events has small set (F latches), else Fp (Table 1 / Def. 4: no
    future is excluded); the root over T and Fp children is Fp if any child is Fp,
    else Tc (A2: a new user may still come and never be small)."""
    tr = tracegen.dropbox_trace(seed=seed, n=60_000, users=800, p_heavy=p_heavy)
    r = oracle.run_offline(tr.formula, tr.keys, tr.letters)
    u, a = tr.keys[0], tr.letters
    users = np.unique(u)
    sat = np.unique(u[(a & 1) == 1])
    t, fp = sat.shape[0], users.shape[0] - sat.shape[0]
    assert r["hist"][1][T] == t and r["hist"][1][Fp] == fp and r["hist"][1].sum() == t + fp
    assert r["verdict"] == (Fp if fp else Tc)
    if p_heavy == 0.0:
        assert fp == 0 or r["verdict"] == Fp


def test_invariance_relabel_and_interleave():
    """Relabeling key values by a bijection, or interleaving events of different
    slices while keeping each slice's order, leaves every count unchanged."""
    tr = tracegen.login_trace(seed=11, n=20_000, users=200, rid_events=2, p_unauth=0.1)
    base = oracle.run_offline(tr.formula, tr.keys, tr.letters)
    u, r = tr.keys
    u2 = np.where(u == tracegen.ABSENT, u, (u ^ np.uint32(0x5bd1e995)) & np.uint32(0x7FFFFFFF))
    r2 = np.where(r == tracegen.ABSENT, r, r * np.uint32(2654435761) + np.uint32(12345))
    assert np.array_equal(oracle.run_offline(tr.formula, [u2, r2], tr.letters)["hist"], base["hist"])
    # stable sort by user interleaves differently but keeps every slice's order
    order = np.argsort(u, kind="stable")
    res = oracle.run_offline(tr.formula, [u[order], r[order]], tr.letters[order])
    assert np.array_equal(res["hist"], base["hist"]) and res["verdict"] == base["verdict"]


def test_online_prefix_equals_offline():
    tr = tracegen.login_trace(seed=2, n=3000, users=40, rid_events=2, p_unauth=0.2)
    m = oracle.Monitor(oracle.Property(tr.formula))
    cuts = [0, 1, 8, 500, 1777, 3000]
    for lo, hi in zip(cuts[:-1], cuts[1:]):
        m.feed([k[lo:hi] for k in tr.keys], tr.letters[lo:hi])
        on = m.evaluate()
        off = oracle.run_offline(tr.formula, [k[:hi] for k in tr.keys], tr.letters[:hi])
        assert on["verdict"] == off["verdict"] and np.array_equal(on["hist"], off["hist"])


def test_sum_of_child_counts():
    tr = tracegen.proxy_trace(seed=2, n=20_000, videos=500)
    r = oracle.run_offline(tr.formula, tr.keys, tr.letters)
    assert r["hist"][0].sum() == 1
    valid = (tr.keys[0] != tracegen.ABSENT) & (tr.keys[1] != tracegen.ABSENT)
    assert r["hist"][1].sum() == np.unique(tr.keys[0][valid]).shape[0]
    pairs = np.unique(np.stack([tr.keys[0][valid], tr.keys[1][valid]]), axis=1)
    assert r["hist"][2].sum() == pairs.shape[1]


# ----------------------------------------------------------------- parser
@pytest.mark.parametrize("text,kind", [
    ("G (forall x : p(x) => r(x))", "noncanonical"),
    ("forall x : p(x) => q(y)", "unbound"),
    ("forall[>=1.5] x : p(x) => q(x)", "range"),
    ("exists[>=-1] x : p(x) => q(x)", "range"),
    ("exists[>=0.5] x : p(x) => q(x)", "range"),
    ("forall x : p(x) => (q(x) &&", "syntax"),
    ("forall x : p(x) => exists y : q(y) => forall z : r(z) => exists w : s(w) => t", "budget"),
    ("forall x : p(x) => (a0 || a1 || a2 || a3 || a4 || a5 || a6 || a7 || a8)", "budget"),
])
def test_parse_errors_S56(text, kind):
    with pytest.raises(oracle.OracleParseError) as e:
        oracle.Property(text)
    assert e.value.kind == kind


def test_parse_defaults_P224():
    p = oracle.Property("forall x : p(x) => exists y : q(y) => F r(x)")
    assert p.quantifier(0) == {"kind": "A", "cmp": "=", "num": 1, "den": 1, "key": "p"}
    assert p.quantifier(1) == {"kind": "E", "cmp": ">=", "num": 1, "den": 1, "key": "q"}
    assert oracle.Property("forall[>=50%] f : intrace(f) => true").quantifier(0)["den"] == 2
    p = oracle.Property("forall x : user(x) => (exists[<=3] r : rid(r) => (login && unauthorized))")
    assert p.levels == 2


# ---------------------------------------------------------------- rule order (A3)
def test_rule_overlapping_rows_golden_A3():
    """Rows of Def. 6 that overlap for '=': the hand-derived verdicts of
    tests/golden/rule_order.txt under reading A3 (SPEC's order is recorded beside)."""
    n = 0
    for line in open(os.path.join(GOLDEN, "rule_order.txt")):
        r = line.split("#")[0].split()
        if not r:
            continue
        h = [int(x) for x in r[3:9]]
        assert oracle.rule(r[0], r[1], int(r[2]), 1, h) == NAME[r[9]], r
        n += 1
    assert n >= 6


# ---------------------------------------------------------------- timing mode
@pytest.mark.parametrize("threads", [2, 3, 8])
def test_threads_mode_identical(threads):
    """the level-0 hash partition over host threads gives the
    same verdict and counts as the sequential run, for every thread count."""
    rng = random.Random(1411 + threads)
    for case in range(25):
        levels = rng.randint(1, 3)
        ops = ["<", "<=", ">", ">=", "="]
        prefix = ""
        for i in range(levels):
            if rng.random() < 0.5:
                prefix += f"forall[{rng.choice(ops)}{rng.choice(['0', '0.5', '1', '0.75'])}] x{i} : k{i}(x{i}) => "
            else:
                prefix += f"exists[{rng.choice(ops)}{rng.randint(0, 3)}] x{i} : k{i}(x{i}) => "
        text = prefix + rng.choice(["a", "F a", "G (a -> F b)", "a U b", "X a && b"])
        keys, letters = tracegen.random_property_trace(case, levels, rng.choice([0, 1, 50, 2000]),
                                                       values=rng.choice([2, 5, 40]), atoms=2)
        a = oracle.run_offline(text, keys, letters)
        b = oracle.run_offline(text, keys, letters, threads=threads)
        assert a["verdict"] == b["verdict"] and np.array_equal(a["hist"], b["hist"]), text
        assert a["events_bound"] == b["events_bound"] and a["events_seen"] == b["events_seen"]


# ---------------------------------------------------------------- three levels (C5)
def _first_events(keys, letters):
    """(key tuples, letter) of the first event of every bound value vector."""
    k = [np.asarray(x) for x in keys]
    ok = np.ones(k[0].shape[0], bool)
    for x in k:
        ok &= x != tracegen.ABSENT
    k = [x[ok] for x in k]
    a = np.asarray(letters)[ok]
    order = np.lexsort((np.arange(a.shape[0]), *k[::-1]))
    sk = [x[order] for x in k]
    first = np.ones(a.shape[0], bool)
    first[1:] = np.any([x[1:] != x[:-1] for x in sk], axis=0) if a.shape[0] else first[1:]
    return [x[first] for x in sk], a[order][first]


def _group_any(keys, flag):
    """per distinct key tuple: any(flag) (keys sorted lexicographically)."""
    order = np.lexsort(keys[::-1])
    sk = [x[order] for x in keys]
    start = np.ones(flag.shape[0], bool)
    start[1:] = np.any([x[1:] != x[:-1] for x in sk], axis=0)
    seg = np.cumsum(start) - 1
    out = np.zeros(int(seg[-1]) + 1 if flag.shape[0] else 0, bool)
    np.logical_or.at(out, seg, flag[order])
    return [x[start] for x in sk], out


def _group_count(keys, flag):
    order = np.lexsort(keys[::-1])
    sk = [x[order] for x in keys]
    start = np.ones(flag.shape[0], bool)
    start[1:] = np.any([x[1:] != x[:-1] for x in sk], axis=0)
    seg = np.cumsum(start) - 1
    return [x[start] for x in sk], np.bincount(seg, weights=flag[order].astype(np.float64)).astype(np.int64)


@pytest.mark.parametrize("seed,p_admin,p_ext", [(0, 0.01, 0.05), (1, 0.0005, 0.01)])
def test_three_level_closed_form_c(seed, p_admin, p_ext):
    """C5 formula (c): A_{>=0.99} h => E_{=0} u => E s => (admin && external).
    Hand-derived: leaf (h,u,s) is T iff the slice's first event has admin & external,
    else F (Def. 4); (h,u) [E, default >= 1, P:226] is T iff one T session, else Fc
    (Table 1 '>=' latch); h [E_{=0}] is F iff one T child (Table 1 '=': > 0),
    else Tc; root [A_{>=0.99}] is Tc iff 100 * #Tc-hosts >= 99 * #hosts, else Fc
    (no A latch for k in (0,1), children are only F / Tc)."""
    tr = tracegen.c5_trace(seed=seed, n=400_000, hosts=64, users=3000, span_events=100_000,
                           p=(0.01, 0.3, 0.3, p_admin, p_ext))
    text = tracegen.C5_FORMULAS[2]
    lk, la = _first_events(tr.keys, tr.letters)
    leaf_t = (la & 0x18) == 0x18               # admin = bit 3, external = bit 4 of the C5 union
    prop = oracle.Property(text)
    assert prop.atoms == ["admin", "external"]
    r = oracle.run_offline(text, tr.keys, ((tr.letters >> 3) & 3).astype(np.uint8))
    hu, hu_t = _group_any(lk[:2], leaf_t)
    h, h_bad = _group_any(hu[:1], hu_t)
    root = Tc if 100 * int((~h_bad).sum()) >= 99 * h_bad.shape[0] else Fc
    assert list(r["hist"][3][[T, F]]) == [leaf_t.sum(), (~leaf_t).sum()] and r["hist"][3].sum() == leaf_t.shape[0]
    assert list(r["hist"][2][[T, Fc]]) == [hu_t.sum(), (~hu_t).sum()] and r["hist"][2].sum() == hu_t.shape[0]
    assert list(r["hist"][1][[F, Tc]]) == [h_bad.sum(), (~h_bad).sum()] and r["hist"][1].sum() == h_bad.shape[0]
    assert r["verdict"] == root


def test_three_level_closed_form_a():
    """C5 formula (a): A_{>=0.95} h => A u => E_{<=2} s => F authfail.
    Leaf T once authfail occurs in the slice, else Fp (Def. 4 of F x);
    (h,u) [E_{<=2}] is F iff > 2 T sessions (Table 1 '<='), else Tc; h [A = A_{=1}]
    is F iff one F child, else Tc; root Tc iff 100 * #Tc >= 95 * #hosts, else Fc."""
    tr = tracegen.c5_trace(seed=3, n=300_000, hosts=32, users=400, span_events=100_000,
                           p=(0.0008, 0.3, 0.3, 0.01, 0.05))
    text = tracegen.C5_FORMULAS[0]
    assert oracle.Property(text).atoms == ["authfail"]
    k = list(tr.keys)
    ok = (k[0] != tracegen.ABSENT) & (k[1] != tracegen.ABSENT) & (k[2] != tracegen.ABSENT)
    lk, leaf_t = _group_any([x[ok] for x in k], (tr.letters[ok] & 1) == 1)
    hu, ntrue = _group_count(lk[:2], leaf_t)
    hu_bad = ntrue > 2
    h, h_bad = _group_any(hu[:1], hu_bad)
    root = Tc if 100 * int((~h_bad).sum()) >= 95 * h_bad.shape[0] else Fc
    r = oracle.run_offline(text, tr.keys, (tr.letters & 1).astype(np.uint8))
    assert list(r["hist"][3][[T, Fp]]) == [leaf_t.sum(), (~leaf_t).sum()]
    assert list(r["hist"][2][[F, Tc]]) == [hu_bad.sum(), (~hu_bad).sum()]
    assert list(r["hist"][1][[F, Tc]]) == [h_bad.sum(), (~h_bad).sum()]
    assert r["verdict"] == root
    assert 0 < h_bad.sum() < h_bad.shape[0]  # both host verdicts occur
