"""CPU tests of the product's host side: the C ABI library loads and exports every
symbol include/ltl4c.h declares; the formula compiler (ltl4c_compile) agrees with
the oracle on parsing, errors, and the LTL4 verdict of EVERY word up to a length
(Def. 5: [u |=_4 psi] = lambda(delta(q0, u)))."""
import ctypes
import itertools
import random
import re

import numpy as np
import pytest

import oracle
import paper_1411_2239_b200 as ltl4c
import tracegen
from tests import ltl_bruteforce as bf

FORMULAS = [tracegen.SOCKET, tracegen.LOGIN, tracegen.PROXY, tracegen.FILES, tracegen.FIG1,
            *tracegen.C5_FORMULAS,
            "forall x : k(x) => X X a", "forall x : k(x) => G F a", "forall x : k(x) => F G a",
            "forall x : k(x) => (a U (b U c))", "forall x : k(x) => X true",
            "forall x : k(x) => !(a U X b) && G(c -> X a)", "forall x : k(x) => true",
            "forall x : k(x) => false", "forall x : k(x) => ((a U b) U c)"]


def run_word(prog, word):
    """Replay the compiled tables (delta, lambda) on one word: a test-side reader of
    the compiler's output (the verification path itself runs on the GPU)."""
    q = prog.initial
    for a in word:
        q = int(prog.delta[q, a])
    return [int(prog.label[f, q]) for f in range(prog.n_formulas)]


def test_library_exports_every_declared_symbol():
    text = open(ltl4c.HEADER).read()
    names = set(re.findall(r"\b(ltl4c_[a-z_]+)\s*\(", text))
    names = {n for n in names if not n.endswith("_t")}
    assert len(names) >= 15
    lib = ctypes.CDLL(ltl4c.LIB_PATH)
    for n in sorted(names):
        assert hasattr(lib, n), n


def test_version_string():
    assert "sm_100a" in ltl4c.version()


@pytest.mark.parametrize("text", FORMULAS)
def test_compiled_monitor_equals_oracle_on_all_words(text):
    prog = ltl4c.compile(text)
    p = oracle.Property(text)
    assert prog.atoms == p.atoms
    assert prog.n_levels == p.levels
    for i in range(p.levels):
        q = p.quantifier(i)
        assert prog.quantifiers[0][i] == q
    na = prog.n_atoms
    maxlen = {0: 3, 1: 7, 2: 6, 3: 4, 4: 3, 5: 2}.get(na, 2)
    for L in range(1, maxlen + 1):
        for w in itertools.product(range(1 << na), repeat=L):
            assert run_word(prog, w)[0] == p.ltl4(list(w)), (text, w)


def test_monitor_traps_and_budget():
    prog = ltl4c.compile(tracegen.FIG1)
    # Fig. 1: states after >= 1 letter are {both alive: Tp, "G a" alive: Tp, "b U c" alive: Fp,
    # T, F}; plus the initial state for u = epsilon (label Fp by reading A14) = 6
    assert prog.n_states == 6
    assert sorted(prog.label[0].tolist()) == [0, 2, 2, 3, 3, 5]
    for q in range(prog.n_states):
        if prog.label[0, q] in (0, 5):
            assert all(prog.delta[q, a] == q for a in range(1 << prog.n_atoms))
    assert ltl4c.compile(tracegen.SOCKET).n_states == 3  # epsilon state, pending (Fp), ok (Tp)
    assert ltl4c.compile(tracegen.LOGIN).n_states == 3


def test_random_formulas_equal_oracle():
    rng = random.Random(2239)
    done = 0
    while done < 40:
        f = bf.random_formula(rng, ["a", "b", "c"], 3)
        if not bf.atoms_in_order(f):
            continue
        text = "forall x : k(x) => " + bf.to_text(f)
        prog = ltl4c.compile(text)
        p = oracle.Property(text)
        na = prog.n_atoms
        for L in range(1, 4 if na < 3 else 3):
            for w in itertools.product(range(1 << na), repeat=L):
                assert run_word(prog, w)[0] == p.ltl4(list(w)), (text, w)
        done += 1


def test_formula_batch_product_projects_to_each_formula():
    prog = ltl4c.compile_batch(tracegen.C5_FORMULAS)
    assert prog.n_formulas == 3 and prog.n_levels == 3
    assert prog.n_states <= 16
    props = [oracle.Property(t) for t in tracegen.C5_FORMULAS]
    gidx = [[prog.atoms.index(a) for a in p.atoms] for p in props]
    rng = np.random.default_rng(5)
    for _ in range(400):
        w = [int(x) for x in rng.integers(0, 1 << prog.n_atoms, size=rng.integers(1, 6))]
        got = run_word(prog, w)
        for f, p in enumerate(props):
            lw = [sum(((a >> g) & 1) << j for j, g in enumerate(gidx[f])) for a in w]
            assert got[f] == p.ltl4(lw)


WIDE = ["forall[>=0.5] x : k(x) => exists[<=2] y : j(y) => ((a1 && a2 && !a3) || (a4 && a5))",
        "exists[>=1] x : k(x) => forall y : j(y) => F (b1 && b2 && b3 && !b4 && b5)",
        "forall x : k(x) => exists y : j(y) => G (c1 || c2)"]


def test_batch_over_more_than_8_atoms_letter_classes():
    """a formula batch over 12 atoms; the batch carries letter
    CODES (ltl4c_tables.letter_class), valuations of one class acting identically.
    Pinned against the oracle's Def. 4 of each formula on the projected valuations
    (every word up to length 3 over a sample of valuations, and random longer words)."""
    prog = ltl4c.compile_batch(WIDE)
    assert prog.n_atoms == 12 and prog.letter_class is not None
    assert prog.letter_class.shape == (1 << 12,) and int(prog.letter_class.max()) < (1 << prog.letter_bits) <= 256
    props = [oracle.Property(t) for t in WIDE]
    gidx = [[prog.atoms.index(a) for a in p.atoms] for p in props]
    rng = np.random.default_rng(12)
    vals = [int(x) for x in rng.integers(0, 1 << 12, size=12)] + [0, (1 << 12) - 1, 0b11011]

    def check(w):
        got = run_word(prog, [int(c) for c in prog.codes(np.array(w))])
        for f, p in enumerate(props):
            lw = [sum(((a >> g) & 1) << j for j, g in enumerate(gidx[f])) for a in w]
            assert got[f] == p.ltl4(lw), (w, f)

    for L in range(1, 4):
        for w in itertools.product(vals, repeat=L):
            check(list(w))
    for _ in range(300):
        check([int(x) for x in rng.integers(0, 1 << 12, size=rng.integers(1, 8))])
    # the classes are exactly the valuations with equal transition columns
    cols = {}
    for v in range(1 << 12):
        col = tuple(prog.delta[:, prog.letter_class[v]])
        cols.setdefault(prog.letter_class[v], col)
        assert cols[prog.letter_class[v]] == col
    assert len(set(cols.values())) == len(cols)
    # budgets: a single formula keeps <= 8 atoms, a batch <= 16
    with pytest.raises(ltl4c.Ltl4cError):
        ltl4c.compile("forall x : k(x) => F (" + " && ".join(f"p{i}" for i in range(9)) + ")")
    with pytest.raises(ltl4c.Ltl4cError, match="16 atoms"):
        ltl4c.compile_batch(["forall x : k(x) => F (" + " && ".join(f"p{i}" for i in range(8)) + ")",
                             "forall x : k(x) => G (" + " || ".join(f"q{i}" for i in range(8)) + ")",
                             "forall x : k(x) => F r0"])


def test_batch_requires_same_keys():
    with pytest.raises(ltl4c.Ltl4cError) as e:
        ltl4c.compile_batch([tracegen.SOCKET, tracegen.LOGIN])
    assert e.value.name == "E_INVALID"


@pytest.mark.parametrize("text,kind", [
    ("G (forall x : p(x) => r(x))", "noncanonical"),
    ("forall x : p(x) => q(y)", "unbound"),
    ("forall[>=1.5] x : p(x) => q(x)", "range"),
    ("exists[>=-1] x : p(x) => q(x)", "range"),
    ("exists[>=0.5] x : p(x) => q(x)", "range"),
    ("forall[>=0.1234567] x : p(x) => q(x)", "range"),
    ("forall x : p(x) => (q(x) &&", "syntax"),
    ("forall x : p(x) => q(x) exists y : r(y) => s", "noncanonical"),
    ("forall x : p(y) => q(x)", "unbound"),
    ("forall x : p(x) => exists y : q(y) => forall z : r(z) => exists w : s(w) => t", "budget"),
    ("forall x : p(x) => (a0 || a1 || a2 || a3 || a4 || a5 || a6 || a7 || a8)", "budget"),
])
def test_parse_errors_match_oracle(text, kind):
    with pytest.raises(oracle.OracleParseError) as oe:
        oracle.Property(text)
    assert oe.value.kind == kind
    with pytest.raises(ltl4c.Ltl4cError) as pe:
        ltl4c.compile(text)
    assert pe.value.name == "E_" + kind.upper()


def test_no_quantifier_is_a_budget_error():
    with pytest.raises(ltl4c.Ltl4cError) as e:
        ltl4c.compile("G (a -> F b)")
    assert e.value.name == "E_BUDGET"


def test_constants_are_exact_fractions():
    for text, num, den in [("forall[>=0.95] s : p(s) => a", 19, 20), ("forall[>=50%] s : p(s) => a", 1, 2),
                           ("forall[<99.5%] s : p(s) => a", 199, 200), ("forall[>0] s : p(s) => a", 0, 1),
                           ("forall[=1.000000] s : p(s) => a", 1, 1)]:
        q = ltl4c.compile(text).quantifiers[0][0]
        assert (q["num"], q["den"]) == (num, den)
        oq = oracle.Property(text).quantifier(0)
        assert (oq["num"], oq["den"]) == (num, den)


def test_state_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    with pytest.raises(ltl4c.Ltl4cError) as e:
        ltl4c.compile(tracegen.LOGIN).state(0)
    assert e.value.name in ("E_CUDA", "E_INVALID")
