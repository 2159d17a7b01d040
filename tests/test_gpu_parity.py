"""GPU parity: the sm_100a path (through the C ABI) against the oracle, bit-exact
on verdicts and per-level counts (integer-only path: SURVEY §8(c), BASELINE.json
"bit-exact verdicts and counts").  Inputs are seeded tracegen workloads."""
import random

import numpy as np
import pytest

import oracle
import tracegen
from tests import ltl_bruteforce as bf

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env(cuda_ok):
    import torch

    import paper_1411_2239_b200 as ltl4c
    return ltl4c, torch, torch.device("cuda:0")


def _dev(torch, dev, keys, letters):
    return ([torch.from_numpy(np.ascontiguousarray(k).view(np.int32)).to(dev) for k in keys],
            torch.from_numpy(np.ascontiguousarray(letters)).to(dev))


def _gpu_offline(env, text, keys, letters):
    ltl4c, torch, dev = env
    st = ltl4c.compile(text).state(0)
    k, l = _dev(torch, dev, keys, letters)
    return st.verify(k, l)


def _assert_same(got, want, ctx=""):
    assert got.verdict == want["verdict"], (ctx, got.verdict, want["verdict"])
    assert np.array_equal(got.hist, want["hist"]), (ctx, got.hist, want["hist"])
    assert got.events_bound == want["events_bound"], ctx


def test_worked_example_offline_and_online(env):
    ltl4c, torch, dev = env
    tr = tracegen.worked_example()
    got = _gpu_offline(env, tr.formula, tr.keys, tr.letters)[0]
    _assert_same(got, oracle.run_offline(tr.formula, tr.keys, tr.letters))
    assert got.verdict == 0 and list(got.hist[1]) == [1, 0, 0, 0, 1, 0]
    st = ltl4c.compile(tr.formula).state(0, online=True)
    verdicts = []
    for j in range(tr.n):
        k, l = _dev(torch, dev, [x[j:j + 1] for x in tr.keys], tr.letters[j:j + 1])
        verdicts.append(st.verify(k, l)[0].verdict)
    assert verdicts == [4, 4, 4, 4, 0]


@pytest.mark.parametrize("seed", range(6))
def test_C1_socket(env, seed):
    tr = tracegen.socket_trace(seed=seed)
    _assert_same(_gpu_offline(env, tr.formula, tr.keys, tr.letters)[0],
                 oracle.run_offline(tr.formula, tr.keys, tr.letters), seed)


@pytest.mark.parametrize("variant,rid_events", [("random", 1), ("clean", 1), ("violator", 1),
                                                ("random", 3)])
def test_C2_login_small(env, variant, rid_events):
    tr = tracegen.login_trace(seed=7, n=300_000, users=3000, variant=variant, rid_events=rid_events,
                              p_unauth=0.04)
    _assert_same(_gpu_offline(env, tr.formula, tr.keys, tr.letters)[0],
                 oracle.run_offline(tr.formula, tr.keys, tr.letters), variant)


def test_C2_login_full_size(env):
    """BASELINE.json configs[1] at full size (10M events, 100k users), as bench.py runs it."""
    tr = tracegen.login_trace(seed=0)
    _assert_same(_gpu_offline(env, tr.formula, tr.keys, tr.letters)[0],
                 oracle.run_offline(tr.formula, tr.keys, tr.letters), "C2 full")


@pytest.mark.parametrize("support,s", [(1 << 12, 1.1), (1 << 16, 1.1)])
def test_C3_zipf_skew(env, support, s):
    """Heavy keys exceed one shared-memory chunk: exercises the chunked global path
    and the warp-level ordered map composition for long slices."""
    tr = tracegen.zipf_socket_trace(seed=1, n=1_000_000, support=support, s=s)
    _assert_same(_gpu_offline(env, tr.formula, tr.keys, tr.letters)[0],
                 oracle.run_offline(tr.formula, tr.keys, tr.letters), support)
    tr = tracegen.zipf_socket_trace(seed=2, n=400_000, support=4096, formula=tracegen.FIG1)
    tr.letters = np.random.default_rng(3).choice(np.array([1, 3, 2, 6, 7, 0], np.uint8), size=tr.n,
                                                 p=[0.6, 0.2, 0.1, 0.05, 0.04, 0.01])
    _assert_same(_gpu_offline(env, tr.formula, tr.keys, tr.letters)[0],
                 oracle.run_offline(tr.formula, tr.keys, tr.letters), "fig1")


def test_C4_proxy(env):
    tr = tracegen.proxy_trace(seed=3, n=1_000_000, videos=20_000, p_ext_cached=0.002)
    _assert_same(_gpu_offline(env, tr.formula, tr.keys, tr.letters)[0],
                 oracle.run_offline(tr.formula, tr.keys, tr.letters), "C4")


@pytest.mark.parametrize("seed,n,users", [(0, 400_000, 5000), (1, 4_000_000, 100_000)])
def test_C6_dropbox(env, seed, n, users):
    """C6 (SURVEY §8(f) NEXT-4 workload): one level, F small(u), uniform users
    (no hot key at 5000 users of 400k events; at 4M events a two-pass cold stream)."""
    tr = tracegen.dropbox_trace(seed=seed, n=n, users=users)
    _assert_same(_gpu_offline(env, tr.formula, tr.keys, tr.letters)[0],
                 oracle.run_offline(tr.formula, tr.keys, tr.letters), ("C6", n))


def _project(letters, prog_atoms, prop_atoms):
    out = np.zeros_like(letters)
    for j, a in enumerate(prop_atoms):
        g = prog_atoms.index(a)
        out |= ((letters >> g) & 1) << j
    return out


def test_C5_formula_batch_online(env):
    ltl4c, torch, dev = env
    tr = tracegen.c5_trace(seed=0, n=300_000, users=2000, hosts=64, span_events=60_000)
    prog = ltl4c.compile_batch(tracegen.C5_FORMULAS)
    st = prog.state(0, online=True)
    props = [oracle.Property(t) for t in tracegen.C5_FORMULAS]
    mons = [oracle.Monitor(p) for p in props]
    cuts = [0, 1000, 50_000, 170_000, 300_000]
    for lo, hi in zip(cuts[:-1], cuts[1:]):
        k, l = _dev(torch, dev, [x[lo:hi] for x in tr.keys], tr.letters[lo:hi])
        got = st.verify(k, l, first_index=lo)
        for f, (p, m) in enumerate(zip(props, mons)):
            m.feed([x[lo:hi] for x in tr.keys], _project(tr.letters[lo:hi], prog.atoms, p.atoms))
            _assert_same(got[f], m.evaluate(), (f, hi))


def test_checkpoint_restore_continues_the_stream(env):
    """an online state's carried state checkpointed after
    some batches and restored into a fresh state (and into a state that had verified
    something else) continues the stream exactly: every later result equals the oracle
    on the prefix; a checkpoint of another program is refused."""
    ltl4c, torch, dev = env
    tr = tracegen.c5_trace(seed=3, n=240_000, users=1500, hosts=48, span_events=50_000)
    prog = ltl4c.compile_batch(tracegen.C5_FORMULAS)
    props = [oracle.Property(t) for t in tracegen.C5_FORMULAS]
    mons = [oracle.Monitor(p) for p in props]
    a = prog.state(0, online=True)
    cuts = [0, 900, 60_000, 110_000, 180_000, 240_000]

    def feed(st, lo, hi, check):
        k, l = _dev(torch, dev, [x[lo:hi] for x in tr.keys], tr.letters[lo:hi])
        got = st.verify(k, l, first_index=lo)
        if check:
            for f, (p, m) in enumerate(zip(props, mons)):
                m.feed([x[lo:hi] for x in tr.keys], _project(tr.letters[lo:hi], prog.atoms, p.atoms))
                _assert_same(got[f], m.evaluate(), ("ckpt", f, hi))
        return got

    for lo, hi in zip(cuts[:3], cuts[1:4]):
        feed(a, lo, hi, True)
    blob = a.checkpoint()
    b = prog.state(0, online=True)
    b.restore(blob)
    c = prog.state(0, online=True)
    feed(c, 0, 900, False)             # c verified another prefix first: restore replaces it
    c.restore(blob)
    a_results = {}
    for lo, hi in zip(cuts[3:-1], cuts[4:]):
        gb = feed(b, lo, hi, True)
        a_results[hi] = (gb[0].verdict, gb[0].hist.copy())
        for st in (a, c):
            g = feed(st, lo, hi, False)
            for f in range(len(props)):
                assert g[f].verdict == gb[f].verdict and np.array_equal(g[f].hist, gb[f].hist)
    other = ltl4c.compile(tracegen.LOGIN).state(0, online=True)
    with pytest.raises(ltl4c.Ltl4cError):
        other.restore(blob)
    # compaction (NEXT-3): the carried tables shrink to the live entries and the stream
    # continues exactly
    d = prog.state(0, online=True)
    d.restore(blob)
    before = len(d.checkpoint())
    d.compact()
    assert len(d.checkpoint()) < before
    for lo, hi in zip(cuts[3:-1], cuts[4:]):
        g = feed(d, lo, hi, False)
        assert g[0].verdict == a_results[hi][0] and np.array_equal(g[0].hist, a_results[hi][1])


def test_node_dump_explains_the_counts(env):
    """ltl4c_state_nodes lists every node of a depth of the online
    tree (Fig. 2) with its verdict; each node's verdict equals the oracle's
    verdict of the same value vector, and the per-verdict counts are the histogram."""
    ltl4c, torch, dev = env
    tr = tracegen.c5_trace(seed=5, n=60_000, users=400, hosts=16, span_events=20_000)
    prog = ltl4c.compile_batch(tracegen.C5_FORMULAS)
    st = prog.state(0, online=True)
    props = [oracle.Property(t) for t in tracegen.C5_FORMULAS]
    mons = [oracle.Monitor(p) for p in props]
    for lo, hi in [(0, 25_000), (25_000, 60_000)]:
        k, l = _dev(torch, dev, [x[lo:hi] for x in tr.keys], tr.letters[lo:hi])
        got = st.verify(k, l, first_index=lo)
        for p, m in zip(props, mons):
            m.feed([x[lo:hi] for x in tr.keys], _project(tr.letters[lo:hi], prog.atoms, p.atoms))
    for f, m in enumerate(mons):
        want = m.evaluate()
        for level in (1, 2, 3):
            keys, ver = st.nodes(level, f)
            assert np.array_equal(np.bincount(ver, minlength=6), got[f].hist[level]), (f, level)
            assert np.array_equal(got[f].hist[level], want["hist"][level]), (f, level)
            pick = np.random.default_rng(level).choice(ver.shape[0], size=min(300, ver.shape[0]), replace=False)
            for j in pick:
                assert m.node_verdict([int(k[j]) for k in keys]) == int(ver[j]), (f, level, j)
    with pytest.raises(ltl4c.Ltl4cError):
        st.nodes(4, 0)


def test_online_batches_equal_offline_prefix(env):
    ltl4c, torch, dev = env
    tr = tracegen.login_trace(seed=9, n=200_000, users=500, rid_events=4, p_unauth=0.05)
    st = ltl4c.compile(tr.formula).state(0, online=True)
    cuts = [0, 7, 5000, 5001, 120_000, 200_000]
    for lo, hi in zip(cuts[:-1], cuts[1:]):
        k, l = _dev(torch, dev, [x[lo:hi] for x in tr.keys], tr.letters[lo:hi])
        got = st.verify(k, l, first_index=lo)[0]
        want = oracle.run_offline(tr.formula, [x[:hi] for x in tr.keys], tr.letters[:hi])
        _assert_same(got, want, hi)


def test_online_rejects_gap_and_reset(env):
    ltl4c, torch, dev = env
    tr = tracegen.worked_example()
    st = ltl4c.compile(tr.formula).state(0, online=True)
    k, l = _dev(torch, dev, [x[:2] for x in tr.keys], tr.letters[:2])
    st.verify(k, l, first_index=0)
    with pytest.raises(ltl4c.Ltl4cError) as e:
        st.verify(k, l, first_index=5)
    assert e.value.name == "E_INVALID"
    st.reset()
    k, l = _dev(torch, dev, tr.keys, tr.letters)
    _assert_same(st.verify(k, l, first_index=0)[0], oracle.run_offline(tr.formula, tr.keys, tr.letters))


def test_edge_cases(env):
    ltl4c, torch, dev = env
    text = tracegen.LOGIN
    empty = [np.zeros(0, np.uint32)] * 2
    _assert_same(_gpu_offline(env, text, empty, np.zeros(0, np.uint8))[0],
                 oracle.run_offline(text, empty, np.zeros(0, np.uint8)), "empty")
    absent = [np.full(100, 0xFFFFFFFF, np.uint32), np.arange(100, dtype=np.uint32)]
    lets = np.full(100, 3, np.uint8)
    _assert_same(_gpu_offline(env, text, absent, lets)[0], oracle.run_offline(text, absent, lets), "absent")
    one = [np.array([5], np.uint32), np.array([6], np.uint32)]
    _assert_same(_gpu_offline(env, text, one, np.array([3], np.uint8))[0],
                 oracle.run_offline(text, one, np.array([3], np.uint8)), "one")
    # key value 0 and 0xFFFFFFFE are ordinary values
    k = [np.array([0, 0xFFFFFFFE, 0], np.uint32), np.array([0, 0, 0xFFFFFFFE], np.uint32)]
    lt = np.array([3, 1, 3], np.uint8)
    _assert_same(_gpu_offline(env, text, k, lt)[0], oracle.run_offline(text, k, lt), "extreme keys")


def test_random_properties_offline_and_online(env):
    """Random formulas (1-3 levels, <= 3 atoms, depth <= 3) x random traces over tiny
    domains, offline and online with random batch splits."""
    ltl4c, torch, dev = env
    rng = random.Random(411)
    ops = ["<", "<=", ">", ">=", "="]
    for case in range(60):
        levels = rng.randint(1, 3)
        f = bf.random_formula(rng, ["a", "b", "c"], 3)
        if not bf.atoms_in_order(f):
            continue
        prefix = ""
        for i in range(levels):
            if rng.random() < 0.5:
                c = rng.choice(["0", "0.25", "0.5", "1", "1/3"]) if False else rng.choice(["0", "0.25", "0.5", "1", "0.75"])
                prefix += f"forall[{rng.choice(ops)}{c}] x{i} : k{i}(x{i}) => "
            else:
                prefix += f"exists[{rng.choice(ops)}{rng.randint(0, 3)}] x{i} : k{i}(x{i}) => "
        text = prefix + bf.to_text(f)
        na = len(bf.atoms_in_order(f))
        n = rng.choice([1, 5, 40, 300, 3000])
        keys, letters = tracegen.random_property_trace(case, levels, n, values=rng.choice([2, 3, 50]),
                                                       atoms=na)
        want = oracle.run_offline(text, keys, letters)
        _assert_same(_gpu_offline(env, text, keys, letters)[0], want, text)
        st = ltl4c.compile(text).state(0, online=True)
        cuts = sorted({0, n, *[rng.randint(0, n) for _ in range(3)]})
        for lo, hi in zip(cuts[:-1], cuts[1:]):
            k, l = _dev(torch, dev, [x[lo:hi] for x in keys], letters[lo:hi])
            got = st.verify(k, l, first_index=lo)[0]
        _assert_same(got, want, ("online", text))


def test_verify_host_equals_device(env):
    ltl4c, torch, dev = env
    tr = tracegen.login_trace(seed=4, n=100_000, users=1000, p_unauth=0.05)
    st = ltl4c.compile(tr.formula).state(0)
    a = st.verify_host(tr.keys, tr.letters)[0]
    k, l = _dev(torch, dev, tr.keys, tr.letters)
    b = st.verify(k, l)[0]
    assert a.verdict == b.verdict and np.array_equal(a.hist, b.hist)


def test_deterministic_reruns(env):
    ltl4c, torch, dev = env
    tr = tracegen.zipf_socket_trace(seed=5, n=500_000, support=1 << 14)
    st = ltl4c.compile(tr.formula).state(0)
    k, l = _dev(torch, dev, tr.keys, tr.letters)
    first = st.verify(k, l)[0]
    for _ in range(3):
        again = st.verify(k, l)[0]
        assert again.verdict == first.verdict and np.array_equal(again.hist, first.hist)


def test_profiling_counts_launches(env):
    ltl4c, torch, dev = env
    tr = tracegen.socket_trace(seed=0)
    st = ltl4c.compile(tr.formula).state(0)
    st.profile(True)
    k, l = _dev(torch, dev, tr.keys, tr.letters)
    st.verify(k, l)
    s = st.stats()
    assert s["launches"] >= 5 and s["kernels"]["bucket_fast"]["launches"] == 1
    assert s["kernels"]["bucket_fast"]["ms"] > 0


def test_exchange_path_single_rank(env):
    """The multi-GPU path (owner partition, NCCL all-gather of counts, grouped
    send/recv, local pipeline, all-reduce, root rule) forced with one rank."""
    import subprocess
    import sys
    code = r'''
import sys, numpy as np, torch
sys.path.insert(0, ".")
import oracle, tracegen, paper_1411_2239_b200 as ltl4c
dev = torch.device("cuda:0")
for tr in (tracegen.login_trace(seed=8, n=200_000, users=2000, rid_events=2, p_unauth=0.05),
           tracegen.zipf_socket_trace(seed=9, n=300_000, support=1 << 12)):
    st = ltl4c.compile(tr.formula).state(0)
    st.comm(None, 1, 0)
    k = [torch.from_numpy(x.view(np.int32)).to(dev) for x in tr.keys]
    got = st.verify(k, torch.from_numpy(tr.letters).to(dev))[0]
    want = oracle.run_offline(tr.formula, tr.keys, tr.letters)
    assert got.verdict == want["verdict"], (got.verdict, want["verdict"])
    assert np.array_equal(got.hist, want["hist"]), (got.hist, want["hist"])
    assert got.events_seen == tr.n and got.events_bound == want["events_bound"]
print("ok")
'''
    env_ = dict(__import__("os").environ, LTL4C_FORCE_EXCHANGE="1")
    r = subprocess.run([sys.executable, "-c", code], env=env_, capture_output=True, text=True, timeout=300,
                       cwd=__import__("os").path.dirname(__import__("os").path.dirname(__file__)))
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


def test_C5_formula_batch_offline(env):
    """K = 3, F = 3 offline: warp, CTA and heavy bucket paths with 3-level tables."""
    ltl4c, torch, dev = env
    for n, users, hosts in [(200_000, 3000, 64), (400_000, 500, 4)]:
        tr = tracegen.c5_trace(seed=2, n=n, users=users, hosts=hosts, span_events=n // 4)
        prog = ltl4c.compile_batch(tracegen.C5_FORMULAS)
        st = prog.state(0)
        k, l = _dev(torch, dev, tr.keys, tr.letters)
        got = st.verify(k, l)
        for f, text in enumerate(tracegen.C5_FORMULAS):
            p = oracle.Property(text)
            want = oracle.run_offline(text, tr.keys, _project(tr.letters, prog.atoms, p.atoms))
            _assert_same(got[f], want, (n, f))


def test_giant_single_slice(env):
    """One value vector with 9M events: > 4096 segments, so the heavy path composes
    the leaf's partial maps in several shared-memory windows."""
    ltl4c, torch, dev = env
    n = 9_000_000
    rng = np.random.default_rng(77)
    keys = [np.full(n, 12345, np.uint32)]
    keys[0][rng.random(n) < 0.001] = 999   # a second, light key in the same stream
    letters = rng.choice(np.array([0, 1, 2, 3], np.uint8), size=n, p=[0.4, 0.3, 0.2, 0.1])
    for text in (tracegen.SOCKET, tracegen.FILES):
        _assert_same(_gpu_offline(env, text, keys, letters)[0], oracle.run_offline(text, keys, letters), text)


def test_online_host_buffers(env):
    ltl4c, torch, dev = env
    tr = tracegen.login_trace(seed=12, n=120_000, users=800, rid_events=3, p_unauth=0.1)
    st = ltl4c.compile(tr.formula).state(0, online=True)
    cuts = [0, 30_000, 30_001, 120_000]
    for lo, hi in zip(cuts[:-1], cuts[1:]):
        got = st.verify_host([x[lo:hi] for x in tr.keys], tr.letters[lo:hi], first_index=lo)[0]
        want = oracle.run_offline(tr.formula, [x[:hi] for x in tr.keys], tr.letters[:hi])
        _assert_same(got, want, hi)


def test_forced_spill_chain():
    """Few, large buckets (bucket bits capped through LTL4C_MAX_BITS in a fresh
    process) route work through every spill tier: warp unit -> warp big ->
    CTA bucket -> heavy path, for K = 1, 2 and 3."""
    import os
    import subprocess
    import sys
    code = r'''
import sys, numpy as np, torch
sys.path.insert(0, ".")
import oracle, tracegen, paper_1411_2239_b200 as ltl4c
dev = torch.device("cuda:0")
def proj(letters, prog_atoms, prop_atoms):
    out = np.zeros_like(letters)
    for j, a in enumerate(prop_atoms):
        out |= ((letters >> prog_atoms.index(a)) & 1) << j
    return out
cases = [tracegen.login_trace(seed=21, n=300_000, users=3000, rid_events=2, p_unauth=0.05),
         tracegen.proxy_trace(seed=22, n=300_000, videos=20_000),
         tracegen.zipf_socket_trace(seed=23, n=300_000, support=1 << 12)]
for tr in cases:
    st = ltl4c.compile(tr.formula).state(0)
    k = [torch.from_numpy(x.view(np.int32)).to(dev) for x in tr.keys]
    got = st.verify(k, torch.from_numpy(tr.letters).to(dev))[0]
    want = oracle.run_offline(tr.formula, tr.keys, tr.letters)
    assert got.verdict == want["verdict"] and np.array_equal(got.hist, want["hist"]), (tr.meta, got.hist, want["hist"])
tr = tracegen.c5_trace(seed=24, n=200_000, users=3000, hosts=64, span_events=50_000)
prog = ltl4c.compile_batch(tracegen.C5_FORMULAS)
k = [torch.from_numpy(x.view(np.int32)).to(dev) for x in tr.keys]
got = prog.state(0).verify(k, torch.from_numpy(tr.letters).to(dev))
for f, text in enumerate(tracegen.C5_FORMULAS):
    p = oracle.Property(text)
    want = oracle.run_offline(text, tr.keys, proj(tr.letters, prog.atoms, p.atoms))
    assert got[f].verdict == want["verdict"] and np.array_equal(got[f].hist, want["hist"]), (f, got[f].hist, want["hist"])
print("ok")
'''
    root = os.path.dirname(os.path.dirname(__file__))
    for bits in ("4", "7", "10"):
        env_ = dict(os.environ, LTL4C_MAX_BITS=bits)
        r = subprocess.run([sys.executable, "-c", code], env=env_, capture_output=True, text=True, timeout=600,
                           cwd=root)
        assert r.returncode == 0 and "ok" in r.stdout, (bits, r.stdout + r.stderr)


def test_online_table_growth(env):
    """Online batches whose distinct leaves outgrow the first carried tables: the
    tables are rehashed into larger ones between batches and nothing is lost."""
    ltl4c, torch, dev = env
    n, b = 1_500_000, 250_000
    tr = tracegen.login_trace(seed=31, n=n, users=3000, p_unauth=0.02)
    st = ltl4c.compile(tr.formula).state(0, online=True)
    st.profile(True)
    for lo in range(0, n, b):
        hi = min(n, lo + b)
        k, l = _dev(torch, dev, [x[lo:hi] for x in tr.keys], tr.letters[lo:hi])
        got = st.verify(k, l, first_index=lo)[0]
        if hi in (2 * b, n):
            _assert_same(got, oracle.run_offline(tr.formula, [x[:hi] for x in tr.keys], tr.letters[:hi]), hi)
    assert st.stats()["kernels"]["rehash"]["launches"] >= 1


@pytest.mark.parametrize("levels,nform", [(1, 2), (2, 2), (2, 4), (1, 4), (3, 2)])
def test_formula_batches(env, levels, nform):
    """Formula batches of F = 2 and 4 (one product monitor, shared guard keys) for
    K = 1, 2, 3: every formula's verdict and counts against the oracle, offline
    (sizes that reach the warp, CTA and heavy paths) and online."""
    ltl4c, torch, dev = env
    rng = random.Random(1000 * levels + nform)
    ops = ["<", "<=", ">", ">=", "="]
    # (the product of the batch must stay within 16 states)
    bodies = (["F a", "G (a -> F b)", "a U b", "(a && b)", "X !a", "G a || (b U c)", "F (a && X c)"] if nform == 2
              else ["F a", "G b", "F (a && b)", "G (a || b)"])
    texts = []
    for f in range(nform):
        prefix = ""
        for i in range(levels):
            if rng.random() < 0.5:
                prefix += f"forall[{rng.choice(ops)}{rng.choice(['0', '0.5', '1', '0.75'])}] x{i} : k{i}(x{i}) => "
            else:
                prefix += f"exists[{rng.choice(ops)}{rng.randint(0, 3)}] x{i} : k{i}(x{i}) => "
        texts.append(prefix + bodies[(f + levels) % len(bodies)])
    prog = ltl4c.compile_batch(texts)
    props = [oracle.Property(t) for t in texts]
    for n, values in [(5000, 40), (300_000, 3000), (400_000, 7)]:
        keys, letters = tracegen.random_property_trace(7 * n + levels, levels, n, values=values,
                                                       atoms=len(prog.atoms))
        k, l = _dev(torch, dev, keys, letters)
        got = prog.state(0).verify(k, l)
        for f, (t, p) in enumerate(zip(texts, props)):
            want = oracle.run_offline(t, keys, _project(letters, prog.atoms, p.atoms))
            _assert_same(got[f], want, (t, n))
        if n == 5000:
            st = prog.state(0, online=True)
            for lo, hi in [(0, 1200), (1200, 1201), (1201, 5000)]:
                kk, ll = _dev(torch, dev, [x[lo:hi] for x in keys], letters[lo:hi])
                got = st.verify(kk, ll, first_index=lo)
            for f, (t, p) in enumerate(zip(texts, props)):
                _assert_same(got[f], oracle.run_offline(t, keys, _project(letters, prog.atoms, p.atoms)), ("online", t))


def test_online_async_pipeline(env):
    """Pipelined online batches (ltl4c_verify_async / ltl4c_result_get) return the
    same result per batch as synchronous verification, with carried tables growing
    while batches are in flight; misuse is rejected."""
    ltl4c, torch, dev = env
    tr = tracegen.c5_trace(seed=41, n=2_400_000, users=3000, hosts=64, span_events=400_000)
    prog = ltl4c.compile_batch(tracegen.C5_FORMULAS)
    sync_st, async_st = prog.state(0, online=True), prog.state(0, online=True)
    k, l = _dev(torch, dev, tr.keys, tr.letters)
    b = 200_000
    tickets, want = [], []
    for i, lo in enumerate(range(0, tr.n, b)):
        hi = min(tr.n, lo + b)
        want.append(sync_st.verify([x[lo:hi] for x in k], l[lo:hi], first_index=lo))
        tickets.append(async_st.verify_async([x[lo:hi] for x in k], l[lo:hi], first_index=lo))
        if len(tickets) > 4:  # read with a lag of 4 batches
            j = len(want) - 5
            got = async_st.result(tickets[j])
            for f in range(len(got)):
                _assert_same(got[f], {"verdict": want[j][f].verdict, "hist": want[j][f].hist,
                                      "events_bound": want[j][f].events_bound}, ("async", j, f))
    for j in range(len(want) - 4, len(want)):
        got = async_st.result(tickets[j])
        for f in range(len(got)):
            assert got[f].verdict == want[j][f].verdict and np.array_equal(got[f].hist, want[j][f].hist)
    for f, text in enumerate(tracegen.C5_FORMULAS):
        p = oracle.Property(text)
        _assert_same(want[-1][f], oracle.run_offline(text, tr.keys, _project(tr.letters, prog.atoms, p.atoms)), f)
    with pytest.raises(ltl4c.Ltl4cError):
        async_st.result(tickets[0])            # already read
    with pytest.raises(ltl4c.Ltl4cError):
        prog.state(0).verify_async([x[:10] for x in k], l[:10])   # offline state
    st = prog.state(0, online=True)
    ts = [st.verify_async([x[i:i + 10] for x in k], l[i:i + 10], first_index=i) for i in range(0, 80, 10)]
    with pytest.raises(ltl4c.Ltl4cError):
        st.verify_async([x[80:90] for x in k], l[80:90], first_index=80)   # 9th outstanding
    for t in ts:
        st.result(t)


def test_records_through_encoder_and_gpu(env):
    """JSON-lines records -> host encoder (ltl4c_encode_jsonl) -> sm_100a path, against
    the oracle reading the SAME records with its own reader: the worked example
    (tests/golden/login_example.jsonl) and a C2-shaped file."""
    import os
    ltl4c, torch, dev = env
    golden = open(os.path.join(os.path.dirname(__file__), "golden", "login_example.jsonl")).read()
    tr = tracegen.login_trace(seed=17, n=300_000, users=3000, rid_events=2, p_unauth=0.05)
    big = tracegen.to_jsonl(tr, ["user", "rid"], ["login", "unauthorized"], [[], []], seed=2, style="mixed")
    sock = tracegen.zipf_socket_trace(seed=18, n=200_000, support=1 << 12)
    sock_txt = tracegen.to_jsonl(sock, ["socket"], ["receive", "respond"], [[0], [0]], seed=3, style="mixed")
    for formula, text in ((tracegen.LOGIN, golden), (tracegen.LOGIN, big), (tracegen.SOCKET, sock_txt)):
        prog = ltl4c.compile(formula)
        keys, letters = prog.encoder().encode(text)
        k, l = _dev(torch, dev, keys, letters)
        got = prog.state(0).verify(k, l)[0]
        want = oracle.run_records(formula, text)
        _assert_same(got, want, (formula, len(text)))
    # online: records streamed in chunks through one encoder (dictionaries persist)
    prog = ltl4c.compile(tracegen.LOGIN)
    enc = prog.encoder()
    st = prog.state(0, online=True)
    lines = big.splitlines(keepends=True)
    mon = oracle.RecordMonitor(oracle.Property(tracegen.LOGIN))
    for lo in range(0, len(lines), 70_000):
        chunk = "".join(lines[lo:lo + 70_000])
        keys, letters = enc.encode(chunk)
        k, l = _dev(torch, dev, keys, letters)
        got = st.verify(k, l)[0]
        mon.feed_records(chunk)
        _assert_same(got, mon.evaluate(), ("online records", lo))


WIDE = ["forall[>=0.5] x : k(x) => exists[<=2] y : j(y) => ((a1 && a2 && !a3) || (a4 && a5))",
        "exists[>=1] x : k(x) => forall y : j(y) => F (b1 && b2 && b3 && !b4 && b5)",
        "forall x : k(x) => exists y : j(y) => G (c1 || c2)"]


def test_batch_over_more_than_8_atoms(env):
    """a formula batch over 12 atoms -- events carry letter
    codes (classes of atom valuations, ltl4c_tables.letter_class); offline and online
    results of every formula equal the oracle on that formula's projected valuations;
    the host encoder emits the codes."""
    ltl4c, torch, dev = env
    prog = ltl4c.compile_batch(WIDE)
    assert prog.n_atoms == 12 and prog.letter_class is not None
    g = np.random.default_rng(121)
    n = 400_000
    keys = [g.integers(0, 3000, n).astype(np.uint32), g.integers(0, 40_000, n).astype(np.uint32)]
    keys[1][g.random(n) < 0.01] = 0xFFFFFFFF
    # valuations: each atom set with its own probability (so every formula sees both outcomes)
    pa = g.uniform(0.2, 0.95, 12)
    vals = np.zeros(n, np.uint32)
    for j in range(12):
        vals |= (g.random(n) < pa[j]).astype(np.uint32) << j
    codes = prog.codes(vals)
    props = [oracle.Property(t) for t in WIDE]
    gidx = [[prog.atoms.index(a) for a in p.atoms] for p in props]

    def proj(v, f):
        out = np.zeros(v.shape[0], np.uint8)
        for j, gg in enumerate(gidx[f]):
            out |= (((v >> gg) & 1) << j).astype(np.uint8)
        return out

    k, l = _dev(torch, dev, keys, codes)
    got = prog.state(0).verify(k, l)
    for f, t in enumerate(WIDE):
        _assert_same(got[f], oracle.run_offline(t, keys, proj(vals, f)), ("wide offline", f))
    st = prog.state(0, online=True)
    for lo, hi in [(0, 1000), (1000, 150_000), (150_000, n)]:
        k, l = _dev(torch, dev, [x[lo:hi] for x in keys], codes[lo:hi])
        got = st.verify(k, l, first_index=lo)
        for f, t in enumerate(WIDE):
            _assert_same(got[f], oracle.run_offline(t, [x[:hi] for x in keys], proj(vals[:hi], f)), ("wide online", f, hi))
    # records: the encoders turn the 12 atoms of a record into the code
    import json as _json
    recs = []
    for j in range(2000):
        r = {"k": int(keys[0][j]), "j": int(keys[1][j])} if keys[1][j] != 0xFFFFFFFF else {"k": int(keys[0][j])}
        for a in range(12):
            if (vals[j] >> a) & 1:
                r[prog.atoms[a]] = True
        recs.append(_json.dumps(r))
    text = "\n".join(recs) + "\n"
    hk, hl = prog.encoder().encode(text)
    assert np.array_equal(hl, codes[:2000])
    dk, dl = prog.device_encoder().encode(text)
    assert np.array_equal(dl.cpu().numpy(), codes[:2000])


def _same_partition(a, b):
    """a and b label the same events with a bijection of ids (equal partitions)."""
    a, b = np.asarray(a, np.int64), np.asarray(b, np.int64)
    if a.shape != b.shape:
        return False
    pairs = np.unique(np.stack([a, b]), axis=1)
    return np.unique(pairs[0]).shape[0] == pairs.shape[1] == np.unique(pairs[1]).shape[0]


def test_device_encoder_matches_host_and_oracle(env):
    """JSON-lines records in device memory encoded on the GPU
    (ltl4c_dencode_jsonl) give the host encoder's letters and, per key, the same
    partition of events by value (ids are a relabelling); verified on the GPU they
    equal the oracle reading the SAME records with its own reader -- the worked
    example, mixed spellings (12 / "12" / 12.0 / 1.2e1, noise keys, blank lines,
    escapes), parametric atoms, three levels, and an online stream in chunks."""
    import os
    ltl4c, torch, dev = env
    golden = open(os.path.join(os.path.dirname(__file__), "golden", "login_example.jsonl")).read()
    tr = tracegen.login_trace(seed=27, n=200_000, users=2000, rid_events=2, p_unauth=0.05)
    big = tracegen.to_jsonl(tr, ["user", "rid"], ["login", "unauthorized"], [[], []], seed=4, style="mixed")
    sock = tracegen.zipf_socket_trace(seed=28, n=150_000, support=1 << 12)
    sock_txt = tracegen.to_jsonl(sock, ["socket"], ["receive", "respond"], [[0], [0]], seed=5, style="mixed")
    c5 = tracegen.c5_trace(seed=6, n=80_000, users=600, hosts=20, span_events=20_000)
    c5_txt = tracegen.to_jsonl(c5, ["host", "user", "session"], ["authfail", "request", "response", "admin", "external"],
                               [[], [], [], [], []], seed=6, style="mixed")
    extra = ('\n{"user": "a\\u00e9", "rid": 1e0, "login": true, "unauthorized": true}\n'
             '   \n{"rid": "1", "user": "a\u00e9", "login": true, "unauthorized": true, "x": {"y": [1, {"z": 2}]}}\n')
    cases = [(tracegen.LOGIN, golden), (tracegen.LOGIN, big + extra), (tracegen.SOCKET, sock_txt),
             ("\n".join(tracegen.C5_FORMULAS), c5_txt)]
    for formula, text in cases:
        prog = ltl4c.compile_batch(formula.split("\n")) if "\n" in formula else ltl4c.compile(formula)
        hk, hl = prog.encoder().encode(text)
        dk, dl = prog.device_encoder().encode(text)
        assert np.array_equal(dl.cpu().numpy(), hl), formula
        for a, b in zip(hk, dk):
            assert _same_partition(a, b.cpu().numpy().view(np.uint32)), formula
        got = prog.state(0).verify(dk, dl)
        texts = formula.split("\n")
        for f, t in enumerate(texts):
            p = oracle.Property(t)
            if len(texts) == 1:
                _assert_same(got[f], oracle.run_records(t, text), ("dev enc", t[:30]))
            else:
                want = oracle.run_offline(t, hk, _project(hl, prog.atoms, p.atoms))
                _assert_same(got[f], want, ("dev enc batch", f))
    # online: chunks through one device encoder (dictionaries persist)
    prog = ltl4c.compile(tracegen.LOGIN)
    enc = prog.device_encoder()
    st = prog.state(0, online=True)
    lines = big.splitlines(keepends=True)
    mon = oracle.RecordMonitor(oracle.Property(tracegen.LOGIN))
    for lo in range(0, len(lines), 60_000):
        chunk = "".join(lines[lo:lo + 60_000])
        k, l = enc.encode(chunk)
        got = st.verify(k, l)[0]
        mon.feed_records(chunk)
        _assert_same(got, mon.evaluate(), ("dev enc online", lo))
    with pytest.raises(ltl4c.Ltl4cError):
        enc.encode('{"user": 1, "rid": 2}\n{"user": 1 "rid": 2}\n')


@pytest.mark.parametrize("shards", [2, 4, 8])
def test_virtual_shards(env, shards):
    """SURVEY §4 T4 / §8(e) on one GPU: LTL4C_VIRTUAL_SHARDS = G runs the multi-GPU
    owner partition (hash of k0) with G logical owners, each owner's events through
    the local pipeline, the per-level histograms summed and the root rule applied
    once -- offline (K = 1, 2, 3) and online batches, against the oracle."""
    import os
    ltl4c, torch, dev = env
    os.environ["LTL4C_VIRTUAL_SHARDS"] = str(shards)
    try:
        for tr in (tracegen.login_trace(seed=51, n=400_000, users=3000, rid_events=3, p_unauth=0.05),
                   tracegen.zipf_socket_trace(seed=52, n=600_000, support=1 << 14),
                   tracegen.proxy_trace(seed=53, n=500_000, videos=3000)):
            _assert_same(_gpu_offline(env, tr.formula, tr.keys, tr.letters)[0],
                         oracle.run_offline(tr.formula, tr.keys, tr.letters), (shards, tr.meta))
        tr = tracegen.c5_trace(seed=54, n=300_000, users=2000, hosts=64, span_events=60_000)
        prog = ltl4c.compile_batch(tracegen.C5_FORMULAS)
        st = prog.state(0, online=True)
        props = [oracle.Property(t) for t in tracegen.C5_FORMULAS]
        for lo, hi in [(0, 1), (1, 70_000), (70_000, 300_000)]:
            k, l = _dev(torch, dev, [x[lo:hi] for x in tr.keys], tr.letters[lo:hi])
            got = st.verify(k, l, first_index=lo)
            for f, p in enumerate(props):
                want = oracle.run_offline(tracegen.C5_FORMULAS[f], [x[:hi] for x in tr.keys],
                                          _project(tr.letters[:hi], prog.atoms, p.atoms))
                _assert_same(got[f], want, (shards, hi, f))
        k, l = _dev(torch, dev, [np.zeros(0, np.uint32)] * 2, np.zeros(0, np.uint8))
        got = ltl4c.compile(tracegen.LOGIN).state(0).verify(k, l)[0]
        _assert_same(got, oracle.run_offline(tracegen.LOGIN, [np.zeros(0, np.uint32)] * 2, np.zeros(0, np.uint8)))
    finally:
        os.environ.pop("LTL4C_VIRTUAL_SHARDS", None)
