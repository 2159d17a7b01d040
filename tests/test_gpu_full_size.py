"""GPU parity at the sizes bench.py publishes (BASELINE.json configs at full size,
in the launch configuration bench.py times): the CUDA path through the C ABI
against the oracle, bit-exact on verdicts and per-level counts.  The oracle runs
in its timing mode (level-0 subtrees over every host thread; pinned identical to
the sequential run by tests/test_oracle_pins.py::test_threads_mode_identical).

Plan coverage (runtime.cu plan_batch): C2 at 12M events needs B = 19 bucket bits,
so three partition passes; C3 (100M, one level: two passes) and C4 (125M, three
passes) have more than 4096 partition tiles, so part_scan takes its multi-sweep
branch; C3/C4 heads go through the heavy (segmented map-scan) path."""
import os

import numpy as np
import pytest

import oracle
import tracegen

pytestmark = pytest.mark.gpu
NPROC = os.cpu_count() or 1


@pytest.fixture(scope="module")
def env(cuda_ok):
    import torch

    import paper_1411_2239_b200 as ltl4c
    return ltl4c, torch, torch.device("cuda:0")


def _verify(env, text, keys, letters, **state_kw):
    ltl4c, torch, dev = env
    st = ltl4c.compile(text).state(0, **state_kw)
    k = [torch.from_numpy(np.ascontiguousarray(x).view(np.int32)).to(dev) for x in keys]
    l = torch.from_numpy(np.ascontiguousarray(letters)).to(dev)
    got = st.verify(k, l)
    if not state_kw.get("online"):
        st.verify(k, l)      # second verify: the captured CUDA graph replays (what bench.py times)
        again = st.verify(k, l)
        assert again[0].verdict == got[0].verdict and np.array_equal(again[0].hist, got[0].hist)
    return got


def _same(got, want, ctx):
    assert got.verdict == want["verdict"], (ctx, got.verdict, want["verdict"])
    assert np.array_equal(got.hist, want["hist"]), (ctx, got.hist, want["hist"])
    assert got.events_bound == want["events_bound"], ctx


def test_C3_full_size_bench_trace(env):
    """BASELINE configs[2]: the 100M-event Zipf(1.1) trace bench.py times (seed 0)."""
    tr = tracegen.zipf_socket_trace(seed=0)
    assert tr.n == 100_000_000
    got = _verify(env, tr.formula, tr.keys, tr.letters)[0]
    _same(got, oracle.run_offline(tr.formula, tr.keys, tr.letters, threads=NPROC), "C3 100M")


def test_C4_full_size_bench_trace(env):
    """C4 at 125M events per GPU (bench.py's extra C4 line, seed 0): three partition
    passes, multi-sweep scan, heavy path with inner levels."""
    tr = tracegen.proxy_trace(seed=0, n=125_000_000)
    got = _verify(env, tr.formula, tr.keys, tr.letters)[0]
    _same(got, oracle.run_offline(tr.formula, tr.keys, tr.letters, threads=NPROC), "C4 125M")


@pytest.mark.parametrize("n,users", [(12_000_000, 120_000), (20_000_000, 200_000)])
def test_C2_shape_three_passes(env, n, users):
    """K = 2 above 11.2M events: B >= 19 bucket bits (three partition passes); 20M
    events also has > 4096 tiles (multi-sweep scan)."""
    tr = tracegen.login_trace(seed=5, n=n, users=users, rid_events=2, p_unauth=0.03)
    got = _verify(env, tr.formula, tr.keys, tr.letters)[0]
    _same(got, oracle.run_offline(tr.formula, tr.keys, tr.letters, threads=NPROC), n)


def test_C2_bench_trace_online_batches_equal_offline(env):
    """The C2 bench trace fed as ten 1M-event online batches: after every batch the
    carried state equals the oracle on the prefix."""
    ltl4c, torch, dev = env
    tr = tracegen.login_trace(seed=0)
    st = ltl4c.compile(tr.formula).state(0, online=True)
    k = [torch.from_numpy(x.view(np.int32)).to(dev) for x in tr.keys]
    l = torch.from_numpy(tr.letters).to(dev)
    b = 1_000_000
    for lo in range(0, tr.n, b):
        got = st.verify([x[lo:lo + b] for x in k], l[lo:lo + b], first_index=lo)[0]
        if lo // b in (0, 1, 4, 9):
            want = oracle.run_offline(tr.formula, [x[:lo + b] for x in tr.keys], tr.letters[:lo + b], threads=NPROC)
            _same(got, want, lo + b)


def _project(letters, prog_atoms, prop_atoms):
    out = np.zeros_like(letters)
    for j, a in enumerate(prop_atoms):
        out |= ((letters >> prog_atoms.index(a)) & 1) << j
    return out


def test_C5_bench_stream_1M_batches(env):
    """BASELINE configs[4] as bench.py runs it: the three C5 formulas (one product
    monitor) online over the bench's 1M-event batches; every formula's verdict and
    counts after each of the first 10 batches and at the end (12 batches)."""
    ltl4c, torch, dev = env
    batch, nb = 1_000_000, 12
    tr = tracegen.c5_trace(seed=0, n=batch * nb)
    prog = ltl4c.compile_batch(tracegen.C5_FORMULAS)
    st = prog.state(0, online=True, capacity=batch)
    k = [torch.from_numpy(x.view(np.int32)).to(dev) for x in tr.keys]
    l = torch.from_numpy(tr.letters).to(dev)
    props = [oracle.Property(t) for t in tracegen.C5_FORMULAS]
    proj = [_project(tr.letters, prog.atoms, p.atoms) for p in props]
    for i in range(nb):
        lo, hi = i * batch, (i + 1) * batch
        got = st.verify([x[lo:hi] for x in k], l[lo:hi], first_index=lo)
        if i < 10 or i == nb - 1:
            for f, text in enumerate(tracegen.C5_FORMULAS):
                want = oracle.run_offline(text, [x[:hi] for x in tr.keys], proj[f][:hi], threads=NPROC)
                _same(got[f], want, (i, f))


def test_many_medium_buckets_through_one_warp(env):
    """Per-lane leaf-verdict counters are 16-bit fields flushed on a bound: push
    8192 medium buckets (~730 events, all-new leaves) through a grid of ONE CTA
    (LTL4C_WARP_GRID=1, LTL4C_MAX_BITS=13): > 4096 buckets per warp, ~23 leaves per
    lane each, so an unbounded 16-bit field would wrap; compare with the oracle."""
    tr = tracegen.login_trace(seed=13, n=6_000_000, users=60_000, p_unauth=0.05)
    old = {k: os.environ.get(k) for k in ("LTL4C_WARP_GRID", "LTL4C_MAX_BITS")}
    os.environ["LTL4C_WARP_GRID"] = "1"
    os.environ["LTL4C_MAX_BITS"] = "13"
    try:
        got = _verify(env, tr.formula, tr.keys, tr.letters)[0]
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    _same(got, oracle.run_offline(tr.formula, tr.keys, tr.letters, threads=NPROC), "one warp")


def test_letters_with_bits_outside_the_program(env):
    """Letter bits of no atom of the program (e.g. letters encoded for a formula
    batch) are ignored, as in the oracle (a letter is read through the atoms)."""
    rng = np.random.default_rng(5)
    tr = tracegen.login_trace(seed=14, n=400_000, users=4000, p_unauth=0.05)
    noisy = (tr.letters | (rng.integers(0, 64, tr.n).astype(np.uint8) << 2)).astype(np.uint8)
    got = _verify(env, tr.formula, tr.keys, noisy)[0]
    _same(got, oracle.run_offline(tr.formula, tr.keys, tr.letters), "masked")
    got = _verify(env, tr.formula, tr.keys, noisy, online=True)[0]
    _same(got, oracle.run_offline(tr.formula, tr.keys, tr.letters), "masked online")


def test_graph_replay_after_reallocation(env):
    """A captured offline graph must not replay on buffers an ungraphed verify
    (profiling on, a larger batch) reallocated in between."""
    ltl4c, torch, dev = env
    small = tracegen.login_trace(seed=15, n=200_000, users=2000, p_unauth=0.05)
    big = tracegen.login_trace(seed=16, n=3_000_000, users=20_000, p_unauth=0.05)
    st = ltl4c.compile(small.formula).state(0)
    ks = [torch.from_numpy(x.view(np.int32)).to(dev) for x in small.keys]
    ls = torch.from_numpy(small.letters).to(dev)
    kb = [torch.from_numpy(x.view(np.int32)).to(dev) for x in big.keys]
    lb = torch.from_numpy(big.letters).to(dev)
    st.verify(ks, ls)
    st.verify(ks, ls)                       # graph captured for the small batch
    st.profile(True)
    _same(st.verify(kb, lb)[0], oracle.run_offline(big.formula, big.keys, big.letters, threads=NPROC), "big")
    st.profile(False)
    _same(st.verify(ks, ls)[0], oracle.run_offline(small.formula, small.keys, small.letters), "small again")


def test_K1_heavy_hitter_path_on_and_off(env):
    """K = 1: the heavy-hitter path (hot.cu; LTL4C_NO_HOT disables it) and the plain
    partition + heavy segmented scan give the oracle's result, on a Zipf head, on a
    single giant key, and on a trace with no key frequent enough to be hot."""
    rng = np.random.default_rng(3)
    n = 20_000_000
    cases = [tracegen.zipf_socket_trace(seed=4, n=n, support=1 << 16, s=1.3),
             tracegen.Trace(tracegen.FILES, [np.where(rng.random(n) < 0.9, 7, rng.integers(0, 1000, n)).astype(np.uint32)],
                            rng.choice(np.array([0, 1, 2, 3], np.uint8), size=n, p=[0.2, 0.7, 0.05, 0.05])),
             tracegen.zipf_socket_trace(seed=5, n=n, support=1 << 24, s=0.5)]
    for tr in cases:
        want = oracle.run_offline(tr.formula, tr.keys, tr.letters, threads=NPROC)
        for off in (False, True):
            if off:
                os.environ["LTL4C_NO_HOT"] = "1"
            try:
                got = _verify(env, tr.formula, tr.keys, tr.letters)[0]
            finally:
                os.environ.pop("LTL4C_NO_HOT", None)
            _same(got, want, (tr.formula, off))


def test_K1_one_pass_mode_and_coarse_overflow(env):
    """K = 1 batches take the one-pass mode when the sample estimates few cold keys
    (seg.cu bucket_coarse: the cold stream partitioned once, a CTA per coarse bucket);
    forced onto ~3M cold keys (LTL4C_FORCE_ONEPASS) every coarse bucket overflows its
    CTA table and goes to the heavy path on the coarse partition; unforced, that trace
    takes the two-pass mode.  All, and LTL4C_NO_COARSE, give the oracle's result."""
    rng = np.random.default_rng(11)
    n = 6_000_000
    hot = rng.random(n) < 0.5
    keys = np.where(hot, rng.integers(0, 8, n), rng.integers(1000, 1 << 31, n)).astype(np.uint32)
    letters = rng.choice(np.array([0, 1, 2, 3], np.uint8), size=n, p=[0.4, 0.3, 0.2, 0.1])
    over = tracegen.Trace(tracegen.FILES, [keys], letters)         # ~3M cold keys: every coarse bucket overflows
    fits = tracegen.zipf_socket_trace(seed=12, n=n, support=1 << 18)  # ~700 cold keys per coarse bucket
    for tr in (over, fits):
        want = oracle.run_offline(tr.formula, tr.keys, tr.letters, threads=NPROC)
        for env_var in (None, "LTL4C_NO_COARSE", "LTL4C_FORCE_ONEPASS"):
            if env_var:
                os.environ[env_var] = "1"
            try:
                got = _verify(env, tr.formula, tr.keys, tr.letters)[0]
            finally:
                if env_var:
                    os.environ.pop(env_var, None)
            _same(got, want, (tr.formula, env_var))


def test_C6_full_size_bench_trace(env):
    """C6 as bench.py --config C6 runs it: 10M events, 10^5 users (seed 0)."""
    tr = tracegen.dropbox_trace(seed=0, n=10_000_000, users=100_000)
    got = _verify(env, tr.formula, tr.keys, tr.letters)[0]
    _same(got, oracle.run_offline(tr.formula, tr.keys, tr.letters, threads=NPROC), "C6 10M")


def test_device_ingest_at_bench_size(env):
    """The records bench.py's extra.ingest encodes (2M C2-shaped records, mixed spellings):
    device encoder == host encoder up to relabelling, and the verdict equals the oracle's."""
    ltl4c, torch, dev = env
    tr = tracegen.login_trace(seed=0, n=2_000_000, users=20_000, rid_events=2)
    text = tracegen.to_jsonl(tr, ["user", "rid"], ["login", "unauthorized"], [[], []], seed=0, style="mixed")
    prog = ltl4c.compile(tr.formula)
    hk, hl = prog.encoder().encode(text)
    dk, dl = prog.device_encoder(max_values=1 << 21).encode(text)
    assert np.array_equal(dl.cpu().numpy(), hl)
    for a, b in zip(hk, dk):
        b = b.cpu().numpy().view(np.uint32)
        pairs = np.unique(np.stack([a.astype(np.int64), b.astype(np.int64)]), axis=1)
        assert np.unique(pairs[0]).shape[0] == pairs.shape[1] == np.unique(pairs[1]).shape[0]
    got = prog.state(0).verify(dk, dl)[0]
    _same(got, oracle.run_offline(tr.formula, hk, hl, threads=NPROC), "ingest 2M")
    # encode_into (what bench.py times): caller buffers, a fresh encoder -> the same events
    d_text = torch.frombuffer(bytearray(text.encode()), dtype=torch.uint8).to(dev)
    ko = [torch.empty(tr.n + 1, dtype=torch.int32, device=dev) for _ in range(2)]
    lo = torch.empty(tr.n + 1, dtype=torch.uint8, device=dev)
    m = prog.device_encoder(max_values=1 << 21).encode_into(d_text, ko, lo)
    assert m == tr.n
    assert torch.equal(lo[:m], dl)
    for a, b in zip(ko, dk):  # (dictionary ids are claimed concurrently: equal up to relabelling)
        pairs = np.unique(np.stack([a[:m].cpu().numpy().astype(np.int64), b.cpu().numpy().astype(np.int64)]), axis=1)
        assert np.unique(pairs[0]).shape[0] == pairs.shape[1] == np.unique(pairs[1]).shape[0]


def test_online_graph_replay_batches_from_host(env):
    """Online batches through ltl4c_verify_host (the state's staging buffers: the same
    layout every call, so the launch sequence is captured as a CUDA graph and replayed,
    the batch id read from device memory): batch = 1 events, then 50k-event batches
    whose leaves outgrow the carried tables (a rehash: a new layout, captured again);
    the carried result equals the oracle on every checked prefix."""
    ltl4c = env[0]
    tr = tracegen.login_trace(seed=21, n=1_400_000, users=30_000, p_unauth=0.05)
    st = ltl4c.compile(tr.formula).state(0, online=True)
    keys = [np.ascontiguousarray(k) for k in tr.keys]
    lets = np.ascontiguousarray(tr.letters)
    pos = 0
    for _ in range(300):                       # batch = 1
        got = st.verify_host([k[pos:pos + 1] for k in keys], lets[pos:pos + 1])[0]
        pos += 1
    _same(got, oracle.run_offline(tr.formula, [k[:pos] for k in keys], lets[:pos]), pos)
    b = 50_000
    checks = {2, 11, 20, 26}
    for i in range(27):                        # ~1.35M leaves: past the first table size
        got = st.verify_host([k[pos:pos + b] for k in keys], lets[pos:pos + b])[0]
        pos += b
        if i in checks:
            _same(got, oracle.run_offline(tr.formula, [k[:pos] for k in keys], lets[:pos], threads=NPROC), pos)


def test_online_graph_replays_across_reset_compact_restore(env):
    """Online streams through verify_host (graph replays) across the operations that change
    the carried state under a captured graph: reset (a new epoch), compact (new tables),
    checkpoint -> restore into the same state and into a fresh one; every result equals
    the oracle on the stream fed since the last reset."""
    ltl4c = env[0]
    tr = tracegen.login_trace(seed=23, n=60_000, users=500, p_unauth=0.05)
    keys = [np.ascontiguousarray(k) for k in tr.keys]
    lets = np.ascontiguousarray(tr.letters)
    prog = ltl4c.compile(tr.formula)
    b = 2_000

    def feed(st, lo, hi):
        got = None
        for p0 in range(lo, hi, b):
            got = st.verify_host([k[p0:p0 + b] for k in keys], lets[p0:p0 + b])[0]
        return got

    def want(lo, hi):
        return oracle.run_offline(tr.formula, [k[lo:hi] for k in keys], lets[lo:hi])

    st = prog.state(0, online=True)
    _same(feed(st, 0, 20_000), want(0, 20_000), "first 20k")
    st.reset()
    _same(feed(st, 0, 10_000), want(0, 10_000), "after reset")
    st.compact()
    _same(feed(st, 10_000, 20_000), want(0, 20_000), "after compact")
    blob = st.checkpoint()
    _same(feed(st, 20_000, 40_000), want(0, 40_000), "continued")
    st.restore(blob)
    _same(feed(st, 20_000, 30_000), want(0, 30_000), "restored in place")
    st2 = prog.state(0, online=True)
    st2.restore(blob)
    _same(feed(st2, 20_000, 60_000), want(0, 60_000), "restored into a fresh state")
