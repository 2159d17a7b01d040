#!/usr/bin/env python
"""Small cases that reach every kernel of the path (partition, bucket_warp,
bucket_warp_big, bucket_fast, heavy path, online leaf/nodes, async ring), each
checked bit-exactly against the oracle.  Run under compute-sanitizer on a GPU box
(scripts/sanitize.sh); sizes are small because the tools slow kernels ~100x."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
import paper_1411_2239_b200 as ltl4c  # noqa: E402

dev = torch.device("cuda:0")
FORMULAS = {
    1: "forall[>=0.5] x0 : k0(x0) => G (a -> F b)",
    2: "forall x0 : k0(x0) => exists[<=3] x1 : k1(x1) => (a U b)",
    3: "exists[>=2] x0 : k0(x0) => forall[>0.25] x1 : k1(x1) => exists x2 : k2(x2) => F (a && X c)",
}


def trace(seed, levels, n, atoms, cards, zipf):
    g = np.random.default_rng(seed)
    keys = []
    for lvl in range(levels):
        if zipf:
            k = (g.zipf(1.3, size=n) % cards[lvl]).astype(np.uint32)
        else:
            k = g.integers(0, cards[lvl], size=n).astype(np.uint32)
        k = ((k * 2654435761 + lvl) & 0xFFFFFFFE).astype(np.uint32)
        k[g.random(n) < 0.01] = 0xFFFFFFFF
        keys.append(k)
    return keys, g.integers(0, 1 << atoms, size=n).astype(np.uint8)


def project(letters, prog_atoms, prop_atoms):
    out = np.zeros_like(letters)
    for j, a in enumerate(prop_atoms):
        out |= ((letters >> prog_atoms.index(a)) & 1) << j
    return out


def check(got, want, tag):
    ok = got.verdict == want["verdict"] and np.array_equal(got.hist, want["hist"])
    print(("ok      " if ok else "MISMATCH"), tag, flush=True)
    if not ok:
        sys.exit(1)


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 40_000
    for levels, text in FORMULAS.items():
        prog = ltl4c.compile(text)
        for bits in (None, "4", "7"):  # default plan, then forced spills / heavy buckets
            if bits is None:
                os.environ.pop("LTL4C_MAX_BITS", None)
            else:
                os.environ["LTL4C_MAX_BITS"] = bits
            for zipf in (False, True):
                keys, letters = trace(levels * 10 + (zipf and 1), levels, n, len(prog.atoms), [50, 300, 5000], zipf)
                want = oracle.run_offline(text, keys, project(letters, prog.atoms, oracle.Property(text).atoms))
                st = prog.state(0)
                got = st.verify([torch.from_numpy(x.view(np.int32)).to(dev) for x in keys],
                                torch.from_numpy(letters).to(dev))[0]
                check(got, want, f"offline K={levels} max_bits={bits} zipf={zipf}")
        os.environ.pop("LTL4C_MAX_BITS", None)
        # online: carried state over uneven batches, then the async ring
        keys, letters = trace(levels * 10 + 5, levels, n, len(prog.atoms), [50, 300, 5000], True)
        want = oracle.run_offline(text, keys, project(letters, prog.atoms, oracle.Property(text).atoms))
        cuts = [0, 7, n // 3, n // 3 + 1, n - 100, n]
        for mode in ("sync", "async"):
            st = prog.state(0, online=True)
            tickets = []
            for lo, hi in zip(cuts[:-1], cuts[1:]):
                k = [torch.from_numpy(x[lo:hi].view(np.int32)).to(dev) for x in keys]
                l = torch.from_numpy(letters[lo:hi]).to(dev)
                if mode == "async":
                    tickets.append(st.verify_async(k, l, first_index=lo))
                else:
                    got = st.verify(k, l, first_index=lo)[0]
            if mode == "async":
                for t in tickets:
                    got = st.result(t)[0]
            check(got, want, f"online K={levels} {mode}")
    # K = 1 modes (hot.cu / seg.cu): dense + one pass (default), two passes + warp units,
    # forced one pass over many cold keys (coarse overflow -> heavy), no hot path
    text = FORMULAS[1]
    prog = ltl4c.compile(text)
    m = max(n, 200_000)
    g = np.random.default_rng(77)
    hot = g.random(m) < 0.6
    k1 = np.where(hot, g.integers(0, 6, m), g.integers(100, 1 << 30, m) % 60_000).astype(np.uint32)
    k1 = ((k1 * 2654435761) & 0xFFFFFFFE).astype(np.uint32)
    l1 = g.integers(0, 1 << len(prog.atoms), size=m).astype(np.uint8)
    want = oracle.run_offline(text, [k1], project(l1, prog.atoms, oracle.Property(text).atoms))
    for knob in (None, "LTL4C_NO_COARSE", "LTL4C_FORCE_ONEPASS", "LTL4C_NO_HOT"):
        if knob:
            os.environ[knob] = "1"
        st = prog.state(0)
        if knob:
            os.environ.pop(knob)
        got = st.verify([torch.from_numpy(k1.view(np.int32)).to(dev)], torch.from_numpy(l1).to(dev))[0]
        check(got, want, f"K=1 modes knob={knob}")
    # device encoder (ingest.cu), checkpoint / restore, node dump
    import tracegen
    tr = tracegen.login_trace(seed=3, n=20_000, users=300, rid_events=2, p_unauth=0.05)
    txt = tracegen.to_jsonl(tr, ["user", "rid"], ["login", "unauthorized"], [[], []], seed=1, style="mixed")
    lp = ltl4c.compile(tracegen.LOGIN)
    dk, dl = lp.device_encoder(max_values=1 << 16).encode(txt)
    check(lp.state(0).verify(dk, dl)[0], oracle.run_records(tracegen.LOGIN, txt), "device encoder")
    st = lp.state(0, online=True)
    st.verify([x[:9000] for x in dk], dl[:9000])
    blob = st.checkpoint()
    st2 = lp.state(0, online=True)
    st2.restore(blob)
    got = st2.verify([x[9000:] for x in dk], dl[9000:])[0]
    check(got, oracle.run_records(tracegen.LOGIN, txt), "checkpoint / restore")
    for level in (1, 2):
        kk, vv = st2.nodes(level)
        assert int(vv.shape[0]) == int(got.hist[level].sum())
    print("ok       node dump", flush=True)
    torch.cuda.synchronize()
    print("sanitize cases done", flush=True)


if __name__ == "__main__":
    main()
