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
    torch.cuda.synchronize()
    print("sanitize cases done", flush=True)


if __name__ == "__main__":
    main()
