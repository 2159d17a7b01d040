#!/usr/bin/env python
"""GPU parity fuzzing: random workload shapes (levels, key cardinalities, skew,
repeated leaves, batch splits, formula batches) through the C ABI, every result
compared bit-exactly with the oracle.  Developer tool (the test suite holds the
fixed cases); run on a GPU box:  python scripts/fuzz_gpu.py [seconds] [seed]"""
import os
import random
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import oracle  # noqa: E402
import paper_1411_2239_b200 as ltl4c  # noqa: E402
import torch  # noqa: E402

dev = torch.device("cuda:0")
BODIES = ["F a", "G (a -> F b)", "a U b", "(a && b)", "X !a", "G a || (b U c)", "F (a && X c)", "G !c", "a"]
OPS = ["<", "<=", ">", ">=", "="]


def formula(rng, levels):
    prefix = ""
    for i in range(levels):
        if rng.random() < 0.5:
            prefix += f"forall[{rng.choice(OPS)}{rng.choice(['0', '0.1', '0.5', '0.95', '1'])}] x{i} : k{i}(x{i}) => "
        else:
            prefix += f"exists[{rng.choice(OPS)}{rng.randint(0, 4)}] x{i} : k{i}(x{i}) => "
    return prefix + rng.choice(BODIES)


def trace(rng, levels, n, atoms):
    g = np.random.default_rng(rng.randrange(1 << 30))
    keys = []
    for lvl in range(levels):
        card = rng.choice([2, 7, 100, 5000, 200_000])
        if rng.random() < 0.4:  # Zipf-skewed key
            k = (g.zipf(rng.choice([1.1, 1.5, 2.0]), size=n) % card).astype(np.uint32)
        else:
            k = g.integers(0, card, size=n).astype(np.uint32)
        k = (k * 2654435761 + lvl) & 0xFFFFFFFE  # arbitrary ids, never 0xFFFFFFFF
        k = k.astype(np.uint32)
        k[g.random(n) < rng.choice([0.0, 0.01, 0.2])] = 0xFFFFFFFF
        keys.append(k)
    letters = g.integers(0, 1 << atoms, size=n).astype(np.uint8)
    return keys, letters


def project(letters, prog_atoms, prop_atoms):
    out = np.zeros_like(letters)
    for j, a in enumerate(prop_atoms):
        out |= ((letters >> prog_atoms.index(a)) & 1) << j
    return out


def main():
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
    rng = random.Random(int(sys.argv[2]) if len(sys.argv) > 2 else 1411)
    t0, cases = time.time(), 0
    while time.time() - t0 < budget:
        levels = rng.randint(1, 3)
        nform = rng.choice([1, 1, 1, 2])
        texts = [formula(rng, levels) for _ in range(nform)]
        try:
            prog = ltl4c.compile_batch(texts) if nform > 1 else ltl4c.compile(texts[0])
        except ltl4c.Ltl4cError:
            continue  # product over the budget
        n = rng.choice([1, 50, 3000, 40_000, 300_000, 1_500_000, 1_500_000, 6_000_000])
        keys, letters = trace(rng, levels, n, len(prog.atoms))
        want = [oracle.run_offline(t, keys, project(letters, prog.atoms, oracle.Property(t).atoms)) for t in texts]
        online = rng.random() < 0.4
        pipelined = online and rng.random() < 0.5  # ltl4c_verify_async, results read with a lag
        # K = 1 mode knobs (read at state creation): forced one-pass / two-pass / no hot path
        knob = rng.choice([None, None, "LTL4C_FORCE_ONEPASS", "LTL4C_NO_COARSE", "LTL4C_NO_HOT"])
        if knob:
            os.environ[knob] = "1"
        st = prog.state(0, online=online)
        if knob:
            os.environ.pop(knob)
        if online:
            cuts = sorted({0, n, *[rng.randint(0, n) for _ in range(rng.randint(0, 12))]})
        else:
            cuts = [0, n]
        tickets = []
        for lo, hi in zip(cuts[:-1], cuts[1:]):
            k = [torch.from_numpy(x[lo:hi].view(np.int32)).to(dev) for x in keys]
            l = torch.from_numpy(letters[lo:hi]).to(dev)
            if pipelined:
                tickets.append(st.verify_async(k, l, first_index=lo))
                if len(tickets) > 3:
                    st.result(tickets.pop(0))
            else:
                got = st.verify(k, l, first_index=lo if online else None)
        for t in tickets:
            got = st.result(t)
        for f, w in enumerate(want):
            ok = got[f].verdict == w["verdict"] and np.array_equal(got[f].hist, w["hist"])
            if not ok:
                print("MISMATCH", texts[f], n, levels, online, pipelined, knob, cuts, got[f].verdict, w["verdict"],
                      got[f].hist.tolist(), w["hist"].tolist(), flush=True)
                sys.exit(1)
        cases += 1
    print(f"fuzz ok: {cases} cases in {time.time() - t0:.0f} s", flush=True)


if __name__ == "__main__":
    main()
