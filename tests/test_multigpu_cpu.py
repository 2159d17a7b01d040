"""World-size-2 gloo tests (CPU) of the multi-GPU host logic.

The library's data path needs GPUs; what is checked here is (1) the id
broadcast and slicing helpers of paper_1411_2239_b200.dist and (2) the sharding
mathematics the library relies on, with the ORACLE: every node below the root
belongs to one level-0 subtree, so routing events by any function of k0,
concatenating each owner's receipts in source-rank order, evaluating each owner
alone and summing the per-level histograms reproduces the single-process result
(root = Def. 6 rule on the summed depth-1 histogram)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle
import tracegen


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, text, q, case):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1411_2239_b200 import dist as ldist
        if case == "id":
            nid = ldist.broadcast_id(lambda: bytes(range(128)))
            q.put((rank, nid))
            return
        tr = {"login": tracegen.login_trace(seed=6, n=40_000, users=300, rid_events=3, p_unauth=0.08),
              "proxy": tracegen.proxy_trace(seed=7, n=30_000, videos=400, p_ext_cached=0.02),
              "c5": tracegen.c5_trace(seed=1, n=20_000, users=200, hosts=16, span_events=5000)}[case]
        keys, letters = tr.keys, tr.letters
        if case == "c5":
            p0 = oracle.Property(tracegen.C5_FORMULAS[0])
            text = tracegen.C5_FORMULAS[0]
            letters = (letters & 1).astype(np.uint8)   # formula 0 has the single atom authfail (bit 0)
            assert p0.atoms == ["authfail"]
        lo, hi = ldist.rank_slice(tr.n, world, rank)
        mine = [k[lo:hi] for k in keys]
        let = letters[lo:hi]
        owner = (mine[0].astype(np.uint64) * np.uint64(2654435761) >> np.uint64(7)) % np.uint64(world)
        # all-to-all of (keys, letters) per owner, preserving order
        outs = []
        for r in range(world):
            sel = (owner == r) & np.all(np.stack([k != tracegen.ABSENT for k in mine]), axis=0)
            outs.append([k[sel] for k in mine] + [let[sel]])
        got = [None] * world
        for r in range(world):
            objs = [None] * world
            dist.all_gather_object(objs, outs[r])
            if r == rank:
                got = objs
        rk = [np.concatenate([g[i] for g in got]) for i in range(len(keys))]
        rl = np.concatenate([g[-1] for g in got])
        res = oracle.run_offline(text, rk, rl)
        h = torch.from_numpy(res["hist"].astype(np.int64))
        dist.all_reduce(h)
        prop = oracle.Property(text)
        qd = prop.quantifier(0)
        root = oracle.rule(qd["kind"], qd["cmp"], qd["num"], qd["den"], h[1].tolist())
        q.put((rank, root, h.numpy()))
    finally:
        dist.destroy_process_group()


def _run(case, text=None):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, text, q, case)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


def test_broadcast_id_gloo():
    out = _run("id")
    assert all(o[1] == bytes(range(128)) for o in out)


@pytest.mark.parametrize("case,text", [("login", tracegen.LOGIN), ("proxy", tracegen.PROXY), ("c5", None)])
def test_sharded_evaluation_equals_single_process(case, text):
    out = _run(case, text)
    tr = {"login": tracegen.login_trace(seed=6, n=40_000, users=300, rid_events=3, p_unauth=0.08),
          "proxy": tracegen.proxy_trace(seed=7, n=30_000, videos=400, p_ext_cached=0.02),
          "c5": tracegen.c5_trace(seed=1, n=20_000, users=200, hosts=16, span_events=5000)}[case]
    if case == "c5":
        text = tracegen.C5_FORMULAS[0]
        want = oracle.run_offline(text, tr.keys, (tr.letters & 1).astype(np.uint8))
    else:
        want = oracle.run_offline(text, tr.keys, tr.letters)
    for rank, root, h in out:
        assert root == want["verdict"]
        assert np.array_equal(h[1:], want["hist"][1:].astype(np.int64))


def test_rank_slice_covers_trace_in_order():
    from paper_1411_2239_b200 import dist as ldist
    for n in (0, 1, 7, 100, 101):
        for world in (1, 2, 4, 8):
            sl = [ldist.rank_slice(n, world, r) for r in range(world)]
            assert sl[0][0] == 0 and sl[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(sl[:-1], sl[1:]))
