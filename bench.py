#!/usr/bin/env python
"""Benchmark of the LTL4-C verification hot path (BASELINE.json metric:
"trace events verified/sec ...; achieved HBM GB/s vs peak").

Default workload (N=1): BASELINE.json configs[1] = C2, the nested property
  A x : user(x) => E_{<=3} r : rid(r) => (login && unauthorized)
over a 10M-event synthetic web-server log with 100k users (tracegen.login_trace).
A step = one ltl4c_verify of the whole 10M-event batch (all of SURVEY §8(a):
epsilon + clustering, dedup, stepping, level reduction, root verdict, result
copy).  Inputs are resident in HBM before the timed region; L2 (126 MB) is
flushed between steps by writing a 256 MiB buffer (the input is 90 MB).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N>1 runs under torch.distributed.run, one rank per GPU, on ONE global trace of
N x 10M events (N x 100k users): rank r holds the contiguous slice r (weak
scaling: 10M events per GPU); ltl4c_verify routes every event to the owner of
its user (hash of k0) with an NCCL all-to-all over NVLink, verifies the owned
subtrees and all-reduces the per-level counts.  Rank 0 prints
one JSON line; time is the max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import tracegen  # noqa: E402

METRIC = "trace events verified/sec"
UNIT = "events/s"
WORKLOAD = ("C2: A x:user(x) => E_{<=3} r:rid(r) => (login && unauthorized), "
            "10M-event synthetic web-server log, 100k users (BASELINE.json configs[1])")
ALG_BYTES_PER_EVENT = 9  # 2 x u32 keys + u8 letter read once
RESULT_BYTES = 928       # sizeof(DevOut) copied device -> host per verify
FLUSH_BYTES = 256 << 20


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = os.path.join("/tmp", f"ltl4c_clocks_{os.getpid()}.csv")

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.2)
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        try:
            rows = [r.split(",") for r in open(self.path).read().strip().splitlines()]
            rows = [[c.strip() for c in r] for r in rows if len(r) >= 8]
        except Exception:
            return None
        if not rows:
            return None
        sm = [float(r[0]) for r in rows]
        mx = max(float(r[1]) for r in rows)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].lower().startswith("active")})
        loaded = [s for s in sm if s > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(rows)}


CONFIGS = {
    "C1": ("C1: A_{>=0.95} s:socket(s) => G(receive(s) -> F respond(s)), 10k events, 100 sockets",
           lambda r: tracegen.socket_trace(seed=r), 5),
    "C2": (WORKLOAD, lambda r: tracegen.login_trace(seed=r), 9),
    "C3": ("C3: socket formula, 100M events, keys Zipf(1.1) over 2^20 ids",
           lambda r: tracegen.zipf_socket_trace(seed=r), 5),
    "C4": ("C4 (single-GPU slice): A v:vid(v) => E_{=0} r:req(r) => (cached(v) && external(r)), "
           "125M events, 10^6 videos Zipf(0.8)",
           lambda r: tracegen.proxy_trace(seed=r, n=125_000_000), 9),
}
CONFIG = "C2"


def make_trace(rank: int):
    return CONFIGS[CONFIG][1](rank)


def run_ours(args, rank, world, local_rank):
    import torch
    import paper_1411_2239_b200 as ltl4c

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    if world > 1:
        # one global trace, rank r holds slice r (same seed on every rank)
        from paper_1411_2239_b200 import dist as ldist
        full = tracegen.login_trace(seed=0, n=10_000_000 * world, users=100_000 * world) if CONFIG == "C2" \
            else make_trace(0)
        lo, hi = ldist.rank_slice(full.n, world, rank)
        tr = tracegen.Trace(full.formula, [k[lo:hi].copy() for k in full.keys], full.letters[lo:hi].copy(), full.meta)
        del full
    else:
        tr = make_trace(rank)
    n = tr.n
    keys = [torch.from_numpy(k.view(np.int32)).to(dev) for k in tr.keys]
    letters = torch.from_numpy(tr.letters).to(dev)
    flush = torch.empty(FLUSH_BYTES // 4, dtype=torch.int32, device=dev)
    prog = ltl4c.compile(tr.formula)
    st = prog.state(local_rank, capacity=n)
    if world > 1:
        ldist.join(st)
    stream = torch.cuda.current_stream(dev)

    def step():
        return st.verify(keys, letters, stream=stream)[0]

    for _ in range(args.warmup):
        flush.zero_()
        res = step()
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize(dev)
    st.stats_reset()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with Clocks(local_rank) as clk:
        for i in range(args.steps):
            flush.zero_()                 # L2 flush, outside the timed interval
            ev[i][0].record(stream)
            res = step()
            ev[i][1].record(stream)
        torch.cuda.synchronize(dev)
    ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = float(sum(ms))
    launches = st.stats()["launches"]
    # kernel-level profile (CUDA events around every library kernel; this runs the
    # launch sequence directly instead of the CUDA graph, so it is a separate pass)
    st.stats_reset()
    st.profile(True)
    for i in range(args.steps):
        flush.zero_()
        step()
    torch.cuda.synchronize(dev)
    st.profile(False)
    stats = st.stats()
    stats["launches"] = launches
    if dist is not None:
        t = torch.tensor([total_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
        dist.barrier()
    # e2e: the same call with HOST (pinned) buffers, H2D copies inside the timed region
    hkeys = [torch.from_numpy(k.view(np.int32)).pin_memory() for k in tr.keys]
    hlet = torch.from_numpy(tr.letters).pin_memory()
    st_h = prog.state(local_rank, capacity=n)
    if world > 1:
        ldist.join(st_h)
    for _ in range(max(1, args.warmup)):
        st_h.verify_host(hkeys, hlet, stream=stream)
    torch.cuda.synchronize(dev)
    e2e_ms = []
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        r2 = st_h.verify_host(hkeys, hlet, stream=stream)[0]   # returns after the D2H result copy
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
    assert r2.verdict == res.verdict
    e2e_total = float(sum(e2e_ms))
    if dist is not None:
        t = torch.tensor([e2e_total], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_total = float(t.item())
    return {"n": n, "total_ms": total_ms, "ms": ms, "stats": stats, "clocks": clk.summary(),
            "verdict": res.verdict, "e2e_total_ms": e2e_total, "tr": tr,
            "h2d": int(sum(k.numel() * 4 for k in hkeys) + hlet.numel())}


def cpu_baseline(tr, max_s=30.0):
    """The oracle as it stands, single-threaded, on the bench trace (or a prefix)."""
    import oracle
    n = tr.n
    t0 = time.perf_counter()
    oracle.run_offline(tr.formula, tr.keys, tr.letters)
    dt = time.perf_counter() - t0
    return {"value": n / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"whole bench trace ({n} events, seed 0), one pass, {dt:.1f} s"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2", choices=sorted(CONFIGS) + ["C5"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    global CONFIG, WORKLOAD, ALG_BYTES_PER_EVENT
    if args.config == "C5":
        return run_c5(args)
    CONFIG = args.config
    WORKLOAD = CONFIGS[CONFIG][0]
    ALG_BYTES_PER_EVENT = CONFIGS[CONFIG][2]
    args.warmup = max(3, args.warmup)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    r = run_ours(args, rank, world, local_rank)
    if rank == 0:
        peak, peak_kind = _peaks()
        n_total = r["n"] * world
        value = n_total * args.steps / (r["total_ms"] / 1e3)
        ks = r["stats"]["kernels"]
        dom = max(ks, key=lambda k: ks[k]["ms"])
        per_launch_ms = ks[dom]["ms"] / max(1, ks[dom]["launches"])
        kernel_ms_step = sum(v["ms"] for v in ks.values()) / args.steps
        alg_bytes = ALG_BYTES_PER_EVENT * r["n"]
        achieved = alg_bytes / (per_launch_ms / 1e3) / 1e9
        traffic = None
        try:
            with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
                traffic = json.load(f).get(dom)
        except Exception:
            traffic = None
        shares = {k: round(v["ms"] / max(1e-9, sum(x["ms"] for x in ks.values())), 4)
                  for k, v in ks.items() if v["launches"]}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": r["total_ms"] / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic (tracegen, seeded)",
            "config": {"workload": WORKLOAD, "events_per_gpu": r["n"], "name": CONFIG,
                       "l2": "flushed between steps (256 MiB write, untimed)",
                       "parallelism": (f"{world} GPUs, one global trace sharded by hash(k0), NCCL all-to-all + "
                                       "all-reduce" if world > 1 else "1 GPU"),
                       "root_verdict": r["verdict"]},
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak,
                         "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic, "alg_bytes_per_launch": alg_bytes,
                         "path_achieved": alg_bytes * args.steps / (r["total_ms"] / 1e3) / 1e9,
                         "kernel_share": shares, "kernel_ms_per_step": kernel_ms_step},
            "e2e": {"value": n_total * args.steps / (r["e2e_total_ms"] / 1e3), "unit": UNIT,
                    "h2d_bytes_per_step": r["h2d"], "d2h_bytes_per_step": RESULT_BYTES},
            "gpu_launches": int(r["stats"]["launches"]),
            "clocks": r["clocks"],
        }
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(r["tr"])
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def run_c5(args):
    """C5: three C5 formulas (one product monitor) in online mode over 1M-event
    batches with carried state; value = events/s over the timed batches."""
    import torch
    import paper_1411_2239_b200 as ltl4c
    dev = torch.device("cuda", 0)
    batch = 1_000_000
    nb = args.warmup + args.steps
    tr = tracegen.c5_trace(seed=0, n=batch * nb)
    keys = [torch.from_numpy(k.view(np.int32)).to(dev) for k in tr.keys]
    letters = torch.from_numpy(tr.letters).to(dev)
    st = ltl4c.compile_batch(tracegen.C5_FORMULAS).state(0, online=True, capacity=batch)
    stream = torch.cuda.current_stream(dev)
    for i in range(args.warmup):
        st.verify([k[i * batch:(i + 1) * batch] for k in keys], letters[i * batch:(i + 1) * batch], stream=stream)
    torch.cuda.synchronize(dev)
    st.stats_reset()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # a stream of batches: each enqueued at once (ltl4c_verify_async), its result read
    # four batches later, so host preparation overlaps the GPU work of earlier batches
    a.record(stream)
    tickets = []
    for i in range(args.warmup, nb):
        tickets.append(st.verify_async([k[i * batch:(i + 1) * batch] for k in keys],
                                       letters[i * batch:(i + 1) * batch], stream=stream))
        if len(tickets) > 4:
            res = st.result(tickets.pop(0))
    for t in tickets:
        res = st.result(t)
    b.record(stream)
    torch.cuda.synchronize(dev)
    ms = a.elapsed_time(b)
    launches = st.stats()["launches"]
    # kernel-level profile: the same batches on a fresh state, every kernel bracketed by events
    sp = ltl4c.compile_batch(tracegen.C5_FORMULAS).state(0, online=True, capacity=batch)
    sp.profile(True)
    for i in range(nb):
        sp.verify([k[i * batch:(i + 1) * batch] for k in keys], letters[i * batch:(i + 1) * batch], stream=stream)
    torch.cuda.synchronize(dev)
    stats = sp.stats()
    stats["launches"] = launches
    line = {"metric": METRIC, "value": batch * args.steps / (ms / 1e3), "unit": UNIT, "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic (tracegen, seeded)",
            "config": {"workload": "C5: 3 three-level formulas, online, 1M-event batches, carried state, "
                                   "pipelined (results read 4 batches behind)",
                       "name": "C5", "verdicts": [r.verdict for r in res]},
            "kernels": {k: v for k, v in stats["kernels"].items() if v["launches"]},
            "gpu_launches": stats["launches"]}
    print(json.dumps(line), flush=True)


def run_reference(args, rank, world):
    """Reference arm: the oracle (oracle/), as it stands, on the host cores; each
    step verifies a bounded 1M-event sample (prefix) of the same C2 workload."""
    if rank != 0:
        return
    import oracle
    tr = make_trace(0)
    m = 1_000_000
    keys = [k[:m] for k in tr.keys]
    letters = tr.letters[:m]
    for _ in range(args.warmup):
        oracle.run_offline(tr.formula, keys, letters)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.run_offline(tr.formula, keys, letters)
    dt = time.perf_counter() - t0
    value = m * args.steps / dt
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dt * 1e3 / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic (tracegen, seeded)",
            "config": {"workload": WORKLOAD, "events_per_gpu": tr.n, "users": 100_000},
            "impl": "reference",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": f"first {m} events of the C2 trace per step"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
