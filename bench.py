#!/usr/bin/env python
"""Benchmark of the LTL4-C verification hot path (BASELINE.json metric:
"trace events verified/sec at 1/2/4/8 B200; achieved HBM GB/s vs peak").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C]

N = 1 (default): BASELINE.json configs[2] = C3, the largest single-GPU config:
  A_{>=0.95} s : socket(s) => G (receive(s) -> F respond(s))
over a 100M-event trace whose socket ids are Zipf(1.1)-skewed over 2^20 ids (a few
huge clusters: the segmented transition-map scan).  The same line carries C2
(configs[1], 10M events, nested login property) and C4 at 125M events per GPU as
extra fields (`extra`).
N > 1: BASELINE.json configs[3] = C4, ONE 1B-event proxy-cache trace
  A v : vid(v) => E_{=0} r : req(r) => (cached(v) && external(r))
sharded over the ranks (rank r holds the contiguous slice r of the trace and
generates only that slice): ltl4c_verify routes every event to the owner of its
video (hash of k0) with NCCL over NVLink, verifies the owned subtrees and
all-reduces the per-level counts.  Strong scaling (total work
fixed); time is the max over ranks.  Without torchrun, `--gpus N` re-launches
itself under `python -m torch.distributed.run --nproc-per-node N`.

A step = one ltl4c_verify of the whole batch (all of SURVEY §8(a): epsilon +
clustering, dedup, stepping, level reduction, root verdict, result copy).  Inputs
are resident in HBM before the timed region; L2 (126 MB) is flushed between steps
by writing a 256 MiB buffer outside the timed interval (C3's input is 500 MB).
"""
from __future__ import annotations

import argparse
import json
import os
import platform
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
RESULT_BYTES = 936       # sizeof(DevOut) copied device -> host per verify
FLUSH_BYTES = 256 << 20

# name -> (workload text, total events, generator(lo, hi), algorithmic bytes per event)
CONFIGS = {
    "C1": ("C1: A_{>=0.95} s:socket(s) => G(receive(s) -> F respond(s)), 10k events, 100 sockets "
           "(BASELINE.json configs[0])", 10_000,
           lambda lo, hi: _cut(tracegen.socket_trace(seed=0), lo, hi), 5),
    "C2": ("C2: A x:user(x) => E_{<=3} r:rid(r) => (login && unauthorized), 10M-event synthetic "
           "web-server log, 100k users (BASELINE.json configs[1])", 10_000_000,
           lambda lo, hi: _cut(tracegen.login_trace(seed=0), lo, hi), 9),
    "C3": ("C3: A_{>=0.95} s:socket(s) => G(receive(s) -> F respond(s)), 100M events, socket ids "
           "Zipf(1.1) over 2^20 (BASELINE.json configs[2])", 100_000_000,
           lambda lo, hi: tracegen.zipf_socket_trace(seed=0, lo=lo, hi=hi), 5),
    "C4": ("C4 (one GPU's share): A v:vid(v) => E_{=0} r:req(r) => (cached(v) && external(r)), "
           "125M events, 10^6 videos Zipf(0.8), unique requests of 1-4 events", 125_000_000,
           lambda lo, hi: tracegen.proxy_trace(seed=0, n=125_000_000, lo=lo, hi=hi), 9),
    "C6": ("C6: A u:user(u) => F small(u), small = avg_chunksize(u) <= maximum (Dropbox fairness, P:1127-1136), "
           "10M events, 10^5 users", 10_000_000,
           lambda lo, hi: _cut(tracegen.dropbox_trace(seed=0, n=10_000_000, users=100_000), lo, hi), 5),
    "C4B": ("C4: A v:vid(v) => E_{=0} r:req(r) => (cached(v) && external(r)), 1B-event proxy-cache "
            "trace, 10^6 videos Zipf(0.8), sharded by hash(video) over the GPUs (BASELINE.json configs[3])",
            1_000_000_000,
            lambda lo, hi: tracegen.proxy_trace(seed=0, n=1_000_000_000, lo=lo, hi=hi), 9),
}


def _cut(tr, lo, hi):
    if lo == 0 and hi == tr.n:
        return tr
    return tracegen.Trace(tr.formula, [k[lo:hi].copy() for k in tr.keys], tr.letters[lo:hi].copy(), tr.meta)


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return platform.processor() or "unknown"


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


def rank_slice(n: int, world: int, rank: int):
    """rank r holds the contiguous events [r n / G, (r+1) n / G)."""
    return n * rank // world, n * (rank + 1) // world


def run_config(name, args, rank, world, local_rank, with_e2e=True, profile=True):
    """Time `args.steps` verifies of config `name` (this rank's slice) after
    `args.warmup` untimed ones; returns the measurements (max over ranks)."""
    import torch
    import paper_1411_2239_b200 as ltl4c

    text, n_total, gen, bpe = CONFIGS[name]
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    lo, hi = rank_slice(n_total, world, rank)
    t0 = time.perf_counter()
    tr = gen(lo, hi)
    gen_s = time.perf_counter() - t0
    n = tr.n
    keys = [torch.from_numpy(k.view(np.int32)).to(dev) for k in tr.keys]
    letters = torch.from_numpy(tr.letters).to(dev)
    flush = torch.empty(FLUSH_BYTES // 4, dtype=torch.int32, device=dev)
    prog = ltl4c.compile(tr.formula)
    st = prog.state(local_rank, capacity=n)
    if world > 1:
        from paper_1411_2239_b200 import dist as ldist
        ldist.join(st)
    stream = torch.cuda.current_stream(dev)
    dist = None
    if world > 1:
        import torch.distributed as dist

    def step():
        return st.verify(keys, letters, stream=stream)[0]

    for _ in range(args.warmup):
        flush.zero_()
        res = step()
    if dist is not None:
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
    stats = None
    if profile:
        # kernel-level profile (CUDA events around every library kernel on the stream it
        # is launched on; the launch sequence runs directly instead of the CUDA graph, so
        # this is a separate pass)
        st.stats_reset()
        st.profile(True)
        for i in range(args.steps):
            flush.zero_()
            step()
        torch.cuda.synchronize(dev)
        st.profile(False)
        stats = st.stats()
    if dist is not None:
        t = torch.tensor([total_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
        dist.barrier()
    out = {"n": n, "n_total": n_total, "total_ms": total_ms, "ms": ms, "stats": stats, "clocks": clk.summary(),
           "verdict": res.verdict, "launches": launches, "gen_s": gen_s, "bpe": bpe, "text": text}
    del keys, letters
    if with_e2e:
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
            if dist is not None:
                dist.barrier()
            t0 = time.perf_counter()
            r2 = st_h.verify_host(hkeys, hlet, stream=stream)[0]   # returns after the D2H result copy
            e2e_ms.append((time.perf_counter() - t0) * 1e3)
        assert r2.verdict == res.verdict
        e2e_total = float(sum(e2e_ms))
        out["e2e_serial_total_ms"] = e2e_total
        if world == 1:
            # the deployment shape of a stream of independent batches: two states on two
            # streams, stepped from two host threads, so one batch's H2D copy overlaps the
            # other's verify (every step still copies its inputs and reads its result back)
            import threading
            st_h2 = prog.state(local_rank, capacity=n)
            streams = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]
            states = [st_h, st_h2]
            for x in range(2):
                for _ in range(max(1, args.warmup)):
                    states[x].verify_host(hkeys, hlet, stream=streams[x])
            torch.cuda.synchronize(dev)
            got = [None, None]

            def worker(x):
                for _ in range(x, args.steps, 2):
                    got[x] = states[x].verify_host(hkeys, hlet, stream=streams[x])[0]

            t0 = time.perf_counter()
            ths = [threading.Thread(target=worker, args=(x,)) for x in range(2)]
            for t in ths:
                t.start()
            for t in ths:
                t.join()
            e2e_total = (time.perf_counter() - t0) * 1e3
            assert all(g is None or g.verdict == res.verdict for g in got)
            out["e2e_streams"] = 2
            del st_h2
        if dist is not None:
            t = torch.tensor([e2e_total], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_total = float(t.item())
        out["e2e_total_ms"] = e2e_total
        out["h2d"] = int(sum(k.numel() * 4 for k in hkeys) + hlet.numel())
        del st_h, hkeys, hlet
    out["tr"] = tr
    del st
    torch.cuda.empty_cache()
    return out


def roofline(r, steps, peak, peak_kind, config):
    """Dominant kernel (largest share of the profiled step): algorithmic bytes per
    launch (bytes/event x the events one launch processes) / its mean
    CUDA-event launch time."""
    ks = r["stats"]["kernels"]
    tot = sum(v["ms"] for v in ks.values())
    dom = max(ks, key=lambda k: ks[k]["ms"])
    per_launch_ms = ks[dom]["ms"] / max(1, ks[dom]["launches"])
    alg = r["bpe"] * r["n"]
    achieved = alg / (per_launch_ms / 1e3) / 1e9
    traffic = None
    try:
        # (the capture of this config's dominant kernel; null when none was taken)
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            traffic = json.load(f).get(config, {}).get(dom)
    except Exception:
        traffic = None
    return {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "peak_kind": peak_kind,
            "unit": "GB/s", "frac": achieved / peak, "traffic": traffic, "alg_bytes_per_launch": alg,
            "path_achieved": alg * steps / (r["total_ms"] / 1e3) / 1e9,
            "path_frac": alg * steps / (r["total_ms"] / 1e3) / 1e9 / peak,
            "kernel_share": {k: round(v["ms"] / max(1e-9, tot), 4) for k, v in ks.items() if v["launches"]},
            "kernel_ms_per_step": tot / steps}


def cpu_baseline(name, tr, max_events=10_000_000):
    """The oracle as it stands on the host cores, on a bounded sample (a prefix) of the
    bench trace: one thread, then every host thread (the oracle's timing mode: level-0
    subtrees partitioned by a hash of k0; identical results)."""
    import oracle
    m = min(tr.n, max_events)
    keys = [k[:m] for k in tr.keys]
    let = tr.letters[:m]
    nproc = os.cpu_count() or 1
    t0 = time.perf_counter()
    r1 = oracle.run_offline(tr.formula, keys, let)
    d1 = time.perf_counter() - t0
    t0 = time.perf_counter()
    rn = oracle.run_offline(tr.formula, keys, let, threads=nproc)
    dn = time.perf_counter() - t0
    assert r1["verdict"] == rn["verdict"] and np.array_equal(r1["hist"], rn["hist"])
    return {"value": m / dn, "unit": UNIT, "cores": nproc, "kind": "oracle",
            "cpu": _cpu_model(), "nproc": nproc,
            "single_thread": {"value": m / d1, "cores": 1, "seconds": round(d1, 2)},
            "sample": f"first {m} events of the {name} bench trace (seed 0), one pass per thread count, "
                      f"{dn:.1f} s on {nproc} threads"}


def line_for(r, args, world, peak, peak_kind, name):
    n_total = r["n_total"] if world > 1 else r["n"]
    value = n_total * args.steps / (r["total_ms"] / 1e3)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": r["total_ms"] / args.steps, "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (tracegen, seeded)",
        "config": {"workload": r["text"], "name": name, "events": n_total, "events_per_gpu": r["n"],
                   "l2": "flushed between steps (256 MiB write, untimed)",
                   "parallelism": (f"{world} GPUs, one global trace sharded by hash(k0): NCCL send/recv + "
                                   "all-reduce" if world > 1 else "1 GPU"),
                   "root_verdict": r["verdict"]},
        "gpu_launches": int(r["launches"]),
        "clocks": r["clocks"],
    }
    if r["stats"] is not None:
        line["roofline"] = roofline(r, args.steps, peak, peak_kind, name)
    if "e2e_total_ms" in r:
        line["e2e"] = {"value": n_total * args.steps / (r["e2e_total_ms"] / 1e3), "unit": UNIT,
                       "h2d_bytes_per_step": r["h2d"] * world, "d2h_bytes_per_step": RESULT_BYTES * world}
        if "e2e_serial_total_ms" in r:
            line["e2e"]["serial_value"] = n_total * args.steps / (r["e2e_serial_total_ms"] / 1e3)
        if r.get("e2e_streams"):
            line["e2e"]["note"] = ("ltl4c_verify_host on pinned host buffers, two states on two streams stepped "
                                   "from two host threads (a batch's copy overlaps the other's verify); "
                                   "serial_value: one call after the other")
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=None, choices=sorted(CONFIGS) + ["C5"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the C2 / C4 extra fields")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # honour --gpus without torchrun: one rank per GPU on this node
        import socket
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and rank == 0:
        print(f"[bench] note: --gpus {args.gpus} but WORLD_SIZE={world}; measuring {world} GPUs", file=sys.stderr)
    name = args.config or ("C3" if world == 1 else "C4B")
    if name == "C5":
        return run_c5(args)
    if args.impl == "reference":
        return run_reference(args, rank, world, name)
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    peak, peak_kind = _peaks()
    r = run_config(name, args, rank, world, local_rank)
    line = line_for(r, args, world, peak, peak_kind, name) if rank == 0 else None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(name, r["tr"])
    r = None
    if world == 1 and not args.no_extra and name == "C3" and rank == 0:
        # extra fields: C2 (configs[1]) and C4 at 125M events on this GPU
        extra = {}
        for x in ("C2", "C4"):
            rx = run_config(x, args, 0, 1, local_rank, with_e2e=False)
            lx = line_for(rx, args, 1, peak, peak_kind, x)
            extra[x] = {k: lx[k] for k in ("value", "ms_per_step", "roofline", "gpu_launches")}
            extra[x]["workload"] = rx["text"]
            extra[x]["root_verdict"] = rx["verdict"]
            rx = None
        extra["C1_sweep"] = c1_sweep(args, local_rank)
        extra["online_batch1"] = online_latency(args, local_rank)
        extra["ingest"] = ingest_rate(args, local_rank)
        line["extra"] = extra
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def c1_sweep(args, local_rank):
    """The paper's size sweep (N = 2^14 ... 2^23) of the C1 socket property:
    per size, the mean latency of one ltl4c_verify (graph replay, inputs in HBM, no
    L2 flush: these inputs are small) and N / latency."""
    import torch
    import paper_1411_2239_b200 as ltl4c
    dev = torch.device("cuda", local_rank)
    out = []
    for lg in range(14, 24):
        tr = tracegen.socket_trace(seed=0, n=1 << lg)
        keys = [torch.from_numpy(k.view(np.int32)).to(dev) for k in tr.keys]
        letters = torch.from_numpy(tr.letters).to(dev)
        st = ltl4c.compile(tr.formula).state(local_rank, capacity=tr.n)
        stream = torch.cuda.current_stream(dev)
        for _ in range(args.warmup):
            st.verify(keys, letters, stream=stream)
        torch.cuda.synchronize(dev)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(args.steps):
            res = st.verify(keys, letters, stream=stream)[0]
        b.record(stream)
        torch.cuda.synchronize(dev)
        ms = a.elapsed_time(b) / args.steps
        out.append({"n": tr.n, "ms": ms, "events_per_s": tr.n / (ms / 1e3), "root_verdict": res.verdict})
        del st, keys, letters
    return out


def ingest_rate(args, local_rank, n=2_000_000):
    """Trace ingest: C2-shaped JSON-lines records (mixed value
    spellings, noise keys) encoded on the GPU from device memory (ltl4c_dencode_jsonl)
    and, for context, by the host encoder on one core."""
    import torch
    import paper_1411_2239_b200 as ltl4c
    dev = torch.device("cuda", local_rank)
    tr = tracegen.login_trace(seed=0, n=n, users=20_000, rid_events=2)
    text = tracegen.to_jsonl(tr, ["user", "rid"], ["login", "unauthorized"], [[], []], seed=0, style="mixed")
    data = text.encode()
    d_text = torch.frombuffer(bytearray(data), dtype=torch.uint8).to(dev)
    prog = ltl4c.compile(tr.formula)
    stream = torch.cuda.current_stream(dev)
    # output buffers allocated once, outside the timed region (encode() would also count
    # the lines with torch and allocate per call)
    cap = tr.n + 1
    k_out = [torch.empty(cap, dtype=torch.int32, device=dev) for _ in range(prog.n_levels)]
    l_out = torch.empty(cap, dtype=torch.uint8, device=dev)
    ms = []
    for i in range(args.warmup + args.steps):
        enc = prog.device_encoder(local_rank, max_values=1 << 21)
        torch.cuda.synchronize(dev)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        m = enc.encode_into(d_text, k_out, l_out, stream=stream)
        b.record(stream)
        torch.cuda.synchronize(dev)
        assert m == tr.n
        if i >= args.warmup:
            ms.append(a.elapsed_time(b))
        del enc
    d_ms = sum(ms) / len(ms)
    t0 = time.perf_counter()
    prog.encoder().encode(data)
    h_s = time.perf_counter() - t0
    return {"records": tr.n, "bytes": len(data), "device_ms": d_ms, "device_records_per_s": tr.n / (d_ms / 1e3),
            "device_GB_per_s": len(data) / (d_ms / 1e3) / 1e9, "host_records_per_s_1core": tr.n / h_s,
            "note": "fresh dictionaries per call, output buffers preallocated; the call includes its own line-count sync"}


def online_latency(args, local_rank, n_events=2000):
    """Per-event verdict stream (SURVEY §8(f) NEXT-4 latency mode): the C2 property
    online, one event per ltl4c_verify (batch = 1, carried state), each result read
    back -- the latency of one event's verdict."""
    import torch
    import paper_1411_2239_b200 as ltl4c
    dev = torch.device("cuda", local_rank)
    tr = tracegen.login_trace(seed=0, n=n_events + 64, users=200)
    keys = [torch.from_numpy(k.view(np.int32)).to(dev) for k in tr.keys]
    letters = torch.from_numpy(tr.letters).to(dev)
    st = ltl4c.compile(tr.formula).state(local_rank, online=True)
    stream = torch.cuda.current_stream(dev)
    for j in range(64):
        st.verify([k[j:j + 1] for k in keys], letters[j:j + 1], stream=stream)
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    for j in range(64, 64 + n_events):
        res = st.verify([k[j:j + 1] for k in keys], letters[j:j + 1], stream=stream)[0]
    dt = time.perf_counter() - t0
    # the same stream arriving from host memory (ltl4c_verify_host: the event copied into
    # the state's staging buffers, so every call has the same layout and the launch
    # sequence replays as a CUDA graph)
    hk = [np.ascontiguousarray(k) for k in tr.keys]
    hl = np.ascontiguousarray(tr.letters)
    st2 = ltl4c.compile(tr.formula).state(local_rank, online=True)
    for j in range(64):
        st2.verify_host([k[j:j + 1] for k in hk], hl[j:j + 1], stream=stream)
    torch.cuda.synchronize(dev)
    t1 = time.perf_counter()
    for j in range(64, 64 + n_events):
        res2 = st2.verify_host([k[j:j + 1] for k in hk], hl[j:j + 1], stream=stream)[0]
    dt2 = time.perf_counter() - t1
    assert res2.verdict == res.verdict and np.array_equal(res2.hist, res.hist)
    return {"events": n_events, "us_per_event": dt2 / n_events * 1e6, "events_per_s": n_events / dt2,
            "device_slices_us_per_event": dt / n_events * 1e6, "root_verdict": res2.verdict,
            "note": "wall clock per ltl4c_verify_host call (event from host memory, verdict on the host); "
                    "device_slices: ltl4c_verify on a new device slice per event (no graph replay)"}


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


def run_reference(args, rank, world, name):
    """Reference arm (tier framing: the oracle is the reference): the oracle, as it
    stands, on the host cores -- every host thread (timing mode, level-0 hash
    partition) -- each step verifying a bounded sample (the first 10M events) of the
    same workload.  Under torchrun only rank 0 runs."""
    if rank != 0:
        return
    import oracle
    text, n_total, gen, _ = CONFIGS[name]
    m = min(n_total, 10_000_000)
    tr = gen(0, m)
    nproc = os.cpu_count() or 1
    for _ in range(args.warmup):
        oracle.run_offline(tr.formula, tr.keys, tr.letters, threads=nproc)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.run_offline(tr.formula, tr.keys, tr.letters, threads=nproc)
    dt = time.perf_counter() - t0
    value = m * args.steps / dt
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dt * 1e3 / args.steps, "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic (tracegen, seeded)",
            "config": {"workload": text, "name": name, "events": n_total, "sample_events": m},
            "impl": "reference",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": nproc, "kind": "oracle", "cpu": _cpu_model(),
                             "sample": f"first {m} events of the {name} trace per step, {nproc} host threads"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
