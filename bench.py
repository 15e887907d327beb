"""Benchmark of the k-hop retrieval hot path (BASELINE.json configs[1], "C2").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one batched retrieval of 1,024 uniform random seeds, k=3 hops,
FRONTIER semantics (the reference default, incidence.py:323), no relation
filter, paths off, over the 407K-entity / 3.4M-triple synthetic UMLS-shaped
graph (workloads.c2_graph).  The step returns every seed's sorted frontier
at hops 1, 2 and 3 (so one k=3 step also yields the k=1 and k=2 answers) and
its per-hop edge counts.  ``value`` = seeds/s with the graph and seeds
already resident in HBM; ``e2e`` = the same through the public API from
pinned host seeds to host-resident results.

Multi-GPU (torchrun): queries are independent, so each rank runs its own
seed batches on a replica of the graph (no data-path collective, weak
scaling); value = total seeds over all ranks / max rank time.

``--impl reference``: the reference algorithm on the host CPU (the oracle
port of triplehop's numpy path, oracle/khop_oracle.py) over a process pool
of every host core, on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

# every kernel is loaded when the library loads, not on its first launch
# inside a timed region (lazy module loading stalled first waves by ms)
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import workloads  # noqa: E402

METRIC = "k-hop seeds/s at k=3 (C2 1024-seed batches; edges/s, k=1/2 and HBM GB/s in extra keys)"
K_HOPS = 3
BATCH = 1024


# ----------------------------------------------------------------- helpers

def load_traffic(group: str, cfg: str = "c2") -> dict:
    """DRAM bytes per step (C2: one k=3 batch; C4: one k=3 wave) of a kernel
    group from the latest committed ncu capture (profiles/r*_<cfg>_traffic.json,
    written by tools/ncu_traffic.py from `ncu --set full`)."""
    files = sorted((ROOT / "profiles").glob(f"r*_{cfg}_traffic.json"))
    if not files:
        return {}
    d = json.loads(files[-1].read_text())
    if group not in d:
        return {}
    return {"bytes": d[group]["bytes"], "ncu_us": d[group].get("us"),
            "source": f"{files[-1].name} (ncu --set full, one {'step' if cfg == 'c2' else 'k=3 wave'})"}


def pull_alg_bytes(n_items: int, n_in_edges: int, W: int, lists: list, modes: list, sem_frontier=True):
    """Algorithmic bytes of the pull hops of a wave (SURVEY 8d restated for
    the dense direction): per pull hop h, the static schedule (12 B per item),
    every in-edge source (4 B), each frontier row once (4W B) and each newly
    reached row's next-layer write (4W B; + its visited row, 4W B, except on
    FRONTIER's last hop)."""
    k = len(lists) - 1
    b = 0
    for h in range(1, k + 1):
        if modes[h]:
            rows_out = lists[h] * (1 if (sem_frontier and h == k) else 2)
            b += 12 * n_items + 4 * n_in_edges + 4 * W * lists[h - 1] + 4 * W * rows_out
    return b


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def load_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured"}
    return {"hbm_gbs": 6650.0, "source": "fallback"}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.lines: list[str] = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (FileNotFoundError, OSError):
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()
        # nvidia-smi's start-up (NVML init) stalls CUDA calls of this process
        # for tens of ms; let it finish before the timed region (a host-driven
        # partitioned wave measured 30 ms instead of 2.6 ms otherwise)
        t0 = time.perf_counter()
        while not self.lines and time.perf_counter() - t0 < 2.0:
            time.sleep(0.01)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if _one_device():
        local = 0
    return world, rank, local


def _one_device() -> bool:
    """TH_BENCH_ONE_DEVICE=1: every rank on cuda:0 with gloo collectives -- a
    check of the multi-rank code path on a one-GPU box, never a measurement
    (NCCL refuses two ranks on one device)."""
    return os.environ.get("TH_BENCH_ONE_DEVICE") == "1"


def _init_dist(dev, rank=None, world=None):
    import torch.distributed as dist

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    kw = {} if rank is None else {"rank": rank, "world_size": world}
    if _one_device():
        dist.init_process_group("gloo", **kw)
    else:
        dist.init_process_group("nccl", device_id=dev, **kw)


def _all_reduce(t, op):
    """In-place all-reduce of a device tensor (through the host under gloo)."""
    import torch.distributed as dist

    if _one_device():
        h = t.cpu()
        dist.all_reduce(h, op=op)
        t.copy_(h)
    else:
        dist.all_reduce(t, op=op)


# --------------------------------------------------------------- CPU side

_G = None  # oracle graph shared with forked workers


def _cpu_worker(args):
    from oracle import khop_oracle as orc

    seeds, k = args
    t0 = time.perf_counter()
    edges = 0
    for s in seeds:
        tr = orc.hop_trace(_G, [int(s)], k, orc.FRONTIER)
        edges += sum(int(a.size) for _, a in tr)
    return len(seeds), edges, time.perf_counter() - t0


def cpu_pool(cores: int):
    """A fork pool of `cores` workers sharing the oracle graph copy-on-write;
    created once, outside every timed region."""
    import multiprocessing as mp

    pool = mp.get_context("fork").Pool(cores)
    pool.map(_cpu_noop, range(cores))  # workers are up before any timing
    return pool


def _cpu_noop(_):
    return 0


def cpu_run(pool, seeds: np.ndarray, k: int, budget_s: float):
    """Oracle k_hop per seed over the pool; stops after ~budget_s."""
    chunk = 4
    done = edges = 0
    t0 = time.perf_counter()
    jobs = [(seeds[i : i + chunk], k) for i in range(0, seeds.size, chunk)]
    it = pool.imap(_cpu_worker, jobs)
    for n, e, _ in it:
        done += n
        edges += e
        if time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    return done, edges, dt


def build_cpu_graph(s, r, o, E, R):
    global _G
    from oracle import khop_oracle as orc

    _G = orc.build_csr(s, r, o, E, R)
    return _G


def run_reference(args, world, rank):
    if rank != 0:
        return
    s, r, o, E, R = workloads.c2_graph()
    build_cpu_graph(s, r, o, E, R)
    cores = os.cpu_count() or 1
    batches = workloads.seed_batches(E, BATCH, 1, seed=100)
    per_step = int(args.ref_step_seeds)
    times, total_seeds, total_edges = [], 0, 0
    pool = cpu_pool(cores)
    for i in range(args.warmup + args.steps):
        sl = batches[0][(i * per_step) % BATCH : (i * per_step) % BATCH + per_step]
        n, e, dt = cpu_run(pool, sl, K_HOPS, 1e9)
        if i >= args.warmup:
            times.append(dt)
            total_seeds += n
            total_edges += e
    pool.terminate()
    t = sum(times)
    value = total_seeds / t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "seeds/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic",
        "config": {"workload": "C2: 407K entities, 3.4M triples, 400 relations, hub-to-hub Zipf 1.2; "
                               f"k={K_HOPS} FRONTIER, uniform seeds", "batch": BATCH,
                   "step_sample_seeds": per_step},
        "edges_per_s": total_edges / t,
        "cpu_baseline": {"value": value, "unit": "seeds/s", "cores": cores, "kind": "port",
                         "cpu_model": cpu_model(),
                         "sample": f"{per_step} seeds of the first C2 batch per step, "
                                   "oracle/khop_oracle.hop_trace per seed, persistent fork pool"},
        "e2e": {"value": value, "unit": "seeds/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------- GPU side

def _timed(stream, fn):
    """Device milliseconds of fn() on `stream` (CUDA events, synchronised)."""
    import torch

    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(stream)
    out = fn()
    b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b), out


def _profiled(ret, steps):
    """Per-kernel-group device ms over a second, profiled pass of `steps`
    (the timed pass runs without the event pairs; the profiled shape is
    captured anew by two untimed runs first)."""
    ret.set_profiling(True)
    for fn in steps[:2]:
        fn()
    ret.profile()
    for fn in steps:
        fn()
    prof = ret.profile()
    ret.set_profiling(False)
    return prof


def run_c3_leg(th, g, s, E, R, stream, peaks):
    """BASELINE configs[2]: relation-constrained k=2 with capped paths on the
    C2 graph; 2,048 uniform + 2,048 top-1% hub seeds, per-seed 32-of-400 masks."""
    import torch

    from paper_2604_18913_b200.retriever import _relation_masks

    seeds, rel_ids = workloads.c3_queries(s, E, R)
    B = seeds.size
    words = _relation_masks(list(rel_ids), B, R)
    dev = g.device
    d_seeds = torch.from_numpy(seeds).to(dev)
    d_masks = torch.from_numpy(words.view(np.int32)).to(dev)
    offs = torch.arange(B + 1, dtype=torch.int32, device=dev)
    ret = th.Retriever(g, stream)

    def step():
        return ret.run(offs, d_seeds, 2, "frontier", d_masks, paths=True, max_paths=10_000,
                       singleton=True, copy=False)

    step()
    step()  # eager run, then the graph capture of this shape
    reps = 3
    times, res = [], None
    for _ in range(reps):
        ms, res = _timed(stream, step)
        times.append(ms)
    prof = _profiled(ret, [step] * reps)
    t = sum(times) / reps
    paths = int(res.path_count.sum().item())
    edges = int(res.edges.sum().item())
    # e2e: host seed/relation lists in, host frontiers + path tids out
    e2e = []
    pinned = {}
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rr = ret.retrieve(seeds, 2, relation_filter=list(rel_ids), paths=True, max_paths=10_000,
                          copy=False)
        d2h = 0
        for name in ("frontier_off", "frontier_len", "frontier_ids", "edges", "path_off", "path_count",
                     "path_tids", "path_truncated"):
            dv = getattr(rr, name)
            buf = pinned.get(name)
            if buf is None or buf.numel() < dv.numel():
                buf = torch.empty(int(dv.numel() * 1.25) + 16, dtype=dv.dtype).pin_memory()
                pinned[name] = buf
            buf[: dv.numel()].copy_(dv.reshape(-1), non_blocking=True)
            d2h += dv.numel() * dv.element_size()
        torch.cuda.synchronize()
        e2e.append(time.perf_counter() - t0)
    return {"workload": "C3 (BASELINE configs[2]): C2 graph, 2,048 uniform + 2,048 top-1% hub seeds, "
                        "per-seed random 32-of-400 relation masks, k=2 FRONTIER, full path "
                        "reconstruction capped at 10,000 paths per seed",
            "seeds_per_s": B / (t / 1e3), "ms_per_batch": t, "paths_per_s": paths / (t / 1e3),
            "paths": paths, "truncated_seeds": int(res.path_truncated.sum().item()),
            "edges_per_s": edges / (t / 1e3),
            "kernel_ms_per_batch": {c: v[0] / reps for c, v in prof.items() if v[0]},
            "e2e": {"value": B / statistics.median(e2e), "unit": "seeds/s",
                    "h2d_bytes_per_step": int(seeds.nbytes + words.nbytes), "d2h_bytes_per_step": d2h}}


def run_c4_leg(th, stream, peaks, n_batches=8, cols=None):
    """BASELINE configs[3] on one GPU: 54.4M entities / 86.5M triples, 8,192
    uniform seeds as 8 waves of 1,024, k=2 and k=3, FRONTIER, frontiers
    materialised per wave (the state and results of a wave are far above L2)."""
    import torch

    t0 = time.perf_counter()
    s, r, o, E, R = cols if cols is not None else workloads.c4_graph()
    gen_s = time.perf_counter() - t0
    stats = workloads.graph_stats(s, o, E)
    n_items = int(((np.bincount(o, minlength=E) + 31) // 32).sum())  # static pull items
    g = th.build_incidence((s, r, o), E, R)
    del s, r, o, cols
    ret = th.Retriever(g, stream)
    batches = torch.from_numpy(workloads.seed_batches(E, BATCH, n_batches, seed=400)).to(g.device)
    offs = torch.arange(BATCH + 1, dtype=torch.int32, device=g.device)
    out = {"workload": "C4 (BASELINE configs[3]) on 1 GPU: 54.4M entities, 86.5M triples, 1,000 "
                       "relations, power law P(w>=x)~x^-1.3 with a shared hub core, 1% isolated; "
                       f"{n_batches * BATCH} uniform seeds in waves of {BATCH}, FRONTIER, no filter",
           "graph": stats, "gen_s": gen_s}
    peaks_leg = peaks
    for k in (2, 3):
        step = lambda i: ret.run(offs, batches[i], k, "frontier", None, singleton=True,  # noqa: E731
                                 copy=False)
        for i in range(n_batches):  # warm-up: every batch once sizes the result buffers
            step(i)
        step(0)  # (stable shape: recorded, then captured as a CUDA graph)
        step(1)
        tot_ms, seeds, edges, ids, lists, pbytes = 0.0, 0, 0, 0, 0, 0
        W = 32
        for i in range(n_batches):
            ms, res = _timed(stream, lambda: step(i))
            tot_ms += ms
            seeds += BATCH
            edges += int(res.edges.sum().item())
            ids += int(res.frontier_len.sum().item())
            wl = ret.wave_lists(k)
            lists += sum(wl[1:])
            pbytes += pull_alg_bytes(n_items, stats["n_triples"], W, wl, ret.wave_modes(k))
        prof = _profiled(ret, [lambda i=i: step(i) for i in range(n_batches)])
        kms = {c: v[0] / n_batches for c, v in prof.items() if v[0]}
        dom = max(("frontier", "pull", "push"), key=lambda c: kms.get(c, 0.0))
        leg = {"seeds_per_s": seeds / (tot_ms / 1e3), "edges_per_s": edges / (tot_ms / 1e3),
               "ms_per_batch": tot_ms / n_batches, "frontier_ids_per_batch": ids / n_batches,
               "kernel_ms_per_batch": kms, "dominant": dom}
        # K4 (frontier materialisation) and the pull hop (the north star's
        # hop kernel), each against its own algorithmic bytes; kernel times
        # are CUDA events on each kernel's own stream in a profiled pass over
        # the same batches (K4 runs on side streams overlapping the next
        # hop, so its event time includes that contention)
        kbytes = 4 * ids + 4 * W * lists + 16 * k * seeds
        for key, group, b, note in (
                ("roofline", "frontier", kbytes, "K4: 4 B per output id + 4W B per nonzero layer row + offsets"),
                ("roofline_pull", "pull", pbytes,
                 "pull hops: 12 B per item + 4 B per in-edge + 4W B per frontier row + 4W B per "
                 "new row (x2 with its visited row)")):
            t = prof[group][0]
            if t <= 0 or b <= 0:
                continue
            a = b / (t / 1e3) / 1e9
            tr = load_traffic(group, "c4") if k == 3 else {}
            leg[key] = {"bound": "hbm", "achieved": a, "peak": peaks_leg["hbm_gbs"], "unit": "GB/s",
                        "frac": a / peaks_leg["hbm_gbs"], "kernel": group,
                        "kernel_ms_per_batch": t / n_batches, "alg_bytes_per_batch": b / n_batches,
                        "traffic": tr.get("bytes"), "traffic_source": tr.get("source"),
                        "note": note}
        out[f"k{k}"] = leg
    del ret
    torch.cuda.empty_cache()
    # streamed e2e (RetrievalPipeline, as the headline's): pinned host seeds
    # in, every wave's per-seed frontiers out to pinned host memory
    from paper_2604_18913_b200.pipeline import RetrievalPipeline

    host = [torch.from_numpy(b).pin_memory() for b in batches.cpu().numpy()]
    pipe = RetrievalPipeline(g, depth=2)
    for k in (2, 3):
        for _ in pipe.run(host, k):  # sizes every buffer; each session records + captures its graph
            pass
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        d2h = 0
        for hb in pipe.run(host, k):
            d2h += hb.nbytes()
        dt = (time.perf_counter() - t0) / len(host)
        out[f"k{k}"]["e2e"] = {"value": BATCH / dt, "unit": "seeds/s", "h2d_bytes_per_step": 4 * BATCH + 4 * (BATCH + 1),
                               "d2h_bytes_per_step": d2h // len(host), "link_GBps": d2h / len(host) / dt / 1e9,
                               "api": "RetrievalPipeline.run, one 1,024-seed wave per step"}
    del pipe, g
    torch.cuda.empty_cache()
    return out


def run_c5_leg(th, stream, n_waves=16):
    """BASELINE configs[4]'s graph on ONE GPU: 200M entities, 1e9 R-MAT
    triples (generated on the device), 2,000 relations; 16,384 seeds in waves
    of 1,024, k=2 FRONTIER, per-seed 64-of-2,000 relation masks.  The config
    names 8 GPUs; this is its single-GPU point (the graph fits one B200's HBM)."""
    import torch

    from paper_2604_18913_b200.retriever import _relation_masks

    t0 = time.perf_counter()
    s, r, o, E, R = workloads.c5_graph_gpu()
    torch.cuda.synchronize()
    gen_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    g = th.build_incidence((s, r, o), E, R)
    del s, r, o
    torch.cuda.empty_cache()
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    seeds, rel = workloads.c5_queries(E, R)
    words = _relation_masks(list(rel), seeds.size, R)
    d_seeds = torch.from_numpy(seeds).to(g.device)
    d_masks = torch.from_numpy(words.view(np.int32)).to(g.device)
    ret = th.Retriever(g, stream)
    offs = torch.arange(BATCH + 1, dtype=torch.int32, device=g.device)

    def wave(w):
        sl = slice(BATCH * w, BATCH * (w + 1))
        return ret.run(offs, d_seeds[sl], 2, "frontier", d_masks[sl], singleton=True, copy=False)

    for w in range(3):  # sizes buffers, records and captures the wave's graph
        wave(w)
    tot_ms, edges, ids = 0.0, 0, 0
    for w in range(n_waves):
        ms, res = _timed(stream, lambda: wave(w))
        tot_ms += ms
        edges += int(res.edges.sum().item())
        ids += int(res.frontier_len.sum().item())
    st = g.stats()
    out = {"workload": "C5 (BASELINE configs[4]) graph on 1 GPU: 200M entities, 1e9 R-MAT triples, 2,000 "
                       f"relations; {n_waves * BATCH} seeds in waves of {BATCH}, k=2 FRONTIER, per-seed "
                       "64-of-2,000 relation masks",
           "gen_s": gen_s, "build_s": build_s, "device_graph_bytes": st.get("device_bytes"),
           "max_out_degree": st.get("max_out_degree"),
           "seeds_per_s": n_waves * BATCH / (tot_ms / 1e3), "edges_per_s": edges / (tot_ms / 1e3),
           "ms_per_wave": tot_ms / n_waves, "frontier_ids_per_wave": ids / n_waves,
           "peak_device_GB": torch.cuda.max_memory_allocated() / 1e9}
    del ret, g, d_seeds, d_masks
    torch.cuda.empty_cache()
    return out


def partitioned_leg(th, cols, E, R, world, rank, ks=(2, 3), n_batches=4, reps=4):
    """BASELINE configs[3] partitioned over the job's ranks (hash owners +
    edge-split top-0.01% hubs, Algorithm 1 per hop with the ranks writing
    into each other's exchange regions): per k, one wave of 1,024 uniform
    seeds per step; seeds/s and edges/s over ALL ranks (strong scaling: the
    wave is the whole job's work), records written to other ranks per hop
    (12 B each: the interconnect bytes), and an e2e through
    ``PartitionedGraph.retrieve`` (host seeds in, merged sorted per-seed
    frontiers back on the host)."""
    import torch

    xch = th.LoopbackExchange(1) if world == 1 else th.DistExchange()
    t0 = time.perf_counter()
    pg = th.PartitionedGraph(cols, E, R, xch)
    build_s = time.perf_counter() - t0
    dev = pg.shards[0].device
    stream = torch.cuda.current_stream(dev)
    batches = workloads.seed_batches(E, BATCH, n_batches, seed=400)
    out = {"workload": f"C4 partitioned over {world} rank(s): hash owners, top-0.01% hubs edge-split "
                       f"({pg.plan.n_hubs} hubs), one wave of {BATCH} uniform seeds per step, FRONTIER",
           "build_s": build_s, "local_triples": [sh.local_triples for sh in pg.shards]}

    def wave(i, k, stats=None):
        q = th.partition.WaveQuery(np.arange(BATCH + 1, dtype=np.int32), batches[i % n_batches], k,
                                   th.HopSemantics.FRONTIER)
        return pg.run(q, stats)

    for k in ks:
        for i in range(n_batches):  # sizes every buffer; every timed wave repeats one of these
            wave(i, k)
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(reps)]
        for i in range(reps):
            evs[i][0].record(stream)
            wave(i, k)
            evs[i][1].record(stream)
        torch.cuda.synchronize()
        t_ms = sum(a.elapsed_time(b) for a, b in evs)
        edges, sent = 0, [0] * k
        for i in range(reps):  # edge totals and interconnect records: the same waves, untimed
            stats = {}
            parts = wave(i, k, stats)
            edges += int(sum(int(p.edges.sum()) for p in parts))
            for per in stats["sent_records"]:
                sent = [x + y for x, y in zip(sent, per)]
        vals = torch.tensor([t_ms, float(edges)] + [float(x) for x in sent], dtype=torch.float64)
        if world > 1:
            vals = vals.to(dev)
            tmax = vals.clone()
            _all_reduce(tmax, torch.distributed.ReduceOp.MAX)
            _all_reduce(vals, torch.distributed.ReduceOp.SUM)
            vals[0] = tmax[0]
            vals = vals.cpu()
        t_ms = float(vals[0])
        per_hop_bytes = [12.0 * float(x) / reps for x in vals[2:].tolist()]
        # e2e: host seeds -> merged per-seed sorted frontiers in pinned host
        # memory (as the C2 e2e: the public API with copy=False, then one
        # non-blocking copy per result tensor)
        e2e, pinned, d2h = [], {}, 0
        for i in range(3):
            torch.cuda.synchronize()
            w0 = time.perf_counter()
            res = pg.retrieve(batches[0], k, copy=False)  # (same shapes: no pinned regrowth)
            d2h = 0
            for name in ("frontier_off", "frontier_len", "frontier_ids", "edges"):
                t = getattr(res, name)
                buf = pinned.get(name)
                if buf is None or buf.numel() < t.numel():
                    buf = torch.empty(int(t.numel() * 1.25) + 16, dtype=t.dtype).pin_memory()
                    pinned[name] = buf
                buf[: t.numel()].copy_(t.reshape(-1), non_blocking=True)
                d2h += t.numel() * t.element_size()
            torch.cuda.synchronize()
            e2e.append(time.perf_counter() - w0)
        e2e = e2e[1:]  # (the first call sizes the pinned buffers)
        out[f"k{k}"] = {
            "seeds_per_s": BATCH * reps / (t_ms / 1e3), "edges_per_s": float(vals[1]) / (t_ms / 1e3),
            "ms_per_wave": t_ms / reps,
            "interconnect": {"bytes_per_hop": per_hop_bytes,
                             "GBps": sum(per_hop_bytes) / (t_ms / reps / 1e3) / 1e9,
                             "peak_per_direction_GBps": 900.0,
                             "note": "records written into other ranks' exchange inboxes (12 B each)"},
            "e2e": {"value": BATCH / statistics.median(e2e), "unit": "seeds/s",
                    "h2d_bytes_per_step": BATCH * 4, "d2h_bytes_per_step": int(d2h),
                    "api": "PartitionedGraph.retrieve(copy=False) (merge of the owners' slices on the "
                           "device) + pinned D2H of the merged results"}}
    del pg
    torch.cuda.empty_cache()
    return out


def run_partitioned(args, world, rank, local):
    """`--partitioned`: only the partitioned C4 leg, as the headline line."""
    import torch
    import torch.distributed as dist

    import paper_2604_18913_b200 as th

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        _init_dist(dev, rank, world)
    s, r, o, E, R = workloads.c4_graph()
    clocks = ClockSampler(local)
    clocks.start()
    leg = partitioned_leg(th, (s, r, o), E, R, world, rank, ks=(args.part_k,),
                          reps=max(args.steps, 1))
    clk = clocks.stop()
    k = args.part_k
    if rank == 0:
        d = leg[f"k{k}"]
        print(json.dumps({
            "metric": f"partitioned C4 k-hop seeds/s at k={k}", "value": d["seeds_per_s"], "unit": "seeds/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": d["ms_per_wave"],
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int32",
            "data": "synthetic", "config": {"workload": leg["workload"], "parallelism": f"graph-partitioned x{world}"},
            "edges_per_s": d["edges_per_s"], "interconnect": d["interconnect"], "e2e": d["e2e"],
            "clocks": clk}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_ours(args, world, rank, local):
    import torch

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        _init_dist(dev)
    import paper_2604_18913_b200 as th

    s, r, o, E, R = workloads.c2_graph()
    stats = workloads.graph_stats(s, o, E)
    g = th.build_incidence((s, r, o), E, R)
    stream = torch.cuda.current_stream(dev)
    ret = th.Retriever(g, stream)
    n_batches = args.warmup + args.steps
    batches = workloads.seed_batches(E, BATCH, n_batches, seed=100 + 7919 * rank)
    d_batches = torch.from_numpy(batches).to(dev)
    offs = torch.arange(BATCH + 1, dtype=torch.int32, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    def step(i, k=K_HOPS):
        ret.run(offs, d_batches[i % n_batches], k, "frontier", None, singleton=True, copy=False,
                collect=False)

    # warm-up (also sizes the result buffers)
    for i in range(args.warmup):
        step(i)
        ret.collect()
    clocks = ClockSampler(local)
    clocks.start()  # (before the barrier: see ClockSampler.start)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    launches0 = ret.launch_count()
    edges = ids = 0
    alg_bytes = 0
    lists_sum = 0
    pull_bytes = 0
    n_items = int(((np.bincount(o, minlength=E) + 31) // 32).sum())  # static pull items
    t_wall0 = time.perf_counter()
    for i in range(args.steps):
        flush.zero_()
        ev[i][0].record(stream)
        step(args.warmup + i)
        ev[i][1].record(stream)
        res = ret.collect()
        e = res.edges.sum().item()
        edges += e
        fl = res.frontier_len
        ids += int(fl.sum().item())
        # SURVEY 8d per-seed algorithmic bytes: 8|X_{h-1}| + 4|T_h| + 4|Out_h|
        xs = torch.cat([torch.ones(1, BATCH, dtype=torch.int64, device=dev), fl[:-1]]).sum().item()
        alg_bytes += 8 * xs + 4 * e + 4 * int(fl.sum().item())
        wl = ret.wave_lists(K_HOPS)
        lists_sum += sum(wl[1:])
        pull_bytes += pull_alg_bytes(n_items, int(s.size), 32, wl, ret.wave_modes(K_HOPS))
    torch.cuda.synchronize()
    wall = time.perf_counter() - t_wall0
    clk = clocks.stop()
    launches = ret.launch_count() - launches0
    times = [a.elapsed_time(b) for a, b in ev]
    # per-kernel-group device times: a profiled pass over the same K batches
    # (event pairs around every kernel group cost ~10% of the step, so the
    # headline is timed without them)
    ret.set_profiling(True)
    for i in range(2):  # the profiled shape is captured anew
        step(args.warmup + i)
        ret.collect()
    ret.profile()
    for i in range(args.steps):
        flush.zero_()
        step(args.warmup + i)
        ret.collect()
    prof = ret.profile()
    ret.set_profiling(False)
    t_ms = sum(times)
    if world > 1:
        import torch.distributed as dist

        tt = torch.tensor([t_ms], dtype=torch.float64, device=dev)
        _all_reduce(tt, dist.ReduceOp.MAX)
        t_ms = float(tt.item())
    seeds_total = BATCH * args.steps * world
    value = seeds_total / (t_ms / 1e3)

    # per-k seeds/s (k=1, 2 are separate, shorter timed runs)
    per_k = {}
    for kk in (1, 2, 3):
        reps = 3
        tk = 0.0
        ek = 0
        for i in range(2):  # eager run + graph capture of this shape
            step(i, kk)
            ret.collect()
        for i in range(reps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            step(i, kk)
            b.record(stream)
            rr = ret.collect()
            tk += a.elapsed_time(b)
            ek += rr.edges.sum().item()
        per_k[f"k{kk}"] = {"seeds_per_s": BATCH * reps / (tk / 1e3), "gteps": ek / (tk / 1e3) / 1e9,
                           "ms_per_batch": tk / reps}

    # roofline of the dominant kernel group
    peaks = load_peaks()
    W = 32
    dominant = max(("frontier", "pull", "push"), key=lambda c: prof[c][0])
    if dominant == "frontier":
        kbytes = 4 * ids + 4 * W * lists_sum + 16 * K_HOPS * BATCH * args.steps
        note = "K4 materialisation: one read of every nonzero layer row + 4 B per output id"
    elif dominant == "pull":
        st = g.stats()
        kbytes =(4 * (E + 1) + 4 * st["n_triples"] + 4 * W * E + 8 * W * lists_sum) * args.steps
        note = "pull hop lower bound: rindptr + in-edge list + visited rows + new rows"
    else:
        kbytes = 4 * edges
        note = "push hop lower bound: 4 B object id per traversed (seed,edge)"
    kms = prof[dominant][0]
    achieved = kbytes / (kms / 1e3) / 1e9 if kms > 0 else 0.0
    traffic = load_traffic(dominant)
    # the pull hop (the north star's hop kernel) against its own bytes
    pms = prof["pull"][0]
    pull_ach = pull_bytes / (pms / 1e3) / 1e9 if pms > 0 else 0.0
    ptraffic = load_traffic("pull")
    roofline_pull = {"bound": "hbm", "achieved": pull_ach, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                     "frac": pull_ach / peaks["hbm_gbs"], "kernel": "pull",
                     "kernel_ms_per_step": pms / args.steps, "alg_bytes_per_step": pull_bytes / args.steps,
                     "traffic": ptraffic.get("bytes"), "traffic_source": ptraffic.get("source"),
                     "note": "pull hops: 12 B per item + 4 B per in-edge + 4W B per frontier row + 4W B "
                             "per new row (x2 with its visited row); C2's 69 MB graph state is L2-resident"}

    # e2e through the public API: pinned host seeds in, host results out
    e2e_times, h2d, d2h = [], 0, 0
    host_seeds = torch.from_numpy(batches[0]).pin_memory()
    pinned = {}
    for i in range(max(2, min(args.steps, 5))):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = ret.retrieve(host_seeds, K_HOPS, copy=False)
        outs = {}
        for name in ("frontier_off", "frontier_len", "frontier_ids", "edges"):
            t = getattr(res, name)
            buf = pinned.get(name)
            if buf is None or buf.numel() < t.numel():
                buf = torch.empty(int(t.numel() * 1.25) + 16, dtype=t.dtype).pin_memory()
                pinned[name] = buf
            buf[: t.numel()].copy_(t.reshape(-1), non_blocking=True)
            outs[name] = t.numel() * t.element_size()
        torch.cuda.synchronize()
        e2e_times.append(time.perf_counter() - t0)
        h2d = host_seeds.numel() * 4 + (BATCH + 1) * 4
        d2h = sum(outs.values())
    e2e_t = statistics.median(e2e_times)
    # streaming e2e (the serving loop): RetrievalPipeline runs batch i+1's
    # hops while batch i's results cross PCIe; every step still moves its
    # pinned seeds in and all of its results out
    from paper_2604_18913_b200.pipeline import RetrievalPipeline

    pipe = RetrievalPipeline(g, depth=2)
    host_batches = [torch.from_numpy(b).pin_memory() for b in batches]
    for _ in pipe.run(host_batches[:4], K_HOPS):  # sizes buffers, captures both sessions' graphs
        pass
    torch.cuda.synchronize()
    n_pipe = len(host_batches)
    t0 = time.perf_counter()
    pipe_d2h = 0
    for hb in pipe.run(host_batches, K_HOPS):
        pipe_d2h += hb.nbytes()
    pipe_t = (time.perf_counter() - t0) / n_pipe
    del pipe
    if world > 1:
        # whole job: every rank's batch over the slowest rank's time
        import torch.distributed as dist

        tt = torch.tensor([e2e_t, pipe_t], dtype=torch.float64, device=dev)
        _all_reduce(tt, dist.ReduceOp.MAX)
        e2e_t, pipe_t = (float(x) for x in tt.tolist())
    e2e_value = BATCH * world / e2e_t
    pipe_value = BATCH * world / pipe_t
    # the e2e's own roofline: one raw pinned D2H of a step's result bytes on
    # this box (the host link, not the kernels, bounds the streamed e2e)
    nb = int(pipe_d2h // n_pipe)
    raw_src = torch.empty(nb // 4 + 1, dtype=torch.int32, device=dev)
    raw_dst = torch.empty(nb // 4 + 1, dtype=torch.int32).pin_memory()
    link_peak = 0.0
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        raw_dst.copy_(raw_src, non_blocking=True)
        torch.cuda.synchronize()
        link_peak = max(link_peak, raw_dst.numel() * 4 / (time.perf_counter() - t0) / 1e9)
    del raw_src, raw_dst

    # CPU baseline: oracle on the host cores, rank 0 at N=1 only
    cpu = None
    if world == 1 and not args.no_cpu:
        cores = os.cpu_count() or 1
        build_cpu_graph(s, r, o, E, R)
        pool = cpu_pool(cores)
        n, e, dt = cpu_run(pool, batches[0], K_HOPS, args.cpu_budget)
        pool.terminate()
        cpu = {"value": n / dt, "unit": "seeds/s", "cores": cores, "kind": "port", "cpu_model": cpu_model(),
               "sample": f"first {n} seeds of the first timed C2 batch (k={K_HOPS} FRONTIER, "
                         f"oracle hop_trace per seed, fork pool, {dt:.1f} s)",
               "edges_per_s": e / dt}

    # the C3 / C4 single-GPU legs run at N=1 only (like the CPU baseline);
    # the partitioned C4 leg runs at every N (all ranks take part)
    c3 = run_c3_leg(th, g, s, E, R, stream, peaks) if (world == 1 and not args.no_c3) else None
    c4 = part = None
    if not args.no_c4:
        del ret, g
        torch.cuda.empty_cache()
        c4_cols = workloads.c4_graph()
        if world == 1:
            c4 = run_c4_leg(th, stream, peaks, cols=c4_cols)
        if not args.no_part:
            part = partitioned_leg(th, c4_cols[:3], c4_cols[3], c4_cols[4], world, rank)
        del c4_cols
    c5 = None
    if world == 1 and not args.no_c5:
        import gc

        gc.collect()  # (the partitioned leg's shards free their device regions on collection)
        torch.cuda.empty_cache()
        try:
            c5 = run_c5_leg(th, stream)
        except (RuntimeError, MemoryError) as e:  # (a leg that cannot run must not lose the line)
            c5 = {"error": f"{type(e).__name__}: {e}"[:300]}
            torch.cuda.empty_cache()

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "seeds/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
            "config": {"workload": "C2 (BASELINE configs[1]): 407K entities, 3.4M triples, 400 relations, "
                                   "hub-to-hub Zipf 1.2 subjects/objects, Zipf 1.0 relations; "
                                   f"{BATCH} uniform seeds per step, k={K_HOPS}, FRONTIER, no filter, "
                                   "paths off, per-seed sorted frontiers materialised for hops 1..3",
                       "batch": BATCH, "k": K_HOPS, "l2": "flushed (256 MB write) before every timed step",
                       "graph": stats, "parallelism": f"seed-sharded replicas x{world}"},
            "edges_per_s": edges * world / (t_ms / 1e3),
            "gteps": edges * world / (t_ms / 1e3) / 1e9,
            "frontier_ids_per_step": ids / args.steps,
            "per_k": per_k,
            "per_seed_equiv": {"bytes_per_step": alg_bytes / args.steps,
                               "GBps": alg_bytes / (t_ms / 1e3) / 1e9,
                               "note": "SURVEY 8d per-seed algorithmic bytes / step time; the bit-parallel "
                                       "engine shares each edge read across up to 1024 seeds"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                         "frac": achieved / peaks["hbm_gbs"], "traffic": traffic.get("bytes"),
                         "traffic_source": traffic.get("source"), "kernel": dominant,
                         "kernel_ms_per_step": kms / args.steps, "alg_bytes_per_step": kbytes / args.steps,
                         "peak_source": peaks["source"], "note": note},
            "roofline_pull": roofline_pull,
            "kernel_ms_per_step": {c: v[0] / args.steps for c, v in prof.items()},
            "kernel_ms_source": "CUDA events around each kernel group, profiled pass over the same K batches",
            "kernel_launches_per_step": {c: v[1] / args.steps for c, v in prof.items()},
            "e2e": {"value": pipe_value, "unit": "seeds/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": pipe_d2h // n_pipe, "steps": n_pipe,
                    "api": "RetrievalPipeline.run (pipeline.py): pinned seeds in, every batch's results "
                           "to pinned host memory, batch i+1's hops overlapping batch i's copy-out",
                    # the host link bounds it: result bytes per second of the whole step
                    "link_GBps": (h2d + pipe_d2h / n_pipe) / pipe_t / 1e9,
                    "link_peak_GBps": link_peak,
                    "link_frac": (h2d + pipe_d2h / n_pipe) / pipe_t / 1e9 / link_peak if link_peak else None,
                    "link_peak_note": "one raw pinned D2H of a step's result bytes, best of 3, same box",
                    "note": "PCIe-bound: every step returns all per-seed frontiers (int32) to the host",
                    "blocking": {"value": e2e_value, "unit": "seeds/s", "h2d_bytes_per_step": h2d,
                                 "d2h_bytes_per_step": d2h,
                                 "api": "Retriever.retrieve + pinned D2H of all results, one batch at a time",
                                 "link_GBps": (h2d + d2h) / e2e_t / 1e9}},
            "gpu_launches": launches,
            "wall_s_timed": wall,
            "clocks": clk,
            "cpu_baseline": cpu,
            "c3": c3,
            "c4": c4,
            "partitioned": part,
            "c5": c5,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--ref-step-seeds", type=int, default=256)
    ap.add_argument("--no-c3", action="store_true", help="skip the C3 (filter + paths) leg")
    ap.add_argument("--no-c4", action="store_true", help="skip the C4 (54.4M-entity) leg")
    ap.add_argument("--no-c5", action="store_true", help="skip the C5 (1e9-triple, one GPU) leg")
    ap.add_argument("--partitioned", action="store_true",
                    help="C4 on a graph partitioned over the ranks (NCCL exchange per hop)")
    ap.add_argument("--part-k", type=int, default=2)
    ap.add_argument("--no-part", action="store_true", help="skip the partitioned C4 leg")
    args = ap.parse_args()
    world, rank, local = dist_env()
    if args.impl == "reference":
        run_reference(args, world, rank)
    elif args.partitioned:
        run_partitioned(args, world, rank, local)
    else:
        run_ours(args, world, rank, local)


if __name__ == "__main__":
    main()
