"""bench.py — simulated MQFQ-Sticky dispatch decisions per second on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl gfq|reference]
                    [--workload c3|c1|c1f10|c2|c4|c5] [--split weak|strong]

A step is one pass of the hot path over one batch: by default the whole C3
sweep (BASELINE configs[2], the configuration the metric's "1/2/4/8 B200" and
the north-star target are quoted on: 4096 MQFQ-Sticky simulations of a
100-flow Azure-shaped Zipf trace, T x alpha x D x 16 seeds) run by one k_sim
launch, including the per-function reducer and latency histograms, plus
(N > 1) the NCCL all-reduce of the histograms and all-gather of the
per-simulation summary rows.

--split weak    (default) each rank simulates its own disjoint block of 16
                seeds: 4096 simulations per GPU, no data-path collective.
--split strong  the ONE fixed 4096-simulation sweep, split over the ranks by
                an a-priori cost model (dist.partition: greedy LPT on
                N_arrivals x F_touched); total work is fixed.
--workload c1   BASELINE configs[0]: the reference's default run (one
                simulation); the line adds per-simulation latencies for the
                stats build and the records/audit build and through the
                public run_simulation drop-in.

value   successful dispatches (DispatchAudit rows) summed over all ranks /
        max-over-ranks device time of the K timed steps, inputs resident in HBM,
        L2 flushed (256 MiB write) before every step.
e2e     the same metric through the public Python API with host buffers: trace
        / flow-table / config / sim-block uploads from pinned memory, launch,
        and the device->host copy of status, counters, summary and per-function
        statistics, every step.
roofline  SM issue (the binding roof): warp-instructions of the
        dominant kernel per launch (from the committed ncu capture of the same
        source build and workload, profiles/ncu_k_sim_<workload>.json) / its
        mean launch time measured here, against 148 SMs x 4 issue slots x the
        SM clock sampled during the run.  roofline_hbm: algorithmic bytes.
cpu_baseline  the C oracle port (oracle/, the reference algorithm restated in
        C; ~100x faster than the reference's Python) on one host core, on a
        bounded random sample of the same sweep, with the engine's exact early
        exit (both arms process the same events).
python_reference  the UNMODIFIED reference (gpufairq, baseline/_ref via
        tools/install_ref.sh) on all host cores, on a bounded random sample.
--impl reference  the oracle port on ALL host cores (rank 0 only).
"""

from __future__ import annotations

import argparse
import json
import os
import random
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "simulated dispatch decisions/s"
UNIT = "dispatches/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="gfq", choices=["gfq", "reference"])
    ap.add_argument("--workload", default="c3", choices=["c3", "c1", "c1f10", "c2", "c4", "c5"])
    ap.add_argument("--split", default="weak", choices=["weak", "strong"])
    ap.add_argument("--emulate-world", type=int, default=0,
                    help="--split strong on ONE GPU: run the part of rank --emulate-rank of a "
                         "sweep split over this many ranks (per-rank time of an N-GPU run)")
    ap.add_argument("--emulate-rank", type=int, default=0)
    ap.add_argument("--py-seconds", type=float, default=15.0,
                    help="wall seconds of the unmodified Python reference sample (0 = skip)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=0)
    ap.add_argument("--seeds", type=int, default=0, help="seeds per GPU (default: the config's)")
    ap.add_argument("--event-capacity", type=int, default=0,
                    help="dynamic event slots per simulation (0 = the engine's default)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


# ---------------------------------------------------------------------------
# CPU side (oracle port) — only bench's cpu_baseline leg and --impl reference

def _oracle_jobs(w, idxs):
    from oracle import oracle as orc
    from paper_2507_08954_b200 import _abi
    jobs = []
    for i in idxs:
        s = w.sims[i]
        tr, tab = w.traces[s.trace], w.tabs[s.flowtab]
        sim = _abi.Sim.from_buffer_copy(s)
        dc = w.dcfgs[s.device_cfg: s.device_cfg + s.n_devices]
        jobs.append((orc, sim, tr, {"warm": tab.warm, "cold": tab.cold, "mem": tab.mem,
                                     "share": tab.share, "weight": tab.weight},
                     [_abi.device_cfg_from(d) for d in dc]))
    return jobs


def _oracle_one(job):
    orc, sim, tr, tab, dc = job
    r = orc.run_packed(sim, tr.arrival, tr.flow, tr.n_flows, tab, dc, want_audit=False,
                       want_dispatch=False, want_records=True, want_stats=True, early_exit=True)
    return len(r["rec_inv"])


def cpu_sample(w, seconds: float, threads: int, seed: int = 0):
    """Run random sims of the workload through the oracle for ~`seconds`."""
    from concurrent.futures import ThreadPoolExecutor
    rng = random.Random(seed)
    order = list(range(len(w.sims)))
    rng.shuffle(order)
    done_disp, done_sims = 0, 0
    t0 = time.perf_counter()
    pos = 0
    with ThreadPoolExecutor(max_workers=threads) as ex:   # ctypes releases the GIL
        while time.perf_counter() - t0 < seconds and pos < len(order):
            chunk = order[pos: pos + 4 * threads]
            pos += len(chunk)
            for n in ex.map(_oracle_one, _oracle_jobs(w, chunk)):
                done_disp += n
                done_sims += 1
    dt = time.perf_counter() - t0
    return done_disp, done_sims, dt


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


_PY_REF = None


def _py_ref_init(src):
    global _PY_REF
    if src not in sys.path:
        sys.path.insert(0, src)
    import gpufairq
    _PY_REF = gpufairq


def _py_ref_one(job):
    """One simulation through the UNMODIFIED reference (engine.py:214-218)."""
    entries, prof_rows, pol, sched, devs = job
    from gpufairq.core import FunctionProfile
    from gpufairq.device import DeviceConfig, DeviceSet
    from gpufairq.engine import run_simulation
    from gpufairq.mqfq import SchedulerConfig
    from gpufairq.policies import make_policy
    from gpufairq.workload import Trace
    profiles = {r[0]: FunctionProfile(*r) for r in prof_rows}
    trace = Trace(entries=entries, duration_s=entries[-1][0] if entries else 0.0)
    policy = make_policy(pol, profiles, SchedulerConfig(**sched))
    res = run_simulation(trace, profiles, policy, DeviceSet([DeviceConfig(**d) for d in devs]))
    return len(res.audit.dispatches)


def python_reference_sample(w, seconds: float, seed: int = 0):
    """The unmodified Python reference (baseline/_ref, tools/install_ref.sh) on
    random sims of the workload, one process per host core, for ~`seconds`."""
    from concurrent.futures import ProcessPoolExecutor, as_completed
    from dataclasses import asdict
    src = os.path.join(ROOT, "baseline", "_ref")
    if seconds <= 0 or not os.path.isfile(os.path.join(src, "gpufairq", "__init__.py")):
        return None
    names = {0: "mqfq", 1: "fcfs", 2: "batch", 3: "sjf", 4: "fcfs_naive"}
    rng = random.Random(seed)
    order = list(range(len(w.sims)))
    rng.shuffle(order)

    def job(i):
        s = w.sims[i]
        tr, tab = w.traces[s.trace], w.tabs[s.flowtab]
        entries = [(float(t), tr.names[f]) for t, f in zip(tr.arrival.tolist(), tr.flow.tolist())]
        rows = [(nm, float(tab.warm[k]), float(tab.cold[k]), float(tab.mem[k]),
                 float(tab.share[k]), float(tab.weight[k])) for k, nm in enumerate(tr.names)]
        sched = {"t_overrun": float(s.t_overrun), "alpha": float(s.alpha),
                 "default_ttl_s": float(s.default_ttl_s)}
        devs = [asdict(d) for d in w.dcfgs[s.device_cfg: s.device_cfg + s.n_devices]]
        return entries, rows, names[int(s.policy)], sched, devs

    cores = os.cpu_count() or 1
    disp = sims = 0
    t0 = time.perf_counter()
    with ProcessPoolExecutor(max_workers=cores, initializer=_py_ref_init, initargs=(src,)) as ex:
        pos, live = 0, set()
        while pos < len(order) and len(live) < 2 * cores:
            live.add(ex.submit(_py_ref_one, job(order[pos]))); pos += 1
        while live:
            done = next(as_completed(live))
            live.discard(done)
            disp += done.result(); sims += 1
            if time.perf_counter() - t0 < seconds and pos < len(order):
                live.add(ex.submit(_py_ref_one, job(order[pos]))); pos += 1
        dt = time.perf_counter() - t0
    return {"value": disp / dt, "unit": UNIT, "cores": cores, "kind": "python",
            "cpu_model": cpu_model(),
            "sample": f"{sims} random sims of the {w.name} workload ({disp} dispatches, "
                      f"{dt:.1f} s wall) through the unmodified reference run_simulation "
                      f"(gpufairq 0.1.0, baseline/_ref), {cores} processes"}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from paper_2507_08954_b200 import sweep
    import oracle.oracle as orc
    orc.build()
    w = sweep.build(args.workload, 0)
    threads = os.cpu_count() or 1
    per_step = max(2.0, 60.0 / max(args.steps + args.warmup, 1))
    for s in range(args.warmup):
        cpu_sample(w, min(per_step, 2.0), threads, seed=1000 + s)
    disp, sims, secs = 0, 0, 0.0
    for s in range(args.steps):
        d, n, dt = cpu_sample(w, per_step, threads, seed=s)
        disp += d; sims += n; secs += dt
    v = disp / secs
    line = {"metric": METRIC, "value": v, "unit": UNIT, "impl": "reference", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps,
            "higher_is_better": True, "scaling": "strong" if args.split == "strong" else "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (gen_zipf traces, default profiles)",
            "config": dict(w.describe, parallelism=f"{threads} host threads"),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "port",
                             "cpu_model": cpu_model(),
                             "sample": f"{sims} random sims of the {args.workload} sweep "
                                       f"({disp} dispatches) through oracle/gfq_oracle.c "
                                       f"with the engine's exact early exit"},
            "python_reference": python_reference_sample(w, args.py_seconds),
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU side

class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.gpu)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        try:
            d = json.load(open(p))
            v = d.get("hbm_gbs") or d.get("hbm_GBps")
            if v:
                return float(v), "measured (MEASURED_PEAKS.json hbm_gbs)"
        except Exception:
            pass
    return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def source_hash() -> str:
    """Hash of the engine sources (csrc + include/gfq.h): ties an ncu capture
    to the build it measured."""
    import glob
    import hashlib
    h = hashlib.sha256()
    files = sorted(glob.glob(os.path.join(ROOT, "paper_2507_08954_b200", "csrc", "*"))) + \
        [os.path.join(ROOT, "include", "gfq.h")]
    for f in files:
        with open(f, "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:12]


def _norm_kernel(name: str) -> str:
    import re
    name = re.sub(r"\bgfq::", "", name).replace("true", "1").replace("false", "0")
    return name.replace(" ", "")


def kernel_sass_hashes(so=None) -> dict:
    """sha256 of each simulation kernel's SASS in libgfq.so, by normalised
    demangled name: ties an ncu capture to the exact machine code measured
    (host-side edits to the engine do not invalidate it)."""
    import hashlib
    import re
    so = so or os.path.join(ROOT, "paper_2507_08954_b200", "libgfq.so")
    try:
        out = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True,
                             timeout=120).stdout
    except (OSError, subprocess.TimeoutExpired):
        return {}
    funcs, cur, buf = {}, None, []
    for ln in out.splitlines():
        m = re.search(r"Function : (\S+)", ln)
        if m:
            if cur:
                funcs[cur] = "\n".join(buf)
            cur, buf = m.group(1), []
        elif cur:
            buf.append(ln)
    if cur:
        funcs[cur] = "\n".join(buf)
    names = [k for k in funcs if "k_sim" in k]
    if not names:
        return {}
    dem = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True,
                         text=True).stdout.splitlines()
    return {_norm_kernel(d): hashlib.sha256(funcs[m].encode()).hexdigest()[:16]
            for m, d in zip(names, dem)}


def ncu_capture(workload: str):
    """The committed ncu --set full numbers of this workload's dominant
    kernel (tools/ncu_summary.py -> profiles/ncu_k_sim_<workload>.json)."""
    p = os.path.join(ROOT, "profiles", f"ncu_k_sim_{workload}.json")
    if os.path.exists(p):
        try:
            return json.load(open(p))
        except Exception:
            return None
    return None


def run_gfq(args):
    import torch
    import torch.distributed as dist
    from paper_2507_08954_b200 import _abi, sweep
    from paper_2507_08954_b200.engine import Engine

    rank, world, local = dist_env()
    # one process per GPU; GFQ_DIST_BACKEND=gloo and ranks > GPUs (ranks then
    # share devices) exist only to exercise the multi-rank path on a 1-GPU box
    backend = os.environ.get("GFQ_DIST_BACKEND", "nccl")
    local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    eng = Engine(local)
    # the sweep's traces come from the GPU trace generator (gfq_generate_traces,
    # bit-identical to gen_zipf); the arrays are also kept on the host for the
    # e2e leg's uploads and the CPU baseline
    if args.split == "strong":
        # ONE fixed sweep (rank 0's seeds on every rank), cost-partitioned
        from paper_2507_08954_b200.dist import partition
        w_full = sweep.build(args.workload, 0, engine=eng,
                             **({"n_seeds": args.seeds} if args.seeds else {}))
        ew = args.emulate_world or world
        er = args.emulate_rank if args.emulate_world else rank
        part = partition(sweep.sim_costs(w_full), ew)[er]
        w = sweep.restrict(w_full, part)
        w.describe["strong_part"] = {"ranks": ew, "rank": er, "sims": len(part),
                                     "emulated_on_one_gpu": bool(args.emulate_world)}
    else:
        w = sweep.build(args.workload, rank, engine=eng,
                        **({"n_seeds": args.seeds} if args.seeds else {}))
    w.upload(eng)
    outputs = _abi.WANT_STATS | _abi.WANT_HIST
    kw = dict(hist_groups=w.groups, hist_rows=w.hist_rows, hist_bins=sweep.HIST_BINS,
              hist_lo_s=sweep.HIST_LO_S, hist_hi_s=sweep.HIST_HI_S,
              event_capacity=args.event_capacity)
    sims = w.sims_array()
    eng.prepare(sims, outputs=outputs, early_exit=True, **kw)
    info = eng.batch_info()
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device="cuda")
    hist_t = summ_t = comm = summ_all = None
    if world > 1 and backend == "nccl":
        # the one collective step through the C ABI
        # (gfq_reduce_nccl): histograms all-reduced, summary rows all-gathered
        # over NVLink; the communicator's id travels over torch.distributed
        from paper_2507_08954_b200.engine import NcclComm
        uid = [NcclComm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = NcclComm(world, rank, uid[0])
        summ_all = torch.empty(world * len(w.sims) * 3, dtype=torch.float64, device="cuda")
    elif world > 1:
        ptr, n = eng.output_device_ptr(_abi.OUT_HIST)
        hist_t = torch.as_tensor(_CudaArray(ptr, n, "<i8"), device="cuda")
        ptr, n = eng.output_device_ptr(_abi.OUT_SUMMARY)
        summ_t = torch.as_tensor(_CudaArray(ptr, n, "<f8"), device="cuda").view(-1, 3)
    from paper_2507_08954_b200.dist import gather_rows

    def step():
        eng.launch(stream)
        if comm is not None:
            eng.reduce_nccl(comm, summ_all, stream)
        elif hist_t is not None:          # gloo (the multi-rank path on one GPU)
            h = hist_t.cpu()
            dist.all_reduce(h)
            hist_t.copy_(h)
            gather_rows(summ_t.cpu())

    for _ in range(max(args.warmup, 0)):
        flush.fill_(1)
        step()
    torch.cuda.synchronize()
    eng.synchronize()
    counters = eng.output(_abi.OUT_COUNTERS).reshape(-1, _abi.NCOUNTERS)
    disp_per_step = int(counters[:, 2].sum())
    calls_per_step = int(counters[:, 1].sum())
    events_per_step = int(counters[:, 0].sum())
    # diagnostic counters exist only in a -DGFQ_DIAG=1 build (zero otherwise)
    scans = {}
    if int(counters[:, 8].sum()):
        scans = {"gvt_scans": int(counters[:, 5].sum()), "refresh_scans": int(counters[:, 6].sum()),
                 "candidate_scans": int(counters[:, 7].sum()), "ticks": int(counters[:, 8].sum()),
                 "window_memo_hits": int(counters[:, 9].sum()),
                 "window_memo_misses": int(counters[:, 10].sum()),
                 "quiet_drains": int(counters[:, 11].sum()),
                 "max_dynamic_events": int(counters[:, 4].max())}

    # ---- timed region (device time, CUDA events on the launch stream)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    eng.kernel_times()                                      # reset the per-launch ring
    with Clocks(local) as clk:
        for k in range(args.steps):
            flush.fill_(k)                                  # evict L2 between steps
            ev[k][0].record(stream)
            step()
            ev[k][1].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    eng.synchronize()
    sim_ms, red_ms = eng.kernel_times()                     # k_sim / k_reduce, per launch
    step_ms = [a.elapsed_time(b) for a, b in ev]
    tot_ms = float(sum(step_ms))
    t = torch.tensor([tot_ms, float(disp_per_step * args.steps)], dtype=torch.float64,
                     device="cuda" if backend == "nccl" else "cpu")
    if world > 1:
        tm = t[:1].clone(); dist.all_reduce(tm, op=dist.ReduceOp.MAX)
        td = t[1:].clone(); dist.all_reduce(td)
        max_ms, all_disp = float(tm.item()), float(td.item())
    else:
        max_ms, all_disp = tot_ms, float(t[1].item())
    value = all_disp / (max_ms / 1e3)

    # ---- e2e through the public API with host buffers
    e2e_steps = args.e2e_steps or max(3, min(args.steps, 10))
    e2e = e2e_run(eng, w, outputs, kw, e2e_steps, world, dist if world > 1 else None)

    if comm is not None:
        torch.cuda.synchronize()
        comm.close()
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    kern_ms = float(statistics.mean(sim_ms)) if len(sim_ms) else statistics.mean(step_ms)
    ck = clk.summary()
    roof, roof_hbm = rooflines(w, args.workload, kern_ms, disp_per_step, events_per_step,
                               calls_per_step, ck, info)
    cpu = pyref = None
    if world == 1 and not args.no_cpu_baseline:
        import oracle.oracle as orc
        orc.build()
        d, n, dt = cpu_sample(w, args.cpu_seconds, 1)
        cpu = {"value": d / dt, "unit": UNIT, "cores": 1, "kind": "port", "cpu_model": cpu_model(),
               "sample": f"{n} random sims of the {args.workload} sweep ({d} dispatches, "
                         f"{dt:.1f} s) through oracle/gfq_oracle.c, 1 thread, with the "
                         f"engine's exact early exit"}
        pyref = python_reference_sample(w, args.py_seconds)
    extra = {}
    if args.workload.startswith("c1"):
        extra = c1_latencies(eng, w, kw, stream, flush, args.steps, step_ms)
    strong = args.split == "strong"
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "higher_is_better": True,
        "scaling": "strong" if strong else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (gen_zipf Azure-shaped traces, default profiles; " + (
            "one fixed sweep cost-partitioned over the ranks)" if strong else "per-rank seed blocks)"),
        "config": dict(w.describe, parallelism=(
                           f"one fixed sweep LPT-partitioned over {world} GPU(s), " if strong else
                           f"sims sharded over {world} GPU(s), ") + (
                           f"CTA ({info['cta_threads']} threads) per simulation"
                           if info["cta_threads"] else "warp per simulation"),
                       l2="flushed (256 MiB write) before every step",
                       outputs="per-function stats + latency histograms",
                       dispatch_calls_per_step=calls_per_step, events_per_step=events_per_step,
                       dispatches_per_step_per_gpu=disp_per_step, **scans),
        "e2e": e2e, "roofline": roof, "roofline_hbm": roof_hbm, "cpu_baseline": cpu,
        "python_reference": pyref,
        "clocks": ck, "gpu_launches": args.steps * info["launches_per_step"],
        "kernel_ms": {"k_sim_mean": kern_ms, "k_reduce_mean": float(statistics.mean(red_ms))
                      if len(red_ms) else None, "step_mean": statistics.mean(step_ms),
                      "step_min": min(step_ms), "step_max": max(step_ms)},
        **extra,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def rooflines(w, workload, kern_ms, disp, events, calls, clocks, info):
    """SM-issue roofline of the dominant kernel (the binding roof, SURVEY
    §8(d)) plus the HBM one.  Warp-instructions per launch come from the
    committed ncu --set full capture of the same source build and workload
    (they are a deterministic function of build and inputs); the launch time
    and SM clock are this run's."""
    import torch
    n_sm = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    nc = ncu_capture(workload) or {}
    mhz = clocks.get("sm_mhz") or clocks.get("sm_max_mhz") or 1965.0
    peak_issue = n_sm * 4 * mhz * 1e6 / 1e9          # G warp-instructions / s
    inst = nc.get("inst_executed_per_launch")
    kern = _norm_kernel(nc.get("kernel", ""))
    same = bool(nc) and nc.get("kernel_sass_hash") == kernel_sass_hashes().get(kern) \
        and nc.get("sims") == len(w.sims)
    roof = {"bound": "sm_issue", "unit": "G warp-inst/s", "peak": peak_issue,
            "peak_source": f"{n_sm} SMs x 4 issue slots x {mhz:.0f} MHz (sampled SM clock)",
            "achieved": None, "frac": None, "traffic": nc.get("dram_bytes_per_launch"),
            "ncu_capture": nc.get("capture"), "ncu_same_build": bool(same)}
    if inst:
        a = inst / (kern_ms / 1e3) / 1e9
        roof.update(achieved=a, frac=a / peak_issue, warp_inst_per_launch=inst,
                    warp_inst_per_dispatch=inst / max(disp, 1),
                    warp_inst_per_event=inst / max(events, 1),
                    warp_inst_per_dispatch_call=inst / max(calls, 1),
                    sm_inst_issued_pct_ncu=nc.get("sm_inst_issued_pct"),
                    warps_active_pct_ncu=nc.get("warps_active_pct"))
    n_arr = w.arrivals
    n_flows = int(sum(w.traces[s.trace].n_flows for s in w.sims))
    alg_bytes = 12 * n_arr + 32 * n_flows + 76 * len(w.sims)
    peak, peak_src = peaks()
    achieved = alg_bytes / (kern_ms / 1e3) / 1e9
    hbm = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
           "frac": achieved / peak, "traffic": nc.get("dram_bytes_per_launch"),
           "peak_source": peak_src, "algorithmic_bytes_per_launch": alg_bytes,
           "note": "12 B per arrival + 32 B per (sim, flow) + 76 B per sim; not binding"}
    return roof, hbm


def c1_latencies(eng, w, kw, stream, flush, steps, stats_ms):
    """BASELINE C1: per-simulation latency of the single default run, in the
    stats build (the timed steps), the records / dispatch / audit / eviction
    build (generic class), and end to end through the public run_simulation
    drop-in (pack, upload, launch, reference-shaped results)."""
    import torch
    from paper_2507_08954_b200 import _abi
    from paper_2507_08954_b200.device import DeviceConfig, DeviceSet
    from paper_2507_08954_b200.engine import run_simulation
    from paper_2507_08954_b200.mqfq import SchedulerConfig
    from paper_2507_08954_b200.policies import make_policy
    from paper_2507_08954_b200.workload import default_profiles, gen_zipf
    rec_out = (_abi.WANT_STATS | _abi.WANT_RECORDS | _abi.WANT_DISPATCH | _abi.WANT_AUDIT |
               _abi.WANT_EVICTIONS)
    eng.prepare(w.sims_array(), outputs=rec_out, early_exit=True)
    ms = []
    for k in range(steps + 2):
        flush.fill_(k)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream); eng.launch(stream); b.record(stream)
        torch.cuda.synchronize()
        if k >= 2:
            ms.append(a.elapsed_time(b))
    d = w.describe
    prof = default_profiles(d["functions"])
    trace = gen_zipf(d["functions"], d["zipf_s"], d["rate_rps"], d["duration_s"], d["seed"],
                     names=list(prof))
    run_simulation(trace, prof, make_policy("mqfq", prof, SchedulerConfig(10.0, 2, 2.0)),
                   DeviceSet([DeviceConfig(d_max=2)]))
    wall = []
    for _ in range(steps):
        pol = make_policy("mqfq", prof, SchedulerConfig(10.0, 2, 2.0))
        t0 = time.perf_counter()
        res = run_simulation(trace, prof, pol, DeviceSet([DeviceConfig(d_max=2)]))
        wall.append(1e3 * (time.perf_counter() - t0))
    # restore the stats launch the caller set up
    eng.prepare(w.sims_array(), outputs=_abi.WANT_STATS | _abi.WANT_HIST, early_exit=True, **kw)
    return {"c1_latency_ms": {
        "stats_build_device": statistics.median(stats_ms),
        "records_audit_build_device": statistics.median(ms),
        "run_simulation_e2e_wall": statistics.median(wall),
        "dispatches": len(res.records),
        "note": "one simulation = one warp: serial event processing, ~1 us per event"}}


class _CudaArray:
    """__cuda_array_interface__ view of an engine-owned device buffer."""

    def __init__(self, ptr, n, typestr):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr,
                                         "data": (ptr, False), "version": 3}


def e2e_run(eng, w, outputs, kw, steps, world, dist):
    """Public-API end-to-end, every step: host->device uploads of the step's
    traces / flow tables / configs / sim blocks from pinned buffers,
    gfq_prepare, launch, and the device->host read of its results (status,
    counters, summary, per-function statistics) into pinned buffers.  Wall
    clock, max over ranks.  Two engine handles alternate (double buffering):
    step k's uploads and step k-1's result reads run on each handle's
    transfer stream while the other handle's kernel runs, so the host work
    hides behind the simulation kernels; every step still moves all of its
    bytes."""
    import torch
    from paper_2507_08954_b200 import _abi
    from paper_2507_08954_b200.engine import Engine

    def pinned(a):
        t = torch.empty(a.shape, dtype=getattr(torch, str(a.dtype)), pin_memory=True)
        t.numpy()[...] = a
        return t.numpy()

    arrival = pinned(np.concatenate([t.arrival for t in w.traces]))
    flow = pinned(np.concatenate([t.flow for t in w.traces]).astype(np.int32))
    toff = pinned(np.concatenate([[0], np.cumsum([t.n for t in w.traces])]).astype(np.int64))
    tnf = pinned(np.array([t.n_flows for t in w.traces], dtype=np.int32))
    cols = [pinned(np.concatenate([getattr(t, c) for t in w.tabs]))
            for c in ("warm", "cold", "mem", "share", "weight")]
    hrow = pinned(np.concatenate([t.hist_row for t in w.tabs]).astype(np.int32))
    tabo = pinned(np.concatenate([[0], np.cumsum([len(t) for t in w.tabs])]).astype(np.int64))
    h2d = (arrival.nbytes + flow.nbytes + toff.nbytes + tnf.nbytes + sum(c.nbytes for c in cols)
           + hrow.nbytes + tabo.nbytes + 88 * len(w.dcfgs) + 96 * len(w.sims))
    sims = w.sims_array()
    engs = [eng, Engine(eng.device)]
    stream = torch.cuda.Stream()                  # both handles' kernels, in order

    res_ids = (_abi.OUT_STATUS, _abi.OUT_COUNTERS, _abi.OUT_SUMMARY, _abi.OUT_FLOW_COUNT,
               _abi.OUT_FLOW_MEAN, _abi.OUT_FLOW_VAR, _abi.OUT_FLOW_COLD_PCT)
    eng.prepare(sims, outputs=outputs, early_exit=True, **kw)
    res_buf = [{oid: pinned(np.zeros(eng.output(oid).shape, dtype=eng.output(oid).dtype))
                for oid in res_ids} for _ in engs]

    def submit(e):
        e.upload_trace_arrays(arrival, flow, toff, tnf)
        e.upload_flowtab_arrays(*cols, hrow, tabo)
        e.upload_device_cfgs(w.dcfgs)
        e.prepare(sims, outputs=outputs, early_exit=True, **kw)
        e.launch(stream)

    def collect(k):
        e, buf = engs[k % 2], res_buf[k % 2]
        e.synchronize()
        n = 0
        for oid in res_ids:
            n += e.output_into(oid, buf[oid]).nbytes
        c = buf[_abi.OUT_COUNTERS].reshape(-1, _abi.NCOUNTERS)
        return int(c[:, 2].sum()), n

    for k in range(2):                            # warm both handles
        submit(engs[k]); collect(k)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    disp = got = 0
    for k in range(steps):
        submit(engs[k % 2])
        if k:
            d, got = collect(k - 1)
            disp += d
    d, got = collect(steps - 1)
    disp += d
    dt = time.perf_counter() - t0
    engs[1].close()
    if dist:
        t = torch.tensor([dt, float(disp)], dtype=torch.float64,
                         device="cuda" if dist.get_backend() == "nccl" else "cpu")
        tm = t[:1].clone(); dist.all_reduce(tm, op=dist.ReduceOp.MAX)
        td = t[1:].clone(); dist.all_reduce(td)
        dt, disp = float(tm.item()), float(td.item())
    return {"value": disp / dt, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(got), "steps": steps,
            "ms_per_step": 1e3 * dt / steps,
            "pipeline": "2 engine handles, double-buffered: step k's uploads + prepare and "
                        "step k-1's result reads overlap the kernels"}


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gfq(args)


if __name__ == "__main__":
    main()
