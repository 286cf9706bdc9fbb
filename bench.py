#!/usr/bin/env python
"""bench.py — CSE substitution steps/s of the B200 search path (BASELINE.json metric).

Workload (BASELINE.json configs[2]): the 4x4x4 rank-49 Strassen(x)Strassen
scheme (tests/golden/schemes/sxs.json, digest 7da4ac65bf44d830), reference
default mixed strategy weights {ga 4, wr 1, gr 2, gi 8, mix 0.1, gp 0.01},
reinit fraction 0.4 (best-pool sharing), N = 16384 processes per component
(the paper's GPU process count for rank < 100), master seed
1, the U, V and W expression sets optimized concurrently.  A STEP is one
optimize_system iteration (parallel_search.hpp:231-271) of all three
components: N processes each run to completion, then the iteration barrier
(incumbent pool update + reinit selection).  Patience is set high so every
timed step is a full iteration (results are bit-identical to the reference
for the same iterations).  The metric counts substitutions selected by
run_cse (cse_engine.hpp:33-40); replayed prefixes are excluded.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

Multi-GPU: torchrun, one rank per GPU; processes are partitioned by global id
(weak: each rank runs N processes per component, total N*world), and the
per-iteration exchange (costs + best record all-gather) keeps the search
identical to a single-process run of N*world processes.
"""
import argparse
import ctypes as C
import json
import os
import re
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

METRIC = "CSE substitution steps/sec (1/2/4/8 B200) & best additions at fixed wall-time"
WORKLOAD = "sxs"


# BASELINE.json configs -> (scheme fixture, forced strategy, processes per GPU)
CONFIGS = {
    0: ("strassen", "greedy", 16384),
    1: ("laderman", "greedy_intersections", 4096),
    2: ("sxs", None, 16384),
    3: ("naive555_f1000", None, 8192),
    4: ("sxl", None, 8192),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="tcse", choices=["tcse", "reference"])
    ap.add_argument("--config", type=int, default=2, choices=range(5),
                    help="BASELINE.json configs[i]: 0 Strassen forced greedy, 1 Laderman gi, 2 S(x)S mixed "
                         "(default, the metric's config), 3 5x5x5 stand-in mixed, 4 6x6x6 stand-in mixed")
    ap.add_argument("--workload", default=None)
    ap.add_argument("--strategy", default=None, help="forced strategy (overrides the config's)")
    ap.add_argument("--processes", type=int, default=None)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--dist-backend", default="auto", choices=["auto", "nccl", "gloo"],
                    help="payload all-gather transport for --gpus > 1: nccl (one rank per GPU, the "
                         "default when ranks <= GPUs) or gloo (stages through host memory; used "
                         "automatically when several ranks share a GPU, which NCCL refuses)")
    args = ap.parse_args()
    wl, strat, procs = CONFIGS[args.config]
    args.workload = args.workload or wl
    args.strategy = args.strategy or strat
    args.processes = args.processes or procs
    return args


def load_systems(name):
    import paper_2512_13365_b200 as T
    s = T.load_scheme(os.path.join(ROOT, "tests", "golden", "schemes", name + ".json"))
    return s, T.extract_systems(s)


def config_block(args, world, scaling="weak"):
    import paper_2512_13365_b200 as T
    s, _ = load_systems(args.workload)
    return {
        "workload": "%s %dx%dx%d:%d, %s, reinit 0.4, %d processes/component/GPU, U/V/W concurrent; "
                    "step = one optimize_system iteration"
                    % (args.workload, s["m"], s["n"], s["p"], s["r"],
                       "forced %s" % args.strategy if args.strategy else "mixed strategies (reference default weights)",
                       args.processes),
        "baseline_config": args.config,
        "scheme_digest": T.scheme_digest(s),
        "processes_per_gpu": args.processes,
        "processes_total": args.processes * world,
        "master_seed": args.seed,
        "parallelism": "process-partition x%d (per-iteration payload all-gather%s)"
                       % (world, "" if world == 1 else (" by the library's ncclAllGather in the iteration graph"
                                                         if getattr(args, "dist_backend", "nccl") == "nccl"
                                                         else " through host memory (gloo; ranks share a GPU)")),
        "l2": "flushed before every timed step (256 MiB write)",
    }


# --------------------------------------------------------------- clocks

class ClockSampler:
    FIELDS = "clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown," \
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS, "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------- reference arm

def run_reference(args, rank, world):
    """The reference's own optimize_system (oracle/_ref, compiled from the
    unmodified headers) on the host cores, same workload, same iterations."""
    if rank != 0:
        return 0
    from oracle_lib import reference
    import paper_2512_13365_b200 as T
    from paper_2512_13365_b200 import _abi
    ref = reference()
    ref.ref_optimize_system_timed.argtypes = [
        C.POINTER(_abi.System), C.POINTER(_abi.SearchConfig), C.c_uint64, C.c_uint32, C.c_double,
        C.POINTER(_abi.Record), C.POINTER(C.c_int32), C.POINTER(C.c_uint64), C.POINTER(C.c_double),
        C.POINTER(C.c_double), C.POINTER(C.c_uint64), C.c_int32]
    threads = os.cpu_count() or 1
    _, systems = load_systems(args.workload)
    # the same process count and iterations as the GPU arm (so the printed
    # substitution_steps of the two arms can be compared); only multi-GPU
    # runs are capped (the CPU's steps/s does not depend on the process count
    # once it exceeds the thread count) to bound the reference's run time
    n_proc = args.processes * args.gpus
    if args.gpus > 1:
        n_proc = min(n_proc, args.processes)
    its = args.warmup + args.steps
    cfg = T.SearchConfig(n_processes=n_proc, patience=1 << 30, master_seed=args.seed, max_iterations=its,
                         forced_strategy=args.strategy).to_c()
    secs = steps = 0.0
    for comp, (nx, rows) in enumerate(systems):
        s = _abi.make_system(nx, rows)
        rec = _abi.make_record(T.naive_cost(rows) + 1)
        it, st, tot = C.c_int32(), C.c_uint64(), C.c_double()
        isecs = (C.c_double * its)()
        isteps = (C.c_uint64 * its)()
        rc = ref.ref_optimize_system_timed(C.byref(s), C.byref(cfg), comp, threads, 0.0, C.byref(rec), C.byref(it),
                                           C.byref(st), C.byref(tot), isecs, isteps, its)
        if rc:
            raise RuntimeError(ref.ref_last_error().decode())
        secs += sum(isecs[args.warmup:its])
        steps += sum(isteps[args.warmup:its])
    value = steps / secs if secs > 0 else 0.0
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "substitution steps/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": secs / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int32", "data": "synthetic (fixed public scheme)",
        "config": config_block(args, args.gpus),
        "cpu_baseline": {"value": value, "unit": "substitution steps/s", "cores": threads, "kind": "reference",
                         "sample": "iterations %d..%d of optimize_system on U, V, W (sequential, as "
                                   "optimize_scheme runs them), %d processes each (GPU arm: %d), threads=%d"
                                   % (args.warmup + 1, its, n_proc, args.processes * args.gpus, threads)},
        "e2e": {"value": value, "unit": "substitution steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "substitution_steps": int(steps),
    }
    print(json.dumps(line))
    return 0


def cpu_baseline_sample(args):
    """Bounded sample of the same workload on the reference CPU path: the
    first optimize_system iteration of U, V and W with every host thread."""
    from oracle_lib import reference
    import paper_2512_13365_b200 as T
    from paper_2512_13365_b200 import _abi
    ref = reference()
    threads = os.cpu_count() or 1
    scheme, systems = load_systems(args.workload)
    # bounded sample (~seconds): large schemes cost far more per process on the CPU
    n_cpu = min(args.processes, 16384 if scheme["r"] < 100 else 512)
    cfg = T.SearchConfig(n_processes=n_cpu, patience=1 << 30, master_seed=args.seed,
                         max_iterations=1, forced_strategy=args.strategy).to_c()
    secs = steps = 0.0
    for comp, (nx, rows) in enumerate(systems):
        s = _abi.make_system(nx, rows)
        rec = _abi.make_record(T.naive_cost(rows) + 1)
        it, st, tot = C.c_int32(), C.c_uint64(), C.c_double()
        rc = ref.ref_optimize_system_counted(C.byref(s), C.byref(cfg), comp, threads, 0.0, C.byref(rec),
                                             C.byref(it), C.byref(st), C.byref(tot))
        if rc:
            raise RuntimeError(ref.ref_last_error().decode())
        secs += tot.value
        steps += st.value
    return {"value": steps / secs if secs > 0 else 0.0, "unit": "substitution steps/s", "cores": threads,
            "kind": "reference",
            "sample": "iteration 1 of optimize_system on U, V, W (%d processes each, %.0f steps, %.1f s), "
                      "threads=%d, oracle/_ref built from the reference headers with its Release flags"
                      % (n_cpu, steps, secs, threads)}


# ----------------------------------------------------------------- GPU arm

def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist
    import paper_2512_13365_b200 as T

    n_dev = max(1, torch.cuda.device_count())
    if args.dist_backend == "auto":
        args.dist_backend = "nccl" if world <= n_dev else "gloo"
    local = local % n_dev  # identity with one rank per GPU
    torch.cuda.set_device(local)
    if world > 1:
        # torch.distributed is plumbing only (unique-id broadcast, barriers,
        # the max-over-ranks timing); the search's own exchange is the
        # library's ncclAllGather inside the iteration graph
        dist.init_process_group("gloo")

    def barrier():
        if world > 1:
            dist.barrier()

    dev = T.Device(local)
    if world > 1 and args.dist_backend == "nccl":
        uid = [T.Device.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        dev.set_nccl(uid[0], rank, world)
    elif world > 1:
        # ranks sharing a GPU (NCCL refuses that): host all-gather over gloo
        def allgather(data):
            parts = [None] * world
            dist.all_gather_object(parts, data)
            return parts
        dev.set_partition(rank, world, allgather)
    stream = torch.cuda.current_stream()
    dev.set_stream(stream.cuda_stream)

    def step(search):
        """One optimize_system iteration; returns the number of active systems."""
        return search.step()
    _, sys_rows = load_systems(args.workload)
    systems = [T.LinearSystem(nx, rows) for nx, rows in sys_rows]
    n_total = args.processes * world
    cfg = T.SearchConfig(n_processes=n_total, patience=1 << 30, master_seed=args.seed, forced_strategy=args.strategy)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    search = T.Search(systems, cfg, [0, 1, 2], device=dev)
    for _ in range(args.warmup):
        step(search)
    torch.cuda.synchronize()
    s0 = search.stats()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.15)
    # each timed step: L2 flush, barrier + synchronize, one iteration (the
    # captured graph: prep, place, search, pack, [all-gather], barrier
    # kernels), synchronize + barrier.  Its device time is the library's CUDA
    # events recorded on the launch stream right before and right after the
    # iteration's launches (stats step_ms); the outer torch events also span
    # the host's synchronisation turnaround and are reported beside it.
    outer_ms = 0.0
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    for _ in range(args.steps):
        flush.zero_()
        barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        step(search)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        outer_ms += e0.elapsed_time(e1)
    s1 = search.stats()
    total_ms = s1["step_ms"] - s0["step_ms"]
    delta = lambda k: s1[k] - s0[k]  # noqa: E731
    steps_local = delta("steps")
    wops = delta("wops")
    group = []  # per launch group: search-kernel span (device clock) and word-ops
    for g in range(s1["n_groups"]):
        group.append({"nt": s1["group_nt"][g], "words": s1["group_words"][g],
                      "ms": s1["group_ms"][g] - s0["group_ms"][g], "wops": s1["group_wops"][g] - s0["group_wops"][g]})
    kernel_ms = delta("kernel_ms")
    exchange_ms = delta("exchange_ms")
    launches_counted = delta("kernel_launches")
    by_strategy = [a - b for a, b in zip(s1["steps_by_strategy"], s0["steps_by_strategy"])]
    results, _ = search.result()
    search.close()

    # ---- e2e: the public session API on the product path (the device-
    # resident loop) over the SAME iterations as `value`: host CSR in (create
    # uploads the systems), W warm-up iterations untimed, iterations W+1..W+K
    # as one run() (graph replays, one host synchronisation), host records
    # out.  Timed: create + run(K) + result, host clock.
    e2e = None
    if not args.no_e2e:
        barrier()
        torch.cuda.synchronize()
        cfg2 = T.SearchConfig(n_processes=n_total, patience=1 << 30, master_seed=args.seed,
                              forced_strategy=args.strategy)
        t0 = time.perf_counter()
        s2 = T.Search(systems, cfg2, [0, 1, 2], device=dev)
        t_create = time.perf_counter() - t0
        s2.run(args.warmup)
        st_w = s2.stats()
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        s2.run(args.steps)
        res2, st2 = s2.result()
        t_run = time.perf_counter() - t1
        s2.close()
        e2e = {"steps": st2["steps"] - st_w["steps"], "secs": t_create + t_run,
               "h2d": st2["h2d_bytes"],  # create's uploads (warm-up iterations copy nothing in)
               "d2h": st2["d2h_bytes"] - st_w["d2h_bytes"], "syncs": st2["host_syncs"] - st_w["host_syncs"],
               "graph": st2["graph_launches"] - st_w["graph_launches"],
               "same_result": [r.cost for r, _ in res2] == [r.cost for r, _ in results]}
    clk = clocks.stop()
    peak_gops = dev.microbench_wordops()
    pipes = dev.microbench_pipes()

    # ---- cross-rank aggregation (max time, summed work)
    vals = torch.tensor([total_ms, float(steps_local), float(wops), kernel_ms,
                         e2e["secs"] if e2e else 0.0, float(e2e["steps"] if e2e else 0)], dtype=torch.float64)
    if world > 1:
        mx = vals.clone()
        sm = vals.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
    else:
        mx = sm = vals
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0
    t_ms = mx[0].item()
    steps_all = sm[1].item()
    value = steps_all / (t_ms / 1e3)
    # roofline of the dominant kernel: the search kernel of the launch group
    # with the longest span (device clock).  achieved = algorithmic word-ops
    # of that group's processes (SURVEY.md 8(d) model, counted by the kernel)
    # / its summed launch span, vs the measured smem word-op peak; the other
    # groups are listed with their own fractions
    for g in group:
        g["achieved_gops"] = g["wops"] / (g["ms"] / 1e3) / 1e9 if g["ms"] > 0 else 0.0
        g["frac"] = g["achieved_gops"] / peak_gops if peak_gops else None
        g["avg_launch_ms"] = g["ms"] / args.steps
        g["kernel"] = "search_kernel<W=%d,NT=%d>" % (g["words"], g["nt"])
    dom = max(group, key=lambda g: g["ms"]) if group else None
    traffic = None
    prof = os.path.join(ROOT, "profiles", "search_kernel_dram.json")
    if os.path.exists(prof):
        with open(prof) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")
    # the binding resource is instruction issue, not smem bandwidth: the
    # newest committed ncu capture of the same kernel gives issue / occupancy
    issue = None
    caps = []
    for name in os.listdir(os.path.join(ROOT, "profiles")):
        m = re.match(r"r(\d+)_v(\d+)_search_kernel_ncu\.json$", name)
        if m:
            caps.append(((int(m.group(1)), int(m.group(2))), name))
    if caps:
        name = max(caps)[1]
        with open(os.path.join(ROOT, "profiles", name)) as f:
            nj = json.load(f)
        pct = lambda k: float(str(nj.get(k, "nan")).split()[0])  # noqa: E731
        issue = {"issue_active_pct": pct("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                 "warps_active_pct": pct("sm__warps_active.avg.pct_of_peak_sustained_active"),
                 "alu_pipe_pct": pct("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
                 "lsu_pipe_pct": pct("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
                 "smem_wavefronts_pct": pct(
                     "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
                 "source": "profiles/" + name}
    line = {
        "metric": METRIC, "value": value, "unit": "substitution steps/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
        "data": "synthetic (fixed public scheme; search randomness from the seed only)",
        "config": config_block(args, world),
        "roofline": {"bound": "smem", "achieved": dom["achieved_gops"] if dom else None, "peak": peak_gops,
                     "unit": "Gword-ops/s", "frac": dom["frac"] if dom else None, "traffic": traffic,
                     "peak_source": "in-repo microbenchmark (tcse_microbench_wordops) on this GPU",
                     "kernel": dom["kernel"] if dom else None,
                     "groups": group,
                     "kernel_share_of_step": kernel_ms / max(1e-9, total_ms),
                     "host_turnaround_ms_per_step": (outer_ms - total_ms) / args.steps,
                     "timing": "device clock (%globaltimer): first block start to last block end of each "
                               "group's search launch, summed over the timed iterations",
                     "ncu_issue": issue,
                     "pipe_peaks_gops": pipes,
                     "pipe_peaks_source": "tcse_microbench_pipes on this GPU: G thread-ops/s of IADD3, LOP3, "
                                          "POPC(+XOR), SHFL, LDS.32, LDS.64 (8 independent chains per thread, "
                                          "every SM at full occupancy)"},
        "clocks": clk,
        # counted by the library while enqueueing the timed iterations: per
        # launch group prep + place + search, per iteration pack + barrier
        "gpu_launches": int(launches_counted),
        "substitution_steps": int(steps_all),
        "steps_by_strategy": dict(zip(T.STRATEGY_SHORT, by_strategy)),
        "exchange_us_per_step": exchange_ms * 1e3 / args.steps,
        "incumbent_costs": [r.cost for r, _ in results],
    }
    if e2e:
        line["e2e"] = {"value": sm[5].item() / mx[4].item(), "unit": "substitution steps/s",
                       "h2d_bytes_per_step": e2e["h2d"] / args.steps, "d2h_bytes_per_step": e2e["d2h"] / args.steps,
                       "call": "tcse_search_create (host CSR in) + tcse_search_run over iterations %d..%d (CUDA "
                               "graph replays, %d host sync) + tcse_search_result (host records out); the %d "
                               "warm-up iterations run untimed in the same session"
                               % (args.warmup + 1, args.warmup + args.steps, e2e["syncs"], args.warmup),
                       "same_incumbents_as_value_run": e2e["same_result"]}
    if world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline_sample(args)
        except Exception as e:  # the checker must not take the bench down
            line["cpu_baseline"] = {"value": None, "error": str(e)}
    print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
