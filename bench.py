"""bench.py -- noisy trajectories/s of config 2 (BASELINE.json configs[1]).

Workload: 20-qubit Sycamore-style random circuit, 14 cycles,
approximate QCS noise model (decay/dephasing triple on every qubit after every
moment, 1q/2q depolarizing after gates, fSim coherent errors, readout errors),
10^4 trajectories per GPU per step (rank r of N runs trajectories r + N j,
j < 10^4: the job's trajectory indices interleave over the ranks),
1 shot per trajectory + <Z_q> for every qubit.  Synthetic, seeded inputs.

A step = one pass of the whole hot path over each rank's 10^4 trajectories: Alg. 2
draws + delayed-inner-product classification + fusion (host, overlapped),
fused tile passes with on-device rho_Q/choose (K1/K2), block sums,
observables (K4), chain-rule sampling + readout (K3), records to the host.
Weak scaling (trajectories are independent units, no data-path
collective; one all-reduce of observable sums per step): per-GPU work is fixed,
value = N * 10^4 trajectories / step time (max over ranks).

At N > 1 the line also carries "strong": C2's own split (10^4 trajectories over
the N GPUs, 10^4 / N per rank).  Extra keys (driver-visible numbers of the other
BASELINE configs): "c1" (GHZ-4, 1000 trajectories), "c3" (26-qubit low-noise grid at
f = 4 and f = 6), "c4" (one 32-qubit noisy trajectory) and the gate-pass HBM sweep at
n = 32 (C4 (i)); "plan" = host planning cost per trajectory (one core) and whether it
hides behind the device work.

`python bench.py --impl reference` times the CPU oracle (plain fp64 C, one
trajectory per host core) on the same workload: the reference arm of this tier.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads  # noqa: E402

CONFIG = 2
TENSOR_CORES = 0  # qt_fuse_opts.tensor_cores (set from --tensor-cores)
TOTAL_TRAJ = 10_000
N_QUBITS = 20
METRIC = "noisy trajectories/s (C2: 20q Sycamore-style depth-14, approximate QCS noise)"
UNIT = "trajectories/s"
CLOCK_QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
               "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
               "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured"
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={CLOCK_QUERY}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        smax = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for i, nm in enumerate(names):
                if len(r) > 5 + i and r[5 + i].lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


def rank_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def my_share(rank, world):
    return rank, world, TOTAL_TRAJ  # traj_begin, stride, count (weak scaling: 10^4 per rank)


def run_oracle_sample(circ, seed, count, begin, stride, threads):
    import oracle
    t0 = time.perf_counter()
    r = oracle.run_trajectories(circ, seed=seed, traj_begin=begin, stride=stride, traj_count=count, shots=1,
                                threads=threads)
    dt = time.perf_counter() - t0
    assert r["rc"] == 0
    return dt


def bench_reference(args):
    rank, world, _ = rank_env()
    if rank != 0:
        return  # rank 0 alone runs the CPU oracle
    circ = workloads.sycamore_grid_qcs(config=CONFIG)
    seed = workloads.trajectory_seed(CONFIG)
    cores = os.cpu_count() or 1
    per_step = cores  # one trajectory per host core per step (bounded sample)
    for w in range(args.warmup):
        run_oracle_sample(circ, seed, per_step, w * 97, 1009, cores)
    tot = 0.0
    for s in range(args.steps):
        tot += run_oracle_sample(circ, seed, per_step, 13 + s * 131, 997, cores)
    value = per_step * args.steps / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded C2 generator)",
        "config": {"workload": "C2 20q sycamore-grid depth14 QCS-noise", "trajectories_per_step": per_step,
                   "l2": "n/a (CPU)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": f"{per_step} trajectory indices per step, one per core, plain fp64 C oracle"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def build_plan(circ, f):
    from paper_2111_02396_b200 import qtraj
    c = qtraj.Circuit.from_description(circ)
    return c, qtraj.Plan(c, max_fused=f, tensor_cores=TENSOR_CORES)


def circuit_bytes(circ):
    b = 0
    for op in circ.ops():
        if hasattr(op, "kraus"):
            b += sum(np.asarray(k).size * 16 for k in op.kraus)
        else:
            b += np.asarray(op.matrix).size * 16
    return b + 2 * 8 * circ.n_qubits


def gate_pass_sweep(ctx, n, dev, hbm_peak, reps=10):
    """Isolated K1 passes of Haar k-qubit gates, k = 1..6, placements all-low,
    all-high and one random mixed; GB/s = 2^(n+4) / t."""
    import torch
    rng = np.random.default_rng(workloads.circuit_seed(4))
    state = torch.zeros(1 << n, dtype=torch.complex64, device=dev)
    state[0] = 1.0
    rows = []
    for k in range(1, 7):
        places = {"low": list(range(k)), "high": list(range(n - k, n)),
                  "mixed": sorted(int(x) for x in rng.choice(n, size=k, replace=False))}
        for name, qs in places.items():
            U = workloads.haar_unitary(rng, 2 ** k)
            ms = ctx.apply_gate(state, qs, U, repeats=reps + 1)  # first application = warm-up
            gbs = 2.0 ** (n + 4) / (ms / 1e3) / 1e9
            rows.append({"k": k, "placement": name, "qubits": qs, "ms": ms, "gbs": gbs, "frac": gbs / hbm_peak})
    torch.cuda.synchronize()
    best = max(r["gbs"] for r in rows)
    med = float(np.median([r["gbs"] for r in rows]))
    return {"n": n, "bytes_per_pass": 2 ** (n + 4), "peak_gbs": hbm_peak, "best_gbs": best, "median_gbs": med,
            "best_frac": best / hbm_peak, "median_frac": med / hbm_peak,
            "min_frac": min(r["frac"] for r in rows),
            "kernel": "gate_stream_kernel<K> (qt_apply_gate: TMA tensor-map tiles, tcgen05 f16 hi/lo GEMM, K = max(k, 5) on n >= 12)",
            "k4_median_frac": float(np.median([r["frac"] for r in rows if r["k"] <= 4])), "rows": rows}


def other_configs(ctx, dev, host_threads):
    """Driver-visible numbers of BASELINE configs 1, 3 and 4 (ii):
    device-timed trajectories/s of one launch sequence each (inputs resident)."""
    import torch
    from paper_2111_02396_b200 import qtraj
    out = {}

    def timed(circ, f, count, batch, seed, reps=2):
        c = qtraj.Circuit.from_description(circ)
        plan = qtraj.Plan(c, max_fused=f)
        st = torch.empty(batch << circ.n_qubits, dtype=torch.complex64, device=dev)
        ctx.run_trajectories(plan, st, seed=seed, traj_count=min(count, batch), shots=1, batch=batch,
                             observables=circ.observables, host_threads=host_threads)  # warm-up
        best = None
        for _ in range(reps):
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            o = ctx.run_trajectories(plan, st, seed=seed, traj_count=count, shots=1, batch=batch,
                                     observables=circ.observables, host_threads=host_threads)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            best = ms if best is None else min(best, ms)
        info = plan.info(seed, 0)
        s = o["stats"]
        del st
        torch.cuda.empty_cache()
        return {"trajectories": count, "ms": best, "traj_per_s": count / (best / 1e3),
                "passes_per_traj": s["passes"] / max(count, 1), "fused_gates_per_traj": s["fused_gates"] / max(count, 1),
                "reductions_per_traj": s["reductions"] / max(count, 1), "tile_bits": int(info["tile_bits"]),
                "kernel": int(info["kernel"])}

    out["c1"] = dict(workload="C1 GHZ-4 + depolarize(0.01)",
                     **timed(workloads.ghz4_depolarized(0.01), 4, 1000, 1000, workloads.trajectory_seed(1)))
    c3 = workloads.low_noise_grid()
    out["c3"] = {"workload": "C3 26q 2x13 low-noise grid, 20 cycles"}
    for f in (4, 6):
        out["c3"][f"f{f}"] = timed(c3, f, 128, 32, workloads.trajectory_seed(3))
    c4 = workloads.low_noise_grid(rows=4, cols=8, config=4, damping="amplitude")
    out["c4"] = dict(workload="C4 (ii) one 32q noisy trajectory (4x8 grid, 20 cycles, depolarize + amplitude damping)",
                     **timed(c4, 4, 1, 1, workloads.trajectory_seed(4), reps=1))
    return out


def bench_gpu(args):
    import torch
    import torch.distributed as dist
    from paper_2111_02396_b200 import dispatch, qtraj
    rank, world, local = rank_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    circ = workloads.sycamore_grid_qcs(config=CONFIG)
    seed = workloads.trajectory_seed(CONFIG)
    obs = circ.observables
    begin, stride, count = my_share(rank, world)
    ctx = qtraj.Context(local)
    _, plan = build_plan(circ, args.fuse)
    batch = args.batch
    state = torch.empty(batch << N_QUBITS, dtype=torch.complex64, device=dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    stream = torch.cuda.current_stream(dev)

    # host planning threads: the node's cores split over the ranks on it (no oversubscription)
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
    host_threads = max(1, (len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else
                           (os.cpu_count() or 1)) // max(local_world, 1))

    def step(profile):
        out = ctx.run_trajectories(plan, state, seed=seed, traj_count=count, traj_begin=begin, traj_stride=stride,
                                   shots=1, batch=batch, observables=obs, profile=profile,
                                   host_threads=host_threads)
        # job output: per-observable sums over this rank's trajectories, reduced over ranks
        sums = torch.tensor(np.concatenate([out["obs"].sum(0), (out["obs"] ** 2).sum(0)]), device=dev,
                            dtype=torch.float64)
        if world > 1:
            dist.all_reduce(sums)
        return out, sums

    for _ in range(args.warmup):
        step(False)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    times, stats = [], []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.fill_(1)  # L2 flush between timed steps (outside the events)
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            out, sums = step(True)
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
            stats.append(out["stats"])
    tot_ms = float(np.sum(times))
    t = torch.tensor([tot_ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    tot_ms = float(t.item())
    value = world * TOTAL_TRAJ * args.steps / (tot_ms / 1e3)

    # ---- strong scaling (C2's own split: 10^4 trajectories over the N GPUs)
    strong = None
    if world > 1:
        sb, ss, sc = dispatch.shard(TOTAL_TRAJ, rank, world)
        s_times = []
        for _ in range(max(1, min(args.steps, 3))):
            flush.fill_(1)
            torch.cuda.synchronize()
            dist.barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ctx.run_trajectories(plan, state, seed=seed, traj_count=sc, traj_begin=sb, traj_stride=ss, shots=1,
                                 batch=batch, observables=obs, host_threads=host_threads)
            e1.record(stream)
            torch.cuda.synchronize()
            s_times.append(e0.elapsed_time(e1))
        ts = torch.tensor([float(np.mean(s_times))], device=dev, dtype=torch.float64)
        dist.all_reduce(ts, op=dist.ReduceOp.MAX)
        strong = {"value": TOTAL_TRAJ / (float(ts.item()) / 1e3), "unit": UNIT, "ms_per_step": float(ts.item()),
                  "trajectories_per_step": TOTAL_TRAJ, "trajectories_per_gpu": TOTAL_TRAJ // world,
                  "scaling": "strong"}

    # ---- e2e: host circuit arrays -> C ABI (upload, fuse, run) -> records of every rank
    # merged through the dispatcher (one all-gather) -> host aggregate (mean, stderr)
    e2e_times = []
    for _ in range(max(1, min(args.steps, 2))):
        flush.fill_(1)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        c2, plan2 = build_plan(circ, args.fuse)

        def runner(b, s_, n_):
            return ctx.run_trajectories(plan2, state, seed=seed, traj_count=n_, traj_begin=b, traj_stride=s_,
                                        shots=1, batch=batch, observables=obs, host_threads=host_threads)
        merged = dispatch.run_sharded(runner, world * TOTAL_TRAJ, device=dev if world > 1 else None)
        mean, se = dispatch.aggregate(merged["obs"])
        e1.record(stream)
        torch.cuda.synchronize()
        e2e_times.append(e0.elapsed_time(e1))
        del c2, plan2, mean, se, merged
    te = torch.tensor([float(np.mean(e2e_times))], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = world * TOTAL_TRAJ / (float(te.item()) / 1e3)

    # ---- host planning cost (Alg. 2 first loop + fusion + passes), one core
    pinfo = plan.info(seed, 0)
    NPL = 1000  # one core, one reused program (as the runtime's per-slot programs); best of 3
    plan_core_ms = min(1e3 * plan.plan_seconds(seed, 17 + NPL * r, NPL) / NPL for r in range(3))
    st0 = stats[-1]
    h2d = circuit_bytes(circ) + st0["h2d_bytes"]  # circuit upload + plan tables + trajectory programs
    d2h = st0["d2h_bytes"]                        # bitstrings, Kraus records, observables, status

    # ---- roofline of the dominant kernel (tile pass), from the timed steps
    peaks, peak_src = load_peaks()
    pass_ms = sum(s["pass_kernel_ms"] for s in stats)
    pass_launches = sum(s["pass_launches"] for s in stats)
    alg_bytes = sum(s["alg_bytes"] for s in stats)
    alg_flops = sum(s["alg_flops"] for s in stats)
    achieved_gbs = alg_bytes / (pass_ms / 1e3) / 1e9
    achieved_tf = alg_flops / (pass_ms / 1e3) / 1e12
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    clocks = clk.summary()
    mhz = clocks["sm_mhz"] or float(peaks.get("clocks_under_load", {}).get("sm_mhz_median", 1320.0))
    fp32_peak_tf = 148 * 128 * 2 * mhz * 1e6 / 1e12  # B200: 148 SMs x 128 FP32 lanes x FMA, at the sampled clock
    frac_hbm = achieved_gbs / hbm_peak
    frac_alu = achieved_tf / fp32_peak_tf
    # With the tensor-core K1 (default for f <= 5) the fused-gate arithmetic is not
    # on the FP32 pipes; the pass is then reported against its HBM roofline (every
    # pass must move 2^(n+4) bytes).  The CUDA-core K1 reports the larger
    # of its FP32-issue and HBM fractions.
    if frac_alu > frac_hbm and not args.tensor_cores_on:
        roof = {"bound": "alu", "achieved": achieved_tf, "peak": fp32_peak_tf, "unit": "TFLOP/s",
                "frac": frac_alu, "traffic": None,
                "peak_source": f"derived: 148 SM x 128 FP32 lanes x 2 flop x {mhz:.0f} MHz (sampled)",
                "hbm": {"achieved_gbs": achieved_gbs, "peak_gbs": hbm_peak, "frac": frac_hbm,
                        "peak_source": peak_src}}
    else:
        roof = {"bound": "hbm", "achieved": achieved_gbs, "peak": hbm_peak, "unit": "GB/s", "frac": frac_hbm,
                "traffic": None, "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_src})",
                "fp32_equivalent": {"achieved_tflops": achieved_tf, "peak_tflops": fp32_peak_tf, "frac": frac_alu,
                                     "note": "fused-gate flops (P:135) vs the FP32 pipes; context only: the tensor-core K1 runs them on tcgen05"}}
    # second in-SM resource of the tensor-core K1: every fused gate's epilogue reads its
    # accumulator D from TMEM -- 16 B per amplitude for the per-tile kernel (64 fp32
    # columns per 16-amplitude row), 8 B for the persistent kernel (32 columns) -- against
    # the measured tcgen05.ld throughput, 415 B/cycle/SM with 8 warps x 4 CTAs
    # (profiles/r2_ubench_sm.txt; the B300 table's 64 B/cycle does not hold on B200)
    if args.tensor_cores_on:
        fused = sum(s["fused_gates"] for s in stats)
        bpa = 8 if pinfo["kernel"] == 13 else 16
        tmem_bytes = fused * (1 << N_QUBITS) * float(bpa)
        tmem_peak = 415.0 * 148 * mhz * 1e6 / 1e9
        tmem_gbs = tmem_bytes / (pass_ms / 1e3) / 1e9
        roof["tmem_read"] = {"achieved_gbs": tmem_gbs, "peak_gbs": tmem_peak, "frac": tmem_gbs / tmem_peak,
                             "bytes_per_amplitude_gate": bpa,
                             "peak_source": f"measured: 415 B/cycle/SM tcgen05.ld (profiles/r2_ubench_sm.txt) x 148 SM x {mhz:.0f} MHz"}
    # traffic: DRAM bytes per launch from the committed ncu --set full capture,
    # scaled to this run's average launch (ratio dram/algorithmic of that capture)
    tpath = os.path.join(ROOT, "profiles", "r2_traffic.json")
    if not os.path.exists(tpath):
        tpath = os.path.join(ROOT, "profiles", "r1_traffic.json")
    if os.path.exists(tpath):
        tr = json.load(open(tpath))
        roof["traffic"] = tr["ratio"] * alg_bytes / max(pass_launches, 1)
        roof["traffic_unit"] = "bytes/launch"
        roof["traffic_source"] = tr["source"]
    roof["alg_bytes_per_launch"] = alg_bytes / max(pass_launches, 1)
    roof["kernel"] = ("tile_pass_v2_kernel (persistent TMEM kernel, 13-qubit tiles)" if pinfo["kernel"] == 13 else
                      ("tile_pass_kernel<12,5,tensor-core,%d>" % pinfo["kernel"]) if pinfo["kernel"] else
                      "tile_pass_kernel<12,4> (CUDA cores)")
    roof["launches_timed"] = int(pass_launches)
    roof["avg_launch_ms"] = pass_ms / max(pass_launches, 1)
    roof["share_of_step"] = pass_ms / tot_ms if tot_ms else None

    # ---- gate-pass HBM GB/s vs peak (second half of the metric; SURVEY 8(d) C4 sweep
    # at n = sweep_n): one fused k-qubit Haar gate per HBM sweep, 2^(n+4) bytes per pass
    sweep = None
    extra = {}
    if rank == 0 and args.sweep_n > 0:
        del state
        torch.cuda.empty_cache()
        sweep = gate_pass_sweep(ctx, args.sweep_n, dev, hbm_peak)
        torch.cuda.empty_cache()
    if rank == 0 and not args.no_configs:
        extra = other_configs(ctx, dev, host_threads)

    # ---- CPU oracle baseline (rank 0, N = 1 only, bounded sample)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cores = os.cpu_count() or 1
        dt = run_oracle_sample(circ, seed, cores, 17, 613, cores)
        cpu = {"value": cores / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
               "sample": f"{cores} C2 trajectory indices (17 + 613 j), one per host core, fp64 C oracle, {dt:.1f} s"}
    if rank == 0:
        st = {k: float(np.mean([s[k] for s in stats])) for k in stats[0]}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": tot_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None,
            "dtype": "complex64 state; gate products as f16 hi/lo splits (x_hi W_hi + x_lo W_hi + x_hi W_lo, "
                     "~22-bit), fp32 accumulate; fp64 reductions",
            "data": "synthetic (seeded C2 generator; SURVEY 8(d))",
            "config": {"workload": "C2 20q sycamore-grid depth14 QCS-noise",
                       "trajectories_per_step": TOTAL_TRAJ * world, "trajectories_per_gpu": TOTAL_TRAJ,
                       "n_qubits": N_QUBITS, "max_fused": args.fuse, "tile_bits": int(pinfo["tile_bits"]),
                       "batch": batch,
                       "shots_per_traj": 1, "observables": len(obs), "parallelism": f"traj{world}",
                       "host_threads_per_rank": host_threads,
                       "l2": "flushed between timed steps (512 MB write)"},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)},
            "gpu_launches": int(sum(s["launches"] for s in stats)),
            "roofline": roof,
            "cpu_baseline": cpu,
            "gate_pass_sweep": sweep,
            "strong": strong,
            "plan": {"core_ms_per_traj": plan_core_ms, "wall_ms_per_step": st["plan_ms"],
                     "host_threads": host_threads, "device_ms_per_step": st["device_ms"],
                     "hidden": st["plan_ms"] < st["device_ms"],
                     "note": "planning of batch i+1 overlaps batch i on the device; core_ms = one host core"},
            "c1": extra.get("c1"), "c3": extra.get("c3"), "c4": extra.get("c4"),
            "clocks": clocks,
            "per_step_stats": {"passes_per_traj": st["passes"] / max(st["trajectories"], 1),
                               "fused_gates_per_traj": st["fused_gates"] / max(st["trajectories"], 1),
                               "reductions_per_traj": st["reductions"] / max(st["trajectories"], 1),
                               "deferral_fraction": st["channels_deferred"] / max(
                                   st["channels_deferred"] + st["channels_conventional"], 1),
                               "plan_ms": st["plan_ms"], "device_ms": st["device_ms"],
                               "pass_kernel_ms": st["pass_kernel_ms"]},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--fuse", type=int, default=4)
    ap.add_argument("--tensor-cores", type=int, default=0, help="0 auto, 1 on, -1 CUDA-core K1")
    ap.add_argument("--batch", type=int, default=384)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sweep-n", type=int, default=32, help="qubits of the gate-pass bandwidth sweep (0 = skip)")
    ap.add_argument("--no-configs", action="store_true", help="skip the C1 / C3 / C4 extra keys")
    args = ap.parse_args()
    global TENSOR_CORES
    TENSOR_CORES = args.tensor_cores
    args.tensor_cores_on = args.tensor_cores >= 0 and args.fuse <= 5  # n = 20 >= 12: auto enables them
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        bench_reference(args)
    else:
        bench_gpu(args)


if __name__ == "__main__":
    main()
