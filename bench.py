#!/usr/bin/env python3
"""Benchmark of the lighting-matrix hot path (arXiv 2202.12567) on B200.

A step = one frame of the whole hot path: lmc_build_slices,
lmc_sample_pass1, lmc_coarsen_cut, lmc_sample_pass2, lmc_complete, lmc_resolve_image (for N > 1
inside it: the NCCL gather of every rank's packed rows to rank 0 and the scatter into the image),
on one batch of seeded synthetic input (scenegen) resident in HBM.  N = 2^k ranks each slice only
the top k levels of the whole G-buffer, then their own subtree.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--solver adm|mals]
  python bench.py --impl reference ...     # the fp64 CPU oracle on a bounded sample

Prints ONE JSON line (rank 0).  metric/unit: BASELINE.json's "ms/frame and lighting-matrix
entries completed/s"; value = sum_s m_s n_s (entries of the completed slice matrices of the
whole frame) / (ms/frame); ms_per_step = ms/frame.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ms/frame and lighting-matrix entries completed/s at 1/2/4/8 B200"
UNIT = "entries/s"
FP32_PEAK_DERIVED = 148 * 128 * 2 * 1.965e9 / 1e12   # 74.4: 148 SMs x 128 FP32 lanes x FMA x max clock


def _microbench(key):
    try:
        return float(json.load(open(os.path.join(ROOT, "profiles", "r01_peaks.json")))[key])
    except Exception:
        return None


def fp32_peak():
    """FP32 roofline peak derived from the unit counts and the max clock (the task's rule for an
    ALU-bound path: MEASURED_PEAKS.json holds no FP32 figure); the FMA microbenchmark of this pool
    (tools/peaks.cu, profiles/r01_peaks.json: 71.0 TF/s, 95% of it) is reported beside it."""
    return FP32_PEAK_DERIVED, "derived: 148 SMs x 128 FP32 FMA lanes x 2 x 1.965 GHz", _microbench("fp32_fma_tflops")


def fp64_peak():
    """FP64 roofline peak derived the same way (half the FP32 rate: 64 FP64 FMA lanes per SM); the
    microbenchmark (34.2 TF/s, 92%) beside it."""
    return FP32_PEAK_DERIVED / 2, "derived: 148 SMs x 64 FP64 FMA lanes x 2 x 1.965 GHz", _microbench("fp64_fma_tflops")


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", default="c4")
    p.add_argument("--solver", default="adm", choices=["adm", "mals"])
    p.add_argument("--impl", default="lmc", choices=["lmc", "reference"])
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-sample-slices", type=int, default=0)
    return p.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu):
        self.gpu = gpu
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([s.strip() for s in line.split(",")])

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.t.join(timeout=2)
        sm = [float(r[1]) for r in self.rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            if len(r) < 9:
                continue
            for k, nm in enumerate(names):
                if r[5 + k].lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


def adm_flops(q, sum_N, sum_m, sum_n, nslices, iters):
    """Algorithmic flops of ADM per frame: per iteration and slice
    6 q N (SDDMM + S Y^T + X^T S) + 6 m q^2 (X update + 2 Grams) + 6 n q^2 (Y update + Gram)
    + 2 q^3 (two q x q SPD inverses)."""
    return iters * (6.0 * q * sum_N + 6.0 * q * q * sum_m + 6.0 * q * q * sum_n + 2.0 * q ** 3 * nslices)


def adm_flops_survey(q, sum_N, sum_m, sum_n, nslices, iters):
    """the SURVEY §8(a) a7 count per iteration and slice: 6 q N + 8 m q^2 + 6 n q^2 + 2/3 q^3 (it
    forms X_k^T G_Y as well; the kernel's reformulation saves that product)"""
    return iters * (6.0 * q * sum_N + 8.0 * q * q * sum_m + 6.0 * q * q * sum_n + (2.0 / 3.0) * q ** 3 * nslices)


def entry_flops_per_entry(x, fr, nslices=8):
    """Mean fp64 operations (+ - * / sqrt, as the oracle's entry function executes them: early exits
    taken, primitives tested until the first hit) over a sample of the pairs this frame evaluated:
    pass 1 + coarsening (rows of every processed candidate x the reps of its two children, from the
    oracle's record of the same slices) and pass 2 (the frame's new samples)."""
    import oracle
    o = oracle.Oracle(x)
    off, rows = fr.slices()
    st = fr.stats()
    s0, s1 = int(st["slice_begin"]), int(st["slice_end"])   # this rank's slices
    ids = sorted(set(np.linspace(s0, s1 - 1, min(nslices, s1 - s0)).astype(int).tolist()))
    t = x.tree
    r1, v1, r2, v2 = [], [], [], []
    for r in o.run_slices(ids, stage=1):
        for k, f in enumerate(r["proc_node"]):
            z = r["rows"][r["proc_zrows"][r["proc_zoff"][k]:r["proc_zoff"][k + 1]]]
            for ch in (t["left"][f], t["right"][f]):
                r1.append(z)
                v1.append(np.full(z.size, t["rep"][ch], np.int32))
    for s in ids:
        sm = fr.samples(s)
        new = sm["carried"] == 0
        cut = fr.cut(s)
        r2.append(rows[off[s] + sm["row"][new]])
        v2.append(t["rep"][cut[sm["col"][new]]].astype(np.int32))
    r1, v1, r2, v2 = (np.concatenate(a) if a else np.zeros(0, np.int32) for a in (r1, v1, r2, v2))
    if x.prims.get("tri") is not None and x.prims["tri"].shape[0]:
        # the oracle tests every triangle (brute force, no BVH): count the frame's arithmetic
        # without the mesh occluders instead — a lower bound of the BVH path's work
        import copy
        xa = copy.copy(x)
        xa.prims = dict(x.prims, tri=np.zeros((0, 9), np.float32))
        o = oracle.Oracle(xa)
    f1 = o.entry_flops(r1, v1) / max(r1.size, 1)
    f2 = o.entry_flops(r2, v2) / max(r2.size, 1)
    return f1, f2, int(r1.size), int(r2.size), len(ids)


def mals_flops(q, sum_N, sum_m, sum_n, nslices, iters):
    """per iteration and slice: Gram + rhs 2 N (q(q+1)/2 + q) twice (rows then columns)
    + (m + n)(q^3/3 + 2 q^2) (Cholesky + two triangular solves)."""
    per_sample = 2.0 * (q * (q + 1) / 2 + q)
    return iters * (2 * per_sample * sum_N + (sum_m + sum_n) * (q ** 3 / 3.0 + 2.0 * q * q))


def cpu_oracle_sample(x, nslices_sample, solver):
    """Time the fp64 oracle (as it stands) on a bounded sample of the workload's slices."""
    import oracle
    o = oracle.Oracle(x, solver=solver)
    off, _ = o.slices()
    S = off.size - 1
    ids = np.linspace(0, S - 1, min(nslices_sample, S)).astype(np.int32)
    t0 = time.perf_counter()
    res = o.run_slices(ids, stage=4)
    dt = time.perf_counter() - t0
    entries = sum(r["m"] * r["n"] for r in res)
    return entries / dt, dt, len(ids), entries


def omp_threads():
    return int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))


def run_reference(args, rank, world):
    """--impl reference: the fp64 oracle on the host cores, each step a bounded sample."""
    if rank != 0:
        return
    import scenegen
    x = scenegen.make_inputs(scenegen.preset(args.config, solver=1 if args.solver == "mals" else 0))
    cores = omp_threads()
    nsamp = args.cpu_sample_slices or max(cores, 8)
    cpu_oracle_sample(x, max(1, nsamp // 4), x.cfg.solver)   # warm-up (page-in, OpenMP pool)
    vals, times = [], []
    for _ in range(args.steps):
        v, dt, k, ent = cpu_oracle_sample(x, nsamp, x.cfg.solver)
        vals.append(v)
        times.append(dt)
    value = statistics.median(vals)
    S = len(__import__("oracle").Oracle(x).slices()[0]) - 1
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": statistics.median(times) * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": f"{args.config}: {x.width}x{x.height} px, {x.vpls['px'].size} VPLs, "
                                   f"{S} slices, q={x.cfg.rank_q}, rate={x.cfg.rate}, solver={args.solver}",
                       "sample": f"{nsamp} of {S} slices per step (whole per-slice pipeline)"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"{nsamp} of {S} slices per step"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import torch
    import torch.distributed as dist

    import scenegen
    from paper_2202_12567_b200 import lmc

    # BENCH_DIST_BACKEND=gloo + BENCH_SAME_DEVICE=1: diagnostic run of the multi-rank path with every
    # rank on GPU 0 (the production path is NCCL, one rank per GPU)
    if os.environ.get("BENCH_SAME_DEVICE") == "1":
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    solver = 1 if args.solver == "mals" else 0
    x = scenegen.make_inputs(scenegen.preset(args.config, solver=solver))
    stream = torch.cuda.current_stream(dev)
    # world > 1 over NCCL: the image gather runs inside the library (lmc_resolve_image: every rank's
    # packed rows to rank 0, one NCCL group); rank 0 makes the NCCL id, torch.distributed broadcasts it
    lib_gather = world > 1 and os.environ.get("BENCH_DIST_BACKEND", "nccl") == "nccl"
    nccl_id = None
    if lib_gather:
        idt = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            idt.copy_(torch.frombuffer(bytearray(lmc.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(idt, 0)
        nccl_id = bytes(idt.cpu().tolist())
    # world > 1: interleaved slices (rank r takes slices r, r + P, ...): the ranks' loads balance
    # (subtree shares differ by up to 1.8x in completion work at P = 8)
    part = int(os.environ.get("BENCH_PARTITION", "1"))
    fr = lmc.Frame(x, rank=rank, world=world, stream=stream, nccl_id=nccl_id, partition=part)
    fr.set_timing(True)
    npix = x.height * x.width
    img = torch.zeros(npix * 3, device=dev)
    st0 = fr.stats()
    rows_local = int(st0["rows"])
    if world > 1 and not lib_gather:   # diagnostic gloo transport (BENCH_DIST_BACKEND=gloo)
        from paper_2202_12567_b200 import dist as pdist
        counts = pdist.row_counts(fr.partition()[1])
        tile = torch.zeros(rows_local * 4, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)   # > L2 (126 MB)

    def frame_once():
        fr.build_slices()
        fr.sample_pass1()
        fr.coarsen_cut()
        fr.sample_pass2()
        fr.complete()
        if world == 1 or lib_gather:
            fr.resolve_image(img)
        else:
            fr.resolve_rows(tile)
            all_rows = pdist.gather_rows(tile, counts)
            if rank == 0:
                fr.scatter_rows(all_rows, img)

    for _ in range(args.warmup):
        frame_once()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    times, solver_ms, eval2_ms = [], [], []
    stage = {k: [] for k in ("slices", "pass1", "coarsen", "pass2", "complete", "resolve")}
    launches0 = fr.stats()["launches"]
    for _ in range(args.steps):
        flush.fill_(1.0)                      # flush L2 between timed frames (outside the events)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        frame_once()
        e1.record(stream)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
        st = fr.stats()
        for k in stage:
            stage[k].append(st["ms_" + k])
        solver_ms.append(st["ms_solver"])   # the completion kernel alone (events around its launch)
        eval2_ms.append(st["ms_eval2"])     # the pass-2 entry kernel alone
    cl = clocks.stop()
    launches = fr.stats()["launches"] - launches0
    ms = statistics.mean(times)
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        tc = torch.tensor([statistics.mean(solver_ms)], device=dev, dtype=torch.float64)
        dist.all_reduce(tc, op=dist.ReduceOp.MAX)
        solver_ms = [float(tc.item())]
    st = fr.stats()
    tot = torch.tensor([st["sum_completed"], st["sum_samples"], st["sum_cols"], st["rows"],
                        st["slice_end"] - st["slice_begin"], st["evals_pass1"] + st["evals_coarsen"] + st["evals_pass2"]],
                       dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tot)
    sum_completed, sum_N, sum_n, sum_m, nsl, evals = [float(v) for v in tot.tolist()]
    value = sum_completed / (ms * 1e-3)
    # roofline of the dominant kernel (the completion kernel) from CUDA events recorded around its
    # launch on the launching stream (lmc_stats.ms_solver), averaged over the timed frames
    ms_c = statistics.mean(solver_ms)
    q = x.cfg.rank_q
    K = x.cfg.max_iter
    fl = (adm_flops if solver == 0 else mals_flops)(q, st["sum_samples"], st["rows"], st["sum_cols"],
                                                     st["slice_end"] - st["slice_begin"], K)
    achieved = fl / (ms_c * 1e-3) / 1e12
    peak, peak_src, peak_mb = fp32_peak() if solver == 0 else fp64_peak()
    fl_survey = adm_flops_survey(q, st["sum_samples"], st["rows"], st["sum_cols"], st["slice_end"] - st["slice_begin"], K) \
        if solver == 0 else fl
    traffic, limiter = None, None
    try:   # DRAM bytes per launch of the dominant kernel from the committed ncu --set full capture
        key = f"{args.config}/{args.solver}/q{x.cfg.rank_q}"
        ent = None
        for fn in ("r02_traffic.json", "r01_traffic.json"):   # the latest capture of this workload
            fp = os.path.join(ROOT, "profiles", fn)
            if ent is None and os.path.exists(fp):
                ent = json.load(open(fp)).get(key)
        traffic = ent["bytes"] if ent else None
        limiter = ent.get("limiter") if ent else None
    except Exception:
        traffic = None
    roof_entry = None
    if rank == 0 and solver in (0, 1) and not os.environ.get("BENCH_NO_ENTRY_ROOFLINE"):
        # entry evaluation (a3): fp64 flops as the oracle executes them x entries evaluated, over the
        # CUDA-event time of the kernels that evaluate them (pass 1 incl. its slice-box kernel,
        # coarsening, the pass-2 entry kernel)
        f1, f2, n1, n2, nsl_s = entry_flops_per_entry(x, fr)
        ev1 = float(st["evals_pass1"] + st["evals_coarsen"])
        ev2 = float(st["evals_pass2"])
        efl = f1 * ev1 + f2 * ev2
        ems = statistics.mean(stage["pass1"]) + statistics.mean(stage["coarsen"]) + statistics.mean(eval2_ms)
        p64, p64_src, p64_mb = fp64_peak()
        ach = efl / (ems * 1e-3) / 1e12
        roof_entry = {"bound": "alu", "kernel": "k_pass1 + k_coarsen + k_eval_new (+ k_slice_bbox)",
                      "achieved": ach, "peak": p64, "unit": "TFLOP/s", "frac": ach / p64, "traffic": None,
                      "peak_source": p64_src + "; FMA counted as 2 flops: the unfused ops of the exact "
                                               "(-fmad=false) path cap the fraction at 0.5",
                      "flops_per_entry": {"pass1+coarsen": f1, "pass2": f2},
                      "entries": {"pass1+coarsen": ev1, "pass2": ev2}, "flops_per_frame": efl, "kernel_ms": ems,
                      "frac_of_microbench_peak": (ach / p64_mb) if p64_mb else None,
                      "sample": f"oracle operation count over {n1} pass-1/coarsening pairs and {n2} pass-2 "
                                f"entries of {nsl_s} slices of this frame"
                                + ("; mesh occluders excluded from the count (BVH work not counted: a lower bound)"
                                   if x.prims.get("tri") is not None and x.prims["tri"].shape[0] else "")}
    e2e = None
    if not args.no_e2e and (world == 1 or lib_gather):
        e2e_id = None
        if world > 1:   # a second context, so its own NCCL communicator (id from rank 0)
            idt = torch.zeros(128, dtype=torch.uint8, device=dev)
            if rank == 0:
                idt.copy_(torch.frombuffer(bytearray(lmc.nccl_unique_id()), dtype=torch.uint8))
            dist.broadcast(idt, 0)
            e2e_id = bytes(idt.cpu().tolist())
        e2e = measure_e2e(x, args, solver, dev, rank, world, e2e_id)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cores = omp_threads()
        nsamp = args.cpu_sample_slices or max(4 * cores, 16)   # ~10-30 s of oracle work
        v, dt, k, ent = cpu_oracle_sample(x, nsamp, solver)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
               "sample": f"{k} of {int(nsl)} slices of {args.config} (full per-slice pipeline, "
                         f"{'literal dense-Z ADM' if solver == 0 else 'masked ALS'}), {dt:.1f} s wall"}
    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32" if solver == 0 else "f64",
        "data": "synthetic",
        "config": {"workload": f"{args.config}: {x.width}x{x.height} px, {x.vpls['px'].size} VPLs, {int(nsl)} slices, "
                               f"q={q}, rate={x.cfg.rate}, K={K}, solver={args.solver}",
                   "l2": "flushed between timed frames (256 MiB write)",
                   "decisions": "f64 (entries, sampling, coarsening)", "completion": "f32" if solver == 0 else "f64"},
        "ms_per_stage": {k: statistics.mean(v) for k, v in stage.items()},
        "completed_entries": sum_completed, "samples": sum_N, "rays_per_pixel": evals / max(sum_m, 1.0),
        "roofline": {"bound": "alu", "kernel": "k_adm" if solver == 0 else "k_mals", "achieved": achieved,
                     "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                     "traffic": traffic, "peak_source": peak_src, "flops_per_launch": fl,
                     "flops_per_launch_survey_count": fl_survey, "frac_survey_count": fl_survey / (ms_c * 1e-3) / 1e12 / peak,
                     "kernel_ms": ms_c, "limiter": limiter,
                     "frac_of_microbench_peak": (achieved / peak_mb) if peak_mb else None},
        "roofline_entry": roof_entry,
        "clocks": cl,
        "gpu_launches": launches,
    }
    if e2e:
        line["e2e"] = e2e
    if cpu:
        line["cpu_baseline"] = cpu
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def measure_e2e(x, args, solver, dev, rank=0, world=1, nccl_id=None):
    """Same metric through the C-ABI with HOST buffers: per step, H2D of the frame's inputs
    (G-buffer + VPLs from pinned memory), the seven calls, D2H of the image.  At N > 1 every rank
    uploads the frame's inputs and renders its slices, rank 0 gathers the image over NCCL inside
    lmc_resolve_image and writes it to host memory; the step time is the max over ranks (host
    clock, barrier-aligned) and the byte counts are the totals over ranks."""
    import torch
    import torch.distributed as dist
    from paper_2202_12567_b200 import lmc
    fr = lmc.Frame(x, memory=lmc.MEM_HOST, stream=torch.cuda.current_stream(dev), rank=rank, world=world,
                   nccl_id=nccl_id, partition=int(os.environ.get("BENCH_PARTITION", "1")))
    npix = x.height * x.width
    host_img = torch.zeros(npix * 3, dtype=torch.float32).pin_memory() if rank == 0 else None
    h2d = (x.m * (14 * 4) + x.vpls["px"].size * 6 * 4) * world
    d2h = npix * 3 * 4

    def step():
        fr.upload_inputs()
        fr.build_slices()
        fr.sample_pass1()
        fr.coarsen_cut()
        fr.sample_pass2()
        fr.complete()
        fr.resolve_image(host_img.numpy() if host_img is not None else None, lmc.MEM_HOST)

    for _ in range(max(1, args.warmup)):
        step()
    ts = []
    for _ in range(args.steps):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        step()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    st = fr.stats()
    fr.close()
    sec = statistics.mean(ts)
    done = float(st["sum_completed"])
    if world > 1:
        t = torch.tensor([sec, done], device=dev, dtype=torch.float64)
        tmax = t[:1].clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        tsum = t[1:].clone()
        dist.all_reduce(tsum)
        sec, done = float(tmax.item()), float(tsum.item())
    return {"value": done / sec, "unit": UNIT, "ms_per_step": sec * 1e3,
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)}


if __name__ == "__main__":
    main()
