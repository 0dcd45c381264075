"""BASELINE.json configs[4]: rank q in {4, 8, 16, 32} x sampling rate in {5, 10, 20}% at the C3 shape
(1024x1024, 300k VPLs, glossy), one B200.  Per setting: ms/frame (CUDA events, L2 flushed between
frames), completed entries/s, the k_adm time and its FP32 roofline fraction, and the completion
quality: relative Frobenius error of U V, and the relative RMS / max error of its row sums (the
rendered pixel luminance of the slice), against the fully evaluated coarsened slice matrix
M~(i, c) = lum(rho_i) lum(I_c) T(i, rep(c)) (all m x n entries, T from the library's fp64 entry
kernel) on a fixed set of slices.  Diagnostic tool (not the bench):

    python tools/sweep_c5.py [frames] [check_slices] > sweep.json
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import scenegen  # noqa: E402
from paper_2202_12567_b200 import lmc  # noqa: E402


def lum(r, g, b):
    return (0.2126 * r + 0.7152 * g) + 0.0722 * b


def slice_error(fr, x, off, rows, s):
    f = fr.factors(s)
    if f["flags"] & (lmc.SLICE_DIRECT | lmc.SLICE_ZERO):
        return None
    cut = fr.cut(s)
    r = rows[off[s]:off[s + 1]]
    m, n = r.size, cut.size
    g, t = x.gbuf, x.tree
    lr = lum(g["rho_r"][r].astype(np.float64), g["rho_g"][r].astype(np.float64), g["rho_b"][r].astype(np.float64))
    lc = lum(t["ir"][cut].astype(np.float64), t["ig"][cut].astype(np.float64), t["ib"][cut].astype(np.float64))
    ii, cc = np.meshgrid(np.arange(m), np.arange(n), indexing="ij")
    T = fr.eval_entries(r[ii.ravel()], t["rep"][cut][cc.ravel()]).reshape(m, n)
    M = (lr[:, None] * lc[None, :]) * T
    # consistency: the observed values of Omega are the same entries
    sm = fr.samples(s)
    om = M[sm["row"], sm["col"]]
    omega_dev = float(np.max(np.abs(om - sm["val"]) / np.maximum(np.abs(om), 1e-30))) if sm["nnz"] else 0.0
    A = f["U"].astype(np.float64) @ f["V"].astype(np.float64)
    nM = np.linalg.norm(M)
    # the rendered quantity: row sums (luminance of the slice's pixels from its columns)
    ra, rm = A.sum(axis=1), M.sum(axis=1)
    floor = 1e-3 * max(float(rm.mean()), 1e-30)
    return {"rel_fro": float(np.linalg.norm(A - M) / nM) if nM > 0 else 0.0,
            "img_rel_rms": float(np.linalg.norm(ra - rm) / max(np.linalg.norm(rm), 1e-30)),
            "img_rel_max": float(np.max(np.abs(ra - rm) / np.maximum(np.abs(rm), floor))),
            "resid_omega": f["resid"], "iters": f["iters"], "omega_value_dev": omega_dev}


def main():
    frames = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    nchk = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    x = scenegen.make_inputs(scenegen.preset("c3"))
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    peak = bench.fp32_peak()[0]
    out = []
    for q in (4, 8, 16, 32):
        for rate in (0.05, 0.10, 0.20):
            fr = lmc.Frame(x, stream=stream, rank_q=q, rate=rate)
            fr.set_timing(True)
            img = torch.zeros(x.height * x.width * 3, device=dev)
            for _ in range(2):
                fr.run(img)
            torch.cuda.synchronize()
            times, solver = [], []
            for _ in range(frames):
                flush.fill_(1.0)
                torch.cuda.synchronize()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                fr.run(img)
                e1.record(stream)
                torch.cuda.synchronize()
                times.append(e0.elapsed_time(e1))
                solver.append(fr.stats()["ms_solver"])
            st = fr.stats()
            ms, msc = statistics.mean(times), statistics.mean(solver)
            fl = bench.adm_flops(q, st["sum_samples"], st["rows"], st["sum_cols"],
                                 st["slice_end"] - st["slice_begin"], x.cfg.max_iter)
            off, rows = fr.slices()
            S = off.size - 1
            errs = [e for e in (slice_error(fr, x, off, rows, int(s))
                                for s in np.linspace(0, S - 1, nchk).astype(int)) if e is not None]
            rec = {"q": q, "rate": rate, "ms_per_frame": ms, "entries_per_s": st["sum_completed"] / (ms * 1e-3),
                   "samples": st["sum_samples"], "k_adm_ms": msc, "k_adm_tflops": fl / (msc * 1e-3) / 1e12,
                   "k_adm_frac_fp32": fl / (msc * 1e-3) / 1e12 / peak,
                   "stage_ms": {k: st["ms_" + k] for k in ("slices", "pass1", "coarsen", "pass2", "complete", "resolve")},
                   "check_slices": len(errs),
                   "rel_fro_mean": float(np.mean([e["rel_fro"] for e in errs])) if errs else None,
                   "rel_fro_max": float(np.max([e["rel_fro"] for e in errs])) if errs else None,
                   "img_rel_rms_mean": float(np.mean([e["img_rel_rms"] for e in errs])) if errs else None,
                   "img_rel_max": float(np.max([e["img_rel_max"] for e in errs])) if errs else None,
                   "resid_omega_mean": float(np.mean([e["resid_omega"] for e in errs])) if errs else None,
                   "omega_value_dev_max": float(np.max([e["omega_value_dev"] for e in errs])) if errs else None}
            out.append(rec)
            print(json.dumps(rec), file=sys.stderr, flush=True)
            fr.close()
            del img
            torch.cuda.empty_cache()
    print(json.dumps({"config": "c5 sweep at the c3 shape (1024x1024, 300k VPLs, glossy, K=100, ADM)",
                      "frames": frames, "results": out}))


if __name__ == "__main__":
    main()
