"""Measured cost of the dense-tile formulation of the ADM iteration on tensor cores (DESIGN.md §6,
"Why not tcgen05 for the streaming part"): the C4 slice shapes (2048 slices of m = 1013 rows,
n = 562 columns -- the mean coarsened cut of the C4 frame --, q = 16, 10% sampling) with every
m x n product dense through cuBLAS batched GEMMs (tensor cores with TF32 / bf16 inputs, or plain
FP32), Z formed densely, K = 100 iterations extrapolated from the per-iteration time.
Diagnostic measurement (library GEMMs, not the product path):

    python tools/dense_tile_bench.py > profiles/r02_dense_tile.json
"""
import json
import sys

import torch


def timeit(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts)


def main():
    S, m, n, q, K = 2048, 1013, 562, 16, 100
    chunk = int(sys.argv[1]) if len(sys.argv) > 1 else 512   # slices per batched call (memory)
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(1)
    X = torch.rand(chunk, m, q, device=dev, generator=g)
    Y = torch.rand(chunk, q, n, device=dev, generator=g)
    M = torch.rand(chunk, m, n, device=dev, generator=g)
    mask = torch.rand(chunk, m, n, device=dev, generator=g) < 0.1
    out = {"shapes": {"slices": S, "m": m, "n": n, "q": q, "K": K, "rate": 0.1, "chunk": chunk},
           "flops_per_iteration_dense": 3 * 2.0 * m * n * q * S}
    res = {}
    for mode in ("fp32", "tf32", "bf16"):
        torch.backends.cuda.matmul.allow_tf32 = mode == "tf32"
        dt = torch.bfloat16 if mode == "bf16" else torch.float32
        Xc, Yc, Mc = X.to(dt), Y.to(dt), M.to(dt)

        def gemms():
            P = torch.bmm(Xc, Yc)                       # X_k Y_k, dense m x n
            Z = torch.where(mask, Mc, P)                # Z_k = P_Omega(M) + P_Omega^c(X_k Y_k)
            a = torch.bmm(Z, Yc.transpose(1, 2))        # Z_k Y_k^T (row update)
            b = torch.bmm(Xc.transpose(1, 2), Z)        # X^T Z_k (column update)
            return a, b

        def only_gemms():
            P = torch.bmm(Xc, Yc)
            a = torch.bmm(P, Yc.transpose(1, 2))
            b = torch.bmm(Xc.transpose(1, 2), P)
            return a, b

        t_all = timeit(gemms) * S / chunk
        t_mm = timeit(only_gemms) * S / chunk
        res[mode] = {"ms_per_iteration": t_all, "ms_per_frame_K100": t_all * K,
                     "ms_per_iteration_gemms_only": t_mm, "ms_per_frame_gemms_only": t_mm * K,
                     "tflops_gemms_only": out["flops_per_iteration_dense"] / (t_mm * 1e-3) / 1e12}
    torch.backends.cuda.matmul.allow_tf32 = False
    # streaming floor of a fused dense kernel that keeps every m x n tile on chip: the dense M^
    # (fp32) read twice per iteration (row and column phase; a 1-bit mask would add 3%)
    t_rd = timeit(lambda: M.sum()) * S / chunk
    res["stream_dense_M_once"] = {"ms_per_iteration": t_rd, "gbytes": 4.0 * S * m * n / 1e9,
                                  "ms_per_frame_two_reads_K100": 2 * t_rd * K}
    out["results"] = res
    out["note"] = ("per frame = per iteration x K = 100 (the sparse kernel k_adm: 137 ms per frame at C4 for "
                   "everything, including the q x q updates and Grams not counted here); 3xTF32 for fp32 "
                   "parity would triple the tf32 GEMM time")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
