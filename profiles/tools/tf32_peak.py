"""TF32 tensor-core denominators and the path's GEMM rates (measurement).

* cuBLAS TF32 dense peak: torch.matmul on 8192^3 fp32 operands with TF32
  allowed, best of 10 (CUDA events) - the library's measured tensor-pipe
  ceiling on this B200, the denominator of the GEMM rows below;
* the layer drivers' own tcgen05 launchers (ht_gemm_rate) at the bench's
  cfg-2 shapes (M = 2.4M rows): z = relu(agg W) 3xTF32, gagg = gz W^T
  1xTF32, dW = agg^T gz.

    python profiles/tools/tf32_peak.py > gpurun_out/r2_tf32_peak.json
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def cublas_tf32(n=8192, reps=10):
    torch.backends.cuda.matmul.allow_tf32 = True
    a = torch.randn(n, n, device="cuda")
    b = torch.randn(n, n, device="cuda")
    for _ in range(3):
        a @ b
    best = 0.0
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        a @ b
        e1.record()
        e1.synchronize()
        best = max(best, 2 * n ** 3 / (e0.elapsed_time(e1) * 1e-3) / 1e12)
    return best


def ours(op, M, K, N, iters=20):
    from paper_2311_14898_b200 import _native as Nat
    out = np.zeros(3)
    Nat.call("ht_gemm_rate", op, 1, M, K, N, iters, Nat.ptr(out))  # 1 = HT_PREC_TF32
    return {"ms": out[0], "tflops_useful": out[1], "gbs_operands": out[2]}


if __name__ == "__main__":
    peak = cublas_tf32()
    res = {"cublas_tf32_tflops_8192": peak,
           "nominal_tf32_dense_tflops": 1100.0,
           "what": "cuBLAS fp32 matmul with TF32 allowed (torch), best of 10, CUDA events"}
    M = 2_400_000
    shapes = {"z_relu_3xtf32_k100_n256": (0, M, 100, 256),
              "z_relu_3xtf32_k256_n256": (0, M, 256, 256),
              "gagg_1xtf32_k100_n256": (2, M, 100, 256),
              "gagg_1xtf32_k256_n256": (2, M, 256, 256),
              "wgrad_k256_n256": (3, M, 256, 256),
              "wgrad_k100_n256": (3, M, 100, 256)}
    for name, (op, m, k, n) in shapes.items():
        r = ours(op, m, k, n)
        mult = 3 if op == 0 else 1  # 3xTF32 issues three MMAs per useful product
        r["tensor_frac_of_cublas_peak"] = r["tflops_useful"] * mult / peak
        res[name] = r
    print(json.dumps(res, indent=1))
