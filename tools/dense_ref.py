"""Library reference points for the dense comparator (cuBLAS through torch.matmul; plumbing only, not
the product): X[N,n] @ A^T[n,k] in TF32 (1xTF32, cublasLt) and in full FP32 (SIMT SGEMM), plus the
same epilogue (+b, /w, floor) in torch, on C1's shape; beside the repo's own tcgen05 K4."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2309_15479_b200 as fl
from fastlsh_inputs import configs, data, e2lsh_arrays


def timed(fn, iters=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


c = configs.get(sys.argv[1] if len(sys.argv) > 1 else "C1")
N = min(c.N, 1_000_000)
X = data.generate(c.data, c.n, 0, N, seed=1, device="cuda")
idx, A, b = e2lsh_arrays(c.n, c.k, c.w, 1)
At = torch.as_tensor(A, device="cuda").t().contiguous()
bt = torch.as_tensor(b, device="cuda")
flops = 2.0 * N * c.n * c.k
for name, tf32 in (("cublas_tf32", True), ("cublas_fp32", False)):
    torch.backends.cuda.matmul.allow_tf32 = tf32
    t_mm = timed(lambda: X @ At)
    t_all = timed(lambda: torch.floor((X @ At + bt) / c.w).to(torch.int32))
    print(f"{c.name} N={N} {name}: GEMM {t_mm:.3f} ms ({flops / t_mm / 1e9:.0f} TFLOP/s), GEMM + epilogue {t_all:.3f} ms")
Pd = fl.Params.e2lsh(c.n, c.k, c.w, seed=1)
for prec in (3, 1):
    t = timed(lambda: fl.e2lsh_hash(Pd, X, precision=prec))
    kpad = (c.k + 255) // 256 * 256
    print(f"{c.name} N={N} K4 tcgen05 {prec}xTF32: {t:.3f} ms ({2.0 * N * c.n * kpad * prec / t / 1e9:.0f} TFLOP/s MMA work)")
