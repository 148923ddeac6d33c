"""Measure a library FP4 (MXFP4, block-32 ue8m0 scales) GEMM peak on this B200 via cuBLASLt
(torch._scaled_mm), for the roofline denominator of the kind::mxf4 numerator GEMM."""
import json, subprocess, sys, torch
dev = torch.device("cuda:0")
print(torch.__version__, hasattr(torch, "float4_e2m1fn_x2"), flush=True)
out = {}
for (M, N, K) in [(8192, 8192, 32768), (16384, 16384, 16384)]:
    try:
        a = torch.randint(0, 256, (M, K // 2), dtype=torch.uint8, device=dev).view(torch.float4_e2m1fn_x2)
        b = torch.randint(0, 256, (N, K // 2), dtype=torch.uint8, device=dev).view(torch.float4_e2m1fn_x2)
        rm = lambda r: (r + 127) // 128 * 128
        rk = lambda k: (k // 32 + 3) // 4 * 4
        sa = torch.full((rm(M) * rk(K),), 127, dtype=torch.uint8, device=dev).view(torch.float8_e8m0fnu)
        sb = torch.full((rm(N) * rk(K),), 127, dtype=torch.uint8, device=dev).view(torch.float8_e8m0fnu)
        import torch.nn.functional as F
        f = lambda: F.scaled_mm(a, b.t(), sa.view(rm(M), rk(K) * 1), F.ScalingType.BlockWise1x32,
                                sb.view(rm(N), rk(K)), F.ScalingType.BlockWise1x32,
                                swizzle_a=F.SwizzleType.SWIZZLE_32_4_4, swizzle_b=F.SwizzleType.SWIZZLE_32_4_4,
                                output_dtype=torch.bfloat16)
        for _ in range(3): f()
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(10):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(); f(); e.record(); torch.cuda.synchronize()
            best = min(best, s.elapsed_time(e))
        # sustained: back to back for ~2 s
        n = max(1, int(2000 / best))
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(n): f()
        e.record(); torch.cuda.synchronize()
        sus = s.elapsed_time(e) / n
        fl = 2.0 * M * N * K
        out[f"{M}x{N}x{K}"] = {"burst_tflops": fl / best / 1e9, "sustained_tflops": fl / sus / 1e9}
        print(M, N, K, out[f"{M}x{N}x{K}"], flush=True)
    except Exception as ex:  # noqa
        print("fail", M, N, K, repr(ex)[:3000], flush=True)
print(json.dumps(out))
