"""Decode-GEMM microbenchmark: the tcgen05 kernels (mirage_decode_gemm, fp32 split
slices; mirage_sk_gemm, persistent stream-K, one fp32 output) vs cuBLASLt (torch bf16 linear) on the decode shapes of the bench models.
Weights are cycled over enough copies to exceed L2; CUDA events around `reps`
launches. Reports weight-streaming GB/s (N*K*2 bytes per GEMM).
Usage: python tools/gemm_bench.py [--batch 16 64 128 256]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2507_11507_b200 import _lib  # noqa: E402

SHAPES = {  # name: (N, K)
    "opt13b_qkv": (15360, 5120), "opt13b_o": (5120, 5120), "opt13b_fc1": (20480, 5120), "opt13b_fc2": (5120, 20480),
    "llama3_8b_qkv": (6144, 4096), "llama3_8b_o": (4096, 4096), "llama3_8b_gateup": (28672, 4096),
    "llama3_8b_down": (4096, 14336),
    "llama70b_tp8_qkv": (1280, 8192), "llama70b_tp8_o": (8192, 1024), "llama70b_tp8_gateup": (7168, 8192),
    "llama70b_tp8_down": (8192, 3584),
}


def timeit(fn, reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for i in range(3):
        fn(i)
    torch.cuda.synchronize()
    e0.record()
    for i in range(reps):
        fn(i)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, nargs="*", default=[16, 64, 128, 256])
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--shape", nargs="*", default=list(SHAPES))
    ap.add_argument("--reduce", action="store_true", help="sum the K splits in the kernel (cluster DSMEM)")
    ap.add_argument("--one-split-cg", type=int, nargs="*", default=[],
                    help="also time the one-split form (the fused TP push GEMM) with these column-group counts")
    a = ap.parse_args()
    for name in a.shape:
        N, K = SHAPES[name]
        copies = max(2, int(3 * 128e6 // (N * K * 2)) + 1)
        ws = [torch.randn((N, K), device="cuda").to(torch.bfloat16) for _ in range(copies)]
        for B in a.batch:
            x = torch.randn((B, K), device="cuda").to(torch.bfloat16)
            y = torch.empty((16, B, N), dtype=torch.float32, device="cuda")
            ns = torch.zeros(1, dtype=torch.int32)
            import ctypes as C
            got = C.c_int32()
            st = torch.cuda.current_stream()

            def ours(i):
                _lib.LIB.mirage_decode_gemm(st.cuda_stream, ws[i % copies].data_ptr(), N, K, x.data_ptr(), B,
                                            y.data_ptr(), 0, int(a.reduce and B <= 128), 0, C.byref(got))

            y1 = torch.empty((B, N), dtype=torch.float32, device="cuda")

            def sk(i):
                _lib.LIB.mirage_sk_gemm(st.cuda_stream, ws[i % copies].data_ptr(), N, K, x.data_ptr(), B,
                                        y1.data_ptr(), None, None, 0)

            def cublas(i):
                torch.nn.functional.linear(x, ws[i % copies])
            one = {}
            for cg in a.one_split_cg:
                def one_split(i, cg=cg):
                    _lib.LIB.mirage_decode_gemm(st.cuda_stream, ws[i % copies].data_ptr(), N, K, x.data_ptr(), B,
                                                y.data_ptr(), 1, 0, cg, C.byref(got))
                t1 = timeit(one_split, a.reps)
                one["cg%d" % cg] = {"us": round(t1 * 1e3, 2), "gbs": round(N * K * 2 / 1e9 / (t1 * 1e-3))}
            t_o = timeit(ours, a.reps)
            t_s = timeit(sk, a.reps)
            t_c = timeit(cublas, a.reps)
            gb = N * K * 2 / 1e9
            print(json.dumps({"shape": name, "N": N, "K": K, "B": B, "splits": got.value,
                              "tcgen05_us": round(t_o * 1e3, 2), "cublas_us": round(t_c * 1e3, 2),
                              "tcgen05_gbs": round(gb / (t_o * 1e-3)), "cublas_gbs": round(gb / (t_c * 1e-3)),
                              "sk_us": round(t_s * 1e3, 2), "sk_gbs": round(gb / (t_s * 1e-3)),
                              "speedup": round(t_c / t_o, 3), "sk_speedup": round(t_c / t_s, 3),
                              "one_split": one}), flush=True)
        del ws
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
