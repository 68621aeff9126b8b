// Legacy mma.sync m16n8k16 bf16 throughput on this GPU: every warp runs 8
// independent accumulator chains; reports TFLOP/s over the whole chip.
// Build/run: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/hmma tools/probes/hmma_probe.cu && /tmp/hmma
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>

__global__ void hmma_loop(float* out, int iters) {
  uint32_t a[4] = {0x3f803f80u, 0x3f803f80u, 0x3f803f80u, 0x3f803f80u};
  uint32_t b[2] = {0x3c003c00u, 0x3c003c00u};
  float d[8][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
          "{%0,%1,%2,%3};"
          : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3])
          : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
  float s = 0.f;
  for (int c = 0; c < 8; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  if (s == 12345.f) out[threadIdx.x] = s;
}

int main() {
  float* out;
  cudaMalloc(&out, 4096);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int warps : {4, 8, 16, 32}) {
    const int iters = 4096;
    hmma_loop<<<sms, warps * 32>>>(out, 16);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    hmma_loop<<<sms, warps * 32>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 16 * 8 * 16 * 8.0 * iters * warps * sms;
    printf("{\"warps_per_sm\": %d, \"ms\": %.3f, \"tflops\": %.1f, \"cycles_per_hmma_per_sm_at_1.9GHz\": %.2f}\n",
           warps, ms, flops / ms / 1e9, ms * 1e-3 * 1.9e9 / (8.0 * iters * warps));
  }
  return 0;
}
