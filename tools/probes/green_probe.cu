// Probe: can an HBM-bound kernel and a tensor-bound GEMM overlap on one B200 when
// each runs in its own SM partition (green contexts)? The question behind a
// micro-batched decode step (DESIGN.md §9 "next"): one half-batch's attention
// (HBM-bound) under the other half's GEMMs (tensor-bound at B = 200).
//   read  : a grid-stride 16-byte-load reduction over a 4 GiB buffer (HBM read stream)
//   gemm  : cuBLAS bf16 GEMM, Y[200 x 20480] = X[200 x 5120] W^T (an OPT-13B FC1 at B = 200), repeated
// Reports each alone on the whole GPU, each alone in its partition, and both together.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o green_probe tools/probes/green_probe.cu -lcuda -lcublas
#include <cublas_v2.h>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#define CKD(x)                                                                    \
  do {                                                                            \
    CUresult r_ = (x);                                                            \
    if (r_ != CUDA_SUCCESS) {                                                     \
      const char* s_ = nullptr;                                                   \
      cuGetErrorString(r_, &s_);                                                  \
      printf("{\"error\": \"%s: %s\"}\n", #x, s_ ? s_ : "?");                     \
      exit(1);                                                                    \
    }                                                                             \
  } while (0)
#define CKR(x)                                                                        \
  do {                                                                                \
    cudaError_t r_ = (x);                                                             \
    if (r_ != cudaSuccess) {                                                          \
      printf("{\"error\": \"%s: %s\"}\n", #x, cudaGetErrorString(r_));                \
      exit(1);                                                                        \
    }                                                                                 \
  } while (0)

__global__ void read_kernel(const uint4* __restrict__ p, size_t n, unsigned* sink) {
  unsigned acc = 0;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p + i));
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678u) *sink = acc;
}

int main(int argc, char** argv) {
  const int nA = argc > 1 ? atoi(argv[1]) : 96;  // SMs for the read stream
  CKD(cuInit(0));
  CUdevice dev;
  CKD(cuDeviceGet(&dev, 0));
  CKR(cudaSetDevice(0));
  CKR(cudaFree(0));
  CUdevResource full;
  CKD(cuDeviceGetDevResource(dev, &full, CU_DEV_RESOURCE_TYPE_SM));
  CUdevResource grpA, rest;
  unsigned n = 1;
  CKD(cuDevSmResourceSplitByCount(&grpA, &n, &full, &rest, 0, nA));
  printf("{\"sms\": %u, \"part_read\": %u, \"part_gemm\": %u}\n", full.sm.smCount, grpA.sm.smCount,
         rest.sm.smCount);
  CUdevResourceDesc dA, dB;
  CKD(cuDevResourceGenerateDesc(&dA, &grpA, 1));
  CKD(cuDevResourceGenerateDesc(&dB, &rest, 1));
  CUgreenCtx gA, gB;
  CKD(cuGreenCtxCreate(&gA, dA, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  CKD(cuGreenCtxCreate(&gB, dB, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  CUstream sA, sB;
  CKD(cuGreenCtxStreamCreate(&sA, gA, CU_STREAM_NON_BLOCKING, 0));
  CKD(cuGreenCtxStreamCreate(&sB, gB, CU_STREAM_NON_BLOCKING, 0));
  cudaStream_t sF;
  CKR(cudaStreamCreateWithFlags(&sF, cudaStreamNonBlocking));

  const size_t bytes = 4ull << 30;
  uint4* buf;
  unsigned* sink;
  CKR(cudaMalloc(&buf, bytes));
  CKR(cudaMemset(buf, 1, bytes));
  CKR(cudaMalloc(&sink, 4));
  const int M = 200, N = 20480, K = 5120, reps = 20;
  __nv_bfloat16 *W, *X, *Y;
  CKR(cudaMalloc(&W, (size_t)N * K * 2));
  CKR(cudaMalloc(&X, (size_t)M * K * 2));
  CKR(cudaMalloc(&Y, (size_t)M * N * 2));
  CKR(cudaMemset(W, 0, (size_t)N * K * 2));
  CKR(cudaMemset(X, 0, (size_t)M * K * 2));
  cublasHandle_t h;
  cublasCreate(&h);
  const float one = 1.f, zero = 0.f;
  auto gemm = [&](cudaStream_t s) {
    cublasSetStream(h, s);
    for (int r = 0; r < reps; ++r)
      cublasGemmEx(h, CUBLAS_OP_T, CUBLAS_OP_N, N, M, K, &one, W, CUDA_R_16BF, K, X, CUDA_R_16BF, K, &zero, Y,
                   CUDA_R_16BF, N, CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT);
  };
  auto read = [&](cudaStream_t s, int reps_r) {
    for (int r = 0; r < reps_r; ++r) read_kernel<<<148 * 8, 256, 0, s>>>(buf, bytes / 16, sink);
  };
  cudaEvent_t e[6];
  for (auto& x : e) CKR(cudaEventCreate(&x));
  auto time1 = [&](auto fn, cudaStream_t s) {
    fn(s);  // warm-up
    CKR(cudaStreamSynchronize(s));
    CKR(cudaEventRecord(e[0], s));
    fn(s);
    CKR(cudaEventRecord(e[1], s));
    CKR(cudaEventSynchronize(e[1]));
    float ms = 0;
    cudaEventElapsedTime(&ms, e[0], e[1]);
    return ms;
  };
  const int rr = 8;  // reads per measurement (8 x 4 GiB)
  float t_read_full = time1([&](cudaStream_t s) { read(s, rr); }, sF);
  float t_gemm_full = time1([&](cudaStream_t s) { gemm(s); }, sF);
  float t_read_A = time1([&](cudaStream_t s) { read(s, rr); }, (cudaStream_t)sA);
  float t_gemm_B = time1([&](cudaStream_t s) { gemm(s); }, (cudaStream_t)sB);
  // both at once: the read stream on partition A, the GEMMs on partition B
  read((cudaStream_t)sA, 1);
  gemm((cudaStream_t)sB);
  CKR(cudaDeviceSynchronize());
  CKR(cudaEventRecord(e[2], (cudaStream_t)sA));
  CKR(cudaStreamWaitEvent((cudaStream_t)sB, e[2], 0));
  read((cudaStream_t)sA, rr);
  gemm((cudaStream_t)sB);
  CKR(cudaEventRecord(e[3], (cudaStream_t)sA));
  CKR(cudaEventRecord(e[4], (cudaStream_t)sB));
  CKR(cudaDeviceSynchronize());
  float t_a = 0, t_b = 0;
  cudaEventElapsedTime(&t_a, e[2], e[3]);
  cudaEventElapsedTime(&t_b, e[2], e[4]);
  const double rd = (double)rr * bytes / 1e9, fl = 2.0 * M * N * K * reps / 1e12;
  printf("{\"read_full_ms\": %.3f, \"read_full_gbs\": %.0f, \"gemm_full_ms\": %.3f, \"gemm_full_tflops\": %.0f, "
         "\"read_partA_ms\": %.3f, \"read_partA_gbs\": %.0f, \"gemm_partB_ms\": %.3f, \"gemm_partB_tflops\": %.0f, "
         "\"both_read_ms\": %.3f, \"both_gemm_ms\": %.3f, \"serial_full_ms\": %.3f, \"both_ms\": %.3f}\n",
         t_read_full, rd / t_read_full * 1e3, t_gemm_full, fl / t_gemm_full * 1e3, t_read_A, rd / t_read_A * 1e3,
         t_gemm_B, fl / t_gemm_B * 1e3, t_a, t_b, t_read_full + t_gemm_full, t_a > t_b ? t_a : t_b);
  return 0;
}
