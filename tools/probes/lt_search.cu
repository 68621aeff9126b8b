// cuBLASLt algorithm-space probe for the decode step's GEMM shapes:
// y[B][N] = x[B][K] W[N][K]^T in the library's layout (A = W as K x N col-major,
// transposed; B = x as K x B; D fp32 or bf16 N x B). Times (1) the heuristic's top
// candidates (what the runtime autotunes over) and (2) every configurable algo id
// x tile x split-K x stages x swizzle combination that cublasLtMatmulAlgoCheck
// accepts, and prints the best of each family as JSON lines.
// Build: nvcc -O2 -arch=sm_100a lt_search.cu -lcublasLt -o lt_search
#include <cublasLt.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                          \
  do {                                                                                 \
    auto e_ = (x);                                                                     \
    if ((int)e_ != 0) {                                                                \
      fprintf(stderr, "%s:%d %s -> %d\n", __FILE__, __LINE__, #x, (int)e_);            \
      exit(1);                                                                         \
    }                                                                                  \
  } while (0)

static cublasLtHandle_t lt;
static void* ws;
static const size_t kWs = 64ull << 20;

struct Prob {
  int N, K, B, out_bf16, relu_bias;
  const char* name;
};

static float time_algo(cublasLtMatmulDesc_t op, cublasLtMatrixLayout_t a, cublasLtMatrixLayout_t b,
                       cublasLtMatrixLayout_t d, const void* W, const void* X, void* Y,
                       const cublasLtMatmulAlgo_t* algo, cudaStream_t s, int reps = 20) {
  const float one = 1.f, zero = 0.f;
  for (int i = 0; i < 3; ++i)
    if (cublasLtMatmul(lt, op, &one, W, a, X, b, &zero, Y, d, Y, d, algo, ws, kWs, s) != CUBLAS_STATUS_SUCCESS)
      return 1e30f;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, s);
  for (int i = 0; i < reps; ++i) cublasLtMatmul(lt, op, &one, W, a, X, b, &zero, Y, d, Y, d, algo, ws, kWs, s);
  cudaEventRecord(e1, s);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (cudaGetLastError() != cudaSuccess) return 1e30f;
  return ms * 1e3f / reps;  // us
}

int main(int argc, char** argv) {
  const int B = argc > 1 ? atoi(argv[1]) : 400;
  std::vector<Prob> probs = {{15360, 5120, B, 0, 0, "opt13b_qkv"},
                             {5120, 5120, B, 0, 0, "opt13b_o"},
                             {20480, 5120, B, 1, 1, "opt13b_fc1"},
                             {5120, 20480, B, 0, 0, "opt13b_fc2"}};
  CK(cublasLtCreate(&lt));
  CK(cudaMalloc(&ws, kWs));
  cudaStream_t s;
  cudaStreamCreate(&s);
  for (const Prob& p : probs) {
    // weights cycled over copies that exceed L2, as in the step
    const int copies = 4;
    std::vector<void*> Ws(copies);
    for (auto& w : Ws) {
      CK(cudaMalloc(&w, (size_t)p.N * p.K * 2));
      cudaMemset(w, 0x3c, (size_t)p.N * p.K * 2);
    }
    void *X, *Y, *bias;
    CK(cudaMalloc(&X, (size_t)p.B * p.K * 2));
    cudaMemset(X, 0x3c, (size_t)p.B * p.K * 2);
    CK(cudaMalloc(&Y, (size_t)p.B * p.N * 4));
    CK(cudaMalloc(&bias, (size_t)p.N * 2));
    cudaMemset(bias, 0, (size_t)p.N * 2);
    cublasLtMatmulDesc_t op;
    CK(cublasLtMatmulDescCreate(&op, CUBLAS_COMPUTE_32F, CUDA_R_32F));
    const cublasOperation_t ta = CUBLAS_OP_T, tb = CUBLAS_OP_N;
    CK(cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSA, &ta, sizeof ta));
    CK(cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSB, &tb, sizeof tb));
    if (p.relu_bias) {
      cublasLtEpilogue_t e = CUBLASLT_EPILOGUE_RELU_BIAS;
      CK(cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_EPILOGUE, &e, sizeof e));
      const cudaDataType_t bt = CUDA_R_16BF;
      CK(cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_BIAS_DATA_TYPE, &bt, sizeof bt));
      CK(cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_BIAS_POINTER, &bias, sizeof bias));
    }
    const cudaDataType_t dt = p.out_bf16 ? CUDA_R_16BF : CUDA_R_32F;
    cublasLtMatrixLayout_t a, b, d;
    CK(cublasLtMatrixLayoutCreate(&a, CUDA_R_16BF, p.K, p.N, p.K));
    CK(cublasLtMatrixLayoutCreate(&b, CUDA_R_16BF, p.K, p.B, p.K));
    CK(cublasLtMatrixLayoutCreate(&d, dt, p.N, p.B, p.N));
    int wi = 0;
    auto timed = [&](const cublasLtMatmulAlgo_t* algo) {
      // rotate the weight copy between timing calls (the first repetitions hit L2 otherwise)
      float best = 1e30f;
      for (int r = 0; r < 2; ++r) best = std::min(best, time_algo(op, a, b, d, Ws[(wi++) % copies], X, Y, algo, s));
      return best;
    };
    const double gflop = 2.0 * p.N * p.K * p.B / 1e9;
    // (1) heuristic candidates
    cublasLtMatmulPreference_t pref;
    CK(cublasLtMatmulPreferenceCreate(&pref));
    CK(cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &kWs, sizeof kWs));
    cublasLtMatmulHeuristicResult_t res[64];
    int n = 0;
    cublasLtMatmulAlgoGetHeuristic(lt, op, a, b, d, d, pref, 64, res, &n);
    float h_best = 1e30f, h_first = 1e30f;
    int h_best_i = -1;
    for (int i = 0; i < n; ++i) {
      if (res[i].state != CUBLAS_STATUS_SUCCESS) continue;
      const float t = timed(&res[i].algo);
      if (i == 0) h_first = t;
      if (t < h_best) {
        h_best = t;
        h_best_i = i;
      }
    }
    printf("{\"shape\": \"%s\", \"B\": %d, \"family\": \"heuristic\", \"candidates\": %d, \"first_us\": %.2f, "
           "\"best_us\": %.2f, \"best_rank\": %d, \"best_tflops\": %.0f}\n",
           p.name, p.B, n, h_first, h_best, h_best_i, gflop / (h_best * 1e-6) / 1e3);
    fflush(stdout);
    // (2) enumerate configurable algos
    int ids[512], nid = 0;
    CK(cublasLtMatmulAlgoGetIds(lt, CUBLAS_COMPUTE_32F, CUDA_R_32F, CUDA_R_16BF, CUDA_R_16BF, dt, dt, 512, ids,
                                &nid));
    float e_best = 1e30f;
    int e_id = -1, e_tile = -1, e_split = -1, e_stage = -1, e_sw = -1, tried = 0;
    for (int ii = 0; ii < nid; ++ii) {
      cublasLtMatmulAlgo_t algo;
      if (cublasLtMatmulAlgoInit(lt, CUBLAS_COMPUTE_32F, CUDA_R_32F, CUDA_R_16BF, CUDA_R_16BF, dt, dt, ids[ii],
                                 &algo) != CUBLAS_STATUS_SUCCESS)
        continue;
      size_t sz = 0;
      std::vector<int> tiles, stages;
      if (cublasLtMatmulAlgoCapGetAttribute(&algo, CUBLASLT_ALGO_CAP_TILE_IDS, nullptr, 0, &sz) ==
              CUBLAS_STATUS_SUCCESS &&
          sz) {
        tiles.resize(sz / sizeof(int));
        cublasLtMatmulAlgoCapGetAttribute(&algo, CUBLASLT_ALGO_CAP_TILE_IDS, tiles.data(), sz, &sz);
      }
      if (tiles.empty()) tiles.push_back(CUBLASLT_MATMUL_TILE_UNDEFINED);
      if (cublasLtMatmulAlgoCapGetAttribute(&algo, CUBLASLT_ALGO_CAP_STAGES_IDS, nullptr, 0, &sz) ==
              CUBLAS_STATUS_SUCCESS &&
          sz) {
        stages.resize(sz / sizeof(int));
        cublasLtMatmulAlgoCapGetAttribute(&algo, CUBLASLT_ALGO_CAP_STAGES_IDS, stages.data(), sz, &sz);
      }
      if (stages.empty()) stages.push_back(CUBLASLT_MATMUL_STAGES_UNDEFINED);
      int splitk = 0, swz = 0;
      cublasLtMatmulAlgoCapGetAttribute(&algo, CUBLASLT_ALGO_CAP_SPLITK_SUPPORT, &splitk, sizeof splitk, &sz);
      cublasLtMatmulAlgoCapGetAttribute(&algo, CUBLASLT_ALGO_CAP_CTA_SWIZZLING_SUPPORT, &swz, sizeof swz, &sz);
      const int splits[] = {1, 2, 3, 4, 6, 8};
      for (int t : tiles)
        for (int st : stages)
          for (int sp : splits) {
            if (sp > 1 && !splitk) continue;
            for (int sw = 0; sw <= (swz ? 1 : 0); ++sw) {
              cublasLtMatmulAlgoConfigSetAttribute(&algo, CUBLASLT_ALGO_CONFIG_TILE_ID, &t, sizeof t);
              cublasLtMatmulAlgoConfigSetAttribute(&algo, CUBLASLT_ALGO_CONFIG_STAGES_ID, &st, sizeof st);
              cublasLtMatmulAlgoConfigSetAttribute(&algo, CUBLASLT_ALGO_CONFIG_SPLITK_NUM, &sp, sizeof sp);
              cublasLtMatmulAlgoConfigSetAttribute(&algo, CUBLASLT_ALGO_CONFIG_CTA_SWIZZLING, &sw, sizeof sw);
              if (sp > 1) {
                int red = CUBLASLT_REDUCTION_SCHEME_OUTPUT_TYPE;
                cublasLtMatmulAlgoConfigSetAttribute(&algo, CUBLASLT_ALGO_CONFIG_REDUCTION_SCHEME, &red, sizeof red);
              }
              cublasLtMatmulHeuristicResult_t chk;
              if (cublasLtMatmulAlgoCheck(lt, op, a, b, d, d, &algo, &chk) != CUBLAS_STATUS_SUCCESS) continue;
              if (chk.workspaceSize > kWs) continue;
              ++tried;
              const float tt = timed(&algo);
              if (tt < e_best) {
                e_best = tt;
                e_id = ids[ii];
                e_tile = t;
                e_split = sp;
                e_stage = st;
                e_sw = sw;
              }
            }
          }
    }
    printf("{\"shape\": \"%s\", \"B\": %d, \"family\": \"configured\", \"algo_ids\": %d, \"configs_timed\": %d, "
           "\"best_us\": %.2f, \"algo\": %d, \"tile\": %d, \"splitk\": %d, \"stages\": %d, \"swizzle\": %d, "
           "\"best_tflops\": %.0f}\n",
           p.name, p.B, nid, tried, e_best, e_id, e_tile, e_split, e_stage, e_sw, gflop / (e_best * 1e-6) / 1e3);
    fflush(stdout);
    cublasLtMatmulPreferenceDestroy(pref);
    cublasLtMatrixLayoutDestroy(a);
    cublasLtMatrixLayoutDestroy(b);
    cublasLtMatrixLayoutDestroy(d);
    cublasLtMatmulDescDestroy(op);
    for (auto w : Ws) cudaFree(w);
    cudaFree(X);
    cudaFree(Y);
    cudaFree(bias);
  }
  return 0;
}
