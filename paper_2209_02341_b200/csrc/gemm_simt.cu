// gemm_simt.cu -- fp32 SIMT GEMM for the fp32 parity mode (BASELINE.json config 1, target 1e-4).
// D[M,N] = A[M,K] . W[N,K]^T (+ bias[N]) (GeLU), fp32 FMA, k ascending per output element.
// Not a performance path: tensor cores (TF32) cannot meet 1e-4, so parity mode stays on the FMA pipe.
#include "common.cuh"
#include "kernels.h"

namespace energon {

constexpr int SG_BM = 64, SG_BN = 64, SG_BK = 16;

__global__ void __launch_bounds__(256) gemm_f32_kernel(const float* __restrict__ A, const float* __restrict__ W,
                                                       const float* __restrict__ bias, float* __restrict__ D, int M,
                                                       int N, int K, int epi) {
  pdl_trigger();
  pdl_wait();
  __shared__ float As[SG_BK][SG_BM + 4];
  __shared__ float Ws[SG_BK][SG_BN + 4];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int m0 = blockIdx.y * SG_BM, n0 = blockIdx.x * SG_BN;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += SG_BK) {
    // 64 x 16 tiles of A and W: 1024 elements each, 4 per thread
    for (int i = threadIdx.x; i < SG_BM * SG_BK; i += 256) {
      const int r = i / SG_BK, c = i % SG_BK;
      const int gm = m0 + r, gn = n0 + r, gk = k0 + c;
      As[c][r] = (gm < M && gk < K) ? A[(int64_t)gm * K + gk] : 0.f;
      Ws[c][r] = (gn < N && gk < K) ? W[(int64_t)gn * K + gk] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < SG_BK; ++kk) {
      float a[4], w[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) w[j] = Ws[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], w[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty * 4 + i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      if (n >= N) continue;
      float v = acc[i][j];
      if (epi >= EPI_BIAS) v += bias[n];
      if (epi == EPI_BIAS_GELU) v = gelu_tanh(v);
      D[(int64_t)m * N + n] = v;
    }
  }
}

void launch_gemm_f32(const float* A, const float* W, const float* bias, float* D, int M, int N, int K, int epi,
                     cudaStream_t st) {
  if (M <= 0 || N <= 0) return;
  dim3 grid((N + SG_BN - 1) / SG_BN, (M + SG_BM - 1) / SG_BM);
  launch_k(gemm_f32_kernel, dim3(grid), dim3(256), 0, st, A, W, bias, D, M, N, K, epi);
}

}  // namespace energon
