// Microbenchmark: shared-memory deposit primitives on B200 (sm_100a).
// Measures throughput of the candidate J-accumulation primitives for the K1 deposit design
// (DESIGN.md "Deposit primitive"): smem int32 atomics (native ATOMS.ADD), smem fp32 atomicAdd
// (CAS loop on sm_100a), plain LDS+FADD+STS read-modify-write, and global REDG.ADD.F32 to L2.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("ERR %s line %d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)
constexpr int NJ = 1088;   // ~ (16+3)^2*3 floats: one tile's J
constexpr int ITERS = 256;

__device__ __forceinline__ unsigned hsh(unsigned x){ x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x; }

template<int MODE>
__global__ void __launch_bounds__(256) kdep(float* out, int spread) {
  __shared__ float sj[NJ];
  __shared__ int si[NJ];
  for (int i = threadIdx.x; i < NJ; i += blockDim.x) { sj[i] = 0.f; si[i] = 0; }
  __syncthreads();
  unsigned h = hsh(threadIdx.x + 977u * blockIdx.x);
  float v = 1e-3f * (threadIdx.x & 7);
  #pragma unroll 4
  for (int it = 0; it < ITERS; ++it) {
    h = hsh(h + it);
    int a = spread ? (int)(h % (NJ - 8)) : (threadIdx.x >> 5);   // spread: random; else: same addr per warp
    #pragma unroll
    for (int k = 0; k < 8; ++k) {        // 8 deposits per "particle"
      int idx = a + k;
      if (MODE == 0) atomicAdd(&si[idx], (int)(v * 1e6f));
      else if (MODE == 1) atomicAdd(&sj[idx], v);
      else if (MODE == 2) { sj[idx] += v; }       // racy RMW (throughput reference only)
      else if (MODE == 3) atomicAdd(&out[(blockIdx.x * 64 + idx) & ((1 << 24) - 1)], v);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] += sj[5] + si[7];
}

__global__ void kcopy(const float4* __restrict__ a, float4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}

int main() {
  float* out; CK(cudaMalloc(&out, (1 << 24) * sizeof(float) + 4096));
  CK(cudaMemset(out, 0, (1 << 24) * sizeof(float)));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks = 148 * 8;
  const char* names[] = {"smem int32 atomicAdd", "smem fp32 atomicAdd(CAS)", "smem fp32 RMW (no atomic)", "global REDG f32"};
  for (int mode = 0; mode < 4; ++mode) for (int spread = 1; spread >= 0; --spread) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      switch (mode) { case 0: kdep<0><<<blocks,256>>>(out, spread); break; case 1: kdep<1><<<blocks,256>>>(out, spread); break;
                      case 2: kdep<2><<<blocks,256>>>(out, spread); break; case 3: kdep<3><<<blocks,256>>>(out, spread); break; }
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double ops = (double)blocks * 256 * ITERS * 8;
      if (rep) printf("%-28s spread=%d: %.3f ms  %.3e lane-ops/s  %.3f lane-ops/cycle/SM (at 1.9GHz)\n", names[mode], spread, ms, ops / (ms * 1e-3),
                      ops / (ms * 1e-3) / 148 / 1.9e9);
    }
  }
  size_t n = (size_t)1 << 28;  // 4 GiB per buffer in float4
  float4 *a, *b; CK(cudaMalloc(&a, n * 16)); CK(cudaMalloc(&b, n * 16)); cudaMemset(a, 0, n * 16);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0); kcopy<<<148 * 16, 256>>>(a, b, n); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("copy: %.1f GB/s\n", 2.0 * n * 16 / (ms * 1e-3) / 1e9);
  }
  CK(cudaGetLastError());
  return 0;
}
