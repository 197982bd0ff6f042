// Probe: a 3D TMA box load of a guard-extended field plane into shared memory, with the tensor
// map in a __grid_constant__ struct parameter (the pattern K1 uses).  Prints mismatches.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>

struct Params {
  CUtensorMap tm;
  int cx, cy;
  float* out;
  const CUtensorMap* gtm;   // a copy in global memory (variant 2)
};

template <int VAR>
__global__ void k(const __grid_constant__ Params p) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) unsigned long long bar;
  const unsigned b = (unsigned)__cvta_generic_to_shared(&bar);
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem);
  constexpr int BYTES = 3 * 18 * 20 * 4;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b) : "memory");
    if (VAR == 0) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    else if (VAR == 1 || VAR == 2) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(BYTES) : "memory");
    if (VAR == 4)
      asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                   ::"r"(d), "l"(reinterpret_cast<uint64_t>(&p.tm)), "r"(p.cx), "r"(p.cy), "r"(0), "r"(b) : "memory");
    else
      asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                   ::"r"(d), "l"(reinterpret_cast<uint64_t>(VAR == 2 ? p.gtm : &p.tm)), "r"(p.cx), "r"(p.cy), "r"(0), "r"(b) : "memory");
  }
  __syncthreads();
  asm volatile("{\n .reg .pred done;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 done, [%0], 0;\n @!done bra WAIT_%=;\n}"
               ::"r"(b) : "memory");
  const float* s = reinterpret_cast<const float*>(smem);
  for (int i = threadIdx.x; i < 3 * 18 * 20; i += blockDim.x) p.out[i] = s[i];
}

int main(int argc, char** argv) {
  const int pitch = 64, rows = 40;
  const long plane = (long)pitch * rows;
  std::vector<float> h(3 * plane);
  for (long i = 0; i < 3 * plane; ++i) h[i] = (float)i;
  float *F, *out;
  cudaMalloc(&F, 3 * plane * 4);
  cudaMalloc(&out, 3 * 18 * 20 * 4);
  cudaMemcpy(F, h.data(), 3 * plane * 4, cudaMemcpyHostToDevice);
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  Params p{};
  const cuuint64_t dims[3] = {(cuuint64_t)pitch, (cuuint64_t)rows, 3};
  const cuuint64_t str[2] = {(cuuint64_t)pitch * 4, (cuuint64_t)plane * 4};
  const cuuint32_t box[3] = {20, 18, 3}, es[3] = {1, 1, 1};
  CUresult r = enc(&p.tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, F, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  p.cx = 51; p.cy = 30; p.out = out;
  CUtensorMap* g;
  cudaMalloc(&g, sizeof(CUtensorMap));
  cudaMemcpy(g, &p.tm, sizeof(CUtensorMap), cudaMemcpyHostToDevice);
  p.gtm = g;
  const int var = argc > 1 ? atoi(argv[1]) : 0;
  if (argc > 2) { p.cx = atoi(argv[2]); p.cy = atoi(argv[3]); }
  {
    cudaMemset(out, 0xff, 3 * 18 * 20 * 4);
    if (var == 0) { cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192); k<0><<<1, 128, 8192>>>(p); }
    else if (var == 1) { cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192); k<1><<<1, 128, 8192>>>(p); }
    else if (var == 2) { cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192); k<2><<<1, 128, 8192>>>(p); }
    else if (var == 3) { cudaFuncSetAttribute(k<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192); k<3><<<1, 128, 8192>>>(p); }
    else { cudaFuncSetAttribute(k<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192); k<4><<<1, 128, 8192>>>(p); }
    cudaError_t e = cudaDeviceSynchronize();
    printf("variant %d: %s\n", var, cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
    std::vector<float> o(3 * 18 * 20);
    cudaMemcpy(o.data(), out, o.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int c = 0; c < 3; ++c)
      for (int y = 0; y < 18; ++y)
        for (int x = 0; x < 20; ++x) {
          const int gx = p.cx + x, gy = p.cy + y;
          const float want = (gx < pitch && gy < rows) ? h[c * plane + (long)gy * pitch + gx] : 0.f;
          if (o[(c * 18 + y) * 20 + x] != want && bad++ < 5) printf("  c%d y%d x%d got %g want %g\n", c, y, x, o[(c * 18 + y) * 20 + x], want);
        }
    printf("variant %d mismatches %d\n", var, bad);
  }
  return 0;
}
