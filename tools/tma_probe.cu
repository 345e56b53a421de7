// Standalone probe: one TMA box load (FP64, no swizzle, padded box) through an mbarrier.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(const __grid_constant__ CUtensorMap map, int c0, int c1, double* out, int nel) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&bar)), "r"(1) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(nel * 8) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
        ::"r"(sa(sm)), "l"(&map), "r"(c0), "r"(c1), "r"(sa(&bar)) : "memory");
  }
  asm volatile(
      "{\n .reg .pred p;\n"
      "W_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra W_%=;\n}\n" ::"r"(sa(&bar)), "r"(0) : "memory");
  for (int i = threadIdx.x; i < nel; i += blockDim.x) out[i] = ((double*)sm)[i];
}

int main() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  const int R = 300, Cn = 200, ld = 300;
  std::vector<double> h((size_t)ld * Cn);
  for (int c = 0; c < Cn; ++c) for (int r = 0; r < R; ++r) h[r + (size_t)c * ld] = r + 1000.0 * c;
  double *d, *o;
  cudaMalloc(&d, h.size() * 8); cudaMalloc(&o, 1 << 20);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  int boxes[3][2] = {{20, 64}, {68, 16}, {20, 256}};
  int bad_total = 0;
  for (auto& b : boxes) {
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)R, (cuuint64_t)Cn};
    cuuint64_t str[1] = {(cuuint64_t)ld * 8};
    cuuint32_t box[2] = {(cuuint32_t)b[0], (cuuint32_t)b[1]};
    cuuint32_t es[2] = {1, 1};
    CUresult rc = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int nel = b[0] * b[1];
    const int c0 = 290, c1 = 190;   // partly out of bounds
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
    probe<<<1, 128, nel * 8 + 1024>>>(m, c0, c1, o, nel);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<double> got(nel);
    cudaMemcpy(got.data(), o, nel * 8, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int y = 0; y < b[1]; ++y) for (int x = 0; x < b[0]; ++x) {
      const int r = c0 + x, c = c1 + y;
      const double exp = (r < R && c < Cn) ? h[r + (size_t)c * ld] : 0.0;
      if (got[x + y * b[0]] != exp) ++bad;
    }
    bad_total += bad;
    printf("{\"probe\":\"tma_box\",\"box\":[%d,%d],\"encode\":%d,\"err\":\"%s\",\"bad\":%d}\n", b[0], b[1], (int)rc,
           cudaGetErrorString(e), bad);
    if (e != cudaSuccess) return 1;
  }
  return bad_total != 0;
}
