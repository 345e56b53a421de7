// FP64 probe for sm_100a: (1) checks the register-fragment layouts assumed for
// mma.sync.aligned.m16n8k{4,8,16}.row.col.f64 against a host matmul, and
// (2) measures DFMA and DMMA throughput per SM.  Harness tool, not product code.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_probe fp64_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

// ---- fragment layout check -------------------------------------------------
// A is 16xK row-major, B is Kx8 (stored as B[k][n]), C 16x8.
template <int K>
__global__ void frag_check(const double* A, const double* B, double* C) {
  int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  double a[K / 2], b[K / 4], c[4] = {0, 0, 0, 0};
  for (int i = 0; i < K / 2; ++i) a[i] = A[(g + 8 * (i & 1)) * K + t + 4 * (i >> 1)];
  for (int i = 0; i < K / 4; ++i) b[i] = B[(t + 4 * i) * 8 + g];
  if (K == 4) {
    asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                 : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]));
  } else if (K == 8) {
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
                 : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
  } else {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                 : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
                 : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                   "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  C[g * 8 + 2 * t] = c[0];
  C[g * 8 + 2 * t + 1] = c[1];
  C[(g + 8) * 8 + 2 * t] = c[2];
  C[(g + 8) * 8 + 2 * t + 1] = c[3];
}

template <int K>
bool run_frag_check() {
  std::vector<double> A(16 * K), B(K * 8), C(128), R(128, 0.0);
  for (int i = 0; i < 16 * K; ++i) A[i] = (double)((i * 7) % 13) - 6.0;
  for (int i = 0; i < K * 8; ++i) B[i] = (double)((i * 5) % 11) - 5.0;
  for (int m = 0; m < 16; ++m)
    for (int n = 0; n < 8; ++n)
      for (int k = 0; k < K; ++k) R[m * 8 + n] += A[m * K + k] * B[k * 8 + n];
  double *dA, *dB, *dC;
  CK(cudaMalloc(&dA, A.size() * 8)); CK(cudaMalloc(&dB, B.size() * 8)); CK(cudaMalloc(&dC, 128 * 8));
  CK(cudaMemcpy(dA, A.data(), A.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size() * 8, cudaMemcpyHostToDevice));
  frag_check<K><<<1, 32>>>(dA, dB, dC);
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(C.data(), dC, 128 * 8, cudaMemcpyDeviceToHost));
  double err = 0;
  for (int i = 0; i < 128; ++i) err = fmax(err, fabs(C[i] - R[i]));
  printf("{\"probe\":\"frag_m16n8k%d\",\"max_err\":%g}\n", K, err);
  cudaFree(dA); cudaFree(dB); cudaFree(dC);
  return err == 0.0;
}

// ---- throughput ------------------------------------------------------------
__global__ void dfma_tput(double* out, int iters) {
  double x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-9 + i;
  const double a = 1.0000001, b = 1e-7;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.0) out[0] = s;
}

template <int K, int NACC>
__global__ void dmma_tput(double* out, int iters) {
  double a[K / 2], b[K / 4], c[NACC][4];
  for (int i = 0; i < K / 2; ++i) a[i] = 1e-3 * (threadIdx.x + i);
  for (int i = 0; i < K / 4; ++i) b[i] = 1e-3 * (threadIdx.x - i);
  for (int j = 0; j < NACC; ++j) for (int i = 0; i < 4; ++i) c[j][i] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < NACC; ++j) {
      if (K == 4)
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                     : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]));
      else if (K == 8)
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
      else
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                     : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                       "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0;
  for (int j = 0; j < NACC; ++j) for (int i = 0; i < 4; ++i) s += c[j][i];
  if (s == 12345.0) out[0] = s;
}

template <typename F>
double time_kernel(F launch, int reps) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  launch();  // warm-up
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(e0));
  for (int r = 0; r < reps; ++r) launch();
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
  return ms / reps;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int nsm = p.multiProcessorCount;
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  printf("{\"probe\":\"device\",\"name\":\"%s\",\"sms\":%d,\"clock_khz\":%d}\n", p.name, nsm, clk_khz);
  bool ok = run_frag_check<4>() & run_frag_check<8>() & run_frag_check<16>();
  printf("{\"probe\":\"frag_all_ok\",\"ok\":%s}\n", ok ? "true" : "false");
  double* out; CK(cudaMalloc(&out, 8));
  const int iters = 4096;
  for (int blocks_per_sm : {1, 2, 4, 8}) {
    int thr = 256;
    double ms = time_kernel([&] { dfma_tput<<<nsm * blocks_per_sm, thr>>>(out, iters); }, 5);
    double flops = 2.0 * 8 * iters * (double)thr * nsm * blocks_per_sm;
    printf("{\"probe\":\"dfma\",\"blocks_per_sm\":%d,\"tflops\":%.3f}\n", blocks_per_sm, flops / ms / 1e9);
  }
  for (int warps : {4, 8, 16}) {
    int thr = 32 * warps;
    double ms;
    ms = time_kernel([&] { dmma_tput<4, 8><<<nsm, thr>>>(out, iters); }, 5);
    printf("{\"probe\":\"dmma_k4\",\"warps\":%d,\"tflops\":%.3f}\n", warps, 2.0 * 16 * 8 * 4 * 8 * iters * (double)warps * nsm / ms / 1e9);
    ms = time_kernel([&] { dmma_tput<8, 8><<<nsm, thr>>>(out, iters); }, 5);
    printf("{\"probe\":\"dmma_k8\",\"warps\":%d,\"tflops\":%.3f}\n", warps, 2.0 * 16 * 8 * 8 * 8 * iters * (double)warps * nsm / ms / 1e9);
    ms = time_kernel([&] { dmma_tput<16, 4><<<nsm, thr>>>(out, iters / 2); }, 5);
    printf("{\"probe\":\"dmma_k16\",\"warps\":%d,\"tflops\":%.3f}\n", warps, 2.0 * 16 * 8 * 16 * 4 * (iters / 2) * (double)warps * nsm / ms / 1e9);
  }
  return 0;
}
