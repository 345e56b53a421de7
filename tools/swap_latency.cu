// Latency of one swap transform evaluation (phase A of the wavefront step) per swap type,
// measured with clock64 in a single thread on a shared-memory block.  Harness tool.
#include <cstdio>
#include "../paper_1905_04975_b200/csrc/sn_swap.cuh"

template <int N1, int N2>
__global__ void lat(const double* blk, long long* cyc, double* sink, int reps) {
  __shared__ double D[16];
  __shared__ double rec[32];
  if (threadIdx.x < 16) D[threadIdx.x] = blk[threadIdx.x];
  __syncthreads();
  if (threadIdx.x != 0) return;
  double acc = 0.0;
  long long t0 = clock64();
  for (int i = 0; i < reps; ++i) {
    bool rj = sn::dev::swap_compute<N1, N2>(D, 4, 0, rec);
    acc += rec[0] + (rj ? 1.0 : 0.0);
    D[0] += acc * 1e-300;   // serialise iterations through the block
  }
  long long t1 = clock64();
  cyc[0] = (t1 - t0) / reps;
  sink[0] = acc;
}

__global__ void lat22p(const double* blk, long long* cyc, double* sink, int reps) {
  __shared__ double D[16];
  if (threadIdx.x < 16) D[threadIdx.x] = blk[threadIdx.x];
  __syncthreads();
  double rec[32];
  double acc = 0.0;
  long long t0 = clock64();
  for (int i = 0; i < reps; ++i) {
    bool rj = sn::dev::swap_compute_22_paired(D, 4, 0, rec, threadIdx.x & 1);
    acc += rec[0] + (rj ? 1.0 : 0.0);
    __syncwarp();
    if (threadIdx.x == 0) D[0] += acc * 1e-300;
    __syncwarp();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = (t1 - t0) / reps; sink[0] = acc; }
}

int main() {
  // a 4x4 quasi-triangular block: [[a b . .],[c a . .],[0 0 e f],[0 0 g e]] etc.
  double h[16] = {2.0, -1.5, 0, 0,  1.2, 2.0, 0, 0,  0.3, -0.7, -3.0, 0.9,  0.4, 0.2, -1.1, -3.0};
  double h11[16] = {2.0, 0, 0, 0, 0.7, -1.0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  double h12[16] = {5.0, 0, 0, 0, 0.3, 1.0, -1.0, 0, -0.7, 1.0, 1.0, 0, 0, 0, 0, 0};
  double h21[16] = {1.0, -1.0, 0, 0, 1.0, 1.0, 0, 0, 0.3, -0.7, 5.0, 0, 0, 0, 0, 0};
  double *d, *sink; long long* c;
  cudaMalloc(&d, 128); cudaMalloc(&c, 8); cudaMalloc(&sink, 8);
  long long cyc;
  auto run = [&](const double* hb, auto kern, const char* name) {
    cudaMemcpy(d, hb, 128, cudaMemcpyHostToDevice);
    kern<<<1, 32>>>(d, c, sink, 200);
    cudaDeviceSynchronize();
    kern<<<1, 32>>>(d, c, sink, 200);
    cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost);
    printf("{\"probe\":\"swap_latency\",\"type\":\"%s\",\"cycles\":%lld}\n", name, cyc);
  };
  run(h11, lat<1, 1>, "1x1");
  run(h12, lat<1, 2>, "1x2");
  run(h21, lat<2, 1>, "2x1");
  run(h, lat<2, 2>, "2x2");
  run(h, lat22p, "2x2_paired");
  return 0;
}
