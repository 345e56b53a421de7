// Phase latencies of the 2x2|2x2 and 1x2 swap transforms (single thread / lane pair), clock64
// around each phase with the results forced through shared memory.  Harness tool.
#include <cstdio>
#include "../paper_1905_04975_b200/csrc/sn_swap.cuh"
using namespace sn::dev;

__global__ void phases22(const double* blk, long long* cyc, double* sink) {
  __shared__ double D[4][4];
  __shared__ volatile double keep[64];
  if (threadIdx.x < 16) D[threadIdx.x / 4][threadIdx.x % 4] = blk[threadIdx.x];
  __syncthreads();
  if (threadIdx.x != 0) return;
  double Db[4][4];
  for (int r = 0; r < 4; ++r) for (int c = 0; c < 4; ++c) Db[r][c] = D[c][r];
  long long t0 = clock64();
  double X[2][2] = {{0, 0}, {0, 0}}, scale;
  sylvester<2, 2>(Db, X, scale);
  keep[0] = X[0][0] + X[1][1] + scale;
  long long t1 = clock64();
  const Refl H1 = reflector(-X[0][0], -X[1][0], keep[0] * 0 + scale);
  const double temp = -H1.tau * (X[0][1] + H1.v1 * X[1][1]);
  const Refl H2 = reflector(-temp * H1.v1 - X[1][1], -temp * H1.v2, scale);
  keep[1] = H1.tau + H2.tau;
  long long t2 = clock64();
  double Dn[4][4];
  for (int r = 0; r < 4; ++r) for (int c = 0; c < 4; ++c) Dn[r][c] = Db[r][c] + keep[1] * 0;
  blk_refl_left<4>(Dn, 0, H1); blk_refl_right<4>(Dn, 0, H1);
  blk_refl_left<4>(Dn, 1, H2); blk_refl_right<4>(Dn, 1, H2);
  keep[2] = Dn[0][0] + Dn[3][3];
  long long t3 = clock64();
  const Std2 s1 = standardize(Dn[0][0] + keep[2] * 0, Dn[0][1], Dn[1][0], Dn[1][1]);
  keep[3] = s1.cs;
  long long t4 = clock64();
  cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3;
  sink[0] = keep[3];
}

int main() {
  double h[16] = {2.0, -1.5, 0, 0,  1.2, 2.0, 0, 0,  0.3, -0.7, -3.0, 0.9,  0.4, 0.2, -1.1, -3.0};
  double *d, *sink; long long* c;
  cudaMalloc(&d, 128); cudaMalloc(&c, 64); cudaMalloc(&sink, 8);
  cudaMemcpy(d, h, 128, cudaMemcpyHostToDevice);
  long long cy[4];
  for (int it = 0; it < 3; ++it) { phases22<<<1, 32>>>(d, c, sink); cudaDeviceSynchronize(); }
  cudaMemcpy(cy, c, 32, cudaMemcpyDeviceToHost);
  printf("{\"probe\":\"swap22_phases\",\"sylvester\":%lld,\"reflectors\":%lld,\"apply\":%lld,\"standardize_one\":%lld}\n",
         cy[0], cy[1], cy[2], cy[3]);
  return 0;
}
