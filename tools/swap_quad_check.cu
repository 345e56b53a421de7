// Bitwise check and latency of the quad 2x2|2x2 transform (sylvester22_quad) against the
// one-thread swap_compute<2,2> and the lane-pair version, on many standardised random blocks
// (equal diagonals in each 2x2 block, so the Kronecker pivot search meets exact ties).
// Harness tool:  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/swap_quad_check tools/swap_quad_check.cu
#include <cstdio>
#include <cstdint>
#include "../paper_1905_04975_b200/csrc/sn_swap.cuh"

__device__ double urand(uint64_t& s) {
  s = s * 6364136223846793005ull + 1442695040888963407ull;
  return ((s >> 11) * (1.0 / 9007199254740992.0)) * 2.0 - 1.0;
}

__device__ void make_block(int idx, double (&Db)[4][4]) {
  uint64_t s = 0x9e3779b97f4a7c15ull * (uint64_t)(idx + 1);
  for (int r = 0; r < 4; ++r) for (int c = 0; c < 4; ++c) Db[r][c] = 0.0;
  const double sc = (idx % 7 == 0) ? 1e-3 : ((idx % 11 == 0) ? 1e3 : 1.0);
  for (int b = 0; b < 2; ++b) {
    const double a = urand(s) * 3.0, x = 0.25 + fabs(urand(s)), y = 0.25 + fabs(urand(s));
    Db[2 * b][2 * b] = a * sc; Db[2 * b + 1][2 * b + 1] = a * sc;
    Db[2 * b][2 * b + 1] = x * sc; Db[2 * b + 1][2 * b] = -y * sc;
  }
  if (idx % 13 == 0) { Db[2][2] = Db[0][0]; Db[3][3] = Db[0][0]; }   // near-common eigenvalues
  for (int r = 0; r < 2; ++r) for (int c = 2; c < 4; ++c) Db[r][c] = urand(s) * sc * ((idx % 5 == 0) ? 0.0 : 1.0);
}

__global__ void check(int nblk, unsigned long long* bad, unsigned long long* badpair) {
  const int lane = threadIdx.x & 31;
  const int gq = (blockIdx.x * blockDim.x + threadIdx.x) >> 2;   // one quad per block
  const int idx = gq < nblk ? gq : 0;
  double Db[4][4];
  make_block(idx, Db);
  double r1[sn::dev::kGen], r2[sn::dev::kGen], r3[sn::dev::kGen];
  const bool j1 = sn::dev::swap_compute_blk<2, 2>(Db, r1);
  const bool j2 = sn::dev::swap_compute_22_paired_blk(Db, r2, lane & 1);
  const bool j3 = sn::dev::swap_compute_22_quad_blk(Db, r3, lane & 3);
  if (gq >= nblk) return;
  bool ok = j1 == j3, okp = j1 == j2;
  if (!j1)
    for (int q = 0; q < sn::dev::kGen; ++q) {
      ok = ok && __double_as_longlong(r1[q]) == __double_as_longlong(r3[q]);
      okp = okp && __double_as_longlong(r1[q]) == __double_as_longlong(r2[q]);
    }
  if (!ok) atomicAdd(bad, 1ull);
  if (!okp) atomicAdd(badpair, 1ull);
}

template <int MODE>
__global__ void lat(long long* cyc, double* sink, int reps) {
  double Db[4][4];
  make_block(3, Db);
  double rec[sn::dev::kGen];
  double acc = 0.0;
  const int lane = threadIdx.x & 31;
  long long t0 = clock64();
  for (int i = 0; i < reps; ++i) {
    bool rj = MODE == 0 ? sn::dev::swap_compute_22_paired_blk(Db, rec, lane & 1)
                        : sn::dev::swap_compute_22_quad_blk(Db, rec, lane & 3);
    acc += rec[0] + (rj ? 1.0 : 0.0);
    Db[0][1] += acc * 1e-300;   // serialise iterations
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = (t1 - t0) / reps; sink[0] = acc; }
}

int main() {
  unsigned long long *bad, hb[2];
  long long* c; double* sink; long long cyc;
  cudaMalloc(&bad, 16); cudaMemset(bad, 0, 16);
  cudaMalloc(&c, 8); cudaMalloc(&sink, 8);
  const int nblk = 1 << 20;
  check<<<(nblk * 4 + 255) / 256, 256>>>(nblk, bad, bad + 1);
  cudaMemcpy(hb, bad, 16, cudaMemcpyDeviceToHost);
  printf("{\"probe\":\"swap_quad_check\",\"blocks\":%d,\"quad_mismatch\":%llu,\"pair_mismatch\":%llu}\n", nblk, hb[0], hb[1]);
  for (int m = 0; m < 2; ++m) {
    if (m == 0) { lat<0><<<1, 32>>>(c, sink, 200); lat<0><<<1, 32>>>(c, sink, 200); }
    else { lat<1><<<1, 32>>>(c, sink, 200); lat<1><<<1, 32>>>(c, sink, 200); }
    cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost);
    printf("{\"probe\":\"swap22_latency\",\"mode\":\"%s\",\"cycles\":%lld}\n", m ? "quad" : "pair", cyc);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("{\"cuda\":\"%s\"}\n", cudaGetErrorString(e));
  return (hb[0] || hb[1] || e != cudaSuccess) ? 1 : 0;
}
