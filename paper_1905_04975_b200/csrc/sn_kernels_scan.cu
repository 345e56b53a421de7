// sn_kernels_scan.cu -- structure scan of S ("upper
// quasi-triangular with 1x1 and 2x2 blocks on the diagonal").
//   subflag[i] = (S[i+1, i] != 0), i < n-1: a 2x2 block starts at i iff set.
//   validate_lower: *bad |= any nonzero strictly below the subdiagonal (n^2/2 reads, one CTA
//   per column, coalesced down the column).
#include "sn_device.cuh"

namespace sn {
namespace {

__global__ void subdiag_kernel(const double* S, int64_t ld, int64_t n, uint8_t* subflag) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i + 1 < n) subflag[i] = S[(i + 1) + i * ld] != 0.0 ? 1 : 0;
  else if (i < n) subflag[i] = 0;
}

__global__ void lower_kernel(const double* S, int64_t ld, int64_t n, int32_t* bad) {
  const int64_t c = blockIdx.x;
  const double* col = S + c * ld;
  int found = 0;
  for (int64_t r = c + 2 + threadIdx.x; r < n; r += blockDim.x) found |= (col[r] != 0.0);
  found = __syncthreads_or(found);
  if (found && threadIdx.x == 0) atomicOr(bad, 1);
}

// sharded S in the extended local layout (sn_dist.h): global column j of rank `rank`'s blocks
__device__ __forceinline__ int64_t ext_lcol(int64_t j, int64_t P, int64_t bc, int64_t hc) {
  const int64_t b = j / bc;
  return (b / P) * (bc + hc) + (j - b * bc);
}

__global__ void subdiag_dist_kernel(const double* Sx, int64_t ld, int64_t n, int64_t P, int64_t bc, int64_t hc,
                                    int64_t rank, uint8_t* subflag) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || (i / bc) % P != rank) return;
  subflag[i] = (i + 1 < n && Sx[(i + 1) + ext_lcol(i, P, bc, hc) * ld] != 0.0) ? 1 : 0;
}

__global__ void lower_dist_kernel(const double* Sx, int64_t ld, int64_t n, int64_t P, int64_t bc, int64_t hc,
                                  int64_t rank, int32_t* bad) {
  const int64_t c = blockIdx.x;
  if ((c / bc) % P != rank) return;
  const double* col = Sx + ext_lcol(c, P, bc, hc) * ld;
  int found = 0;
  for (int64_t r = c + 2 + threadIdx.x; r < n; r += blockDim.x) found |= (col[r] != 0.0);
  found = __syncthreads_or(found);
  if (found && threadIdx.x == 0) atomicOr(bad, 1);
}

}  // namespace

void launch_scan_dist(const double* Sx, int64_t ldx, int64_t n, int64_t P, int64_t bc, int64_t hc, int64_t rank,
                      int32_t validate_lower, uint8_t* subflag, int32_t* bad, cudaStream_t st) {
  if (n <= 0) return;
  subdiag_dist_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(Sx, ldx, n, P, bc, hc, rank, subflag);
  if (validate_lower && n > 2)
    lower_dist_kernel<<<(unsigned)(n - 2), 256, 0, st>>>(Sx, ldx, n, P, bc, hc, rank, bad);
}

void launch_scan(const double* S, int64_t ldS, int64_t n, int32_t validate_lower, uint8_t* subflag,
                 int32_t* bad, cudaStream_t st) {
  if (n <= 0) return;
  subdiag_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(S, ldS, n, subflag);
  if (validate_lower && n > 2) lower_kernel<<<(unsigned)(n - 2), 256, 0, st>>>(S, ldS, n, bad);
}

}  // namespace sn
