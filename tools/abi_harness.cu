// Calls libsn_b200.so through its C ABI from a plain CUDA program (no torch): a random upper
// triangular S (1x1 blocks), Q = I, the trailing half selected.  Prints rc and the residual.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include "sn_reorder.h"

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 300;
  const int w = argc > 2 ? atoi(argv[2]) : 64;
  std::vector<double> S((size_t)n * n, 0.0), Q((size_t)n * n, 0.0);
  srand(3);
  for (int j = 0; j < n; ++j) {
    for (int i = 0; i < j; ++i) S[i + (size_t)j * n] = rand() / (double)RAND_MAX - 0.5;
    S[j + (size_t)j * n] = 20.0 * (rand() / (double)RAND_MAX) - 10.0;
    Q[j + (size_t)j * n] = 1.0;
  }
  std::vector<int32_t> sel(n);
  for (int i = 0; i < n; ++i) sel[i] = i >= n / 2;
  double *dS, *dQ;
  cudaMalloc(&dS, S.size() * 8); cudaMalloc(&dQ, Q.size() * 8);
  cudaMemcpy(dS, S.data(), S.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dQ, Q.data(), Q.size() * 8, cudaMemcpyHostToDevice);
  sn_opts o; sn_default_opts(&o); o.window = w; o.lookahead = 0; o.q_stream_overlap = 0; o.serialize = 1;
  int64_t m = 0; sn_stats st;
  int rc = sn_reorder_schur_ex(&o, n, dS, n, dQ, n, sel.data(), &m, nullptr, &st, nullptr);
  printf("{\"probe\":\"abi_harness\",\"n\":%d,\"w\":%d,\"rc\":%d,\"m\":%lld,\"windows\":%lld,\"err\":\"%s\"}\n", n, w, rc,
         (long long)m, (long long)st.windows, cudaGetErrorString(cudaDeviceSynchronize()));
  return rc != 0;
}
