// Standalone check of the TMA panel kernels on one synthetic window (no torch, no plan):
// left/right/Q products against a CPU triple loop.  Build: see tools/gpu_tma_probe.sh.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_1905_04975_b200/csrc/sn_kernels_panel_tma.cu"

using namespace sn;

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 300;
  const int k = argc > 2 ? atoi(argv[2]) : 64;
  const int j1 = argc > 3 ? atoi(argv[3]) : 100;
  const int mt = k <= 64 ? 64 : (k <= 128 ? 128 : 256);
  const int ld = n;
  std::vector<double> S((size_t)ld * n), Z((size_t)kZslot, 0.0);
  srand(1);
  for (auto& x : S) x = rand() / (double)RAND_MAX - 0.5;
  for (int c = 0; c < k; ++c) for (int r = 0; r < k; ++r) Z[r + c * kZld] = rand() / (double)RAND_MAX - 0.5;
  std::vector<int16_t> zr(kZrange);
  for (int c = 0; c < kZld; ++c) { zr[c] = c < k ? 0 : 255; zr[kZld + c] = c < k ? k - 1 : 0; }
  double *dS, *dZ; int16_t* dzr; WinDev* dw; int32_t *dst, *dpref;
  cudaMalloc(&dS, S.size() * 8); cudaMalloc(&dZ, Z.size() * 8); cudaMalloc(&dzr, zr.size() * 2);
  cudaMalloc(&dw, sizeof(WinDev)); cudaMalloc(&dst, 4); cudaMalloc(&dpref, 8);
  cudaMemcpy(dZ, Z.data(), Z.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dzr, zr.data(), zr.size() * 2, cudaMemcpyHostToDevice);
  WinDev w{}; w.j1 = j1; w.k = k; w.slot = 0; w.coff = 0; w.sidx = 0;
  cudaMemcpy(dw, &w, sizeof(w), cudaMemcpyHostToDevice);
  int one = 1; cudaMemcpy(dst, &one, 4, cudaMemcpyHostToDevice);
  PanelMaps pm;
  bool ok = panel_maps_init(&pm, dZ, 1, dS, n, n, ld);
  printf("maps ok %d\n", (int)ok);
  int fails = 0;
  for (int kind = 0; kind < 3; ++kind) {
    cudaMemcpy(dS, S.data(), S.size() * 8, cudaMemcpyHostToDevice);
    const int ns = kind == 0 ? (n - j1 - k + 63) / 64 : kind == 1 ? (j1 + 63) / 64 : (n + 63) / 64;
    int pref[2] = {0, ns};
    cudaMemcpy(dpref, pref, 8, cudaMemcpyHostToDevice);
    PanelArgs a{};
    a.wins = dw; a.nwin = 1; a.base = 0; a.prefix = dpref; a.strips = nullptr; a.part = 0; a.vec16 = 1;
    a.status = dst; a.M = dS; a.ld = ld; a.n = n; a.Z = dZ; a.zrange = dzr; a.maps = &pm;
    launch_panel_tma(kind, mt, a, ns, pm, 0);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<double> got(S.size());
    cudaMemcpy(got.data(), dS, S.size() * 8, cudaMemcpyDeviceToHost);
    double err = 0;
    if (e == cudaSuccess) {
      std::vector<double> ref = S;
      if (kind == 0) {
        for (int c = j1 + k; c < n; ++c) for (int m = 0; m < k; ++m) {
          double acc = 0; for (int q = 0; q < k; ++q) acc += Z[q + m * kZld] * S[(j1 + q) + (size_t)c * ld];
          ref[(j1 + m) + (size_t)c * ld] = acc;
        }
      } else {
        const int rows = kind == 1 ? j1 : n;
        for (int r = 0; r < rows; ++r) for (int m = 0; m < k; ++m) {
          double acc = 0; for (int q = 0; q < k; ++q) acc += S[r + (size_t)(j1 + q) * ld] * Z[q + m * kZld];
          ref[r + (size_t)(j1 + m) * ld] = acc;
        }
      }
      for (size_t i = 0; i < S.size(); ++i) err = fmax(err, fabs(ref[i] - got[i]));
    }
    printf("{\"probe\":\"tma_panel\",\"kind\":%d,\"mt\":%d,\"n\":%d,\"k\":%d,\"err\":\"%s\",\"maxdiff\":%.3g}\n", kind, mt,
           n, k, cudaGetErrorString(e), err);
    if (e != cudaSuccess || err > 1e-12) ++fails;
    if (e != cudaSuccess) return 2;
  }
  return fails;
}
