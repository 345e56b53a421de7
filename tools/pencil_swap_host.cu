// Host-side check of the pencil swap transform of sn_pencil.cu (its __host__ __device__
// functions compiled for the CPU) against the oracle's or_gswap, on random small pencils.
// Build: nvcc -std=c++17 -I include -I oracle tools/pencil_swap_host.cu oracle/sn_oracle.c
//        -L paper_1905_04975_b200 -lsn_b200 -o tools/pencil_swap_host   (debug tool)
#include "../paper_1905_04975_b200/csrc/sn_pencil.cu"
extern "C" {
#include "sn_oracle.h"
}
#include <random>

int main() {
  std::mt19937_64 g(7);
  std::normal_distribution<double> N(0.0, 1.0);
  std::uniform_real_distribution<double> U(0.0, 1.0);
  double worst = 0.0;
  int rej = 0, cnt = 0;
  for (int n1 = 1; n1 <= 2; ++n1)
    for (int n2 = 1; n2 <= 2; ++n2)
      for (int trial = 0; trial < 2000; ++trial) {
        const int m = n1 + n2;
        double A[16] = {0}, B[16] = {0};
        for (int c = 0; c < m; ++c)
          for (int r = 0; r <= c; ++r) { A[r + 4 * c] = N(g); B[r + 4 * c] = N(g); }
        int r0 = 0;
        for (int q = 0; q < 2; ++q) {
          const int sz = q == 0 ? n1 : n2;
          if (sz == 1) { A[r0 * 5] = -10 + 20 * U(g); B[r0 * 5] = 0.5 + 1.5 * U(g); }
          else {
            const double a = -10 + 20 * U(g), b = (0.5 + 2.5 * U(g)) * (U(g) < 0.5 ? 1 : -1);
            const double cc = -(b > 0 ? 1 : -1) * (0.5 + 2.5 * U(g));
            A[r0 * 5] = A[(r0 + 1) * 5] = a; A[r0 + 4 * (r0 + 1)] = b; A[(r0 + 1) + 4 * r0] = cc;
            B[r0 * 5] = B[(r0 + 1) * 5] = 0.5 + 1.5 * U(g); B[r0 + 4 * (r0 + 1)] = 0.0;
          }
          r0 += sz;
        }
        double Uu[16], V[16], An[16], Bn[16];
        const bool ok = sn::pl_swap(A, B, n1, n2, Uu, V, An, Bn);
        // oracle on the same block as a full m x m pencil
        double S[16], T[16], Ql[16], Zr[16];
        for (int c = 0; c < m; ++c)
          for (int r = 0; r < m; ++r) {
            S[r + m * c] = A[r + 4 * c]; T[r + m * c] = B[r + 4 * c];
            Ql[r + m * c] = Zr[r + m * c] = (r == c);
          }
        const int orc = or_gswap(m, S, m, T, m, 0, n1, n2, Ql, m, m, Zr, m, m);
        if (!ok || orc) { ++rej; if (ok != (orc == 0)) { printf("reject mismatch %d %d\n", n1, n2); return 1; } continue; }
        double d = 0.0;
        for (int c = 0; c < m; ++c)
          for (int r = 0; r < m; ++r) {
            d = fmax(d, fabs(An[r + 4 * c] - S[r + m * c]));
            d = fmax(d, fabs(Bn[r + 4 * c] - T[r + m * c]));
            d = fmax(d, fabs(Uu[r + 4 * c] - Ql[r + m * c]));
            d = fmax(d, fabs(V[r + 4 * c] - Zr[r + m * c]));
          }
        worst = fmax(worst, d);
        ++cnt;
      }
  printf("pencil swap host check: %d swaps, %d rejected (both), max |device - oracle| = %.3g\n", cnt, rej, worst);
  return worst < 1e-10 ? 0 : 1;
}
