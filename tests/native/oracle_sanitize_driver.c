/* Host sanitizer driver for the oracle (host half): links oracle/lofp_oracle.c
 * built with -fsanitize=address,undefined and calls every exported function on small
 * random circuits (local and non-local, with gates).  Exit code 0 = no sanitizer report. */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

void oracle_bs_element(double theta, double phi, int x1, int x2, int y1, int y2, double out[2]);
int oracle_naive_permanent(int n, const double *a, double out[2]);
int oracle_ryser_permanent(int n, const double *a, double out[2]);
int oracle_circuit_unitary(int M, int D, const int *bpl, const int *ma, const int *mb, const double *th,
                           const double *ph, double *out);
int oracle_amplitude_permanent(int M, int D, const int *bpl, const int *ma, const int *mb, const double *th,
                               const double *ph, const int *S, long B, const int *T, int naive, int nt,
                               double *out);
int oracle_path_sum_gates(int M, int D, const int *bpl, const int *ma, const int *mb, const double *th,
                          const double *ph, const int *S, long B, const int *T, int prune, int nt, int ng,
                          const int *gm, const int *gl, const double *ga, const double *gb, double *out,
                          uint64_t *leaves);
int oracle_reachable(int M, int D, const int *bpl, const int *ma, const int *mb, const int *S, long B,
                     const int *T, int nt, uint8_t *out);
int oracle_count_paths(int M, int D, const int *bpl, const int *ma, const int *mb, const int *S, long B,
                       const int *T, int nt, long max_states, uint64_t *out, int *status);

static double urand(void) { return rand() / (double)RAND_MAX; }

int main(void) {
  srand(7);
  double out[2];
  for (int n = 0; n <= 12; ++n)
    for (int x1 = 0; x1 <= n; ++x1) oracle_bs_element(0.3 + 0.1 * n, 1.1, x1, n - x1, n / 2, n - n / 2, out);
  double A[2 * 36];
  for (int i = 0; i < 72; ++i) A[i] = urand() - 0.5;
  oracle_naive_permanent(6, A, out);
  oracle_ryser_permanent(6, A, out);
  for (int trial = 0; trial < 40; ++trial) {
    const int M = 2 + rand() % 6, D = rand() % 5, nonlocal = trial % 2;
    int bpl[8], ma[64], mb[64], nb = 0;
    double th[64], ph[64];
    for (int l = 0; l < D; ++l) {
      int used[8] = {0}, cnt = 0;
      for (int a = 0; a < M; ++a) {
        int b = nonlocal ? rand() % M : a + 1;
        if (b >= M || b == a || used[a] || used[b] || urand() < 0.3) continue;
        used[a] = used[b] = 1;
        ma[nb] = a;
        mb[nb] = b;
        th[nb] = urand() * 1.5;
        ph[nb] = urand() * 6.0;
        ++nb;
        ++cnt;
      }
      bpl[l] = cnt;
    }
    int S[8] = {0}, T[8 * 16] = {0}, N = rand() % 5;
    for (int i = 0; i < N; ++i) S[rand() % M]++;
    const int B = 16;
    for (int q = 0; q < B; ++q)
      for (int i = 0; i < N; ++i) T[q * M + rand() % M]++;
    double U[2 * 64], amps[2 * 16];
    uint64_t leaves[16], cnt2[32];
    uint8_t reach[16];
    int st[16], gm[2] = {0, M - 1}, gl[2] = {0, D};
    double ga[2] = {0.3, -0.7}, gb[2] = {0.1, 0.2};
    oracle_circuit_unitary(M, D, bpl, ma, mb, th, ph, U);
    oracle_amplitude_permanent(M, D, bpl, ma, mb, th, ph, S, B, T, 0, 1, amps);
    for (int prune = 0; prune <= 2; ++prune)
      oracle_path_sum_gates(M, D, bpl, ma, mb, th, ph, S, B, T, prune, 1, 2, gm, gl, ga, gb, amps, leaves);
    oracle_reachable(M, D, bpl, ma, mb, S, B, T, 1, reach);
    oracle_count_paths(M, D, bpl, ma, mb, S, B, T, 1, 1 << 16, cnt2, st);
  }
  puts("oracle sanitize driver: ok");
  return 0;
}
