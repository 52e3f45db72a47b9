/*
 * oracle/lofp_oracle.c — CPU ORACLE FOR THE LOFP PATH SUM.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load this library.  The product path (paper_2510_26408_b200/) never
 * includes, links or calls anything here, and this file includes nothing from it.
 *
 * Everything is plain, slow and written from the paper (arXiv 2510.26408, PAPER.md
 * lines "P:n"); arithmetic is `long double` (x87 80-bit) complex, except the
 * Appendix-A element, which is summed in __float128 (113-bit significand) because its
 * alternating t-sum cancels catastrophically at high photon numbers (DESIGN.md reading
 * R18: a precision choice only; the formula is the paper's).
 *
 *   oracle_bs_element      Appendix A, the printed factorial (y1-x2+t)!
 *                          of P:406 read as (x2-y1+t)! (reading R1); summed
 *                          in __float128 (reading R18).
 *   oracle_naive_permanent definition of the permanent, sum over all n!
 *                          permutations.
 *   oracle_ryser_permanent Ryser's formula in Gray-code order.
 *   oracle_circuit_unitary U = U_D ... U_1 from eq. bs_matrix.
 *   oracle_amplitude_permanent  <T|U_P|S> = Per(U[T,S]) / sqrt(prod S! prod T!)
 *                          (P:41): rows of U repeated by T, columns by S.
 *   oracle_path_sum        eq. (1): recursion over the BS in layer order,
 *                          summing the product of Appendix-A elements of every valid
 *                          path.  prune 0 = none (final check against T only),
 *                          1 = the paper's past/future light-cone upper bounds,
 *                          2 = the cumulative light-cone box (reading R5).
 *   oracle_path_sum_gates  the same recursion with photon-number-preserving phase gates
 *                          exp(i (a n + b n^2)) on a mode after a layer (reading
 *                          R19), multiplied in when the layer that precedes them ends.
 *   oracle_cone_bound      the per-waveguide bound of P:164.
 *   oracle_count_paths     exact number of valid paths (the number of terms of eq. (1))
 *                          by a transfer over cuts with explicit constraint checks
 *                          (reading R6); pinned against oracle_path_sum's leaf
 *                          count in tests/.
 *   oracle_reachable       structural reachability (the box test, reading R5).
 *
 * Every pin lives in tests/test_oracle_*.py.  No function here is "parity unpinned".
 */
#include <complex.h>
#include <math.h>
#include <quadmath.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef long double R;
typedef long double complex C;

#define ORACLE_MAXM 256
#define ORACLE_MAXD 64
#define ORACLE_MAXN 120 /* photons (uint8-safe; the ABI's LOFP_MAX_PHOTONS) */

/* ------------------------------------------------------------------------- */
/* small helpers                                                              */
/* ------------------------------------------------------------------------- */

static R fact(int n) {
  R f = 1.0L;
  for (int i = 2; i <= n; ++i) f *= (R)i;
  return f;
}

/* eq. bs_matrix: BS = [[cos t, -e^{-i phi} sin t], [e^{i phi} sin t, cos t]]. */
static void bs_matrix(double theta, double phi, C u[4]) {
  R c = cosl((R)theta), s = sinl((R)theta);
  C e = cosl((R)phi) + I * sinl((R)phi);
  u[0] = c;               /* U11 */
  u[1] = -conjl(e) * s;   /* U12 */
  u[2] = e * s;           /* U21 */
  u[3] = c;               /* U22 */
}

/* Appendix A.  <y1,y2|BS|x1,x2> =
 *   1/sqrt(x1!x2!y1!y2!) * sum_t [y1! x1! / (t! (y1-t)!)] [y2! x2! / ((x1-t)! (x2-y1+t)!)]
 *                         U11^t U12^(y1-t) U21^(x1-t) U22^(x2-y1+t)
 * with max(0, y1-x2, x1-y2) <= t <= min(x1, y1).  Zero when photon number
 * is not conserved ("valid path").  Summed term by term in __float128 (reading
 * R18): the terms alternate in sign and exceed the result by up to ~1e17 at 120
 * photons, which a 64-bit significand cannot absorb. */
typedef __float128 Q;
typedef __complex128 QC;

static Q QFACT[ORACLE_MAXN + 1]; /* n! in __float128, filled when the library loads */

__attribute__((constructor)) static void qfact_init(void) {
  QFACT[0] = 1.0Q;
  for (int i = 1; i <= ORACLE_MAXN; ++i) QFACT[i] = QFACT[i - 1] * (Q)i;
}

static Q qfact(int n) { return QFACT[n]; }

static void bs_matrix_q(double theta, double phi, QC u[4]) {
  Q c = cosq((Q)theta), s = sinq((Q)theta);
  QC e = cosq((Q)phi) + 1.0Qi * sinq((Q)phi);
  u[0] = c;              /* U11 */
  u[1] = -conjq(e) * s;  /* U12 */
  u[2] = e * s;          /* U21 */
  u[3] = c;              /* U22 */
}

/* The t-sum of Appendix A with the powers U_ij^p tabulated (p <= n; 0^0 = 1). */
static QC bs_element_q(const QC u[4], int x1, int x2, int y1, int y2) {
  if (x1 < 0 || x2 < 0 || y1 < 0 || y2 < 0 || x1 + x2 != y1 + y2) return 0.0Q;
  int n = x1 + x2;
  QC pw[4][ORACLE_MAXN + 1];
  for (int k = 0; k < 4; ++k) {
    pw[k][0] = 1.0Q;
    for (int p = 1; p <= n; ++p) pw[k][p] = pw[k][p - 1] * u[k];
  }
  int tlo = 0;
  if (y1 - x2 > tlo) tlo = y1 - x2;
  if (x1 - y2 > tlo) tlo = x1 - y2;
  int thi = x1 < y1 ? x1 : y1;
  QC per = 0.0Q;
  for (int t = tlo; t <= thi; ++t) {
    Q comb = (qfact(y1) * qfact(x1) / (qfact(t) * qfact(y1 - t))) *
             (qfact(y2) * qfact(x2) / (qfact(x1 - t) * qfact(x2 - y1 + t)));
    per += comb * pw[0][t] * pw[1][y1 - t] * pw[2][x1 - t] * pw[3][x2 - y1 + t];
  }
  return per / sqrtq(qfact(x1) * qfact(x2) * qfact(y1) * qfact(y2));
}

static C bs_element_theta(double theta, double phi, int x1, int x2, int y1, int y2) {
  QC u[4];
  bs_matrix_q(theta, phi, u);
  QC a = bs_element_q(u, x1, x2, y1, y2);
  return (R)crealq(a) + I * (R)cimagq(a);
}

void oracle_bs_element(double theta, double phi, int x1, int x2, int y1, int y2, double out[2]) {
  if (x1 + x2 > ORACLE_MAXN || y1 + y2 > ORACLE_MAXN) { out[0] = out[1] = NAN; return; }
  C a = bs_element_theta(theta, phi, x1, x2, y1, y2);
  out[0] = (double)creall(a);
  out[1] = (double)cimagl(a);
}

/* ------------------------------------------------------------------------- */
/* permanents                                                                 */
/* ------------------------------------------------------------------------- */

/* Definition: Per(A) = sum over permutations sigma of prod_i a_{i,sigma(i)}. */
static C naive_perm_rec(int n, const C *A, int row, uint32_t used) {
  if (row == n) return 1.0L;
  C s = 0.0L;
  for (int j = 0; j < n; ++j)
    if (!(used & (1u << j))) s += A[row * n + j] * naive_perm_rec(n, A, row + 1, used | (1u << j));
  return s;
}

/* Ryser's formula Per(A) = (-1)^n sum_{S subset [n]} (-1)^{|S|} prod_i sum_{j in S} a_ij,
 * visiting the subsets in Gray-code order so one column is added or removed per step
 * (P:41). */
static C ryser_perm(int n, const C *A) {
  if (n == 0) return 1.0L;
  C rowsum[64];
  for (int i = 0; i < n; ++i) rowsum[i] = 0.0L;
  C total = 0.0L;
  uint64_t g_prev = 0;
  uint64_t nsub = 1ull << n;
  for (uint64_t k = 1; k < nsub; ++k) {
    uint64_t g = k ^ (k >> 1);
    uint64_t diff = g ^ g_prev;
    int j = __builtin_ctzll(diff);
    R sgn = (g & diff) ? 1.0L : -1.0L; /* column j entered (+) or left (-) the subset */
    for (int i = 0; i < n; ++i) rowsum[i] += sgn * A[i * n + j];
    C prod = 1.0L;
    for (int i = 0; i < n; ++i) prod *= rowsum[i];
    int sz = __builtin_popcountll(g);
    total += ((sz & 1) ? -1.0L : 1.0L) * prod;
    g_prev = g;
  }
  return ((n & 1) ? -1.0L : 1.0L) * total;
}

static void unpack_matrix(int n, const double *a, C *A) {
  for (int i = 0; i < n * n; ++i) A[i] = (R)a[2 * i] + I * (R)a[2 * i + 1];
}

int oracle_naive_permanent(int n, const double *a /* [n][n][2] */, double out[2]) {
  if (n < 0 || n > 10) return -1;
  C A[100];
  unpack_matrix(n, a, A);
  C p = naive_perm_rec(n, A, 0, 0);
  out[0] = (double)creall(p);
  out[1] = (double)cimagl(p);
  return 0;
}

int oracle_ryser_permanent(int n, const double *a, double out[2]) {
  if (n < 0 || n > 40) return -1;
  C *A = (C *)malloc(sizeof(C) * (size_t)(n > 0 ? n * n : 1));
  unpack_matrix(n, a, A);
  C p = ryser_perm(n, A);
  free(A);
  out[0] = (double)creall(p);
  out[1] = (double)cimagl(p);
  return 0;
}

/* ------------------------------------------------------------------------- */
/* circuits                                                                   */
/* ------------------------------------------------------------------------- */

/* A circuit is D layers; layer l holds bs_per_layer[l] beam splitters, listed
 * layer-major in (mode_a, mode_b, theta, phi).  mode_a is BS port 1 (the "upper"
 * waveguide of P:92): x1 = occupation of mode_a, x2 = occupation of mode_b. */
typedef struct {
  int M, D, nbs;
  const int *bs_per_layer;
  const int *ma, *mb;
  const double *theta, *phi;
} circuit_t;

static int circuit_check(const circuit_t *c) {
  if (c->M < 1 || c->M > ORACLE_MAXM || c->D < 0 || c->D > ORACLE_MAXD) return -1;
  int n = 0;
  for (int l = 0; l < c->D; ++l) {
    if (c->bs_per_layer[l] < 0) return -1;
    int used[ORACLE_MAXM];
    memset(used, 0, sizeof(used));
    for (int i = 0; i < c->bs_per_layer[l]; ++i, ++n) {
      int a = c->ma[n], b = c->mb[n];
      if (a < 0 || b < 0 || a >= c->M || b >= c->M || a == b) return -1;
      if (used[a] || used[b]) return -1;
      used[a] = used[b] = 1;
    }
  }
  return n;
}

/* U = U_D ... U_1: layer unitaries act on output creation operators, later
 * layers on the left.  U[i][j] = amplitude for input mode j -> output mode i, so the
 * BS block is U[a][a]=U11, U[a][b]=U12, U[b][a]=U21, U[b][b]=U22 (rows = outputs as
 * in the Appendix-A expansion). */
static void circuit_unitary(const circuit_t *c, C *U) {
  int M = c->M;
  for (int i = 0; i < M * M; ++i) U[i] = 0.0L;
  for (int i = 0; i < M; ++i) U[i * M + i] = 1.0L;
  C *T = (C *)malloc(sizeof(C) * (size_t)M * M);
  int n = 0;
  for (int l = 0; l < c->D; ++l) {
    memcpy(T, U, sizeof(C) * (size_t)M * M);
    for (int i = 0; i < c->bs_per_layer[l]; ++i, ++n) {
      int a = c->ma[n], b = c->mb[n];
      C u[4];
      bs_matrix(c->theta[n], c->phi[n], u);
      for (int j = 0; j < M; ++j) {
        C ra = T[a * M + j], rb = T[b * M + j];
        U[a * M + j] = u[0] * ra + u[1] * rb;
        U[b * M + j] = u[2] * ra + u[3] * rb;
      }
    }
  }
  free(T);
}

int oracle_circuit_unitary(int M, int D, const int *bs_per_layer, const int *ma, const int *mb,
                           const double *theta, const double *phi, double *out /* [M][M][2] */) {
  circuit_t c = {M, D, 0, bs_per_layer, ma, mb, theta, phi};
  if (circuit_check(&c) < 0) return -1;
  C *U = (C *)malloc(sizeof(C) * (size_t)M * M);
  circuit_unitary(&c, U);
  for (int i = 0; i < M * M; ++i) {
    out[2 * i] = (double)creall(U[i]);
    out[2 * i + 1] = (double)cimagl(U[i]);
  }
  free(U);
  return 0;
}

/* <T|U_P|S> = Per(U[T,S]) / sqrt(prod_i S_i! prod_j T_j!). */
static C amplitude_permanent(int M, const C *U, const int *S, const int *T, int use_naive) {
  int nS = 0, nT = 0;
  for (int i = 0; i < M; ++i) { nS += S[i]; nT += T[i]; }
  if (nS != nT) return 0.0L;
  int n = nS;
  int rows[64], cols[64];
  int r = 0, q = 0;
  for (int i = 0; i < M; ++i) for (int k = 0; k < T[i]; ++k) rows[r++] = i;
  for (int j = 0; j < M; ++j) for (int k = 0; k < S[j]; ++k) cols[q++] = j;
  C *A = (C *)malloc(sizeof(C) * (size_t)(n > 0 ? n * n : 1));
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) A[i * n + j] = U[rows[i] * M + cols[j]];
  C p = use_naive ? naive_perm_rec(n, A, 0, 0) : ryser_perm(n, A);
  free(A);
  R norm = 1.0L;
  for (int i = 0; i < M; ++i) norm *= fact(S[i]) * fact(T[i]);
  return p / sqrtl(norm);
}

int oracle_amplitude_permanent(int M, int D, const int *bs_per_layer, const int *ma, const int *mb,
                               const double *theta, const double *phi, const int *S, long B,
                               const int *T /* [B][M] */, int use_naive, int nthreads,
                               double *out /* [B][2] */) {
  circuit_t c = {M, D, 0, bs_per_layer, ma, mb, theta, phi};
  if (circuit_check(&c) < 0) return -1;
  int nS = 0;
  for (int i = 0; i < M; ++i) { if (S[i] < 0) return -1; nS += S[i]; }
  if (nS > 40 || (use_naive && nS > 10)) return -2;
  C *U = (C *)malloc(sizeof(C) * (size_t)M * M);
  circuit_unitary(&c, U);
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1)
#endif
  for (long b = 0; b < B; ++b) {
    C a = amplitude_permanent(M, U, S, T + b * M, use_naive);
    out[2 * b] = (double)creall(a);
    out[2 * b + 1] = (double)cimagl(a);
  }
  free(U);
  return 0;
}

/* ------------------------------------------------------------------------- */
/* light cones                                                    */
/* ------------------------------------------------------------------------- */

/* Past light cone of waveguide (mode m, segment j) -- segment j is the output of
 * layer j, j = 0 the input: the input modes connected to it through
 * layers j..1.  Future cone: the output modes connected to it through layers
 * j+1..D.  Bound = min(sum of S over the past cone, sum of T over the future cone). */
static int cone_bound(const circuit_t *c, const int *layer_start, const int *S, const int *T, int m,
                      int j) {
  int M = c->M;
  unsigned char in[ORACLE_MAXM];
  memset(in, 0, sizeof(in));
  in[m] = 1;
  for (int l = j - 1; l >= 0; --l)
    for (int i = layer_start[l]; i < layer_start[l + 1]; ++i)
      if (in[c->ma[i]] || in[c->mb[i]]) in[c->ma[i]] = in[c->mb[i]] = 1;
  int past = 0;
  for (int i = 0; i < M; ++i) if (in[i]) past += S[i];
  memset(in, 0, sizeof(in));
  in[m] = 1;
  for (int l = j; l < c->D; ++l)
    for (int i = layer_start[l]; i < layer_start[l + 1]; ++i)
      if (in[c->ma[i]] || in[c->mb[i]]) in[c->ma[i]] = in[c->mb[i]] = 1;
  int fut = 0;
  for (int i = 0; i < M; ++i) if (in[i]) fut += T[i];
  return past < fut ? past : fut;
}

/* Exposed for the P:164 worked-example pin: the past and future cone membership. */
int oracle_cone_sets(int M, int D, const int *bs_per_layer, const int *ma, const int *mb, int m,
                     int j, int *past /* [M] */, int *future /* [M] */) {
  circuit_t c = {M, D, 0, bs_per_layer, ma, mb, NULL, NULL};
  if (circuit_check(&c) < 0 || m < 0 || m >= M || j < 0 || j > D) return -1;
  int ls[ORACLE_MAXD + 1];
  ls[0] = 0;
  for (int l = 0; l < D; ++l) ls[l + 1] = ls[l] + bs_per_layer[l];
  for (int i = 0; i < M; ++i) past[i] = future[i] = 0;
  past[m] = 1;
  for (int l = j - 1; l >= 0; --l)
    for (int i = ls[l]; i < ls[l + 1]; ++i)
      if (past[ma[i]] || past[mb[i]]) past[ma[i]] = past[mb[i]] = 1;
  future[m] = 1;
  for (int l = j; l < D; ++l)
    for (int i = ls[l]; i < ls[l + 1]; ++i)
      if (future[ma[i]] || future[mb[i]]) future[ma[i]] = future[mb[i]] = 1;
  return 0;
}

/* ------------------------------------------------------------------------- */
/* cumulative light-cone box (reading R5; requires nearest-neighbour pairs)    */
/* ------------------------------------------------------------------------- */

/* Cut k (1..M-1) sits between modes k-1 and k; F(k) = photons in modes < k.  A BS on
 * modes {k-1, k} in layer l is "active at cut k".  Box: lo_D(k) = hi_D(k) = G(k) =
 * sum_{i<k} T_i; going back through layer l: lo_{l-1}(k) = lo_l(k-1), hi_{l-1}(k) =
 * hi_l(k+1) for cuts active in l, unchanged otherwise.  lo/hi are [D+1][M+1]. */
static int is_nn(const circuit_t *c) {
  for (int i = 0; i < c->nbs; ++i) if (abs(c->ma[i] - c->mb[i]) != 1) return 0;
  return 1;
}

static void build_box(const circuit_t *c, const int *layer_start, const int *T, int *lo, int *hi) {
  int M = c->M, D = c->D, W = M + 1;
  int G = 0;
  for (int k = 0; k <= M; ++k) {
    lo[D * W + k] = hi[D * W + k] = G;
    if (k < M) G += T[k];
  }
  for (int l = D; l >= 1; --l) {
    unsigned char act[ORACLE_MAXM + 1];
    memset(act, 0, sizeof(act));
    for (int i = layer_start[l - 1]; i < layer_start[l]; ++i) {
      int k = c->ma[i] > c->mb[i] ? c->ma[i] : c->mb[i];
      act[k] = 1;
    }
    for (int k = 0; k <= M; ++k) {
      if (act[k]) {
        lo[(l - 1) * W + k] = lo[l * W + k - 1];
        hi[(l - 1) * W + k] = hi[l * W + k + 1];
      } else {
        lo[(l - 1) * W + k] = lo[l * W + k];
        hi[(l - 1) * W + k] = hi[l * W + k];
      }
    }
  }
}

/* ------------------------------------------------------------------------- */
/* eq. (1): the Feynman path sum                        */
/* ------------------------------------------------------------------------- */

typedef struct {
  const circuit_t *c;
  const int *layer_start;
  const int *T;
  int N;
  int prune;
  const int *bound;   /* prune 1: [D+1][M] cone bounds */
  const int *lo, *hi; /* prune 2: [D+1][M+1] box */
  const C *elem;      /* per-BS element cache [nbs][tri(N)] */
  const int *tri_off; /* offset of photon number n inside a BS's cache */
  int tri_size;
  int ngates;         /* photon-number-preserving phase gates */
  const int *g_mode, *g_after;
  const double *g_a, *g_b;
  int occ[ORACLE_MAXM];
  C acc;
  uint64_t leaves;
} pathsum_t;

/* Appendix-A element of BS b for (x1, x2) -> (y1, x1+x2-y1), from the cache. */
static C elem_of(const pathsum_t *p, int b, int x1, int x2, int y1) {
  int n = x1 + x2;
  return p->elem[(size_t)b * p->tri_size + p->tri_off[n] + x1 * (n + 1) + y1];
}

/* Phase gates ("nonlinear phase gates are also photon-number preserving"): a
 * gate on mode m after layer j (j = 0: on the input) multiplies the path by
 * exp(i (a n + b n^2)), n = the photons in mode m after layer j.  b = 0 is a linear
 * phase shifter, b != 0 a Kerr-type nonlinear phase (reading R19). */
static C gate_factor(const pathsum_t *p, int after_layer) {
  C f = 1.0L;
  for (int g = 0; g < p->ngates; ++g) {
    if (p->g_after[g] != after_layer) continue;
    R n = (R)p->occ[p->g_mode[g]];
    R arg = (R)p->g_a[g] * n + (R)p->g_b[g] * n * n;
    f *= cosl(arg) + I * sinl(arg);
  }
  return f;
}

/* Recursion over the BS in layer order ("a systematic way to enumerate all possible
 * valid paths"): BS b gets every output split y1 = 0..x1+x2 (photon number is
 * conserved at each BS); the product of BS elements along the path is
 * carried down ("multiply these individual amplitudes"); at the end a path is
 * valid only if the occupations equal T and its product is added (eq. 1). */
static void pathsum_rec(pathsum_t *p, int layer, int b, C prod) {
  const circuit_t *c = p->c;
  if (b == p->layer_start[layer + 1]) { /* layer finished */
    ++layer;
    if (p->ngates) prod *= gate_factor(p, layer);
    if (layer == c->D) {
      for (int i = 0; i < c->M; ++i) if (p->occ[i] != p->T[i]) return; /* invalid path */
      p->acc += prod;
      p->leaves++;
      return;
    }
    pathsum_rec(p, layer, b, prod);
    return;
  }
  int a = c->ma[b], bb = c->mb[b];
  int x1 = p->occ[a], x2 = p->occ[bb];
  int n = x1 + x2;
  for (int y1 = 0; y1 <= n; ++y1) {
    int y2 = n - y1;
    if (p->prune == 1) { /* occupation <= min(past-cone input, future-cone output) */
      if (y1 > p->bound[(layer + 1) * c->M + a] || y2 > p->bound[(layer + 1) * c->M + bb]) continue;
    }
    p->occ[a] = y1;
    p->occ[bb] = y2;
    if (p->prune == 2) { /* reading R5: F_l(k) inside the cumulative box */
      int k = a > bb ? a : bb, F = 0;
      for (int i = 0; i < k; ++i) F += p->occ[i];
      if (F < p->lo[(layer + 1) * (c->M + 1) + k] || F > p->hi[(layer + 1) * (c->M + 1) + k]) {
        p->occ[a] = x1;
        p->occ[bb] = x2;
        continue;
      }
    }
    pathsum_rec(p, layer, b + 1, prod * elem_of(p, b, x1, x2, y1));
    p->occ[a] = x1;
    p->occ[bb] = x2;
  }
}

/* Largest photon number that can enter BS i (of layer l, 0-based): the input photons
 * of its past light cone, capped at N.  Sizes the element cache only. */
static int bs_cap(const circuit_t *c, const int *layer_start, const int *S, int l, int i, int N) {
  unsigned char in[ORACLE_MAXM];
  memset(in, 0, sizeof(in));
  in[c->ma[i]] = in[c->mb[i]] = 1;
  for (int k = l - 1; k >= 0; --k)
    for (int j = layer_start[k]; j < layer_start[k + 1]; ++j)
      if (in[c->ma[j]] || in[c->mb[j]]) in[c->ma[j]] = in[c->mb[j]] = 1;
  int s = 0;
  for (int m = 0; m < c->M; ++m) if (in[m]) s += S[m];
  return s < N ? s : N;
}

/* Batch entry: amplitudes (and leaf counts = number of valid paths reached) for B
 * output patterns, with optional phase gates.  Returns 0, or -1 bad circuit / -2 bad
 * state / -3 prune 2 on a non-nearest-neighbour circuit / -5 bad gate. */
int oracle_path_sum_gates(int M, int D, const int *bs_per_layer, const int *ma, const int *mb,
                          const double *theta, const double *phi, const int *S, long B,
                          const int *T /* [B][M] */, int prune, int nthreads, int ngates,
                          const int *g_mode, const int *g_after, const double *g_a, const double *g_b,
                          double *out /* [B][2] */, uint64_t *leaves /* [B] or NULL */) {
  circuit_t c = {M, D, 0, bs_per_layer, ma, mb, theta, phi};
  int nbs = circuit_check(&c);
  if (nbs < 0) return -1;
  c.nbs = nbs;
  if (prune == 2 && !is_nn(&c)) return -3;
  int N = 0;
  for (int i = 0; i < M; ++i) { if (S[i] < 0) return -2; N += S[i]; }
  if (N > ORACLE_MAXN) return -2;
  for (int g = 0; g < ngates; ++g)
    if (g_mode[g] < 0 || g_mode[g] >= M || g_after[g] < 0 || g_after[g] > D) return -5;
  int ls[ORACLE_MAXD + 1];
  ls[0] = 0;
  for (int l = 0; l < D; ++l) ls[l + 1] = ls[l] + bs_per_layer[l];
  /* per-BS cache of Appendix-A elements for every (x1, x2, y1) with x1 + x2 <= cap(BS) */
  int *tri_off = (int *)malloc(sizeof(int) * (size_t)(N + 2));
  tri_off[0] = 0;
  for (int n = 0; n <= N; ++n) tri_off[n + 1] = tri_off[n] + (n + 1) * (n + 1);
  int tri = tri_off[N + 1];
  int *cap = (int *)malloc(sizeof(int) * (size_t)(nbs > 0 ? nbs : 1));
  for (int l = 0; l < D; ++l)
    for (int i = ls[l]; i < ls[l + 1]; ++i) cap[i] = bs_cap(&c, ls, S, l, i, N);
  C *elem = (C *)malloc(sizeof(C) * (size_t)(nbs > 0 ? nbs : 1) * tri);
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for collapse(2) schedule(dynamic, 1)
#endif
  for (int b = 0; b < nbs; ++b)
    for (int n = 0; n <= N; ++n) {
      if (n > cap[b]) continue;
      for (int x1 = 0; x1 <= n; ++x1)
        for (int y1 = 0; y1 <= n; ++y1)
          elem[(size_t)b * tri + tri_off[n] + x1 * (n + 1) + y1] =
              bs_element_theta(theta[b], phi[b], x1, n - x1, y1, n - y1);
    }
  int rc = 0;
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic, 1)
#endif
  for (long q = 0; q < B; ++q) {
    const int *Tq = T + q * M;
    int NT = 0, bad = 0;
    for (int i = 0; i < M; ++i) { if (Tq[i] < 0) bad = 1; NT += Tq[i]; }
    out[2 * q] = out[2 * q + 1] = 0.0;
    if (leaves) leaves[q] = 0;
    if (bad) { out[2 * q] = out[2 * q + 1] = NAN; continue; }
    if (NT != N) continue; /* photon number is conserved: exact zero (R9) */
    pathsum_t *p = (pathsum_t *)calloc(1, sizeof(pathsum_t));
    int *bound = NULL, *lo = NULL, *hi = NULL;
    p->c = &c;
    p->layer_start = ls;
    p->T = Tq;
    p->N = N;
    p->prune = prune;
    p->elem = elem;
    p->tri_off = tri_off;
    p->tri_size = tri;
    p->ngates = ngates;
    p->g_mode = g_mode;
    p->g_after = g_after;
    p->g_a = g_a;
    p->g_b = g_b;
    if (prune == 1) {
      bound = (int *)malloc(sizeof(int) * (size_t)(D + 1) * M);
      for (int j = 0; j <= D; ++j)
        for (int m = 0; m < M; ++m) bound[j * M + m] = cone_bound(&c, ls, S, Tq, m, j);
      p->bound = bound;
    } else if (prune == 2) {
      lo = (int *)malloc(sizeof(int) * (size_t)(D + 1) * (M + 1));
      hi = (int *)malloc(sizeof(int) * (size_t)(D + 1) * (M + 1));
      build_box(&c, ls, Tq, lo, hi);
      p->lo = lo;
      p->hi = hi;
    }
    for (int i = 0; i < M; ++i) p->occ[i] = S[i];
    p->acc = 0.0L;
    C start = ngates ? gate_factor(p, 0) : 1.0L;
    if (D == 0) {
      int same = 1;
      for (int i = 0; i < M; ++i) if (S[i] != Tq[i]) same = 0;
      if (same) { p->acc = start; p->leaves = 1; }
    } else {
      pathsum_rec(p, 0, 0, start);
    }
    out[2 * q] = (double)creall(p->acc);
    out[2 * q + 1] = (double)cimagl(p->acc);
    if (leaves) leaves[q] = p->leaves;
    free(bound); free(lo); free(hi);
    free(p);
  }
  free(elem);
  free(cap);
  free(tri_off);
  return rc;
}

int oracle_path_sum(int M, int D, const int *bs_per_layer, const int *ma, const int *mb,
                    const double *theta, const double *phi, const int *S, long B,
                    const int *T /* [B][M] */, int prune, int nthreads, double *out /* [B][2] */,
                    uint64_t *leaves /* [B] or NULL */) {
  return oracle_path_sum_gates(M, D, bs_per_layer, ma, mb, theta, phi, S, B, T, prune, nthreads, 0,
                               NULL, NULL, NULL, NULL, out, leaves);
}

/* ------------------------------------------------------------------------- */
/* structural reachability and exact path counts (readings R5, R6)            */
/* ------------------------------------------------------------------------- */

/* T is structurally reachable from S  <=>  sum S = sum T and F_0 = cum(S) lies in the
 * time-0 box (reading R5). */
int oracle_reachable(int M, int D, const int *bs_per_layer, const int *ma, const int *mb,
                     const int *S, long B, const int *T, int nthreads, uint8_t *out /* [B] */) {
  circuit_t c = {M, D, 0, bs_per_layer, ma, mb, NULL, NULL};
  int nbs = circuit_check(&c);
  if (nbs < 0) return -1;
  c.nbs = nbs;
  if (!is_nn(&c)) return -3;
  int ls[ORACLE_MAXD + 1];
  ls[0] = 0;
  for (int l = 0; l < D; ++l) ls[l + 1] = ls[l] + bs_per_layer[l];
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel
#endif
  {
    int *lo = (int *)malloc(sizeof(int) * (size_t)(D + 1) * (M + 1));
    int *hi = (int *)malloc(sizeof(int) * (size_t)(D + 1) * (M + 1));
#ifdef _OPENMP
#pragma omp for schedule(static)
#endif
    for (long q = 0; q < B; ++q) {
      const int *Tq = T + q * M;
      int nS = 0, nT = 0, ok = 1;
      for (int i = 0; i < M; ++i) { nS += S[i]; nT += Tq[i]; if (Tq[i] < 0) ok = 0; }
      if (nS != nT) ok = 0;
      if (ok) {
        build_box(&c, ls, Tq, lo, hi);
        int F = 0;
        for (int k = 0; k <= M; ++k) {
          if (F < lo[k] || F > hi[k]) { ok = 0; break; }
          if (k < M) F += S[k];
        }
      }
      out[q] = (uint8_t)ok;
    }
    free(lo);
    free(hi);
  }
  return 0;
}

/* Number of valid paths = number of integer arrays F[t][k] (t = 0..D, k = 0..M) with
 *   F[t][0] = 0, F[t][M] = N, F[0][k] = cum(S)(k), F[D][k] = cum(T)(k),
 *   F[t][k] = F[t-1][k] for cuts k not active in layer t,
 *   F[t-1][k-1] <= F[t][k] <= F[t-1][k+1] for cuts active in layer t (conservation and
 *   non-negative BS outputs), F[t][k] <= F[t][k+1] (non-negative occupations).
 * Every such array is one valid path and vice versa.  Counted by a transfer over
 * columns k = 1..M (reading R6): a column is its values after each of its active
 * layers; each candidate value ranges over the cumulative box (a superset of the
 * valid values, reading R5) and every constraint between adjacent columns is checked
 * explicitly, so the count does not rely on the box being tight.  Counts are exact
 * unsigned 128-bit integers, returned as (lo64, hi64) pairs.  -4 = state space too big. */
typedef unsigned __int128 u128;

static int count_one(const circuit_t *c, const int *ls, const int *S, const int *T, u128 *result,
                     long max_states) {
  int M = c->M, D = c->D, W = M + 1;
  int N = 0, NT = 0;
  for (int i = 0; i < M; ++i) { N += S[i]; NT += T[i]; }
  *result = 0;
  if (N != NT) return 0;
  int *lo = (int *)malloc(sizeof(int) * (size_t)(D + 1) * W);
  int *hi = (int *)malloc(sizeof(int) * (size_t)(D + 1) * W);
  build_box(c, ls, T, lo, hi);
  /* active layers (1-based) of every cut */
  unsigned char *act = (unsigned char *)calloc((size_t)(D + 1) * W, 1);
  for (int l = 1; l <= D; ++l)
    for (int i = ls[l - 1]; i < ls[l]; ++i) {
      int k = c->ma[i] > c->mb[i] ? c->ma[i] : c->mb[i];
      act[l * W + k] = 1;
    }
  int cumS[ORACLE_MAXM + 1], cumT[ORACLE_MAXM + 1];
  cumS[0] = cumT[0] = 0;
  for (int k = 0; k < M; ++k) { cumS[k + 1] = cumS[k] + S[k]; cumT[k + 1] = cumT[k] + T[k]; }
  /* previous column: list of full F_t vectors (t = 0..D) with their counts */
  int rc = 0;
  long nprev = 1;
  int *prevF = (int *)malloc(sizeof(int) * (size_t)(D + 1));
  u128 *prevN = (u128 *)malloc(sizeof(u128));
  for (int t = 0; t <= D; ++t) prevF[t] = 0;
  prevN[0] = 1;
  for (int k = 1; k <= M && nprev > 0; ++k) {
    /* enumerate candidate columns for cut k */
    int al[ORACLE_MAXD], m = 0;
    for (int l = 1; l <= D; ++l) if (k < M && act[l * W + k]) al[m++] = l;
    long ncand = 1;
    int rlo[ORACLE_MAXD], rn[ORACLE_MAXD];
    for (int i = 0; i < m; ++i) {
      rlo[i] = lo[al[i] * W + k];
      rn[i] = hi[al[i] * W + k] - rlo[i] + 1;
      if (rn[i] <= 0) { ncand = 0; break; }
      ncand *= rn[i];
      if (ncand > max_states) { rc = -4; break; }
    }
    if (rc) break;
    int *curF = (int *)malloc(sizeof(int) * (size_t)(ncand > 0 ? ncand : 1) * (D + 1));
    u128 *curN = (u128 *)calloc((size_t)(ncand > 0 ? ncand : 1), sizeof(u128));
    long ncur = 0;
    for (long idx = 0; idx < ncand; ++idx) {
      int u[ORACLE_MAXD];
      long r = idx;
      for (int i = m - 1; i >= 0; --i) { u[i] = rlo[i] + (int)(r % rn[i]); r /= rn[i]; }
      int *F = curF + ncur * (D + 1);
      int val = (k == M) ? N : cumS[k], ai = 0;
      for (int t = 0; t <= D; ++t) {
        if (ai < m && al[ai] == t) val = u[ai++];
        F[t] = val;
      }
      if (F[D] != cumT[k]) continue; /* must end on T */
      ++ncur;
    }
    /* transfer: explicit adjacent-column constraints */
    long long pairs = (long long)ncur * nprev;
    if (pairs > (long long)max_states * 64) { rc = -4; free(curF); free(curN); break; }
    for (long a = 0; a < ncur; ++a) {
      const int *Fc = curF + a * (D + 1);
      u128 s = 0;
      for (long b = 0; b < nprev; ++b) {
        const int *Fp = prevF + b * (D + 1);
        int ok = 1;
        for (int t = 0; t <= D && ok; ++t) {
          if (Fp[t] > Fc[t]) ok = 0;                                              /* monotone */
          if (t >= 1 && k < M && act[t * W + k] && Fp[t - 1] > Fc[t]) ok = 0;      /* F[t-1][k-1] <= F[t][k] */
          if (t >= 1 && k - 1 >= 1 && act[t * W + k - 1] && Fp[t] > Fc[t - 1]) ok = 0; /* F[t][k-1] <= F[t-1][k] */
        }
        if (ok) s += prevN[b];
      }
      curN[a] = s;
    }
    free(prevF);
    free(prevN);
    prevF = curF;
    prevN = curN;
    nprev = ncur;
  }
  if (rc == 0 && nprev == 1) *result = prevN[0];
  free(prevF);
  free(prevN);
  free(lo); free(hi); free(act);
  return rc;
}

int oracle_count_paths(int M, int D, const int *bs_per_layer, const int *ma, const int *mb,
                       const int *S, long B, const int *T, int nthreads, long max_states,
                       uint64_t *out /* [B][2] = (lo64, hi64) */, int *status /* [B] */) {
  circuit_t c = {M, D, 0, bs_per_layer, ma, mb, NULL, NULL};
  int nbs = circuit_check(&c);
  if (nbs < 0) return -1;
  c.nbs = nbs;
  if (!is_nn(&c)) return -3;
  for (int i = 0; i < M; ++i) if (S[i] < 0) return -2;
  int ls[ORACLE_MAXD + 1];
  ls[0] = 0;
  for (int l = 0; l < D; ++l) ls[l + 1] = ls[l] + bs_per_layer[l];
  if (max_states <= 0) max_states = 1L << 22;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1)
#endif
  for (long q = 0; q < B; ++q) {
    u128 r = 0;
    int bad = 0;
    for (int i = 0; i < M; ++i) if (T[q * M + i] < 0) bad = 1;
    int rc = bad ? -2 : count_one(&c, ls, S, T + q * M, &r, max_states);
    status[q] = rc;
    out[2 * q] = (uint64_t)r;
    out[2 * q + 1] = (uint64_t)(r >> 64);
  }
  return 0;
}
