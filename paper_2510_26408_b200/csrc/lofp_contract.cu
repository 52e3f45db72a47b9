// lofp_contract.cu — the strip tensor contraction (NEXT-1) with one warp per
// output, for nearest-neighbour circuits.
//
// The paper contracts the circuit block by block, keeping for every tuple of occupation
// numbers that crosses from one block to the next its partial amplitude.  The
// blocks here are the cuts: the state crossing cut k is the column pair
// (c_{k-1}, c_k), and
//     A_{k+1}(c_k, c_{k+1}) = sum_{c_{k-1}} A_k(c_{k-1}, c_k) f_k(c_{k-1}, c_k, c_{k+1})
// with f_k the cut factor (the product of cut k's BS elements, eq. (1)).  The
// amplitude is the sum of the last level.
//
// Why a warp per output: on the paper's workloads a column holds tens of states and a cut
// a few hundred terms (configs[3]: <= 60 states, ~730 terms per cut), far too little for
// a 256-thread block per output with a barrier per cut (lofp_contract_kernel, which stays
// the fallback for larger state spaces and for non-local circuits).  Here 8 outputs share
// a block, each warp walks its output's cuts with no block barrier, and a warp's lanes
// split a level's entries evenly.
//
// Layout (no index arithmetic on a dense n x n square): for a nearest-neighbour mesh,
// F_t(k-1) <= F_t(k) for every t is, for a fixed state of column k, an upper bound per
// segment of column k-1 — the compatible states of column k-1 form a sub-box of its
// mixed-radix state box, starting at the box's lower corner.  Level k stores, for every
// state s of column k (a "row"), one entry per state of that sub-box in odometer order
// (segment 0 fastest).  A row is walked by incrementing the packed segment values, so no
// state is ever decoded inside the term loop.  Segment values are bytes packed in a u64
// (<= 8 segments per column, i.e. <= 7 active layers per cut).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "lofp_internal.h"

using namespace lofp;

namespace {

typedef unsigned long long ull;

#ifdef LOFP_DEBUG
#define DCHECK_C(cond)                                                                         \
  do {                                                                                         \
    if (!(cond)) {                                                                             \
      printf("LOFP_DEBUG contraction check failed at line %d block %d\n", __LINE__, blockIdx.x); \
      __trap();                                                                                \
    }                                                                                          \
  } while (0)
#else
#define DCHECK_C(cond) \
  do {                 \
  } while (0)
#endif

#ifdef LOFP_CPROF  // phase clocks and level statistics of the warp kernel (A/B experiments only)
#define CPROF(x) x
#else
#define CPROF(x)
#endif

#ifndef LOFP_CW
#define LOFP_CW 4
#endif
constexpr int kCW = LOFP_CW;       // warps (outputs in flight) per block
#ifndef LOFP_CWPS
#define LOFP_CWPS 16               // resident warps per SM the register cap is set for (128 registers)
#endif
constexpr int kCSeg = 8;           // segments per column: one byte each of a packed u64
constexpr int kCMaxN = 4096;       // states per column (as the block kernel)
constexpr int kCMaxStates = 16384; // states of all columns of one output
constexpr int kCFac = 32;          // phase gates of one cut staged in shared memory

constexpr int kLB = 32;            // row-length classes of the entry schedule
constexpr int kCF = kCSeg - 1;     // BS of one cut (<= 7 active layers: 8 segments)
constexpr int kCCmp = 2 * kCSeg;   // CmpPair checks between two columns

struct GateW {           // one phase gate folded into the cut
  int row;               // gate_tab row
  uint8_t col_off;       // 0: it reads columns k-1 and k, 1: columns k and k+1
  uint8_t seg_lo, seg_hi;
  uint8_t slot;          // col_off 0: the byte of the entries' gather holding F(k-1)
};

template <int MM>          // MM: the most modes of a circuit this instantiation takes
struct CWarpT {          // shared state of one lane group's output
  uint64_t lo[MM + 1];             // packed lower corner of each column's box
  uint64_t hi[MM + 1];             // packed upper corner
  uint32_t vbase[MM + 1];          // first packed state of each column in the scratch
  uint16_t n[MM + 1];              // states per column
  uint8_t nseg[MM + 1];
  int16_t G[MM + 1];               // cum(T)
  // cut k being contracted (staged once per cut)
  int ftab[kCF];                   // Appendix-A block of each of its BS (offset in the x1-linear table)
  uint8_t fcap[kCF];               // its photon cap (the block's extent)
  uint32_t fsh[kCF];               // segments it reads: i (column k) | sC << 8 (column k+1)
  GateW gat[kCFac];
};

struct CCirc {           // the circuit's column data, cached once per block
  SegInfo seg[kMaxModes + 1][kCSeg];   // light-cone maps of each segment
  uint16_t cmp[kMaxModes + 1][kCCmp];  // CmpPairs of column k: sa | sb << 8
  uint8_t nseg[kMaxModes + 1], ncmp[kMaxModes + 1];
  uint8_t ok[kMaxModes + 1];           // within the warp kernel's limits
};

__device__ void cache_circuit(const CallParams &p, CCirc &cc) {
  for (int k = threadIdx.x; k <= p.M; k += blockDim.x) {
    const ColInfo ci = p.col[k];
    int slots = ci.nfac;
    for (int g = 0; g < ci.ngate; ++g) slots += p.gat[ci.gate_base + g].col_off ? 0 : 1;
    const bool ok = ci.nseg <= kCSeg && ci.nfac <= kCF && ci.ngate <= kCFac && ci.ncmp <= kCCmp && slots <= kCSeg;
    cc.ok[k] = ok;
    cc.nseg[k] = ci.nseg;
    cc.ncmp[k] = ci.ncmp;
    if (!ok) continue;
    for (int i = 0; i < ci.nseg; ++i) cc.seg[k][i] = p.seg[ci.seg_base + i];
    for (int c = 0; c < ci.ncmp; ++c) {
      const CmpPair pr = p.cmp[ci.cmp_base + c];
      cc.cmp[k][c] = (uint16_t)(pr.sa | pr.sb << 8);
    }
  }
}

// byte j (0..7) of a packed state: one PRMT (selector nibble j picks the byte of the two
// words) and a mask, instead of a 64-bit funnel shift (16 % of the warp kernel's instructions)
__device__ __forceinline__ int byte_at(uint64_t v, int j) {
#ifdef LOFP_DEBUG
  if ((unsigned)j >= 8u) __trap();
#endif
#ifdef LOFP_BYTE_SHIFT
  return (int)((v >> (8 * j)) & 0xffu);
#else
  return (int)(__byte_perm((uint32_t)v, (uint32_t)(v >> 32), (uint32_t)j) & 0xffu);
#endif
}

// floor(x / d) for the mixed-radix decodes (d <= 121 photons + 1, x d < 2^32): one multiply
// by ceil(2^32 / d) from a shared table (exact in that range) instead of a division
__device__ __forceinline__ uint32_t div_small(const uint32_t *inv, uint32_t x, uint32_t d) {
#ifdef LOFP_DIV_PLAIN
  (void)inv;
  return x / d;
#else
  DCHECK_C(d >= 2u && d < 128u && (unsigned long long)x * d < (1ull << 32));
  return __umulhi(x, inv[d]);
#endif
}

__device__ __forceinline__ uint64_t set_byte(uint64_t v, int j, int b) {
  const int s = 8 * j;
  return (v & ~(0xffull << s)) | ((uint64_t)(uint32_t)b << s);
}

__device__ __forceinline__ ull sat_add_c(ull a, ull b) {
  const ull c = a + b;
  return c < a ? ~0ull : c;
}

// A group of G consecutive lanes of a warp that evaluates one output (G = 32: the whole
// warp; G = 8: four small outputs per warp).  Groups of one warp run different outputs, so
// every collective names the group's lanes only.
template <int G>
struct Grp {
  int lane;       // lane within the group
  unsigned mask;  // the group's lanes
  __device__ __forceinline__ Grp() {
    const int l = threadIdx.x & 31;
    lane = l % G;
    mask = G == 32 ? 0xffffffffu : (((1u << (G & 31)) - 1u) << (l - lane));
  }
  template <class T>
  __device__ __forceinline__ T scan(T v) const {  // inclusive prefix sum over the group
#pragma unroll
    for (int d = 1; d < G; d <<= 1) {
      const T u = __shfl_up_sync(mask, v, d, G);
      if (lane >= d) v += u;
    }
    return v;
  }
  template <class T>
  __device__ __forceinline__ T last(T v) const { return __shfl_sync(mask, v, G - 1, G); }
  template <class T>
  __device__ __forceinline__ T first(T v) const { return __shfl_sync(mask, v, 0, G); }
  __device__ __forceinline__ bool any(bool b) const { return (__ballot_sync(mask, b) & mask) != 0u; }
  __device__ __forceinline__ void sync() const { __syncwarp(mask); }
  __device__ __forceinline__ double sum(double v) const {  // fixed-order tree (deterministic)
#pragma unroll
    for (int d = G / 2; d > 0; d >>= 1) v += __shfl_down_sync(mask, v, d, G);
    return v;
  }
  __device__ __forceinline__ ull sum_sat(ull v) const {
#pragma unroll
    for (int d = G / 2; d > 0; d >>= 1) v = sat_add_c(v, __shfl_down_sync(mask, v, d, G));
    return v;
  }
};

// Upper corner of the sub-box of column k-1 compatible with state vr of column k:
// F_t(k-1) <= F_t(k) on every time interval (CmpPair list of column k).
template <class W>
__device__ __forceinline__ uint64_t sub_hi(const CCirc &cc, const W &w, int k, uint64_t vr) {
  uint64_t h = w.hi[k - 1];
  for (int c = 0; c < cc.ncmp[k]; ++c) {
    const int sa = cc.cmp[k][c] & 0xff, v = byte_at(vr, cc.cmp[k][c] >> 8);
    if (v < byte_at(h, sa)) h = set_byte(h, sa, v);
  }
  return h;
}

__device__ __forceinline__ uint32_t box_count(uint64_t lo, uint64_t hi, int ns) {
  uint32_t c = 1;
  for (int j = 0; j < ns; ++j) {
    const int d = byte_at(hi, j) - byte_at(lo, j) + 1;
    c = d > 0 ? c * (uint32_t)d : 0u;
  }
  return c;
}

// sub_hi with the column's CmpPairs staged in shared memory
__device__ __forceinline__ uint64_t sub_hi_s(uint64_t h, const uint16_t *cmp, int ncmp, uint64_t vr) {
  for (int c = 0; c < ncmp; ++c) {
    const int sa = cmp[c] & 0xff, v = byte_at(vr, cmp[c] >> 8);
    if (v < byte_at(h, sa)) h = set_byte(h, sa, v);
  }
  return h;
}

// The bytes of a column-(c-1) state that cut c's factor reads ("gather" slots): F_{l-1}(c-1)
// for each BS of cut c in order, then the column-(c-1) end of each gate folded into cut c
// with col_off 0.  Every level entry carries its row-side state's gather for the next cut,
// so the term loop reads A = F_{l-1}(c-1) as byte f of one register.  Built once per block
// for every cut (the circuit's, not the output's).
__device__ void gather_lists(const CallParams &p, uint8_t (*gseg)[kCSeg], uint8_t *ngs) {
  for (int c = threadIdx.x; c <= p.M; c += blockDim.x) {
    int n = 0;
    if (c >= 1 && c <= p.M - 1) {
      const ColInfo cc = p.col[c];
      for (int f = 0; f < cc.nfac && n < kCSeg; ++f) gseg[c][n++] = p.fac[cc.fac_base + f].sA;
      for (int g = 0; g < cc.ngate && n < kCSeg; ++g) {
        const GateInfo gi = p.gat[cc.gate_base + g];
        if (!gi.col_off) gseg[c][n++] = gi.seg_lo;
      }
    }
    ngs[c] = (uint8_t)n;
  }
}

__device__ __forceinline__ uint64_t gather(uint64_t v, const uint8_t *gseg, int ngs) {
  uint64_t g = 0;
  for (int j = 0; j < ngs; ++j) g |= (uint64_t)byte_at(v, gseg[j]) << (8 * j);
  return g;
}

// Rows of the level whose rows are the states of column k (entries: the compatible
// sub-box of column k-1): exclusive offsets into roff[0..n_k], returns the entry count.
// hrow[s] keeps the sub-box's upper corner of row s (the entry pass reads it per row).
template <int G, class W>
__device__ uint32_t level_rows(const CCirc &cc, const W &w, const uint64_t *vals, int k, uint32_t *roff,
                               uint64_t *hrow, const Grp<G> &g) {
  const int nk = w.n[k], ns = w.nseg[k - 1];
  uint32_t run = 0;
  for (int base = 0; base < nk; base += G) {
    const int s = base + g.lane;
    uint32_t c = 0;
    if (s < nk) {
      const uint64_t h = sub_hi(cc, w, k, vals[w.vbase[k] + s]);
      hrow[s] = h;
      c = box_count(w.lo[k - 1], h, ns);
    }
    const uint32_t incl = g.scan(c);
    if (s < nk) roff[s] = run + incl - c;
    run += g.last(incl);
  }
  if (g.lane == 0) roff[nk] = run;
  g.sync();
  return run;
}

// Per-output setup: G = cum(T), the light-cone box of every column (readings R5, R15),
// the packed states.  Returns kStatusOk / Zero / Bad / Deferred (warp-uniform).
template <int G, class W>
__device__ int setup_warp(const CallParams &p, const CCirc &cc, W &w, uint64_t *vals, const uint32_t *inv, int q,
                          const Grp<G> &g) {
  const int M = p.M;
  // G = cum(T); negative entries make the row bad, totals other than N an exact zero
  int bad = 0, run = 0;
  if (g.lane == 0) w.G[0] = 0;
  for (int base = 0; base < M; base += G) {
    const int i = base + g.lane;
    int t = 0;
    if (i < M) {
      t = p.T[(long long)q * M + i];
      if (t < 0) bad = 1;
      t = min(max(t, 0), 255);
    }
    const int incl = g.scan(t);
    if (i < M) w.G[i + 1] = (int16_t)min(run + incl, 32767);
    run += g.last(incl);
  }
  if (g.any(bad)) return kStatusBad;
  if (run != p.N) return kStatusZero;  // photon number (reading R9)
  g.sync();
  // segment boxes: backward (T) and forward (S) light cones intersected
  int zero = 0, defer = 0;
  for (int k = g.lane; k <= M; k += G) {
    if (!cc.ok[k]) {
      defer = 1;
      w.n[k] = 0;
      continue;
    }
    const int nseg = cc.nseg[k];
    uint64_t lo = 0, hi = 0;
    uint32_t n = 1;
    for (int i = 0; i < nseg; ++i) {
      const SegInfo si = cc.seg[k][i];
      const int l = max((int)w.G[si.rho], (int)p.cumS[si.rhop]);
      const int h = min((int)w.G[si.sig], (int)p.cumS[si.sigp]);
      if (h < l) {
        n = 0;
      } else {
        lo = set_byte(lo, i, l);
        hi = set_byte(hi, i, h);
        n = min(n * (uint32_t)(h - l + 1), (uint32_t)kCMaxN + 1);
      }
    }
    if (n == 0) zero = 1;
    if (n > (uint32_t)kCMaxN) defer = 1;
    w.lo[k] = lo;
    w.hi[k] = hi;
    w.n[k] = (uint16_t)min(n, (uint32_t)kCMaxN);
    w.nseg[k] = (uint8_t)nseg;
  }
  const bool any_zero = g.any(zero), any_defer = g.any(defer);
  if (any_zero) return kStatusZero;  // a column with no state: structurally unreachable (R5)
  if (any_defer || p.tabA_off[p.nbs] > 0x7fffffffll) return kStatusDeferred;  // (int32 table offsets)
  g.sync();
  // first packed state of each column
  uint32_t tot = 0;
  for (int base = 0; base <= M; base += G) {
    const int k = base + g.lane;
    const uint32_t c = k <= M ? w.n[k] : 0u;
    const uint32_t incl = g.scan(c);
    if (k <= M) w.vbase[k] = tot + incl - c;
    tot += g.last(incl);
  }
  if (tot > (uint32_t)kCMaxStates) return kStatusDeferred;
  g.sync();
  if (g.lane == 0) atomicMax(&p.ctr->max_states, (ull)tot);
  // packed segment values of every state (mixed radix, segment 0 fastest); lanes over the
  // states of all columns (column by a search over vbase)
  for (uint32_t x = g.lane; x < tot; x += G) {
    int lo_k = 0, hi_k = M;
    while (lo_k < hi_k) {
      const int mid = (lo_k + hi_k + 1) >> 1;
      if (w.vbase[mid] <= x) lo_k = mid; else hi_k = mid - 1;
    }
    const int k = lo_k, ns = w.nseg[k];
    const uint64_t lo = w.lo[k], hi = w.hi[k];
    uint64_t v = lo;
    uint32_t r = x - w.vbase[k];
    for (int i = 0; i < ns; ++i) {
      const uint32_t rad = (uint32_t)(byte_at(hi, i) - byte_at(lo, i) + 1);
      if (rad == 1) continue;
      const uint32_t qd = div_small(inv, r, rad);
      v += (uint64_t)(r - qd * rad) << (8 * i);
      r = qd;
    }
    vals[x] = v;
  }
  g.sync();
  return kStatusOk;
}

// Cut factor of one term (eq. (1)): for every BS f of the cut, the Appendix-A element
// <y1, n-y1|BS|x1, n-x1> with x1 = Bm - A, y1 = Bp - A, n = C - A, where A = F_{l-1}(k-1)
// is byte f of the entry's gather g and C, Bm, Bp are fixed by the entry (cb).  In the
// x1-linear table (lofp_tableA_kernel) x2 = C - Bm and y2 = C - Bp are fixed by the entry too,
// so the element sits at pidx[f] - A with pidx[f] = block (x2, y2) + Bm, set once per entry.
// A vacuum BS (n = 0) reads its block's element (0, 0, 0), exactly 1 (reading R16).
template <int NF, bool FULL>
__device__ __forceinline__ double2 cut_fac(const double2 *__restrict__ tableA, const int (&pidx)[NF],
                                           const uint32_t (&cb)[NF], int nfac, uint64_t g) {
  // FULL (every cut of the circuit carries NF BS): no predicates, so the NF table loads are
  // independent and issue back to back
  double2 e[NF];
#pragma unroll
  for (int f = 0; f < NF; ++f) {
    e[f] = make_double2(1.0, 0.0);
    if (FULL || f < nfac) {
      const int A = (int)((g >> (8 * f)) & 0xffu);
      DCHECK_C(((cb[f] >> 8) & 0xff) >= (uint32_t)A && (cb[f] & 0xff) >= ((cb[f] >> 8) & 0xff) &&
               (cb[f] >> 16) >= (uint32_t)A && (cb[f] >> 16) <= (cb[f] & 0xff));
      e[f] = __ldg(tableA + (pidx[f] - A));
    }
  }
  (void)cb;
  // product as a balanced tree (depth log2 NF instead of NF dependent multiplications);
  // the unused slots hold exactly 1
#pragma unroll
  for (int st = 1; st < NF; st *= 2)
#pragma unroll
    for (int f = 0; f + st < NF; f += 2 * st)
      e[f] = make_double2(e[f].x * e[f + st].x - e[f].y * e[f + st].y, e[f].x * e[f + st].y + e[f].y * e[f + st].x);
  return e[0];
}

// phase gates of the cut on (column k-1, column k): n = F(k) - F(k-1) at their time
template <class W>
__device__ __forceinline__ double2 gates_a(const CallParams &p, const W &w, int ngate, uint64_t vb, uint64_t g,
                                           double2 fac, ull &cm) {
  for (int gi = 0; gi < ngate; ++gi) {
    const GateW gw = w.gat[gi];
    if (gw.col_off) continue;
    const double2 ge = p.gate_tab[gw.row * (p.N + 1) + byte_at(vb, gw.seg_hi) - (int)((g >> (8 * gw.slot)) & 0xffu)];
    fac = make_double2(fac.x * ge.x - fac.y * ge.y, fac.x * ge.y + fac.y * ge.x);
    ++cm;
  }
  return fac;
}

// The sum over one row of level k (the states of column k-1 compatible with sb) of
// A_k(c_{k-1}, sb) f_k(c_{k-1}, sb, sc): kRowU entries per step, their loads first.
#ifndef LOFP_ROW_UNROLL
#define LOFP_ROW_UNROLL 3
#endif
constexpr int kRowU = LOFP_ROW_UNROLL;

template <int NF, bool CNT, bool FULL, class W>
__device__ __forceinline__ void row_sum(const double2 *__restrict__ table, const int (&pidx)[NF],
                                        const uint32_t (&cb)[NF], int nfac, double2 gfix, const CallParams &p,
                                        const W &w, int ngate, uint64_t vb, const double2 *__restrict__ Ac,
                                        const uint64_t *__restrict__ Gc, const ull *__restrict__ Cc, uint32_t r0,
                                        uint32_t r1, double &sx, double &sy, ull &csum, ull &cm, ull &terms) {
  uint32_t r = r0;
  for (; r + kRowU <= r1; r += kRowU) {
    double2 a[kRowU], f[kRowU];
    uint64_t gg[kRowU];
#pragma unroll
    for (int u = 0; u < kRowU; ++u) {
      a[u] = Ac[r + u];
      gg[u] = Gc[r + u];
    }
    if (CNT)
#pragma unroll
      for (int u = 0; u < kRowU; ++u) csum = sat_add_c(csum, Cc[r + u]);
#pragma unroll
    for (int u = 0; u < kRowU; ++u) f[u] = cut_fac<NF, FULL>(table, pidx, cb, nfac, gg[u]);
    if (ngate)
#pragma unroll
      for (int u = 0; u < kRowU; ++u) f[u] = gates_a(p, w, ngate, vb, gg[u], f[u], cm);
#pragma unroll
    for (int u = 0; u < kRowU; ++u) {
      sx = fma(a[u].x, f[u].x, fma(-a[u].y, f[u].y, sx));
      sy = fma(a[u].x, f[u].y, fma(a[u].y, f[u].x, sy));
    }
  }
  for (; r < r1; ++r) {
    const double2 a0 = Ac[r];
    const uint64_t g0 = Gc[r];
    if (CNT) csum = sat_add_c(csum, Cc[r]);
    double2 f0 = cut_fac<NF, FULL>(table, pidx, cb, nfac, g0);
    if (ngate) f0 = gates_a(p, w, ngate, vb, g0, f0, cm);
    sx = fma(a0.x, f0.x, fma(-a0.y, f0.y, sx));
    sy = fma(a0.x, f0.y, fma(a0.y, f0.x, sy));
  }
  // every term of the row is a live (c_{k-1}, c_k, c_{k+1}) triple: nfac - 1 multiplications
  // of Appendix-A elements and one multiply-accumulate each
  terms += r1 - r0;
  cm += (ull)(r1 - r0) * (ull)(nfac > 1 ? nfac - 1 : 0);
  if (ngate) {  // the gates on (column k, column k+1) are fixed along the row: applied to its sum
    ++cm;
    const double tx = sx * gfix.x - sy * gfix.y;
    sy = sx * gfix.y + sy * gfix.x;
    sx = tx;
  }
}

}  // namespace

// NF: the most BS any cut carries (<= 7; loops unrolled to it), CNT: exact path counts too,
// G: lanes per output (32, or 8 for small circuits in large batches), MM: most modes
template <int NF, bool CNT, int G, int MM>
__global__ void __launch_bounds__(32 * kCW, LOFP_CWPS / kCW) lofp_contract_warp_kernel(const __grid_constant__ CallParams p) {
  constexpr int kGroups = kCW * (32 / G);  // outputs in flight per block
  __shared__ CWarpT<MM> sw[kGroups];
  __shared__ uint8_t s_gseg[kMaxModes + 1][kCSeg], s_ngs[kMaxModes + 1];  // gather slots per cut
  __shared__ CCirc cc;
  __shared__ uint32_t s_hist[kGroups][kLB];  // entries per row-length class (the cut's schedule)
  __shared__ uint32_t s_inv[128];  // ceil(2^32 / d) (div_small)
  for (int d = threadIdx.x; d < 128; d += blockDim.x) s_inv[d] = d >= 2 ? 0xffffffffu / (uint32_t)d + 1u : 0u;
  gather_lists(p, s_gseg, s_ngs);
  cache_circuit(p, cc);
  __syncthreads();
  const Grp<G> g;
  const int gib = threadIdx.x / G;  // group in the block
  CWarpT<MM> &w = sw[gib];
  const int M = p.M;
  constexpr bool with_counts = CNT;
  // group scratch: packed states, row corners, two row-offset arrays, two levels (values, gathers [, counts])
  char *ws = p.slab + ((long long)blockIdx.x * kGroups + gib) * p.cw_bytes;
  uint64_t *vals = (uint64_t *)ws;
  uint64_t *const hrow = vals + kCMaxStates;  // sub-box corner per row of the level being built
  uint32_t *const roff0 = (uint32_t *)(hrow + kCMaxN), *const roff1 = roff0 + (kCMaxN + 1);
  char *lv0 = (char *)(roff1 + kCMaxN + 1);
  lv0 = (char *)(((uintptr_t)lv0 + 15) & ~(uintptr_t)15);
  const long long per = with_counts ? 32 : 24;
  const long long capE = (p.cw_bytes - (lv0 - ws)) / (2 * per + 16);
  double2 *const lvA = (double2 *)lv0, *const lvB = lvA + capE;
  uint64_t *const lgA = (uint64_t *)(lvB + capE), *const lgB = lgA + capE;
  uint64_t *const rec_t = lgB + capE, *const rec_s = rec_t + capE;  // the cut's entry records
  ull *const lcA = (ull *)(rec_s + capE), *const lcB = lcA + capE;
  uint32_t *const hist = s_hist[gib];
#define ROFF(i) ((i) ? roff1 : roff0)
#define LV(i) ((i) ? lvB : lvA)
#define LG(i) ((i) ? lgB : lgA)
#define LC(i) ((i) ? lcB : lcA)
  ull cm = 0, terms = 0;
  while (true) {
    int q = 0;
    if (g.lane == 0) q = (int)atomicAdd(&p.ctr->cticket, 1ull);
    q = g.first(q);
    if (q >= p.B) break;
    CPROF(long long c0 = clock64();)
    int st = setup_warp(p, cc, w, vals, s_inv, q, g);
    CPROF(if (g.lane == 0) atomicAdd(&p.ctr->phase[0], (ull)(clock64() - c0));)
    double re = 0.0, im = 0.0;
    ull count = 0;
    int cur = 0;
    if (st == kStatusOk) {
      // level 1: rows = states of column 1, entries = the single state of column 0
      double2 root = make_double2(1.0, 0.0);
      if (M == 1)
        for (int g = 0; g < p.ngate; ++g) {
          const double2 e = p.gate_tab[g * (p.N + 1) + p.N];
          root = make_double2(root.x * e.x - root.y * e.y, root.x * e.y + root.y * e.x);
        }
      const uint32_t tot = level_rows(cc, w, vals, 1, roff0, hrow, g);
      if (tot > (uint64_t)capE) st = kStatusDeferred;
      if (st == kStatusOk) {
        const uint64_t g0 = gather(vals[w.vbase[0]], s_gseg[1], s_ngs[1]);
        for (uint32_t t = g.lane; t < tot; t += G) {
          lvA[t] = root;
          lgA[t] = g0;
          if (with_counts) lcA[t] = 1ull;
        }
        g.sync();
      }
    }
    // cuts 1..M-1: level k (rows: column k, entries: column k-1) -> level k+1
    for (int k = 1; k <= M - 1 && st == kStatusOk; ++k) {
      const int nxt = cur ^ 1;
      CPROF(long long c1 = clock64();)
      const uint32_t totn = level_rows(cc, w, vals, k + 1, ROFF(nxt), hrow, g);
      if (totn > (uint64_t)capE) {
        st = kStatusDeferred;
        break;
      }
      const ColInfo ck = p.col[k];
      const int nfac = ck.nfac, ngate = ck.ngate, ncR = cc.ncmp[k + 1];
      (void)ncR;
      for (int f = g.lane; f < nfac; f += G) {
        const FacInfo fi = p.fac[ck.fac_base + f];
        const BSInfo bi = p.bsi[fi.bs];
        w.ftab[f] = (int)p.tabA_off[fi.bs];
        w.fcap[f] = (uint8_t)min(p.N, (int)p.cumS[bi.cap_hi] - (int)p.cumS[bi.cap_lo]);  // (bs_cap)
        w.fsh[f] = (uint32_t)fi.i | (uint32_t)fi.sC << 8;
      }
      g.sync();
      if (g.lane == 0) {
        int slot = nfac;  // the gather order of gather_lists
        for (int gt = 0; gt < ngate; ++gt) {
          const GateInfo gi = p.gat[ck.gate_base + gt];
          GateW gw;
          gw.row = gi.gate;
          gw.col_off = gi.col_off;
          gw.seg_lo = gi.seg_lo;
          gw.seg_hi = gi.seg_hi;
          gw.slot = gi.col_off ? 0 : (uint8_t)slot++;
          w.gat[gt] = gw;
        }
      }
      g.sync();
      const double2 *__restrict__ table = p.tableA;
      int tbo[NF], tc1[NF];
#pragma unroll
      for (int f = 0; f < NF; ++f) {
        tbo[f] = f < nfac ? w.ftab[f] : 0;
        tc1[f] = f < nfac ? (int)w.fcap[f] + 1 : 1;
      }
      const uint32_t *rn = ROFF(nxt), *rc = ROFF(cur);
      const double2 *Ac = LV(cur);
      const uint64_t *Gc = LG(cur);
      const ull *Cc = LC(cur);
      double2 *An = LV(nxt);
      uint64_t *Gn = LG(nxt);
      ull *Cn = LC(nxt);
      const uint64_t loB = w.lo[k], hiB = w.hi[k];
      const int nsB = w.nseg[k];
      const uint32_t vbC = w.vbase[k + 1];
      // Pass 1 — the cut's entry records: entry t of the next level is (row sc = a state of
      // column k+1, the pos-th state sb of its sub-box of column k); its sum runs over row sb
      // of the current level.  Rows differ in length (the sub-box of column k-1 under sb), and
      // lanes that take entries in storage order wait for the longest row of their round
      // (configs[3]: 30 % of the lane-steps of the row loop did work).  So levels of more than
      // two rounds are scheduled by row length, longest first (a counting sort over kLB length
      // classes): the entries of a round have rows of about one length.  Each entry's value
      // is formed exactly as before and stored at its own t, so the results do not depend on
      // the schedule (bitwise the same).
      const bool sorted = totn > 2u * G && !p.contract_nosort;
      if (sorted) {
        for (int b = g.lane; b < kLB; b += G) hist[b] = 0u;
        g.sync();
      }
      {
        int sc = 0, sc_last = -1;
        uint64_t hB = 0;
        for (uint32_t t = g.lane; t < totn; t += G) {
          while (rn[sc + 1] <= t) ++sc;
          if (sc != sc_last) {  // the row's state (column k+1) bounds its sub-box of column k
            hB = hrow[sc];
            DCHECK_C(hB == sub_hi_s(hiB, cc.cmp[k + 1], ncR, vals[vbC + sc]));
            sc_last = sc;
          }
          // entry t = the pos-th state of the sub-box (odometer order, segment 0 fastest)
          uint32_t pos = t - rn[sc];
          uint32_t sb = 0, stride = 1;  // sb: the state's index in column k's full box
          for (int j = 0; j < nsB; ++j) {
            const int l = byte_at(loB, j), rad = byte_at(hB, j) - l + 1;
            if (rad > 1) {
              const uint32_t qd = div_small(s_inv, pos, (uint32_t)rad);
              sb += (pos - qd * (uint32_t)rad) * stride;
              pos = qd;
            }
            stride *= (uint32_t)(byte_at(hiB, j) - l + 1);
          }
          DCHECK_C(sb < (uint32_t)w.n[k] && sc < (int)w.n[k + 1]);
          const uint32_t len = rc[sb + 1] - rc[sb];
          const uint32_t cls = len < 24u ? len : min(24u + ((len - 24u) >> 3), (uint32_t)kLB - 1u);
          rec_t[t] = (uint64_t)t | (uint64_t)sc << 32 | (uint64_t)sb << 44 | (uint64_t)cls << 56;
          if (sorted) atomicAdd(&hist[cls], 1u);
        }
      }
      g.sync();
      const uint64_t *recs = rec_t;
      if (sorted) {
        if (g.lane == 0) {  // first slot of each class, longest rows first
          uint32_t run = 0;
          for (int b = kLB - 1; b >= 0; --b) {
            const uint32_t c = hist[b];
            hist[b] = run;
            run += c;
          }
        }
        g.sync();
        for (uint32_t t = g.lane; t < totn; t += G) {
          const uint64_t rec = rec_t[t];
          const uint32_t slot = atomicAdd(&hist[rec >> 56], 1u);
          DCHECK_C(slot < totn);
          rec_s[slot] = rec;
        }
        g.sync();
        recs = rec_s;
      }
      const uint64_t *const valsB = vals + w.vbase[k];
      CPROF(long long c2 = clock64(); if (g.lane == 0) { atomicAdd(&p.ctr->phase[1], (ull)(c2 - c1));
                                                         atomicAdd(&p.ctr->phase[4], (ull)totn);
                                                         atomicAdd(&p.ctr->phase[7], 1ull); })
      for (uint32_t it = g.lane; it < totn; it += G) {
        const uint64_t rec = recs[it];
        const uint32_t t = (uint32_t)rec, sb = (uint32_t)(rec >> 44) & 0xfffu;
        const uint64_t vc = vals[vbC + ((uint32_t)(rec >> 32) & 0xfffu)], vb = valsB[sb];
        // per BS f the photon numbers fixed by (sb, sc): C = F_{l-1}(k+1), Bm = F_{l-1}(k),
        // Bp = F_l(k); only A = F_{l-1}(k-1) varies along the row
        uint32_t cb[NF];
#pragma unroll
        for (int f = 0; f < NF; ++f) {
          const uint32_t sh = f < nfac ? w.fsh[f] : 0u;
          const int i = sh & 0xff;
          cb[f] = (uint32_t)byte_at(vc, sh >> 8) | (uint32_t)byte_at(vb, i) << 8 | (uint32_t)byte_at(vb, i + 1) << 16;
        }
        int pidx[NF];  // x1-linear block (x2, y2) of each BS, offset by Bm: element at pidx - A
#pragma unroll
        for (int f = 0; f < NF; ++f) {
          const int C = cb[f] & 0xff, Bm = (cb[f] >> 8) & 0xff, Bp = cb[f] >> 16;
          const int x2 = C - Bm, y2 = C - Bp, c1 = tc1[f];
          pidx[f] = f < nfac ? tbo[f] + c1 * (x2 * c1 - ((x2 * (x2 - 1)) >> 1)) + y2 * (c1 - x2) + Bm : 0;
          DCHECK_C(f >= nfac || (x2 >= 0 && y2 >= 0 && x2 < c1 && y2 < c1));
        }
        double2 gfix = make_double2(1.0, 0.0);  // gates on (column k, column k+1): fixed too
        for (int gt = 0; gt < ngate; ++gt) {
          const GateW gw = w.gat[gt];
          if (!gw.col_off) continue;
          const double2 ge = p.gate_tab[gw.row * (p.N + 1) + byte_at(vc, gw.seg_hi) - byte_at(vb, gw.seg_lo)];
          gfix = make_double2(gfix.x * ge.x - gfix.y * ge.y, gfix.x * ge.y + gfix.y * ge.x);
          ++cm;
        }
        // sum over row sb of level k: the states of column k-1 compatible with sb
        const uint32_t r0 = rc[sb], r1 = rc[sb + 1];
        CPROF({
          const unsigned am = __activemask();
          const uint32_t mx = __reduce_max_sync(am, r1 - r0);
          if ((threadIdx.x & 31) == __ffs(am) - 1) atomicAdd(&p.ctr->phase[5], (ull)mx);
          atomicAdd(&p.ctr->phase[6], (ull)(r1 - r0));
        })
        // (two entries per step, loads first; an entry whose value is 0 contributes 0)
        double sx = 0.0, sy = 0.0;
        ull csum = 0;
        if (nfac == NF)
          row_sum<NF, CNT, true>(table, pidx, cb, nfac, gfix, p, w, ngate, vb, Ac, Gc, Cc, r0, r1, sx, sy, csum, cm,
                                 terms);
        else
          row_sum<NF, CNT, false>(table, pidx, cb, nfac, gfix, p, w, ngate, vb, Ac, Gc, Cc, r0, r1, sx, sy, csum,
                                  cm, terms);
        An[t] = make_double2(sx, sy);
        Gn[t] = gather(vb, s_gseg[k + 1], s_ngs[k + 1]);  // what cut k+1 reads of sb
        if (with_counts) Cn[t] = csum;
      }
      g.sync();
      CPROF(if (g.lane == 0) atomicAdd(&p.ctr->phase[2], (ull)(clock64() - c2));)
      cur = nxt;
    }
    if (st == kStatusOk) {
      // the last level: one row (column M has one state); its sum is the amplitude
      const uint32_t e = ROFF(cur)[1];
      const double2 *Al = LV(cur);
      const ull *Cl = LC(cur);
      for (uint32_t t = g.lane; t < e; t += G) {
        re += Al[t].x;
        im += Al[t].y;
        if (with_counts) count = sat_add_c(count, Cl[t]);
      }
    }
    // fixed-order group reduction (deterministic)
    re = g.sum(re);
    im = g.sum(im);
    count = g.sum_sat(count);
    if (g.lane == 0) {
      if (st == kStatusOk && with_counts && count == 0) st = kStatusZero;
      if (st == kStatusDeferred) {
        atomicAdd(&p.ctr->cdeferred, 1ull);
      } else {
        double2 a = make_double2(re, im);
        if (st == kStatusBad) a = make_double2(__longlong_as_double(0x7ff8000000000000ll),
                                               __longlong_as_double(0x7ff8000000000000ll));
        if (st != kStatusOk) a = st == kStatusBad ? a : make_double2(0.0, 0.0);
        p.amps[q] = a;
        if (with_counts) p.counts[q] = st == kStatusOk ? count : 0ull;
        if (st == kStatusOk) atomicAdd(&p.ctr->feasible, 1ull);
        if (st == kStatusBad) atomicAdd(&p.ctr->bad_rows, 1ull);
      }
      p.status[q] = (uint8_t)st;
    }
    g.sync();
  }
  __syncwarp();
  const int lane = threadIdx.x & 31;
  for (int d = 16; d > 0; d >>= 1) {
    cm += __shfl_down_sync(0xffffffffu, cm, d);
    terms += __shfl_down_sync(0xffffffffu, terms, d);
  }
  if (lane == 0) {
    atomicAdd(&p.ctr->cmuls, cm);
    atomicAdd(&p.ctr->contractions, terms);
  }
}

template <int NF, bool CNT, int G, int MM>
static int launch_nf(const CallParams *p, int grid, cudaStream_t stream) {
  static int per_sm[32] = {0};
  static int nsm[32] = {0};
  constexpr int kGroups = kCW * (32 / G);
  int dev = 0;
  cudaGetDevice(&dev);
  dev &= 31;
  if (!per_sm[dev]) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[dev], lofp_contract_warp_kernel<NF, CNT, G, MM>, 32 * kCW, 0);
    cudaDeviceGetAttribute(&nsm[dev], cudaDevAttrMultiProcessorCount, dev);
    if (per_sm[dev] < 1) per_sm[dev] = 1;
  }
  long long blocks = (long long)per_sm[dev] * nsm[dev];
  const long long need = ((long long)p->B + kGroups - 1) / kGroups;
  if (need < blocks) blocks = need;
  if (blocks < 1) return 0;
  CallParams q = *p;
  const long long total = (long long)grid * p->slab_bytes;
  q.cw_bytes = (total / (blocks * kGroups)) & ~255ll;
  const long long fixed = (long long)kCMaxStates * 8 + (long long)kCMaxN * 8 + 2ll * (kCMaxN + 1) * 4 + 16;
  if (q.cw_bytes < fixed + 64 * 1024) return -1;  // scratch too small (LOFP_SLAB_MB): not launched
  lofp_contract_warp_kernel<NF, CNT, G, MM><<<(int)blocks, 32 * kCW, 0, stream>>>(q);
  return (int)cudaGetLastError();
}

// Small circuits (<= 32 modes, <= 4 BS per cut) in batches that fill the GPU four times over
// run with 8 lanes per output (four outputs per warp): their levels hold a few entries per
// lane of a full warp (configs[1]-sized outputs: lanes mostly idle).
constexpr int kSmallM = 32;

template <int NF>
static int launch_cnt(const CallParams *p, int grid, cudaStream_t stream) {
  if constexpr (NF <= 4) {
    const bool small = p->M <= kSmallM && (long long)p->B >= 4ll * 32 * grid;
    if (p->contract_group == 8 || (p->contract_group == 0 && small && p->M <= kSmallM)) {
      if (p->M <= kSmallM)
        return p->counts ? launch_nf<NF, true, 8, kSmallM>(p, grid, stream)
                         : launch_nf<NF, false, 8, kSmallM>(p, grid, stream);
    }
    if (p->contract_group == 16 && p->M <= kSmallM)
      return p->counts ? launch_nf<NF, true, 16, kSmallM>(p, grid, stream)
                       : launch_nf<NF, false, 16, kSmallM>(p, grid, stream);
  }
  return p->counts ? launch_nf<NF, true, 32, kMaxModes>(p, grid, stream)
                   : launch_nf<NF, false, 32, kMaxModes>(p, grid, stream);
}

// Launch: blocks of kCW warps, as many as are resident at once (the warps pull outputs from
// a ticket counter); each warp's scratch is carved from the slab of the block kernels
// (grid x slab_bytes), which runs after it on the same stream.  Instantiated per the most
// BS a cut carries (outputs of circuits with more than 7 per cut are deferred anyway).
// Returns 0 (launched), -1 (not launched: the caller runs the block kernel on every output)
// or a CUDA error.
extern "C" int lofp_launch_contract_warp(const CallParams *p, int grid, void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  switch (p->max_nfac) {
    case 0:
    case 1: return launch_cnt<1>(p, grid, st);
    case 2: return launch_cnt<2>(p, grid, st);
    case 3: return launch_cnt<3>(p, grid, st);
    case 4: return launch_cnt<4>(p, grid, st);
    case 5: return launch_cnt<5>(p, grid, st);
    case 6: return launch_cnt<6>(p, grid, st);
    default: return launch_cnt<7>(p, grid, st);
  }
}
