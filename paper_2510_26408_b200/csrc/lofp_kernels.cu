// lofp_kernels.cu — sm_100a kernels of liblofp (the LOFP path sum of arXiv 2510.26408).
//
// Pipeline of one lofp_amplitudes call (all on the caller's stream, no host sync):
//   lofp_table_off_kernel   per-BS Appendix-A block sizes from the input's past light cones
//                            and the phase-gate tables
//   lofp_table_kernel       Appendix-A elements <y1,y2|BS|x1,x2> by the stable
//                           four-term creation-operator recurrence (reading R1/R18)
//   lofp_plan_kernel        per output: column states inside the light-cone box (R5, R15),
//                           exact path counts by a transfer over columns (R6), and the split
//                           of the path tree into units of <= thr paths (a prefix split,
//                           BASELINE north_star "splits the path tree ... into prefixes")
//   lofp_scan_kernel        unit numbering
//   lofp_units_kernel       the hot path: per unit, the column-split enumeration (R20):
//                           half-path lists on both sides of a column pair, then every path
//                           formed as (left half-path) x (right half-path), one complex
//                           multiply-accumulate per path on the FP64 pipe
//   lofp_final_kernel       per output: sum of its units in a fixed order (deterministic)
//
// Notation: column k holds F_t(k), t = 0..D (photons in modes < k after layer t) as a
// tuple of segment values; see lofp_internal.h.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "lofp_internal.h"

using namespace lofp;

// Debug build (-DLOFP_DEBUG, liblofp_debug.so): bounds checks that name the failing site.
#ifdef LOFP_DEBUG
#include <cstdio>
#define DCHECK(cond, tag)                                                                        \
  do {                                                                                           \
    if (!(cond)) {                                                                               \
      printf("LOFP_DEBUG %s failed at line %d block %d thread %d\n", tag, __LINE__, blockIdx.x,   \
             threadIdx.x);                                                                       \
      __trap();                                                                                  \
    }                                                                                            \
  } while (0)
#else
#define DCHECK(cond, tag) \
  do {                    \
  } while (0)
#endif

namespace {

typedef unsigned long long ull;

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

__device__ __forceinline__ ull sat_add(ull a, ull b) {
  ull c = a + b;
  return c < a ? ~0ull : c;
}

__device__ __forceinline__ long long lin_dev(int cap) {  // lin_entries (lofp_internal.h)
  const long long c = cap + 1;
  return c * c * (c + 1) / 2;
}

__device__ __forceinline__ long long tri_dev(int n) {  // sum_{m<n} (m+1)^2
  return (long long)n * (n + 1) * (2 * n + 1) / 6;
}

// ---- scratch layout of one block (global memory, L1/L2 resident) -------------------
struct Seg {             // one (predecessor, state) pair of a BFS level or a column pair
  uint32_t dst, src, len;
  uint16_t p, s;
};

struct StackEnt {
  int32_t j;
  uint16_t sjm1, sj;
  double re, im;
  ull pad;
};

struct SplitEnt {         // a node of the split kernel's frontier: columns 0..j fixed
  uint16_t sjm1, sj;
  uint32_t pad;
  double re, im;           // product of the cut factors of cuts 1..j-1
};

constexpr long long kOffSegs = 0;
constexpr long long kOffFL = kOffSegs + (long long)kMaxSegments * sizeof(Seg);
constexpr long long kOffFR = kOffFL + (long long)kMaxStates * 16;
constexpr long long kOffStack = kOffFR + (long long)kMaxStates * 16;
constexpr long long kOffA = kOffStack + (long long)kStackMax * sizeof(StackEnt);
constexpr long long kOffB = kOffA + (long long)kMaxStates * 4;
constexpr long long kOffTmp = kOffB + (long long)kMaxStates * 4;
constexpr long long kOffTmp2 = kOffTmp + (long long)kMaxStates * 4;
constexpr int kSegSlots = 8192;  // segment descriptors of all columns of one output
constexpr long long kOffSegLo = kOffTmp2 + (long long)kMaxStates * 4;
constexpr long long kOffSegRad = kOffSegLo + kSegSlots;
constexpr long long kOffSegStr = kOffSegRad + kSegSlots;
constexpr long long kOffVar = kOffSegStr + (long long)kSegSlots * 4;  // vals, cL, cR, lists

struct Block {           // per-block views (pointers into the slab) + shared-memory state
  char *slab;
  Seg *segs;
  double2 *FL, *FR;
  StackEnt *stack;
  uint32_t *offA, *offB, *tmp, *tmp2;
  uint8_t *segLo, *segRad;
  int32_t *segStr;
  uint8_t *vals;
  ull *cL, *cR;
  char *lists;
  long long list_bytes;
};

struct Shared {
  ColInfo col[kMaxModes + 1];
  int G[kMaxModes + 1];
  int T[kMaxModes];
  int n[kMaxModes + 1];    // states per column
  int raw[kMaxModes + 1];  // non-local circuits: raw combinations of a filtered column
  int vb[kMaxModes + 1];   // vals base
  int cb[kMaxModes + 1];   // count base
  ull NL[kMaxModes + 1], NR[kMaxModes + 1];
  uint32_t scan[kThreads];
  int status;
  int ks;
  int nsegs;
  uint32_t total;
  int sp;                  // stack pointer
  StackEnt top;
  int q_cached;
  int cr_q;                // output whose cR counts are in the slab
  int unit;
  ull ph[8];               // thread 0's SM clock per phase (lofp_stats phase_cycles)
  ull tph;
};

// phase timer of thread 0 (block time split: lofp_run_stats::phase_cycles)
#define PHASE(sh, i)                          \
  do {                                        \
    if (threadIdx.x == 0) {                   \
      const ull now_ = clock64();             \
      (sh).ph[i] += now_ - (sh).tph;          \
      (sh).tph = now_;                        \
    }                                         \
  } while (0)

// slab carve of one output: vals, cL, cR, then the half-path lists (needs sh.n/vb/cb)
__device__ __forceinline__ void carve(const CallParams &p, Block &b, const Shared &sh) {
  const int M = p.M;
  const long long vb = sh.vb[M] + (long long)sh.n[M] * sh.col[M].nvar;
  const long long cb = sh.cb[M] + sh.n[M];
  const long long vbytes = (vb + 15) & ~15ll;
  b.vals = (uint8_t *)(b.slab + kOffVar);
  b.cL = (ull *)(b.slab + kOffVar + vbytes);
  b.cR = b.cL + cb;
  const long long used = kOffVar + vbytes + 16 * cb;
  b.lists = b.slab + used;
  b.list_bytes = p.slab_bytes - used;
}

__device__ __forceinline__ const uint8_t *vrow(const Block &b, const Shared &sh, int k, int s) {
  return b.vals + sh.vb[k] + s * sh.col[k].nvar;
}

// F(k-1) <= F(k) at every time (non-negative occupations of mode k-1)
__device__ __forceinline__ bool compat(const CallParams &p, const Block &b, const Shared &sh, int k, int sa, int sb) {
  const ColInfo &ck = sh.col[k];
  const uint8_t *va = vrow(b, sh, k - 1, sa);
  const uint8_t *vb = vrow(b, sh, k, sb);
  for (int c = 0; c < ck.ncmp; ++c) {
    const CmpPair pr = p.cmp[ck.cmp_base + c];
    if (va[pr.sa] > vb[pr.sb]) return false;
  }
  for (int e = 0; e < ck.neq; ++e) {  // non-local circuits: conservation / carried variables
    const EqCon ec = p.eqc[ck.eq_base + e];
    int sum = 0;
    for (int t = 0; t < ec.nterm; ++t) {
      const int v = (ec.var[t] & 0x80) ? vb[ec.var[t] & 0x7f] : va[ec.var[t] & 0x7f];
      sum += ec.coef[t] * v;
    }
    if (sum != 0) return false;
  }
  return true;
}

__device__ __forceinline__ bool live(const Block &b, const Shared &sh, int k, int s) {
  return b.cL[sh.cb[k] + s] != 0 && b.cR[sh.cb[k] + s] != 0;
}

// Cut factor of cut c: the product of the Appendix-A elements of the BS on modes (c-1, c)
// (eq. (1)) for columns c-1, c, c+1 in states sa, sb, sc, times the phase gates
// folded into cut c.  Vacuum BS (x1 + x2 = 0) contribute exactly 1.
__device__ double2 cut_factor(const CallParams &p, const Block &b, const Shared &sh, int c, int sa, int sb, int sc,
                              ull &cm) {
  double2 f = make_double2(1.0, 0.0);
  if (c < 1 || c > p.M - 1) return f;
  const ColInfo &cc = sh.col[c];
  const uint8_t *va = vrow(b, sh, c - 1, sa);
  const uint8_t *vb = vrow(b, sh, c, sb);
  const uint8_t *vc = vrow(b, sh, c + 1, sc);
  for (int t = 0; t < cc.nfac; ++t) {
    const FacInfo fi = p.fac[cc.fac_base + t];
    int x1, x2, y1;
    if (fi.kind == 0) {  // BS on (c-1, c): x1, x2 before it, y1 after it
      const int A = va[fi.sA], Bm = vb[fi.i], Bp = vb[fi.i + 1], C = vc[fi.sC];
      x1 = Bm - A;
      x2 = C - Bm;
      y1 = Bp - A;
    } else {  // carried BS (a, c): x1, y1 of mode a carried in column c; x2 of mode c
      x1 = vb[fi.i];
      y1 = vb[fi.sA];
      x2 = vc[fi.sC] - vb[fi.sB];
    }
    const int n = x1 + x2;
    if (n == 0) continue;
    const long long idx = p.tab_off[fi.bs] + tri_dev(n) + (long long)x1 * (n + 1) + y1;
    if (x1 < 0 || x2 < 0 || y1 < 0 || y1 > n || idx >= p.tab_off[fi.bs + 1]) {
      atomicAdd(&p.ctr->table_error, 1ull);
      continue;
    }
    f = cmul(f, p.table[idx]);
    ++cm;
  }
  for (int t = 0; t < cc.ngate; ++t) {
    const GateInfo gi = p.gat[cc.gate_base + t];
    const uint8_t *lo = gi.col_off ? vb : va;
    const uint8_t *hi = gi.col_off ? vc : vb;
    const int n = (int)hi[gi.seg_hi] - (int)lo[gi.seg_lo];
    f = cmul(f, p.gate_tab[gi.gate * (p.N + 1) + n]);
    ++cm;
  }
  return f;
}

// ---- block-wide helpers --------------------------------------------------------------
// exclusive scan of in[0..n) into out[0..n) (slab arrays); returns the total (all threads)
__device__ uint32_t block_scan(Shared &sh, const uint32_t *in, uint32_t *out, int n) {
  const int per = (n + kThreads - 1) / kThreads;
  const int a = threadIdx.x * per, e = min(n, a + per);
  uint32_t s = 0;
  for (int i = a; i < e; ++i) s += in[i];
  sh.scan[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    uint32_t loc[kThreads / 32];
    uint32_t tot = 0;
#pragma unroll
    for (int i = 0; i < kThreads / 32; ++i) {
      loc[i] = sh.scan[lane * (kThreads / 32) + i];
      tot += loc[i];
    }
    uint32_t incl = tot;
    for (int d = 1; d < 32; d <<= 1) {
      uint32_t v = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += v;
    }
    uint32_t run = incl - tot;
#pragma unroll
    for (int i = 0; i < kThreads / 32; ++i) {
      sh.scan[lane * (kThreads / 32) + i] = run;
      run += loc[i];
    }
    if (lane == 31) sh.total = incl;
  }
  __syncthreads();
  uint32_t run = sh.scan[threadIdx.x];
  for (int i = a; i < e; ++i) {
    const uint32_t v = in[i];
    out[i] = run;
    run += v;
  }
  const uint32_t total = sh.total;
  __syncthreads();
  return total;
}

// The same scan as a call: inlined into the level-synchronous split kernel, nvcc 12.9
// emitted code that raised "illegal instruction" on sm_100a (warp 0's shuffles after a
// barrier); as a call it is correct (the unit kernel keeps the inlined form: measured
// 2.5 % faster on configs[4]).
__device__ __noinline__ uint32_t block_scan_call(Shared &sh, const uint32_t *in, uint32_t *out, int n) {
  return block_scan(sh, in, out, n);
}

__device__ __forceinline__ ull warp_sum_sat(ull v) {
  for (int d = 16; d > 0; d >>= 1) v = sat_add(v, __shfl_down_sync(0xffffffffu, v, d));
  return v;
}

__device__ __forceinline__ Block make_block(const CallParams &p) {
  Block b;
  b.slab = p.slab + (long long)blockIdx.x * p.slab_bytes;
  b.segs = (Seg *)(b.slab + kOffSegs);
  b.FL = (double2 *)(b.slab + kOffFL);
  b.FR = (double2 *)(b.slab + kOffFR);
  b.stack = (StackEnt *)(b.slab + kOffStack);
  b.offA = (uint32_t *)(b.slab + kOffA);
  b.offB = (uint32_t *)(b.slab + kOffB);
  b.tmp = (uint32_t *)(b.slab + kOffTmp);
  b.tmp2 = (uint32_t *)(b.slab + kOffTmp2);
  b.segLo = (uint8_t *)(b.slab + kOffSegLo);
  b.segRad = (uint8_t *)(b.slab + kOffSegRad);
  b.segStr = (int32_t *)(b.slab + kOffSegStr);
  b.vals = nullptr;
  b.cL = b.cR = nullptr;
  b.lists = nullptr;
  b.list_bytes = 0;
  return b;
}

// value of variable g (slot seg_base + i) in the raw mixed-radix combination r
__device__ __forceinline__ int raw_val(const Block &b, int g, int r) {
  return b.segLo[g] + (r / b.segStr[g]) % b.segRad[g];
}

// non-local circuits: the column's own equalities (the jump of F(k) at a layer equals the
// summed y1 - x1 of the carried BS crossing cut k) for raw combination r
__device__ bool intra_ok(const CallParams &p, const Block &b, const ColInfo &ci, int r) {
  for (int e = 0; e < ci.nintra; ++e) {
    const EqCon ec = p.eqc[ci.intra_base + e];
    int sum = 0;
    for (int t = 0; t < ec.nterm; ++t) sum += ec.coef[t] * raw_val(b, ci.seg_base + (ec.var[t] & 0x7f), r);
    if (sum != 0) return false;
  }
  return true;
}

// ---- per-output column setup (readings R5, R15) --------------------------------------
// Returns kStatusOk / kStatusZero / kStatusBad / kStatusUnsupported (block-uniform).
__device__ int setup_output(const CallParams &p, Block &b, Shared &sh, int q) {
  const int M = p.M, tid = threadIdx.x;
  for (int i = tid; i < M; i += kThreads) sh.T[i] = p.T[(long long)q * M + i];
  if (tid == 0) sh.cr_q = -1;
  __syncthreads();
  if (tid == 0) {
    int st = kStatusOk, g = 0;
    sh.G[0] = 0;
    for (int i = 0; i < M; ++i) {
      const int t = sh.T[i];
      if (t < 0) st = kStatusBad;
      g += t > 0 ? t : 0;
      if (g > 255) g = 255;
      sh.G[i + 1] = g;
    }
    if (st == kStatusOk && sh.G[M] != p.N) st = kStatusZero;  // photon number (reading R9)
    sh.status = st;
  }
  __syncthreads();
  if (sh.status != kStatusOk) return sh.status;
  if (p.force_generic) return kStatusUnsupported;  // test hook: every output to the generic engine
  // segment ranges: intersection of the backward (T) and forward (S) light-cone boxes
  int my_bad = 0;
  for (int k = tid; k <= M; k += kThreads) {
    const ColInfo ci = sh.col[k];
    long long n = 1;
    for (int i = 0; i < ci.nvar; ++i) {
      int lo, hi;
      if (!p.general) {
        const SegInfo si = p.seg[ci.seg_base + i];
        lo = max(sh.G[si.rho], (int)p.cumS[si.rhop]);
        hi = min(sh.G[si.sig], (int)p.cumS[si.sigp]);
      } else {  // non-local circuit: cone sums over mode sets
        const BoundInfo &bi = p.bnd[ci.seg_base + i];
        int sum[4];
        for (int w = 0; w < 4; ++w) {
          int acc = 0;
          for (int h = 0; h < 2; ++h) {
            uint64_t m = bi.m[w][h];
            while (m) {
              const int md = 64 * h + __ffsll((long long)m) - 1;
              m &= m - 1;
              acc += (w < 2) ? (int)p.cumS[md + 1] - (int)p.cumS[md] : sh.G[md + 1] - sh.G[md];
            }
          }
          sum[w] = acc;
        }
        hi = min(sum[0], sum[2]);
        lo = max(0, max(p.N - sum[1], p.N - sum[3]));
      }
      const int rad = hi - lo + 1;
      b.segLo[ci.seg_base + i] = (uint8_t)max(lo, 0);
      b.segRad[ci.seg_base + i] = (uint8_t)max(rad, 0);
      b.segStr[ci.seg_base + i] = (int)n;
      n = rad > 0 ? n * rad : 0;
      if (n > kMaxRawStates) { n = kMaxRawStates + 1; }
    }
    // local circuits: every raw combination is a state; non-local ones filter by the
    // column's conservation equalities below (ColInfo::nintra)
    const int lim = (p.general && ci.nintra) ? kMaxRawStates : kMaxStates;
    if (n > lim) my_bad = 1;
    sh.n[k] = (int)n;
  }
  my_bad = __syncthreads_or(my_bad);
  if (p.general && !my_bad) {
    // count the raw combinations of each constrained column that satisfy its equalities
    for (int k = 0; k <= M; ++k) {
      const ColInfo ci = sh.col[k];
      if (!ci.nintra) continue;  // (block-uniform)
      if (tid == 0) sh.total = 0;
      __syncthreads();
      uint32_t c = 0;
      for (int r = tid; r < sh.n[k]; r += kThreads) c += intra_ok(p, b, ci, r) ? 1u : 0u;
      atomicAdd(&sh.total, c);
      __syncthreads();
      if (tid == 0) sh.raw[k] = sh.n[k], sh.n[k] = (int)sh.total;
      __syncthreads();
      if (sh.n[k] > kMaxStates) my_bad = 1;
    }
  }
  if (tid == 0) {
    int st = my_bad ? kStatusUnsupported : kStatusOk;
    long long vb = 0, cb = 0;
    for (int k = 0; k <= M && st == kStatusOk; ++k) {
      if (sh.n[k] == 0) st = kStatusZero;  // structurally unreachable (reading R5)
      sh.vb[k] = (int)vb;
      sh.cb[k] = (int)cb;
      vb += (long long)sh.n[k] * sh.col[k].nvar;
      cb += sh.n[k];
    }
    if (st == kStatusOk && cb > kMaxStatesTotal) st = kStatusUnsupported;
    if (st == kStatusOk) {
      const long long used = kOffVar + ((vb + 15) & ~15ll) + 16 * cb;
      if (p.slab_bytes - used < 4096) st = kStatusUnsupported;
      if (p.general && used > p.slab_bytes - 8ll * kMaxRawStates) st = kStatusUnsupported;
      atomicMax(&p.ctr->max_states, (ull)cb);
    }
    sh.status = st;
  }
  __syncthreads();
  if (sh.status != kStatusOk) return sh.status;
  carve(p, b, sh);
  // segment values of every column state (mixed radix over the segments)
  for (int k = 0; k <= M; ++k) {
    const ColInfo ci = sh.col[k];
    if (p.general && ci.nintra) {  // the raw combinations that satisfy the equalities, in order
      uint32_t *flag = (uint32_t *)(b.slab + p.slab_bytes - 8ll * kMaxRawStates);
      uint32_t *pos = flag + kMaxRawStates;
      const int R = sh.raw[k];
      for (int r = tid; r < R; r += kThreads) flag[r] = intra_ok(p, b, ci, r) ? 1u : 0u;
      __syncthreads();
      block_scan(sh, flag, pos, R);
      for (int r = tid; r < R; r += kThreads) {
        if (!flag[r]) continue;
        uint8_t *row = b.vals + sh.vb[k] + pos[r] * ci.nvar;
        for (int i = 0; i < ci.nvar; ++i) row[i] = (uint8_t)raw_val(b, ci.seg_base + i, r);
      }
      __syncthreads();
      continue;
    }
    for (int s = tid; s < sh.n[k]; s += kThreads) {
      uint8_t *row = b.vals + sh.vb[k] + s * ci.nvar;
      for (int i = 0; i < ci.nvar; ++i) {
        const int g = ci.seg_base + i;
        row[i] = (uint8_t)(b.segLo[g] + (s / b.segStr[g]) % b.segRad[g]);
      }
    }
  }
  __syncthreads();
  return kStatusOk;
}

// ---- exact path counts by a transfer over columns (reading R6) -----------------------
// cL[k][s]: partial paths from column j (state sj) to column k ending in s;
// cR[k][s]: completions from column k (state s) to column M.  Columns >= j.
__device__ void dp_counts(const CallParams &p, Block &b, Shared &sh, int j, int sj, bool need_right,
                          bool need_left = true) {
  const int M = p.M, tid = threadIdx.x;
  if (need_left)
    for (int s = tid; s < sh.n[j]; s += kThreads) b.cL[sh.cb[j] + s] = (s == sj) ? 1ull : 0ull;
  if (need_right)
    for (int s = tid; s < sh.n[M]; s += kThreads) b.cR[sh.cb[M] + s] = 1ull;
  __syncthreads();
  // the right counts depend on the output only: computed for every column (they are cached
  // across the units of one output); the left counts from column j
  const int iters = need_right ? M : M - j;
  for (int i = 1; i <= iters; ++i) {
    const int kL = j + i, kR = M - i;
    const int nL = (need_left && kL <= M) ? sh.n[kL] : 0, nR = need_right ? sh.n[kR] : 0;
    for (int t = tid; t < nL + nR; t += kThreads) {
      ull sum = 0;
      if (t < nL) {
        const int n0 = sh.n[kL - 1];
        const ull *src = b.cL + sh.cb[kL - 1];
        for (int pp = 0; pp < n0; ++pp) {
          const ull c = src[pp];
          if (c && compat(p, b, sh, kL, pp, t)) sum = sat_add(sum, c);
        }
        b.cL[sh.cb[kL] + t] = sum;
      } else {
        const int s = t - nL;
        const int n1 = sh.n[kR + 1];
        const ull *src = b.cR + sh.cb[kR + 1];
        for (int sp = 0; sp < n1; ++sp) {
          const ull c = src[sp];
          if (c && compat(p, b, sh, kR + 1, s, sp)) sum = sat_add(sum, c);
        }
        b.cR[sh.cb[kR] + s] = sum;
      }
    }
    __syncthreads();
  }
}

// NL[k] / NR[k]: half-path list sizes if the split were at column k (live states only)
__device__ void list_sizes(Block &b, Shared &sh, int j, int M) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int k = j + warp; k <= M; k += kThreads / 32) {
    ull sl = 0, sr = 0;
    for (int s = lane; s < sh.n[k]; s += 32) {
      const ull l = b.cL[sh.cb[k] + s], r = b.cR[sh.cb[k] + s];
      if (l && r) {
        sl = sat_add(sl, l);
        sr = sat_add(sr, r);
      }
    }
    sl = warp_sum_sat(sl);
    sr = warp_sum_sat(sr);
    if (lane == 0) {
      sh.NL[k] = sl;
      sh.NR[k] = sr;
    }
  }
  __syncthreads();
}

// Segment list of one BFS level: for every live state s of column kd (in order), its live
// neighbours p in column ks_ (in order); dst offsets from offD, src offsets from offS.
// left = true: kd = ks_ + 1, compat(kd, p, s); else kd = ks_ - 1, compat(ks_, s, p).
__device__ int build_segments(const CallParams &p, Block &b, Shared &sh, int kd, int kn, bool left,
                              const uint32_t *offS, const uint32_t *offD) {
  const int nd = sh.n[kd], nn = sh.n[kn], tid = threadIdx.x;
  const ull *cnt = left ? b.cL : b.cR;
  for (int s = tid; s < nd; s += kThreads) {
    uint32_t c = 0;
    if (live(b, sh, kd, s))
      for (int pp = 0; pp < nn; ++pp)
        if (live(b, sh, kn, pp) && (left ? compat(p, b, sh, kd, pp, s) : compat(p, b, sh, kn, s, pp))) ++c;
    b.tmp[s] = c;
  }
  __syncthreads();
  const uint32_t nsegs = block_scan(sh, b.tmp, b.tmp2, nd);
  if (nsegs > (uint32_t)kMaxSegments) return -1;
  for (int s = tid; s < nd; s += kThreads) {
    if (!live(b, sh, kd, s)) continue;
    uint32_t e = b.tmp2[s], d = offD[s];
    for (int pp = 0; pp < nn; ++pp) {
      if (!live(b, sh, kn, pp)) continue;
      if (!(left ? compat(p, b, sh, kd, pp, s) : compat(p, b, sh, kn, s, pp))) continue;
      const uint32_t len = (uint32_t)cnt[sh.cb[kn] + pp];
      Seg g;
      g.dst = d;
      g.src = offS[pp];
      g.len = len;
      g.p = (uint16_t)pp;
      g.s = (uint16_t)s;
      DCHECK(e < (uint32_t)kMaxSegments, "segs");
      b.segs[e++] = g;
      d += len;
    }
  }
  __syncthreads();
  return (int)nsegs;
}

__device__ __forceinline__ int find_seg(const Seg *segs, int nsegs, uint32_t t) {
  int lo = 0, hi = nsegs - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (segs[mid].dst <= t) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// Bucket offsets of column k: exclusive scan of the live counts (cL or cR).
__device__ uint32_t bucket_offsets(Block &b, Shared &sh, int k, bool left, uint32_t *off) {
  const ull *cnt = left ? b.cL : b.cR;
  for (int s = threadIdx.x; s < sh.n[k]; s += kThreads)
    b.tmp[s] = live(b, sh, k, s) ? (uint32_t)cnt[sh.cb[k] + s] : 0u;
  __syncthreads();
  return block_scan(sh, b.tmp, off, sh.n[k]);
}

// ---- the outer product: every path = X_i * Y_j, one complex FMA pair per path --------
// A warp holds kKX X values per lane (a tile of kXT = 32 kKX) in registers and streams a
// tile of up to kYT Y values from its shared-memory slice (broadcast reads): per Y value
// 1 LDS.128 and 4 kKX DFMA per lane.
#define LOFP_CFMA(v, KX)                           \
  _Pragma("unroll") for (int r = 0; r < KX; ++r) { \
    acc[r].x = fma(x[r].x, (v).x, acc[r].x);        \
    acc[r].y = fma(x[r].x, (v).y, acc[r].y);        \
    acc[r].x = fma(-x[r].y, (v).y, acc[r].x);       \
    acc[r].y = fma(x[r].y, (v).x, acc[r].y);        \
  }

// KX <= kKX: only the first KX X slots of each lane hold values (a pair's last X tile with
// at most 32 KX elements left): the other slots would multiply zeros
template <int KX>
__device__ __forceinline__ void fma_block(const double2 (&x)[kKX], const double2 *__restrict__ sW, uint32_t len,
                                          double2 (&acc)[kKX]) {
  uint32_t y = 0;
  for (; y + 3 < len; y += 4) {  // four Y values loaded ahead of their 16 KX DFMA
    const double2 v0 = sW[y], v1 = sW[y + 1], v2 = sW[y + 2], v3 = sW[y + 3];
    LOFP_CFMA(v0, KX)
    LOFP_CFMA(v1, KX)
    LOFP_CFMA(v2, KX)
    LOFP_CFMA(v3, KX)
  }
  for (; y < len; ++y) {
    const double2 v0 = sW[y];
    LOFP_CFMA(v0, KX)
  }
}

struct PairInfo {        // one column pair (a, b) of a unit: X = the longer list
  uint32_t xoff, yoff, nX, nY;
  uint32_t nxt;          // X tiles
  uint32_t swap;         // 1: X is the right list
};

// One BFS level of a half-path list: element t of the new level extends element src of
// the old one by one column; its product gains one cut factor.  Elements of one segment
// (predecessor p, state s) differ only in their context state (the column beyond p), so
// when cheaper the factors are tabulated per (segment, context) first (nseg * nctx cut
// factors instead of one per element).  Warps take 32 consecutive elements: one binary
// search per warp, then a short forward scan per lane.
//   left:  dst column k+1, src column k, factor of cut k  = f(ctx @ k-1, p @ k, s @ k+1)
//   right: dst column k,   src column k+1, factor of cut k+1 = f(s @ k, p @ k+1, ctx @ k+2)
template <bool LEFT>
__device__ void expand_level(const CallParams &p, Block &b, Shared &sh, int k, int nsegs, uint32_t total,
                             const double2 *__restrict__ srcP, const uint16_t *__restrict__ srcC,
                             double2 *__restrict__ dstP, uint16_t *__restrict__ dstC, double2 *Fseg,
                             long long fcap, ull &cm) {
  const int M = p.M, tid = threadIdx.x;
  const int cut = LEFT ? k : k + 1;
  const bool has_factor = cut >= 1 && cut <= M - 1;
  const int nctx = LEFT ? (k >= 1 ? sh.n[k - 1] : 1) : (k + 2 <= M ? sh.n[k + 2] : 1);
  const long long ntab = (long long)nsegs * nctx;
  const bool use_table = has_factor && ntab <= fcap && ntab < (long long)total;
  if (use_table) {
    for (long long t = tid; t < ntab; t += kThreads) {
      const int e = (int)(t / nctx), c = (int)(t - (long long)e * nctx);
      const Seg g = b.segs[e];
      double2 f = make_double2(0.0, 0.0);
      if (LEFT) {
        if (compat(p, b, sh, k, c, g.p)) f = cut_factor(p, b, sh, k, c, g.p, g.s, cm);
      } else {
        if (k + 2 > M || compat(p, b, sh, k + 2, g.p, c)) f = cut_factor(p, b, sh, k + 1, g.s, g.p, c, cm);
      }
      Fseg[t] = f;
    }
    __syncthreads();
  }
  const int warp = tid >> 5, lane = tid & 31;
  for (uint32_t base = (uint32_t)warp * 32; base < total; base += kThreads) {
    int e = 0;
    if (lane == 0) e = find_seg(b.segs, nsegs, base);
    e = __shfl_sync(0xffffffffu, e, 0);
    const uint32_t t = base + lane;
    if (t < total) {
      while (e + 1 < nsegs && b.segs[e + 1].dst <= t) ++e;
      const Seg g = b.segs[e];
      const uint32_t src = g.src + (t - g.dst);
      DCHECK(t >= g.dst && t - g.dst < g.len, "bfs segment");
      const int ctx = srcC[src];
      double2 f = make_double2(1.0, 0.0);
      if (use_table) {
        DCHECK(ctx < nctx, "bfs ctx");
        f = Fseg[(long long)e * nctx + ctx];
      } else if (has_factor) {
        f = LEFT ? cut_factor(p, b, sh, k, ctx, g.p, g.s, cm) : cut_factor(p, b, sh, k + 1, g.s, g.p, ctx, cm);
      }
      dstP[t] = cmul(srcP[src], f);
      dstC[t] = g.p;
      ++cm;
    }
  }
  __syncthreads();
}

// ---- one unit: column-split enumeration of its subtree (reading R20) ------------------
// Paths below the prefix (columns 0..j fixed) = sum over column-pair states (a, b) at
// columns (ks, ks+1) of L(a) x R(b): L(a) = partial paths j..ks ending in a (products of
// cut factors j..ks-1), R(b) = partial paths ks+1..M starting in b (cuts ks+2..M-1); the
// cut factors of ks and ks+1 scale the two lists per pair.  Both lists are built level by
// level (BFS with exact bucket offsets from the counts: deterministic, no atomics).
__device__ void process_stack(const CallParams &p, Block &b, Shared &sh, double2 *sY, double2 (&acc)[kKX],
                              ull &npaths, ull &cm, ull &nelem, ull &tstage, ull &tfma) {
  const int M = p.M, tid = threadIdx.x;
  while (true) {
    if (tid == 0) {
      if (sh.sp > 0) sh.top = b.stack[--sh.sp];
      else sh.top.j = -1;
    }
    __syncthreads();
    const StackEnt top = sh.top;
    if (top.j < 0) break;
    const int j = top.j, sj = top.sj, sjm1 = top.sjm1;
    const double2 pi = make_double2(top.re, top.im);
    const bool need_right = sh.cr_q != sh.q_cached;  // cR depends on the output only
    PHASE(sh, 7);
    dp_counts(p, b, sh, j, sj, need_right);
    if (tid == 0) sh.cr_q = sh.q_cached;
    list_sizes(b, sh, j, M);
    // choose the split column pair: smallest L + R lists that fit the scratch
    if (tid == 0) {
      int best = -1;
      ull bcost = ~0ull;
      for (int k = j; k <= M - 1; ++k) {
        const ull c = sat_add(sh.NL[k], sh.NR[k + 1]);
        // lists (two buffers each side, 18 B per element) + room for 16 pairs' scaling tables
        const long long nctx = (k >= 1 ? sh.n[k - 1] : 1) + (k + 2 <= M ? sh.n[k + 2] : 1);
        const long long reserve = 64 + 16 * ((long long)sizeof(PairInfo) + 16 * nctx);
        if (c < (ull)(b.list_bytes / 36) && 36ll * (long long)c + reserve <= b.list_bytes && c < bcost) {
          bcost = c;
          best = k;
        }
      }
      sh.ks = best;
    }
    __syncthreads();
    const int ks = sh.ks;
    if (ks < 0) {
      // lists over capacity: split by fixing column j+1 and process the children in turn
      if (tid == 0) {
        atomicAdd(&p.ctr->subsplits, 1ull);
        const int n1 = sh.n[j + 1];
        for (int s = n1 - 1; s >= 0; --s) {
          if (!live(b, sh, j + 1, s) || !compat(p, b, sh, j + 1, sj, s)) continue;
          ull c2 = 0;
          const double2 f = cut_factor(p, b, sh, j, sjm1, sj, s, c2);
          const double2 np = cmul(pi, f);
          if (sh.sp < kStackMax) {
            StackEnt e;
            e.j = j + 1;
            e.sjm1 = (uint16_t)sj;
            e.sj = (uint16_t)s;
            e.re = np.x;
            e.im = np.y;
            e.pad = 0;
            b.stack[sh.sp++] = e;
          } else {
            atomicAdd(&p.ctr->unsupported, 1ull);
          }
        }
      }
      __syncthreads();
      continue;
    }
    PHASE(sh, 1);
    const ull NLk = sh.NL[ks], NRk = sh.NR[ks + 1];
    const ull capL = NLk, capR = NRk;
    double2 *Lp[2], *Rp[2];
    uint16_t *Lc[2], *Rc[2];
    {
      char *q = b.lists;
      Lp[0] = (double2 *)q; q += 16 * capL;
      Lp[1] = (double2 *)q; q += 16 * capL;
      Rp[0] = (double2 *)q; q += 16 * capR;
      Rp[1] = (double2 *)q; q += 16 * capR;
      Lc[0] = (uint16_t *)q; q += 2 * capL;
      Lc[1] = (uint16_t *)q; q += 2 * capL;
      Rc[0] = (uint16_t *)q; q += 2 * capR;
      Rc[1] = (uint16_t *)q;
    }
    // scratch after the lists: per-(segment, context) factor tables of the BFS levels
    double2 *Fscratch = (double2 *)(((uintptr_t)(b.lists + 36ll * (long long)(NLk + NRk)) + 15) & ~(uintptr_t)15);
    const long long fcap = ((b.lists + b.list_bytes) - (char *)Fscratch) / 16 - 1;
    // ---- left lists: levels j..ks
    uint32_t *offS = b.offA, *offD = b.offB;
    int cur = 0;
    if (tid == 0) {
      Lp[0][0] = make_double2(1.0, 0.0);
      Lc[0][0] = (uint16_t)sjm1;
    }
    for (int s = tid; s < sh.n[j]; s += kThreads) offS[s] = 0;
    __syncthreads();
    bool ok = true;
    for (int k = j; k < ks && ok; ++k) {
      const uint32_t total = bucket_offsets(b, sh, k + 1, true, offD);
      const int nsegs = build_segments(p, b, sh, k + 1, k, true, offS, offD);
      if (nsegs < 0) { ok = false; break; }
      DCHECK(total <= capL, "left level size");
      expand_level<true>(p, b, sh, k, nsegs, total, Lp[cur], Lc[cur], Lp[cur ^ 1], Lc[cur ^ 1], Fscratch, fcap, cm);
      nelem += (total + kThreads - 1 - tid) / kThreads;
      cur ^= 1;
      uint32_t *tt = offS; offS = offD; offD = tt;
    }
    PHASE(sh, 2);
    const int curL = cur;
    uint32_t *offL = offS;  // bucket offsets of column ks
    // ---- right lists: levels M..ks+1 (the other offset buffer pair)
    uint32_t *offS2 = (offL == b.offA) ? b.offB : b.offA;
    cur = 0;
    if (tid == 0) {
      Rp[0][0] = make_double2(1.0, 0.0);
      Rc[0][0] = 0;
    }
    for (int s = tid; s < sh.n[M]; s += kThreads) offS2[s] = 0;
    __syncthreads();
    // the right BFS needs three offset arrays besides offL: use FR's storage as scratch
    uint32_t *rA = offS2, *rB = (uint32_t *)b.FR;
    for (int k = M - 1; k >= ks + 1 && ok; --k) {
      const uint32_t total = bucket_offsets(b, sh, k, false, rB);
      const int nsegs = build_segments(p, b, sh, k, k + 1, false, rA, rB);
      if (nsegs < 0) { ok = false; break; }
      DCHECK(total <= capR, "right level size");
      expand_level<false>(p, b, sh, k, nsegs, total, Rp[cur], Rc[cur], Rp[cur ^ 1], Rc[cur ^ 1], Fscratch, fcap, cm);
      nelem += (total + kThreads - 1 - tid) / kThreads;
      cur ^= 1;
      uint32_t *tt = rA; rA = rB; rB = tt;
    }
    const int curR = cur;
    uint32_t *offR = rA;  // bucket offsets of column ks+1
    if (offR == (uint32_t *)b.FR) {
      // move the offsets out of FR's storage (FR is rebuilt per pair)
      uint32_t *dst = (offL == b.offA) ? b.offB : b.offA;
      for (int s = tid; s < sh.n[ks + 1]; s += kThreads) dst[s] = offR[s];
      __syncthreads();
      offR = dst;
    }
    if (!ok) {
      if (tid == 0) atomicAdd(&p.ctr->unsupported, 1ull);
      __syncthreads();
      continue;
    }
    if (tid == 0) {
      atomicMax(&p.ctr->max_list, (ull)max(NLk, NRk));
    }
    PHASE(sh, 3);
    // ---- column pairs (a at ks, b at ks+1): all pairs' scaling tables, then warp tiles
    {
      // reuse build_segments with kd = ks+1 (b), kn = ks (a), left = true: offsets unused
      const int npairs = build_segments(p, b, sh, ks + 1, ks, true, b.offA /*unused*/, b.tmp /*unused*/);
      if (npairs < 0) {
        if (tid == 0) atomicAdd(&p.ctr->unsupported, 1ull);
        __syncthreads();
        continue;
      }
      if (tid == 0) atomicAdd(&p.ctr->pairs, (ull)npairs);
      const int nctxL = ks >= 1 ? sh.n[ks - 1] : 1;
      const int nctxR = ks + 2 <= M ? sh.n[ks + 2] : 1;
      char *pq = b.lists + 36ll * (long long)(NLk + NRk);
      pq = (char *)(((uintptr_t)pq + 15) & ~(uintptr_t)15);
      const long long room = (b.lists + b.list_bytes) - pq;
      const long long per_pair = (long long)sizeof(PairInfo) + 16ll * (nctxL + nctxR);
      const int batch = (int)min((long long)min(npairs, kMaxStates), (room - 16) / per_pair);
      DCHECK(batch >= 1, "pair batch");
      PairInfo *pinfo = (PairInfo *)pq;
      double2 *FLall = (double2 *)(((uintptr_t)(pq + (long long)sizeof(PairInfo) * batch) + 15) & ~(uintptr_t)15);
      double2 *FRall = FLall + (long long)nctxL * batch;
      for (int e0 = 0; e0 < npairs; e0 += batch) {
        const int e1 = min(npairs, e0 + batch), ne = e1 - e0;
        for (int e = tid; e < ne; e += kThreads) {
          const Seg g = b.segs[e0 + e];
          const int a = g.p, bb = g.s;
          const uint32_t nL = (uint32_t)b.cL[sh.cb[ks] + a];
          const uint32_t nR = (uint32_t)b.cR[sh.cb[ks + 1] + bb];
          PairInfo pi_;
          pi_.swap = nL < nR;
          pi_.nX = pi_.swap ? nR : nL;
          pi_.nY = pi_.swap ? nL : nR;
          pi_.xoff = pi_.swap ? offR[bb] : offL[a];
          pi_.yoff = pi_.swap ? offL[a] : offR[bb];
          pi_.nxt = (pi_.nX + kXT - 1) / kXT;
          b.tmp[e] = pi_.nxt * ((pi_.nY + kYT - 1) / kYT);
          pinfo[e] = pi_;
        }
        for (int t = tid; t < ne * nctxL; t += kThreads) {
          const int e = t / nctxL, al = t - e * nctxL;
          const Seg g = b.segs[e0 + e];
          double2 f = pi;
          if (ks >= 1) {
            if (compat(p, b, sh, ks, al, g.p)) f = cmul(pi, cut_factor(p, b, sh, ks, al, g.p, g.s, cm));
            else f = make_double2(0.0, 0.0);
          }
          FLall[t] = f;
        }
        for (int t = tid; t < ne * nctxR; t += kThreads) {
          const int e = t / nctxR, be = t - e * nctxR;
          const Seg g = b.segs[e0 + e];
          double2 f = make_double2(1.0, 0.0);
          if (ks + 1 <= M - 1) {
            if (compat(p, b, sh, ks + 2, g.s, be)) f = cut_factor(p, b, sh, ks + 1, g.p, g.s, be, cm);
            else f = make_double2(0.0, 0.0);
          }
          FRall[t] = f;
        }
        __syncthreads();
        const uint32_t ntiles = block_scan(sh, b.tmp, b.tmp2, ne);  // tile offsets per pair
        PHASE(sh, 4);
        // every warp takes every (kThreads/32)-th tile: a static, deterministic assignment
        const int warp = tid >> 5, lane = tid & 31;
        double2 *sW = sY + warp * kYT;
        int last_lo = -1;
        uint32_t last_yt = 0;
        for (uint32_t t = warp; t < ntiles; t += kThreads / 32) {
          int lo = 0, hi = ne - 1;
          while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (b.tmp2[mid] <= t) lo = mid; else hi = mid - 1;
          }
          const PairInfo pr = pinfo[lo];
          DCHECK(lo >= 0 && lo < ne && t >= b.tmp2[lo], "tile pair");
          DCHECK((pr.swap ? (ull)pr.xoff + pr.nX <= capR && (ull)pr.yoff + pr.nY <= capL
                          : (ull)pr.xoff + pr.nX <= capL && (ull)pr.yoff + pr.nY <= capR), "tile lists");
          const uint32_t local = t - b.tmp2[lo];
          const uint32_t xt = local % pr.nxt, yt = local / pr.nxt;
          const double2 *Xp = (pr.swap ? Rp[curR] : Lp[curL]) + pr.xoff;
          const uint16_t *Xc = (pr.swap ? Rc[curR] : Lc[curL]) + pr.xoff;
          const double2 *FX = pr.swap ? FRall + (long long)lo * nctxR : FLall + (long long)lo * nctxL;
          const double2 *Yp = (pr.swap ? Lp[curL] : Rp[curR]) + pr.yoff;
          const uint16_t *Yc = (pr.swap ? Lc[curL] : Rc[curR]) + pr.yoff;
          const double2 *FY = pr.swap ? FLall + (long long)lo * nctxL : FRall + (long long)lo * nctxR;
          const long long tc0 = clock64();
          const uint32_t y0 = yt * kYT, len = min((uint32_t)kYT, pr.nY - y0);
          // the warp's previous tile had the same pair and Y slice (the tiles of a pair go
          // X-tile fastest, so a warp's consecutive tiles often share it): already staged
          if (lo != last_lo || yt != last_yt) {
#pragma unroll
            for (int r = 0; r < kYT / 32; ++r) {
              const uint32_t jj = lane + 32 * r;
              if (jj < len) {
                DCHECK(Yc[y0 + jj] < (pr.swap ? nctxL : nctxR), "Y ctx");
                sW[jj] = cmul(Yp[y0 + jj], FY[Yc[y0 + jj]]);
              }
            }
            cm += (len + 31 - lane) / 32;
            last_lo = lo;
            last_yt = yt;
          }
          const uint32_t x0 = xt * kXT;
          double2 x[kKX];
          int nv = 0;
#pragma unroll
          for (int r = 0; r < kKX; ++r) {
            const uint32_t i = x0 + lane + 32 * r;
            if (i < pr.nX) {
              DCHECK(Xc[i] < (pr.swap ? nctxR : nctxL), "X ctx");
              x[r] = cmul(Xp[i], FX[Xc[i]]);
              ++nv;
            } else {
              x[r] = make_double2(0.0, 0.0);
            }
          }
          cm += nv;
          __syncwarp();
          const long long tc1 = clock64();
          // X slots in use: the tile's X elements rounded up to 32 lanes, then to a power of 2
          const uint32_t xs = (min((uint32_t)kXT, pr.nX - x0) + 31) / 32;
          if (xs > kKX / 2) fma_block<kKX>(x, sW, len, acc);
          else if (xs > kKX / 4) fma_block<kKX / 2>(x, sW, len, acc);
          else if (xs > kKX / 8) fma_block<kKX / 4>(x, sW, len, acc);
          else fma_block<kKX / 8>(x, sW, len, acc);
          npaths += (ull)nv * len;
          __syncwarp();
          if (lane == 0) {
            tstage += (ull)(tc1 - tc0);
            tfma += (ull)(clock64() - tc1);
          }
        }
        PHASE(sh, 5);
        __syncthreads();
        PHASE(sh, 6);
      }
    }
  }
}

__device__ void reduce_block(Shared &sh, double2 (&acc)[kKX], double2 *out, ull np, ull *np_out) {
  double re = 0.0, im = 0.0;
#pragma unroll
  for (int r = 0; r < kKX; ++r) {
    re += acc[r].x;
    im += acc[r].y;
  }
  for (int d = 16; d > 0; d >>= 1) {
    re += __shfl_down_sync(0xffffffffu, re, d);
    im += __shfl_down_sync(0xffffffffu, im, d);
    np += __shfl_down_sync(0xffffffffu, np, d);
  }
  __shared__ double rre[kThreads / 32], rim[kThreads / 32];
  __shared__ ull rnp[kThreads / 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    rre[warp] = re;
    rim[warp] = im;
    rnp[warp] = np;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, c = 0.0;
    ull n = 0;
    for (int w = 0; w < kThreads / 32; ++w) {
      a += rre[w];
      c += rim[w];
      n += rnp[w];
    }
    *out = make_double2(a, c);
    *np_out = n;
  }
  __syncthreads();
}

__device__ void load_cols(const CallParams &p, Shared &sh) {
  for (int k = threadIdx.x; k <= p.M; k += kThreads) sh.col[k] = p.col[k];
  if (threadIdx.x == 0) sh.q_cached = -1;
  __syncthreads();
}

}  // namespace

// ---- Appendix-A tables ---------------------------------------------------------------
// photons that can enter BS i: its inputs' past light cone, at most N
__device__ __forceinline__ int bs_cap(const CallParams &p, int i) {
  const BSInfo &bi = p.bsi[i];
  int c;
  if (!p.general) {
    c = (int)p.cumS[bi.cap_hi] - (int)p.cumS[bi.cap_lo];
  } else {
    c = 0;
    for (int h = 0; h < 2; ++h) {
      uint64_t m = bi.capmask[h];
      while (m) {
        const int md = 64 * h + __ffsll((long long)m) - 1;
        m &= m - 1;
        c += (int)p.cumS[md + 1] - (int)p.cumS[md];
      }
    }
  }
  return min(p.N, c);
}

__global__ void lofp_table_off_kernel(const __grid_constant__ CallParams p) {
  // one block: per-BS block sizes (past light cone of its inputs) and offsets
  __shared__ long long part[kThreads];
  const int nb = p.nbs, tid = threadIdx.x;
  const int per = (nb + kThreads - 1) / kThreads;
  const int a = tid * per, e = min(nb, a + per);
  long long s = 0;
  for (int i = a; i < e; ++i) s += tri_dev(bs_cap(p, i) + 1);
  part[tid] = s;
  __syncthreads();
  if (tid == 0) {
    long long run = 0;
    for (int i = 0; i < kThreads; ++i) {
      const long long v = part[i];
      part[i] = run;
      run += v;
    }
    p.tab_off[nb] = run;
    if (run > p.table_cap) atomicAdd(&p.ctr->table_error, 1ull);
  }
  __syncthreads();
  long long run = part[tid];
  for (int i = a; i < e; ++i) {
    p.tab_off[i] = run;
    run += tri_dev(bs_cap(p, i) + 1);
  }
  if (p.tableA) {  // the contraction's x1-linear layout: offsets by the same two-pass scan
    __syncthreads();
    s = 0;
    for (int i = a; i < e; ++i) s += lin_dev(bs_cap(p, i));
    part[tid] = s;
    __syncthreads();
    if (tid == 0) {
      long long r = 0;
      for (int i = 0; i < kThreads; ++i) {
        const long long v = part[i];
        part[i] = r;
        r += v;
      }
      p.tabA_off[nb] = r;
      if (r > p.tableA_cap) atomicAdd(&p.ctr->table_error, 1ull);
    }
    __syncthreads();
    long long r = part[tid];
    for (int i = a; i < e; ++i) {
      p.tabA_off[i] = r;
      r += lin_dev(bs_cap(p, i));
    }
  }
  // phase gates exp(i (a n + b n^2)) for n = 0..N (reading R19)
  for (int t = tid; t < p.ngate * (p.N + 1); t += kThreads) {
    const int g = t / (p.N + 1), n = t % (p.N + 1);
    const double arg = p.gate_ab[2 * g] * n + p.gate_ab[2 * g + 1] * (double)n * n;
    double sn, cs;
    sincos(arg, &sn, &cs);
    p.gate_tab[t] = make_double2(cs, sn);
  }
}

// Appendix-A elements of BS blockIdx.x for every photon number n <= cap:
// the real Wigner-type factor d_n(x1, y1) of <y1, n-y1| BS |x1, n-x1> from the four-term
// recurrence  n d_n(x, y) = sum_{i,k} sqrt(x_i y_k) u_ki d_{n-1}(x - e_i, y - e_k)  with
// u = [[c, -s], [s, c]] (reading R18), then the phase e^{i phi (x1 - y1)}
// (SURVEY A.1).  Stable to ~1e-15 at 120 photons, unlike the alternating t-sum.
__global__ void __launch_bounds__(kThreads) lofp_table_kernel(const __grid_constant__ CallParams p) {
  const int bs = blockIdx.x, tid = threadIdx.x;
  if (p.tab_off[p.nbs] > p.table_cap) return;
  const BSInfo bi = p.bsi[bs];
  const int cap = bs_cap(p, bs);
  double2 *tb = p.table + p.tab_off[bs];
  const double c = bi.c, s = bi.s;
  if (tid == 0) tb[0] = make_double2(1.0, 0.0);
  __syncthreads();
  for (int n = 1; n <= cap; ++n) {
    const double2 *prev = tb + tri_dev(n - 1);
    double2 *curr = tb + tri_dev(n);
    const double inv_n = 1.0 / n;
    for (int idx = tid; idx < (n + 1) * (n + 1); idx += kThreads) {
      const int x1 = idx / (n + 1), y1 = idx - x1 * (n + 1);
      const int x2 = n - x1, y2 = n - y1;
      double v = 0.0;
      if (x1 > 0) {  // remove a photon from input mode 1 (row x1-1 of level n-1)
        if (y1 > 0) v += sqrt((double)(x1 * y1)) * c * prev[(x1 - 1) * n + (y1 - 1)].x;
        if (y2 > 0) v += sqrt((double)(x1 * y2)) * s * prev[(x1 - 1) * n + y1].x;
      }
      if (x2 > 0) {  // remove a photon from input mode 2 (row x1 of level n-1)
        if (y1 > 0) v -= sqrt((double)(x2 * y1)) * s * prev[x1 * n + (y1 - 1)].x;
        if (y2 > 0) v += sqrt((double)(x2 * y2)) * c * prev[x1 * n + y1].x;
      }
      curr[idx] = make_double2(v * inv_n, 0.0);
    }
    __syncthreads();
  }
  // phases: <y1,y2|BS(theta,phi)|x1,x2> = e^{i phi (x1 - y1)} d; the 2 cap + 1
  // distinct phases are tabulated once (a sincos per element was most of this kernel at
  // 100 photons)
  __shared__ double2 ph[2 * kMaxPhotons + 1];
  for (int d = tid; d <= 2 * cap; d += kThreads) {
    double sn, cs;
    sincos(bi.phi * (double)(d - cap), &sn, &cs);
    ph[d] = make_double2(cs, sn);
  }
  __syncthreads();
  for (int n = 1; n <= cap; ++n) {
    double2 *curr = tb + tri_dev(n);
    for (int idx = tid; idx < (n + 1) * (n + 1); idx += kThreads) {
      const int x1 = idx / (n + 1), y1 = idx - x1 * (n + 1);
      if (x1 == y1) continue;
      const double2 e = ph[x1 - y1 + cap];
      const double d = curr[idx].x;
      curr[idx] = make_double2(d * e.x, d * e.y);
    }
  }
}

// The contraction's copy of each BS block in the x1-linear layout: element (x2, y2, x1), i.e.
// <y1, y2|BS|x1, x2> with y1 = x1 + x2 - y2, at (cap+1) R(x2) + y2 (cap+1-x2) + x1 where
// R(x2) = sum_{x' < x2} (cap+1-x') (lin_base).  A term of the contraction fixes x2 and y2 per
// entry and varies x1 with one byte of its row (lofp_contract.cu), so its index is one
// subtraction.  Elements with y1 < 0 do not exist (0; never read).
__global__ void __launch_bounds__(kThreads) lofp_tableA_kernel(const __grid_constant__ CallParams p) {
  // block (bs, x2): the run of x2, c1 (c1 - x2) entries starting at c1 R(x2) (one block per
  // BS walked to its x2 entry by entry: 1.2 ms of a 2.6 ms call at 100 photons)
  const int bs = blockIdx.x, x2 = blockIdx.y;
  if (p.tab_off[p.nbs] > p.table_cap || p.tabA_off[p.nbs] > p.tableA_cap) return;
  const int cap = bs_cap(p, bs), c1 = cap + 1;
  if (x2 > cap) return;
  const double2 *src = p.table + p.tab_off[bs];
  const int w = c1 - x2;
  double2 *dst = p.tableA + p.tabA_off[bs] + (long long)c1 * ((long long)x2 * c1 - ((long long)x2 * (x2 - 1)) / 2);
  const int tot = c1 * w;
  for (int off = threadIdx.x; off < tot; off += kThreads) {
    const int y2 = off / w, x1 = off - y2 * w;
    const int n = x1 + x2, y1 = n - y2;
    dst[off] = y1 >= 0 ? src[tri_dev(n) + (long long)x1 * (n + 1) + y1] : make_double2(0.0, 0.0);
  }
}

// ---- plan: per output, the column states and the exact path count ---------------------
__global__ void __launch_bounds__(kThreads) lofp_plan_kernel(const __grid_constant__ CallParams p) {
  __shared__ Shared sh;
  Block b = make_block(p);
  load_cols(p, sh);
  const int tid = threadIdx.x;
  for (int q = blockIdx.x; q < p.B; q += gridDim.x) {
    int st = setup_output(p, b, sh, q);
    if (st == kStatusOk) {
      dp_counts(p, b, sh, 0, 0, true);
      if (b.cR[sh.cb[0]] == 0) st = kStatusZero;
    }
    if (st == kStatusOk && p.path_budget && b.cR[sh.cb[0]] > p.path_budget) st = kStatusOverBudget;
    if (tid == 0) {
      p.pdone[q] = 0;
      p.status[q] = (uint8_t)st;
      p.pexp[q] = st == kStatusOk ? b.cR[sh.cb[0]] : 0ull;
      if (st == kStatusOk) atomicAdd(&p.ctr->feasible, 1ull);
      if (st == kStatusOverBudget) atomicAdd(&p.ctr->over_budget, 1ull);
      if (st == kStatusBad) atomicAdd(&p.ctr->bad_rows, 1ull);
      if (st == kStatusUnsupported) atomicAdd(&p.ctr->unsupported, 1ull);
    }
    __syncthreads();
  }
}

// unit size: the batch's paths spread over ~8 units per block of the unit kernel, at least
// p.thr (so small batches still split their big trees, north_star "prefixes")
__global__ void lofp_thr_kernel(const __grid_constant__ CallParams p, int grid) {
  __shared__ ull part[kThreads];
  ull s = 0;
  for (int q = threadIdx.x; q < p.B; q += kThreads) s = sat_add(s, p.pexp[q]);
  part[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    ull tot = 0;
    for (int i = 0; i < kThreads; ++i) tot = sat_add(tot, part[i]);
    ull t = tot / (ull)(p.units_per_block * grid);
    p.ctr->thr = t > p.thr ? t : p.thr;
  }
}

// split: an output above the unit size becomes the prefix subtrees (columns 0..j fixed)
// of at most that many paths, in depth-first order; every other feasible output is one unit
__global__ void __launch_bounds__(kThreads) lofp_split_kernel(const __grid_constant__ CallParams p) {
  __shared__ Shared sh;
  Block b = make_block(p);
  load_cols(p, sh);
  const int M = p.M, tid = threadIdx.x;
  for (int q = blockIdx.x; q < p.B; q += gridDim.x) {
    const int st0 = p.status[q];
    const ull P = p.pexp[q];
    Unit *U = p.units + (long long)q * p.budget;
    // root product: phase gates that no cut carries (M == 1: the single mode holds N)
    double2 root = make_double2(1.0, 0.0);
    if (M == 1)
      for (int g = 0; g < p.ngate; ++g) root = cmul(root, p.gate_tab[g * (p.N + 1) + p.N]);
    ull thr = p.ctr->thr;
    if (st0 != kStatusOk || P <= thr) {
      if (tid == 0) {
        if (st0 == kStatusOk) {
          Unit u;
          u.q = q; u.j = 0; u.sjm1 = 0; u.sj = 0; u.pad = 0; u.re = root.x; u.im = root.y; u.paths = P;
          U[0] = u;
        }
        p.nunits[q] = st0 == kStatusOk ? 1 : 0;
      }
      continue;  // (block-uniform)
    }
    setup_output(p, b, sh, q);
    dp_counts(p, b, sh, 0, 0, true);
    // Level-synchronous expansion of the prefix tree (all threads): a node (columns 0..j
    // fixed) whose subtree holds at most thr paths -- or that reached column M-1 -- becomes
    // a unit; every other node is replaced by its live, compatible children at column j+1.
    // Units are numbered level by level, in frontier order (deterministic).  If the units
    // exceed the output's slots, the unit size grows 4x and the expansion restarts; if a
    // frontier outgrows the scratch, its nodes become (larger) units.
    SplitEnt *fr[2];
    uint32_t *cnt, *off, *flag;
    long long cap;
    {
      char *q0 = (char *)(((uintptr_t)b.lists + 15) & ~(uintptr_t)15);
      cap = (b.list_bytes - 64) / (2 * (long long)sizeof(SplitEnt) + 12);
      fr[0] = (SplitEnt *)q0;
      fr[1] = fr[0] + cap;
      cnt = (uint32_t *)(fr[1] + cap);
      off = cnt + cap;
      flag = off + cap;
    }
    while (true) {
      if (tid == 0) {
        SplitEnt e;
        e.sjm1 = 0; e.sj = 0; e.re = root.x; e.im = root.y;
        fr[0][0] = e;
      }
      __syncthreads();
      uint32_t nf = 1, units = 0;
      int cur = 0;
      for (int j = 0; nf > 0; ++j) {
        const bool last = j >= M - 1;
        // children per node (0 for a unit); a unit is marked with bit 31
        for (uint32_t i = tid; i < nf; i += kThreads) {
          const SplitEnt t = fr[cur][i];
          DCHECK(j <= M && t.sj < sh.n[j] && (j == 0 || t.sjm1 < sh.n[j - 1]), "split node");
          const ull below = b.cR[sh.cb[j] + t.sj];
          uint32_t c = 0;
          if (!(below <= thr || last)) {
            const int n1 = sh.n[j + 1];
            for (int s1 = 0; s1 < n1; ++s1)
              if (live(b, sh, j + 1, s1) && compat(p, b, sh, j + 1, t.sj, s1)) ++c;
          }
          cnt[i] = c ? c : 0x80000000u;
        }
        __syncthreads();
        // units of this level: nodes with bit 31; children: the rest (scan of the low bits)
        for (uint32_t i = tid; i < nf; i += kThreads) flag[i] = cnt[i] >> 31;
        __syncthreads();
        const uint32_t nunit = block_scan_call(sh, flag, off, (int)nf);
        for (uint32_t i = tid; i < nf; i += kThreads) {
          if (!(cnt[i] >> 31)) continue;
          const uint32_t k = units + off[i];
          if (k < (uint32_t)p.budget) {
            const SplitEnt t = fr[cur][i];
            Unit u;
            u.q = q; u.j = (int16_t)j; u.sjm1 = t.sjm1; u.sj = t.sj; u.pad = 0;
            u.re = t.re; u.im = t.im; u.paths = b.cR[sh.cb[j] + t.sj];
            U[k] = u;
          }
        }
        units += nunit;
        __syncthreads();
        for (uint32_t i = tid; i < nf; i += kThreads) flag[i] = (cnt[i] >> 31) ? 0u : cnt[i];
        __syncthreads();
        const uint32_t nchild = block_scan_call(sh, flag, off, (int)nf);
        if ((long long)nchild > cap) {
          // the next frontier does not fit: the remaining nodes become units as they are
          for (uint32_t i = tid; i < nf; i += kThreads) flag[i] = (cnt[i] >> 31) ? 0u : 1u;
          __syncthreads();
          const uint32_t nrest = block_scan_call(sh, flag, off, (int)nf);
          for (uint32_t i = tid; i < nf; i += kThreads) {
            if (cnt[i] >> 31) continue;
            const uint32_t k = units + off[i];
            if (k < (uint32_t)p.budget) {
              const SplitEnt t = fr[cur][i];
              Unit u;
              u.q = q; u.j = (int16_t)j; u.sjm1 = t.sjm1; u.sj = t.sj; u.pad = 0;
              u.re = t.re; u.im = t.im; u.paths = b.cR[sh.cb[j] + t.sj];
              U[k] = u;
            }
          }
          units += nrest;
          __syncthreads();
          break;
        }
        // children in node order, states of column j+1 in increasing order
        for (uint32_t i = tid; i < nf; i += kThreads) {
          if (cnt[i] >> 31) continue;
          const SplitEnt t = fr[cur][i];
          const double2 pr = make_double2(t.re, t.im);
          uint32_t o = off[i];
          const int n1 = sh.n[j + 1];
          for (int s1 = 0; s1 < n1; ++s1) {
            if (!live(b, sh, j + 1, s1) || !compat(p, b, sh, j + 1, t.sj, s1)) continue;
            ull c2 = 0;
            const double2 np = cmul(pr, cut_factor(p, b, sh, j, t.sjm1, t.sj, s1, c2));
            SplitEnt e;
            e.sjm1 = t.sj; e.sj = (uint16_t)s1; e.re = np.x; e.im = np.y;
            DCHECK(o < nchild && (long long)o < cap, "split child");
            fr[cur ^ 1][o++] = e;
          }
        }
        __syncthreads();
        nf = nchild;
        cur ^= 1;
      }
      if (units <= (uint32_t)p.budget) {
        if (tid == 0) p.nunits[q] = (int)units;
        break;
      }
      thr = thr > (~0ull >> 2) ? ~0ull : thr * 4;  // too many units for the slots: coarser
      __syncthreads();
    }
    __syncthreads();
  }
}

// slot of unit u: output q = the last with ubase[q] <= u (ubase[B] = the unit count)
__device__ __forceinline__ long long unit_slot(const CallParams &p, int u) {
  int lo = 0, hi = p.B - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (p.ubase[mid] <= u) lo = mid; else hi = mid - 1;
  }
  return (long long)lo * p.budget + (u - p.ubase[lo]);
}

// exclusive scan of nunits -> ubase, total -> ctr->total_units; then the schedule: units
// by decreasing size class (floor log2 of their path count), largest first (one block)
__global__ void lofp_scan_kernel(const __grid_constant__ CallParams p) {
  __shared__ long long part[kThreads];
  __shared__ unsigned int hist[65], base[65];
  const int B = p.B, tid = threadIdx.x;
  const int per = (B + kThreads - 1) / kThreads;
  const int a = tid * per, e = min(B, a + per);
  long long s = 0;
  for (int i = a; i < e; ++i) s += p.nunits[i];
  part[tid] = s;
  if (tid < 65) hist[tid] = 0;
  __syncthreads();
  if (tid == 0) {
    long long run = 0;
    for (int i = 0; i < kThreads; ++i) {
      const long long v = part[i];
      part[i] = run;
      run += v;
    }
    p.ubase[B] = (int)run;
    p.ctr->total_units = (ull)run;
  }
  __syncthreads();
  long long run = part[tid];
  for (int i = a; i < e; ++i) {
    p.ubase[i] = (int)run;
    run += p.nunits[i];
  }
  __syncthreads();
  const int U = (int)p.ctr->total_units;
  // size class of every unit (unit u of output q is slot q*budget + u - ubase[q]); threads
  // over the units, so that one output split into thousands of units is not one thread's
  for (int u = tid; u < U; u += kThreads) {
    const ull P = p.units[unit_slot(p, u)].paths;
    atomicAdd(&hist[64 - (P ? 64 - __clzll(P) : 0)], 1u);
  }
  __syncthreads();
  if (tid == 0) {
    unsigned int r = 0;
    for (int c = 0; c < 65; ++c) {
      base[c] = r;
      r += hist[c];
    }
  }
  __syncthreads();
  for (int u = tid; u < U; u += kThreads) {
    const ull P = p.units[unit_slot(p, u)].paths;
    const unsigned int pos = atomicAdd(&base[64 - (P ? 64 - __clzll(P) : 0)], 1u);
    if ((int)pos < U) p.sched[pos] = u;
  }
}

// ---- the hot path ----------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads, 2) lofp_units_kernel(const __grid_constant__ CallParams p) {
  __shared__ Shared sh;
  extern __shared__ double2 sY[];
  Block b = make_block(p);
  load_cols(p, sh);
  const int tid = threadIdx.x;
  ull cm = 0, nelem = 0, tstage = 0, tfma = 0;
  if (tid == 0) {
    for (int i = 0; i < 8; ++i) sh.ph[i] = 0;
    sh.tph = clock64();
  }
  while (true) {
    if (tid == 0) sh.unit = (int)atomicAdd(&p.ctr->ticket, 1ull);
    __syncthreads();
    const int k_ = sh.unit;
    if ((ull)k_ >= p.ctr->total_units) break;
#ifdef LOFP_UNIT_CLOCKS
    const long long uc0 = clock64();
#endif
    const int u = p.sched[k_];
    DCHECK(u >= 0 && u < (int)p.ctr->total_units, "sched");
    // unit u -> output q (binary search over ubase) -> slot
    int lo = 0, hi = p.B - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (p.ubase[mid] <= u) lo = mid; else hi = mid - 1;
    }
    const int q = lo;
    DCHECK(u - p.ubase[q] >= 0 && u - p.ubase[q] < p.nunits[q] && p.nunits[q] <= p.budget, "unit slot");
    const Unit un = p.units[(long long)q * p.budget + (u - p.ubase[q])];
    if (sh.q_cached != q) {
      const int st = setup_output(p, b, sh, q);
      if (st != kStatusOk) {  // cannot happen: units exist only for feasible outputs
        if (tid == 0) {
          atomicAdd(&p.ctr->table_error, 1ull);
          p.partial[u] = make_double2(0.0, 0.0);
        }
        __syncthreads();
        continue;
      }
      if (tid == 0) sh.q_cached = q;
    } else {
      carve(p, b, sh);  // columns of q are still in the slab from an earlier unit
    }
    if (tid == 0) {
      StackEnt e;
      e.j = un.j; e.sjm1 = un.sjm1; e.sj = un.sj; e.re = un.re; e.im = un.im; e.pad = 0;
      b.stack[0] = e;
      sh.sp = 1;
    }
    __syncthreads();
    double2 acc[kKX];
#pragma unroll
    for (int r = 0; r < kKX; ++r) acc[r] = make_double2(0.0, 0.0);
    ull np = 0;
    process_stack(p, b, sh, sY, acc, np, cm, nelem, tstage, tfma);
    ull np_tot = 0;
    reduce_block(sh, acc, &p.partial[u], np, &np_tot);
#ifdef LOFP_UNIT_CLOCKS  // experiment (scripts/unit_clocks.py): the unit's partial replaced by
                         // (its SM clocks + block / 1024, its end time in ns)
    __syncthreads();
    if (tid == 0) {
      unsigned long long gt;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
      p.partial[u] = make_double2((double)(clock64() - uc0) + blockIdx.x / 1024.0, (double)gt);
    }
    __syncthreads();
#endif
    if (tid == 0) {
      atomicAdd(&p.pdone[q], np_tot);
      atomicAdd(&p.ctr->paths, np_tot);
      atomicAdd(&p.ctr->units, 1ull);
    }
  }
  // statistics
  PHASE(sh, 0);
  if (tid == 0)
    for (int i = 0; i < 8; ++i) atomicAdd(&p.ctr->phase[i], sh.ph[i]);
  for (int d = 16; d > 0; d >>= 1) {
    cm += __shfl_down_sync(0xffffffffu, cm, d);
    nelem += __shfl_down_sync(0xffffffffu, nelem, d);
  }
  if ((tid & 31) == 0) {
    atomicAdd(&p.ctr->cmuls, cm);
    atomicAdd(&p.ctr->elements, nelem);
    atomicAdd(&p.ctr->tile_stage, tstage);
    atomicAdd(&p.ctr->tile_fma, tfma);
  }
}

// per output: the sum of its units (a warp per output: lane-strided partial sums in unit
// order, then a fixed shuffle tree -- deterministic), exact 0 / NaN otherwise
__global__ void lofp_final_kernel(const __grid_constant__ CallParams p) {
  const int lane = threadIdx.x & 31;
  const int w0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (int q = w0; q < p.B; q += nw) {
    const int st = p.status[q];
    double2 a = make_double2(0.0, 0.0);
    if (st == kStatusOk)
      for (int u = p.ubase[q] + lane; u < p.ubase[q + 1]; u += 32) {
        const double2 v = p.partial[u];
        a.x += v.x;
        a.y += v.y;
      }
    for (int d = 16; d > 0; d >>= 1) {
      a.x += __shfl_down_sync(0xffffffffu, a.x, d);
      a.y += __shfl_down_sync(0xffffffffu, a.y, d);
    }
    if (lane == 0) {
      if (st == kStatusOk) {
        if (p.pdone[q] != p.pexp[q]) atomicAdd(&p.ctr->table_error, 1ull);  // every path exactly once
      } else if (st == kStatusBad || st == kStatusUnsupported || st == kStatusOverBudget) {
        a = make_double2(__longlong_as_double(0x7ff8000000000000ll), __longlong_as_double(0x7ff8000000000000ll));
      } else {
        a = make_double2(0.0, 0.0);
      }
      p.amps[q] = a;
      if (p.counts) p.counts[q] = p.pdone[q];
    }
  }
}

__global__ void __launch_bounds__(kThreads) lofp_generic_kernel(const __grid_constant__ CallParams p);

// ---- launchers -------------------------------------------------------------------------
extern "C" int lofp_units_grid(int device) {
  int nsm = 0;
  if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return -1;
  return 2 * nsm;
}

extern "C" int lofp_launch_tables(const CallParams *p, void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  lofp_table_off_kernel<<<1, kThreads, 0, st>>>(*p);
  if (p->nbs > 0) lofp_table_kernel<<<p->nbs, kThreads, 0, st>>>(*p);
  return (int)cudaGetLastError();
}

extern "C" int lofp_launch_paths(const CallParams *p, int grid, void *stream, void *ev0, void *ev1) {
  cudaStream_t st = (cudaStream_t)stream;
  const int smem = kCY * (int)sizeof(double2);
  static int attr_device_mask = 0;  // set once per device, outside any stream capture
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(attr_device_mask & (1 << (dev & 31)))) {
    cudaFuncSetAttribute(lofp_units_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr_device_mask |= 1 << (dev & 31);
  }
  const int pgrid = p->B < grid ? p->B : grid;
#define LOFP_CHECK_STEP(name)                                                                  \
  if (getenv("LOFP_SYNC_EACH")) {                                                              \
    const cudaError_t e_ = cudaStreamSynchronize(st);                                          \
    if (e_ != cudaSuccess) {                                                                   \
      fprintf(stderr, "liblofp: %s failed: %s\n", name, cudaGetErrorString(e_));               \
      return (int)e_;                                                                          \
    }                                                                                          \
  }
  lofp_plan_kernel<<<pgrid, kThreads, 0, st>>>(*p);
  LOFP_CHECK_STEP("plan")
  lofp_thr_kernel<<<1, kThreads, 0, st>>>(*p, grid);
  lofp_split_kernel<<<pgrid, kThreads, 0, st>>>(*p);
  LOFP_CHECK_STEP("split")
  lofp_scan_kernel<<<1, kThreads, 0, st>>>(*p);
  LOFP_CHECK_STEP("scan")
  if (ev0) cudaEventRecord((cudaEvent_t)ev0, st);
  lofp_units_kernel<<<grid, kThreads, smem, st>>>(*p);
  if (ev1) cudaEventRecord((cudaEvent_t)ev1, st);
  LOFP_CHECK_STEP("units")
  lofp_final_kernel<<<(p->B + 7) / 8 < 1184 ? (p->B + 7) / 8 : 1184, 256, 0, st>>>(*p);  // a warp per output
  LOFP_CHECK_STEP("final")
  lofp_generic_kernel<<<grid, kThreads, 0, st>>>(*p);  // outputs over the column limits
  return (int)cudaGetLastError();
}

// ---- NEXT-1: the strip tensor contraction --------------------------------
// The paper contracts the circuit block by block from top to bottom, storing for every
// tuple l_{k,j} of occupation numbers crossing from block C_k to C_{k+1} its partial
// amplitude.  Here the blocks are the cuts: the state crossing cut k is the
// column pair (c_{k-1}, c_k) (the photon counts left of the cut over all layers), and
//   A_{k+1}(c_k, c_{k+1}) = sum_{c_{k-1}} A_k(c_{k-1}, c_k) f_k(c_{k-1}, c_k, c_{k+1})
// with f_k the cut factor (the BS of cut k, eq. (1)); the amplitude is the sum of the last
// level ("the last contraction block ... gives us the wanted amplitude").  Only
// light-cone-live states are carried ("upper bounds ... using the light cones").
__global__ void __launch_bounds__(kThreads) lofp_contract_kernel(const __grid_constant__ CallParams p) {
  __shared__ Shared sh;
  __shared__ double red_re[kThreads / 32], red_im[kThreads / 32];
  if (p.deferred_only && p.ctr->cdeferred == 0) return;  // the warp kernel did every output
  Block b = make_block(p);
  load_cols(p, sh);
  const int M = p.M, tid = threadIdx.x;
  ull cm = 0, terms = 0;
  for (int q = blockIdx.x; q < p.B; q += gridDim.x) {
    if (p.deferred_only && p.status[q] != kStatusDeferred) continue;  // done by the warp kernel (uniform)
    int st = setup_output(p, b, sh, q);
    const bool with_counts = p.counts != nullptr;
    if (st == kStatusOk && with_counts) {
      dp_counts(p, b, sh, 0, 0, true, false);  // completions: the exact path count, and pruning
      if (b.cR[sh.cb[0]] == 0) st = kStatusZero;
    }
    long long need = 0;
    if (st == kStatusOk)
      for (int k = 1; k <= M; ++k) need = max(need, (long long)sh.n[k - 1] * sh.n[k]);
    if (st == kStatusOk && 2 * 16 * need > b.list_bytes) st = kStatusUnsupported;
    double re = 0.0, im = 0.0;
    if (st == kStatusOk) {
      double2 *A = (double2 *)b.lists, *Bn = A + need;
      // level 1: the pair (c_0, c_1), c_0 the single state of column 0
      double2 root = make_double2(1.0, 0.0);
      if (M == 1)
        for (int g = 0; g < p.ngate; ++g) root = cmul(root, p.gate_tab[g * (p.N + 1) + p.N]);
      // nz[s] == k+1: state s of column k+1 has a nonzero entry in the level being built
      // (generation stamps: no clearing; two arrays alternate between the columns)
      uint32_t *nzc = b.tmp, *nzn = b.tmp2;
      for (int s = tid; s < kMaxStates; s += kThreads) nzc[s] = 0u;
      __syncthreads();
      for (int s1 = tid; s1 < sh.n[1]; s1 += kThreads) {
        const bool on = (!with_counts || b.cR[sh.cb[1] + s1] != 0) && compat(p, b, sh, 1, 0, s1);
        A[s1] = on ? root : make_double2(0.0, 0.0);
        nzc[s1] = on ? 1u : 0u;
      }
      for (int s = tid; s < kMaxStates; s += kThreads) nzn[s] = 0u;
      __syncthreads();
      for (int k = 1; k <= M - 1; ++k) {  // contract cut k: level (k-1, k) -> (k, k+1)
        const int nA = sh.n[k - 1], nB = sh.n[k], nC = sh.n[k + 1];
        for (int t = tid; t < nB * nC; t += kThreads) {
          const int sb = t / nC, sc = t - sb * nC;
          double2 sum = make_double2(0.0, 0.0);
          if (nzc[sb] == (uint32_t)k && (!with_counts || b.cR[sh.cb[k + 1] + sc] != 0) &&
              compat(p, b, sh, k + 1, sb, sc)) {
            for (int sa = 0; sa < nA; ++sa) {
              const double2 a = A[sa * nB + sb];
              if (a.x == 0.0 && a.y == 0.0) continue;
              const double2 f = cut_factor(p, b, sh, k, sa, sb, sc, cm);
              sum.x = fma(a.x, f.x, fma(-a.y, f.y, sum.x));
              sum.y = fma(a.x, f.y, fma(a.y, f.x, sum.y));
              ++terms;
            }
          }
          Bn[t] = sum;
          if (sum.x != 0.0 || sum.y != 0.0) nzn[sc] = (uint32_t)(k + 1);  // (same value from all writers)
        }
        __syncthreads();
        double2 *tt = A; A = Bn; Bn = tt;
        uint32_t *tz = nzc; nzc = nzn; nzn = tz;
      }
      // the last level (c_{M-1}, c_M): its sum is the amplitude
      const int nL = sh.n[M - 1] * sh.n[M];
      for (int t = tid; t < nL; t += kThreads) {
        re += A[t].x;
        im += A[t].y;
      }
    }
    // fixed-order block reduction (deterministic)
    for (int d = 16; d > 0; d >>= 1) {
      re += __shfl_down_sync(0xffffffffu, re, d);
      im += __shfl_down_sync(0xffffffffu, im, d);
    }
    if ((tid & 31) == 0) {
      red_re[tid >> 5] = re;
      red_im[tid >> 5] = im;
    }
    __syncthreads();
    if (tid == 0) {
      double2 a = make_double2(0.0, 0.0);
      for (int w = 0; w < kThreads / 32; ++w) {
        a.x += red_re[w];
        a.y += red_im[w];
      }
      if (st == kStatusBad || st == kStatusUnsupported)
        a = make_double2(__longlong_as_double(0x7ff8000000000000ll), __longlong_as_double(0x7ff8000000000000ll));
      p.amps[q] = a;
      p.status[q] = (uint8_t)st;
      if (with_counts) p.counts[q] = st == kStatusOk ? b.cR[sh.cb[0]] : 0ull;
      if (st == kStatusOk) atomicAdd(&p.ctr->feasible, 1ull);
      if (st == kStatusBad) atomicAdd(&p.ctr->bad_rows, 1ull);
      if (st == kStatusUnsupported) atomicAdd(&p.ctr->unsupported, 1ull);
    }
    __syncthreads();
  }
  for (int d = 16; d > 0; d >>= 1) {
    cm += __shfl_down_sync(0xffffffffu, cm, d);
    terms += __shfl_down_sync(0xffffffffu, terms, d);
  }
  if ((tid & 31) == 0) {
    atomicAdd(&p.ctr->cmuls, cm);
    atomicAdd(&p.ctr->contractions, terms);
  }
}

extern "C" int lofp_launch_contract(const CallParams *p, int grid, void *stream) {
  const int g = p->B < grid ? p->B : grid;
  CallParams q = *p;
  // nearest-neighbour circuits: one warp per output first (lofp_contract.cu); this block
  // kernel then takes only the outputs it deferred (state spaces over the warp limits)
  q.deferred_only = 0;
  if (!p->general && !p->force_generic && !p->contract_block_only && p->tableA) {
    if (p->nbs > 0) lofp_tableA_kernel<<<dim3(p->nbs, p->N + 1), kThreads, 0, (cudaStream_t)stream>>>(*p);
    const int e = lofp_launch_contract_warp(p, grid, stream);
    if (e > 0) return e;
    q.deferred_only = e == 0 ? 1 : 0;  // (-1: not launched, the block kernel takes every output)
  }
  lofp_contract_kernel<<<g, kThreads, 0, (cudaStream_t)stream>>>(q);
  lofp_generic_kernel<<<grid, kThreads, 0, (cudaStream_t)stream>>>(*p);  // outputs over the column limits
  return (int)cudaGetLastError();
}

// ---- NEXT-2: every output pattern of N photons in M modes ----------------------
// Pattern r (0 <= r < C(N+M-1, M-1)) in the order of decreasing T_0, then decreasing T_1,
// ...: unranked independently per thread from the binomial counts of the suffixes.
__global__ void lofp_outputs_kernel(int M, int N, long long count, int32_t *T) {
  for (long long r0 = blockIdx.x * (long long)blockDim.x + threadIdx.x; r0 < count;
       r0 += (long long)gridDim.x * blockDim.x) {
    ull r = (ull)r0;
    int rem = N;
    int32_t *row = T + r0 * M;
    for (int i = 0; i < M - 1; ++i) {
      // patterns of the remaining m + 1 modes holding rem - v photons: c = C(rem - v + m, m),
      // stepped with v by C(n + 1, m) = C(n, m) (n + 1) / (n + 1 - m) (exact; one division per
      // step instead of m: the kernel was 10 % of the distribution call)
      const int m = M - i - 2;
      int v = rem, n = m;
      ull c = 1;
      for (; v > 0; --v) {
        if (r < c) break;
        r -= c;
        c = c * (ull)(n + 1) / (ull)(n + 1 - m);
        ++n;
      }
      row[i] = v;
      rem -= v;
    }
    row[M - 1] = rem;
  }
}

extern "C" int lofp_launch_outputs(int M, int N, long long count, int32_t *T, void *stream) {
  const long long blocks = (count + 255) / 256;
  lofp_outputs_kernel<<<(int)(blocks < 4096 ? (blocks > 0 ? blocks : 1) : 4096), 256, 0, (cudaStream_t)stream>>>(
      M, N, count, T);
  return (int)cudaGetLastError();
}

// ---- the generic engine: the paper's own recursion ------------------
// For any output the column model cannot hold (a non-local circuit whose columns exceed the
// state limits, or any over-limit output): the path tree in the paper's order, BS by BS in
// layer-major order, each BS choosing y1 within the waveguides' light-cone bounds (P:164:
// photons in a waveguide <= min(sum of S over its past cone, sum of T over its future
// cone)); a leaf is a valid path iff it lands on T.  One block per output: the tree is
// expanded breadth-first into >= 4 prefixes per thread (the north_star's prefix split), then
// every thread walks its prefixes depth-first with an explicit stack (fixed order: the sum
// is deterministic).
namespace {

constexpr int kGenMaxBS = 1024;      // levels of the generic tree (BS count)
constexpr int kGenFront = 8192;      // frontier entries of the prefix split
constexpr ull kGenNodeBudget = 1ull << 22;  // tree nodes per thread before an output is given up (~5 s)

struct GenEntry {
  double re, im;
  int32_t level;
  int32_t pad;
};

__device__ __forceinline__ double2 gen_gates(const CallParams &p, int l0, int l1, const uint8_t *occ) {
  double2 f = make_double2(1.0, 0.0);
  if (p.ngate == 0 || l0 >= l1) return f;
  for (int g = 0; g < p.ngate; ++g) {
    const int a = p.gate_after[g];
    if (a >= l0 && a < l1) f = cmul(f, p.gate_tab[g * (p.N + 1) + occ[p.gate_mode[g]]]);
  }
  return f;
}

__device__ __forceinline__ void gen_range(const CallParams &p, const uint8_t *bnd, const SeqBS &s, const uint8_t *occ,
                                          int &ylo, int &yhi) {
  const int M = p.M, n = occ[s.lo] + occ[s.hi];
  const int ba = bnd[s.layer * M + s.lo], bb = bnd[s.layer * M + s.hi];
  ylo = max(0, n - bb);
  yhi = min(n, ba);
}

}  // namespace

__global__ void __launch_bounds__(kThreads) lofp_generic_kernel(const __grid_constant__ CallParams p) {
  __shared__ uint8_t bnd[(kMaxLayers + 1) * kMaxModes];
  __shared__ int sT[kMaxModes];
  __shared__ double rre[kThreads / 32], rim[kThreads / 32];
  __shared__ ull rnp[kThreads / 32];
  __shared__ int s_front, s_level, s_done;
  const int M = p.M, D = p.D, L = p.nbs, tid = threadIdx.x;
  // no output over the column limits (an unsupported output keeps the counter above 0
  // until this kernel evaluates it)
  if (p.ctr->unsupported == 0) return;
  char *slab = p.slab + (long long)blockIdx.x * p.slab_bytes;
  GenEntry *fe[2] = {(GenEntry *)slab, (GenEntry *)slab + kGenFront};
  uint8_t *fo[2] = {(uint8_t *)((GenEntry *)slab + 2 * kGenFront),
                    (uint8_t *)((GenEntry *)slab + 2 * kGenFront) + (long long)kGenFront * M};
  // per-thread DFS state (occupations + stack) after the frontier
  char *tstate = (char *)(fo[1] + (long long)kGenFront * M);
  tstate = (char *)(((uintptr_t)tstate + 15) & ~(uintptr_t)15);
  const long long per_thread = (24ll * L + M + 64 + 15) & ~15ll;
  uint8_t *occ = (uint8_t *)(tstate + per_thread * tid);
  double2 *prodst = (double2 *)(((uintptr_t)(occ + M) + 15) & ~(uintptr_t)15);
  int16_t *yst = (int16_t *)(prodst + L + 1);  // y1 chosen per level
  int16_t *yhs = yst + L;                        // its upper end
  ull cm = 0;
  for (int q = blockIdx.x; q < p.B; q += gridDim.x) {
    if (p.status[q] != kStatusUnsupported || L > kGenMaxBS || D > kMaxLayers ||
        (long long)(2 * kGenFront) * (16 + M) + per_thread * kThreads + 64 > p.slab_bytes)
      continue;  // (block-uniform)
    for (int i = tid; i < M; i += kThreads) sT[i] = p.T[(long long)q * M + i];
    __syncthreads();
    // light-cone bounds of every waveguide (mode m after layer t)
    for (int w = tid; w < (D + 1) * M; w += kThreads) {
      const uint64_t *c = p.cone + 4ll * w;
      int ps = 0, ft = 0;
      for (int h = 0; h < 2; ++h) {
        uint64_t m = c[h];
        while (m) {
          const int md = 64 * h + __ffsll((long long)m) - 1;
          m &= m - 1;
          ps += (int)p.cumS[md + 1] - (int)p.cumS[md];
        }
        m = c[2 + h];
        while (m) {
          const int md = 64 * h + __ffsll((long long)m) - 1;
          m &= m - 1;
          ft += sT[md];
        }
      }
      bnd[w] = (uint8_t)min(255, min(ps, ft));
    }
    // root
    if (tid == 0) {
      for (int m = 0; m < M; ++m) fo[0][m] = (uint8_t)((int)p.cumS[m + 1] - (int)p.cumS[m]);
      const double2 g = gen_gates(p, 0, p.seq_gl0, fo[0]);
      fe[0][0].re = g.x;
      fe[0][0].im = g.y;
      fe[0][0].level = 0;
      s_front = 1;
      s_level = 0;
    }
    __syncthreads();
    // breadth-first prefix split until every thread has ~4 prefixes (or the tree ends)
    int cur = 0;
    while (s_front < 4 * kThreads && s_level < L) {
      const int nf = s_front, lev = s_level;
      const SeqBS sb = p.seq[lev];
      // count children per entry (thread 0: the frontier is small)
      if (tid == 0) {
        int tot = 0;
        for (int e = 0; e < nf; ++e) {
          int ylo, yhi;
          gen_range(p, bnd, sb, fo[cur] + (long long)e * M, ylo, yhi);
          tot += max(0, yhi - ylo + 1);
        }
        s_done = tot;
      }
      __syncthreads();
      if (s_done > kGenFront || s_done == 0) break;  // (uniform)
      if (tid == 0) {
        int o = 0;
        for (int e = 0; e < nf; ++e) {
          const uint8_t *src = fo[cur] + (long long)e * M;
          int ylo, yhi;
          gen_range(p, bnd, sb, src, ylo, yhi);
          const int x1 = src[sb.lo], x2 = src[sb.hi], n = x1 + x2;
          for (int y1 = ylo; y1 <= yhi; ++y1) {
            uint8_t *dst = fo[cur ^ 1] + (long long)o * M;
            for (int m = 0; m < M; ++m) dst[m] = src[m];
            dst[sb.lo] = (uint8_t)y1;
            dst[sb.hi] = (uint8_t)(n - y1);
            double2 f = make_double2(1.0, 0.0);
            if (n > 0) {
              f = p.table[p.tab_off[sb.bs] + tri_dev(n) + (long long)x1 * (n + 1) + y1];
              ++cm;
            }
            double2 pr = cmul(make_double2(fe[cur][e].re, fe[cur][e].im), f);
            pr = cmul(pr, gen_gates(p, sb.gl0, sb.gl1, dst));
            fe[cur ^ 1][o].re = pr.x;
            fe[cur ^ 1][o].im = pr.y;
            fe[cur ^ 1][o].level = lev + 1;
            ++o;
          }
        }
        s_front = o;
        s_level = lev + 1;
      }
      __syncthreads();
      cur ^= 1;
    }
    // depth-first walk of every prefix
    double are = 0.0, aim = 0.0;
    ull np = 0, nodes = 0;
    bool over = false;
    const int nf = s_front;
    for (int e = tid; e < nf && !over; e += kThreads) {
      for (int m = 0; m < M; ++m) occ[m] = fo[cur][(long long)e * M + m];
      const int l0 = fe[cur][e].level;
      prodst[l0] = make_double2(fe[cur][e].re, fe[cur][e].im);
      int lev = l0;
      bool down = true;  // entering level lev fresh
      while (true) {
        if (lev == L) {  // leaf: a valid path iff it lands on T
          bool ok = true;
          for (int m = 0; m < M; ++m) ok &= (occ[m] == sT[m]);
          if (ok) {
            are += prodst[L].x;
            aim += prodst[L].y;
            ++np;
          }
          --lev;
          down = false;
          if (lev < l0) break;
        }
        const SeqBS sb = p.seq[lev];
        if (++nodes > kGenNodeBudget) {  // keep the GPU responsive: give the output up (NaN)
          over = true;
          break;
        }
        int y1;
        if (down) {
          int ylo, yhi;
          gen_range(p, bnd, sb, occ, ylo, yhi);
          if (ylo > yhi) {  // dead end
            --lev;
            down = false;
            if (lev < l0) break;
            continue;
          }
          yst[lev] = (int16_t)(occ[sb.lo] + occ[sb.hi]);  // n, kept with y1 below
          yhs[lev] = (int16_t)yhi;
          y1 = ylo;
          // remember x1 in the high byte of yst (n <= 240, x1 <= 120)
          yst[lev] = (int16_t)(yst[lev] | (occ[sb.lo] << 8));
        } else {
          y1 = occ[sb.lo] + 1;  // next choice
          if (y1 > yhs[lev]) {  // exhausted: restore the inputs and go up
            const int n = yst[lev] & 0xff, x1 = (yst[lev] >> 8) & 0xff;
            occ[sb.lo] = (uint8_t)x1;
            occ[sb.hi] = (uint8_t)(n - x1);
            --lev;
            if (lev < l0) break;
            continue;
          }
        }
        const int n = yst[lev] & 0xff, x1 = (yst[lev] >> 8) & 0xff;
        occ[sb.lo] = (uint8_t)y1;
        occ[sb.hi] = (uint8_t)(n - y1);
        double2 f = make_double2(1.0, 0.0);
        if (n > 0) {
          f = p.table[p.tab_off[sb.bs] + tri_dev(n) + (long long)x1 * (n + 1) + y1];
          ++cm;
        }
        double2 pr = cmul(prodst[lev], f);
        if (sb.gl1 > sb.gl0) pr = cmul(pr, gen_gates(p, sb.gl0, sb.gl1, occ));
        prodst[lev + 1] = pr;
        ++lev;
        down = true;
      }
    }
    // deterministic block reduction
    const int any_over = __syncthreads_or(over ? 1 : 0);
    for (int d = 16; d > 0; d >>= 1) {
      are += __shfl_down_sync(0xffffffffu, are, d);
      aim += __shfl_down_sync(0xffffffffu, aim, d);
      np += __shfl_down_sync(0xffffffffu, np, d);
    }
    if ((tid & 31) == 0) {
      rre[tid >> 5] = are;
      rim[tid >> 5] = aim;
      rnp[tid >> 5] = np;
    }
    __syncthreads();
    if (tid == 0 && !any_over) {
      double a = 0.0, b2 = 0.0;
      ull n = 0;
      for (int w = 0; w < kThreads / 32; ++w) {
        a += rre[w];
        b2 += rim[w];
        n += rnp[w];
      }
      p.amps[q] = make_double2(a, b2);
      if (p.counts) p.counts[q] = n;
      p.status[q] = kStatusOk;
      atomicAdd(&p.ctr->paths, n);
      atomicAdd(&p.ctr->generic, 1ull);
      atomicAdd(&p.ctr->unsupported, ~0ull);  // (-1: the output is evaluated after all)
    }
    __syncthreads();
  }
  for (int d = 16; d > 0; d >>= 1) cm += __shfl_down_sync(0xffffffffu, cm, d);
  if ((tid & 31) == 0) atomicAdd(&p.ctr->cmuls, cm);
}

extern "C" int lofp_launch_generic(const CallParams *p, int grid, void *stream) {
  lofp_generic_kernel<<<grid, kThreads, 0, (cudaStream_t)stream>>>(*p);
  return (int)cudaGetLastError();
}
