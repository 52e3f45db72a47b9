// lofp_kernels.cu — sm_100a kernels of the LOFP path sum (arXiv 2510.26408).
//
//   lofp_prep_kernel   per output row: validity, photon number, per-mode max of T.
//   lofp_table_kernel  Appendix-A BS elements for every (x1, x2, y1) inside
//                      the paper's light-cone caps, fp64.
//   lofp_plan_kernel   per output: G = cum(T), exact light-cone reachability (reading
//                      R5), the output's DFS levels (free "green" waveguides)
//                      and attached factors, and the product of the constant factors.
//   lofp_enum_kernel   persistent path enumeration (eq. (1)): one warp per work
//                      item (a subtree of one output), one iterative DFS per lane over
//                      the item's levels with its state in shared memory, fp64 complex
//                      products of Appendix-A factors staged in shared memory, subtrees
//                      handed between lanes of a warp (shared memory) and between warps
//                      (a global atomic work queue); warp-shuffle reduction per item.
//
// The arithmetic follows the paper; the data layout is described in lofp_internal.h
// and DESIGN.md.  No code here is shared with oracle/.
#include <cuda_runtime.h>
#include <stdint.h>

#include "lofp_internal.h"

namespace {

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  // (a.x + i a.y)(b.x + i b.y): 2 DMUL + 2 DFMA
  double2 r;
  r.x = fma(a.x, b.x, -a.y * b.y);
  r.y = fma(a.x, b.y, a.y * b.x);
  return r;
}

// ---------------------------------------------------------------------------
// prep: row validity, photon number, per-mode max of T over the batch
// ---------------------------------------------------------------------------
__global__ void lofp_prep_kernel(CallArgs a) {
  int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= a.B) return;
  const int32_t *t = a.T + q * a.M;
  int sum = 0, bad = 0;
  for (int m = 0; m < a.M; ++m) {
    int v = t[m];
    if (v < 0) bad = 1;
    sum += v;
  }
  uint8_t f = 0;
  if (bad) {
    f = 2;
    atomicAdd(&a.ctr->bad_rows, 1ull);
  } else if (sum == a.N) {
    f = 1;
    for (int m = 0; m < a.M; ++m) {
      int v = t[m];
      if (v > 0) atomicMax(&a.ctr->tmax[m], v);
    }
  }
  a.flags[q] = f;
  const double nan = __longlong_as_double(0x7ff8000000000000ll);
  a.amps[2 * q] = bad ? nan : 0.0;
  a.amps[2 * q + 1] = bad ? nan : 0.0;
  if (a.counts) a.counts[q] = 0;
}

// ---------------------------------------------------------------------------
// Appendix A: <y1,y2|BS|x1,x2> = e^{i phi (x1 - y1)} sqrt(x1! x2! y1! y2!)
//   * sum_t (-1)^{y1-t} c^{x2-y1+2t} s^{x1+y1-2t} / (t! (y1-t)! (x1-t)! (x2-y1+t)!)
// with max(0, y1-x2, x1-y2) <= t <= min(x1, y1).  This is the paper's t-sum
// (factorial read as (x2-y1+t)!, reading R1) with U11 = U22 = c,
// U12 = -e^{-i phi} s, U21 = e^{i phi} s substituted (eq. bs_matrix).
// ---------------------------------------------------------------------------
__device__ double dfact(int n) {
  double f = 1.0;
  for (int i = 2; i <= n; ++i) f *= (double)i;
  return f;
}

__device__ double ipow(double x, int n) {  // x^n, n >= 0, 0^0 = 1
  double r = 1.0;
  for (int i = 0; i < n; ++i) r *= x;
  return r;
}

__global__ void lofp_table_kernel(CallArgs a) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.nentries) return;
  EntryDesc e = a.edesc[i];
  const double *cs = a.bs_cs + 4 * e.bs;
  double c = cs[0], s = cs[1], cph = cs[2], sph = cs[3];
  int x1 = e.x1, x2 = e.x2, y1 = e.y1, y2 = x1 + x2 - y1;
  int tlo = max(0, max(y1 - x2, x1 - y2)), thi = min(x1, y1);
  double sum = 0.0;
  for (int t = tlo; t <= thi; ++t) {
    double term = ipow(c, x2 - y1 + 2 * t) * ipow(s, x1 + y1 - 2 * t) /
                  (dfact(t) * dfact(y1 - t) * dfact(x1 - t) * dfact(x2 - y1 + t));
    sum += ((y1 - t) & 1) ? -term : term;
  }
  double d = sum * sqrt(dfact(x1) * dfact(x2) * dfact(y1) * dfact(y2));
  // phase e^{i phi (x1 - y1)} by repeated multiplication of (cos phi, sin phi)
  int k = x1 - y1;
  double pr = 1.0, pi = 0.0;
  double sgn = k < 0 ? -1.0 : 1.0;
  for (int j = 0; j < (k < 0 ? -k : k); ++j) {
    double nr = pr * cph - pi * (sgn * sph);
    double ni = pr * (sgn * sph) + pi * cph;
    pr = nr;
    pi = ni;
  }
  a.entries[2 * i] = d * pr;
  a.entries[2 * i + 1] = d * pi;
}

// ---------------------------------------------------------------------------
// plan: per output, levels + attached factors + root product
// ---------------------------------------------------------------------------
// A reference to F_t(k) while sweeping the layers: a level slot, or a constant.
struct Ref {
  int slot;  // -1 = constant
  int cst;
};

// A factor before sorting: input slots (-1 = constant), attachment level, folded table
// coordinates.
struct __align__(16) FacTmp {
  int8_t s[4];
  int16_t at, stride;
  int32_t base;
  int16_t dy, dx;
};
static_assert(sizeof(FacTmp) == 16, "FacTmp layout");

__global__ void lofp_plan_kernel(CallArgs a) {
  int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= a.B) return;
  if (a.flags[q] != 1) return;  // amps already 0 (photon number) or NaN (bad row)
  const int M = a.M, D = a.D, W = M + 1;
  const int32_t *t = a.T + q * M;
  uint8_t G[LOFP_MAX_CUTS];
  {
    int g = 0;
    for (int k = 0; k <= M; ++k) {
      G[k] = (uint8_t)g;
      if (k < M) g += t[k];
    }
  }
  const uint8_t *rho = a.maps, *sig = a.maps + (D + 1) * W;
  const uint8_t *frho = a.maps + 2 * (D + 1) * W, *fsig = a.maps + 3 * (D + 1) * W;
  // exact reachability: cum(S) inside the time-0 box (reading R5)
  for (int k = 0; k <= M; ++k) {
    int f = a.cumS[k];
    if (f < G[rho[k]] || f > G[sig[k]]) return;  // structural zero
  }
  unsigned char *plan = a.plans + (size_t)q * a.plan_stride;
  PlanHead *head = reinterpret_cast<PlanHead *>(plan);
  PlanLevel *lev = reinterpret_cast<PlanLevel *>(plan + sizeof(PlanHead));
  // plan layout: head | levels [Lg] | factors [nbs] | scatter u16 [4 nbs] | scratch
  PlanFactor *fac = reinterpret_cast<PlanFactor *>(plan + sizeof(PlanHead) + (size_t)a.Lg * sizeof(PlanLevel));
  uint16_t *scat = reinterpret_cast<uint16_t *>(fac + a.nbs);
  FacTmp *tmp = reinterpret_cast<FacTmp *>((reinterpret_cast<uintptr_t>(scat + 4 * (size_t)a.nbs) + 15) &
                                           ~uintptr_t(15));  // unsorted factors
  uint32_t *stmp = reinterpret_cast<uint32_t *>(tmp + a.nbs);         // unsorted scatter
  const uint16_t zero_off = LOFP_ZERO_OFF;
  const double2 *ent = reinterpret_cast<const double2 *>(a.entries);

  Ref cur[LOFP_MAX_CUTS];
  for (int k = 0; k <= M; ++k) cur[k] = Ref{-1, (int)a.cumS[k]};
  uint8_t lev_layer[LOFP_MAX_LEVELS];
  int8_t lev_rl[LOFP_MAX_LEVELS], lev_rr[LOFP_MAX_LEVELS];
  int L = 0, nf = 0;
  double2 root = make_double2(1.0, 0.0);
  for (int b = 0; b < a.nbs; ++b) {
    int l = a.bs_lk[2 * b], k = a.bs_lk[2 * b + 1];
    Ref A = cur[k - 1], Bv = cur[k], C = cur[k + 1];
    int idx = l * W + k;
    int lo = max((int)G[rho[idx]], (int)a.cumS[frho[idx]]);
    int hi = min((int)G[sig[idx]], (int)a.cumS[fsig[idx]]);
    if (lo > hi) return;  // empty box: no valid path (cannot happen once reachable)
    Ref Y;
    if (lo == hi) {
      Y = Ref{-1, lo};
    } else {
      Y = Ref{L, 0};
      PlanLevel pl;
      pl.ol = A.slot < 0 ? zero_off : lofp_level_off(A.slot);
      pl.cl = (uint8_t)(A.slot < 0 ? A.cst : 0);
      pl.or_ = C.slot < 0 ? zero_off : lofp_level_off(C.slot);
      pl.cr = (uint8_t)(C.slot < 0 ? C.cst : 0);
      pl.lo = (uint8_t)lo;
      pl.hi = (uint8_t)hi;
      pl.fbeg = pl.fend = 0;
      pl.sbeg = pl.send = 0;
      lev[L] = pl;
      lev_layer[L] = (uint8_t)l;
      lev_rl[L] = (int8_t)A.slot;
      lev_rr[L] = (int8_t)C.slot;
      ++L;
    }
    cur[k] = Y;
    // the element <y1, y2| BS_b |x1, x2>
    int at = max(max(A.slot, Bv.slot), max(C.slot, Y.slot));
    int ca = A.slot < 0 ? A.cst : 0, cb = Bv.slot < 0 ? Bv.cst : 0, cc = C.slot < 0 ? C.cst : 0,
        cy = Y.slot < 0 ? Y.cst : 0;
    int stride = a.bs_stride[b];
    if (at < 0) {  // all inputs constant: multiply into the root product
      int x1 = cb - ca, x2 = cc - cb, y1 = cy - ca;
      if (x1 + x2 == 0) continue;  // vacuum: the element is 1
      int o = a.offsets[a.bs_base[b] + x1 * stride + x2] + y1;
      root = cmul(root, ent[o]);
      continue;
    }
    if (A.slot < 0 && C.slot < 0 && cc == ca) continue;  // always vacuum
    FacTmp ft;
    ft.s[0] = (int8_t)A.slot;
    ft.s[1] = (int8_t)Bv.slot;
    ft.s[2] = (int8_t)C.slot;
    ft.s[3] = (int8_t)Y.slot;
    ft.at = (int16_t)at;
    ft.stride = (int16_t)stride;
    ft.base = a.bs_base[b] + stride * (cb - ca) + (cc - cb);
    ft.dy = (int16_t)(cy - ca);
    ft.dx = (int16_t)(cc - ca);
    tmp[nf] = ft;
    ++nf;
  }
  // counting sort of the factors by level; factor f (sorted) owns key word f
  uint16_t cnt[LOFP_MAX_LEVELS + 1];
  for (int j = 0; j <= L; ++j) cnt[j] = 0;
  for (int f = 0; f < nf; ++f) cnt[tmp[f].at + 1]++;
  for (int j = 0; j < L; ++j) cnt[j + 1] += cnt[j];
  for (int j = 0; j < L; ++j) {
    lev[j].fbeg = cnt[j];
    lev[j].fend = cnt[j + 1];
  }
  // the chain: the last free layer's levels, if their ranges and factors qualify (R17)
  int jb = L;
  if (L >= LOFP_CHAIN_MIN) {
    int cand = L - 1;
    while (cand > 0 && lev_layer[cand - 1] == lev_layer[L - 1]) --cand;
    if (cand < L - 32) cand = L - 32;  // one lane per chain level in the engine
    bool ok = true;
    for (int m = cand; m < L; ++m)
      if (lev_rl[m] >= cand || lev_rr[m] >= cand) ok = false;
    for (int f = 0; f < nf && ok; ++f) {
      const int at = tmp[f].at;
      if (at < cand) continue;
      for (int p = 0; p < 4; ++p) {
        const int sl = tmp[f].s[p];
        if (sl >= cand && sl != at && sl != at - 1) ok = false;
      }
    }
    // worth a warp only when the chain's box admits many paths (the box product bounds
    // the paths of every chain subtree of this output)
    double rbox = 1.0;
    for (int m = cand; m < L; ++m) rbox *= (double)((int)lev[m].hi - (int)lev[m].lo + 1);
    if (ok && L - cand >= LOFP_CHAIN_MIN) {
      atomicAdd(&a.ctr->nchain_ok, 1);
      if (rbox >= LOFP_CHAIN_MODE_RBOX) atomicAdd(&a.ctr->nchain_big, 1);
      atomicAdd(&a.ctr->rbox_log16, (unsigned long long)(16.0 * log2(rbox)));
    }
    if (ok && L - cand >= LOFP_CHAIN_MIN && rbox >= a.chain_rbox) jb = cand;
  }
  // scatter entries per level: those of chain factors go last (<= 15 per level, and the
  // whole list < 4096 entries, else no chain for this output)
  if (jb < L) {
    uint8_t chc[LOFP_MAX_LEVELS];
    for (int j = 0; j < L; ++j) chc[j] = 0;
    int tot = 0;
    bool fits = true;
    for (int f = 0; f < nf; ++f)
      for (int p = 0; p < 4; ++p)
        if (tmp[f].s[p] >= 0) {
          ++tot;
          if (tmp[f].at >= jb && ++chc[tmp[f].s[p]] > 15) fits = false;
        }
    if (!fits || tot >= 4096) jb = L;
  }
  int ns = 0;
  for (int f = 0; f < nf; ++f) {
    const FacTmp ft = tmp[f];
    int w = cnt[ft.at]++;
    uint32_t chain = 0x3210u;  // identity byte selector
    if (ft.at >= jb)
      for (int p = 0; p < 4; ++p)
        if (ft.s[p] >= jb)  // a chain value: the level's own (4) or the previous one's (5)
          chain = (chain & ~(15u << (4 * p))) | ((ft.s[p] == ft.at ? 4u : 5u) << (4 * p));
    PlanFactor pf;
    pf.crow = (int32_t)(((uint32_t)(uint8_t)(int8_t)(-ft.stride)) | ((uint32_t)(uint8_t)(int8_t)(ft.stride - 1) << 8) |
                        (1u << 16));
    pf.base = ft.base;
    pf.dy = (int8_t)ft.dy;
    pf.dx = (int8_t)ft.dx;
    pf.chain = (uint16_t)chain;
    for (int p = 0; p < 4; ++p) pf.slot[p] = (uint8_t)ft.s[p];  // -1 -> 0xff
    fac[w] = pf;
    const uint32_t isch = ft.at >= jb ? 1u : 0u;
    for (int p = 0; p < 4; ++p)
      if (ft.s[p] >= 0) stmp[ns++] = ((2u * (uint32_t)ft.s[p] + isch) << 16) | (uint32_t)(w * 128 + p);
  }
  // counting sort of the scatter entries by (level, chain factor)
  uint16_t cnt2[2 * LOFP_MAX_LEVELS + 1];
  for (int j = 0; j <= 2 * L; ++j) cnt2[j] = 0;
  for (int i = 0; i < ns; ++i) cnt2[(stmp[i] >> 16) + 1]++;
  for (int j = 0; j < 2 * L; ++j) cnt2[j + 1] += cnt2[j];
  for (int j = 0; j < L; ++j) {
    const int nch = cnt2[2 * j + 2] - cnt2[2 * j + 1];
    lev[j].sbeg = cnt2[2 * j];
    lev[j].send = (uint16_t)((cnt2[2 * j + 2] & 0xfff) | (jb < L ? nch << 12 : 0));
  }
  for (int i = 0; i < ns; ++i) scat[cnt2[stmp[i] >> 16]++] = (uint16_t)(stmp[i] & 0xffff);
  const int nkeys = jb < L ? (int)lev[jb].fbeg : nf;  // non-chain factors (they come first)
  PlanHead h;
  h.root[0] = root.x;
  h.root[1] = root.y;
  h.L = (uint16_t)L;
  h.nfac = (uint16_t)nf;
  h.nscat = (uint16_t)ns;
  h.jb = (uint16_t)jb;
  h.pad1 = 0;
  *head = h;
  if (L == 0) {  // a single valid path (eq. (10))
    a.amps[2 * q] = root.x;
    a.amps[2 * q + 1] = root.y;
    if (a.counts) a.counts[q] = 1;
    return;
  }
  atomicMax(&a.ctr->maxL, L);
  atomicMax(&a.ctr->maxF, nf);
  atomicMax(&a.ctr->maxS, ns);
  atomicMax(&a.ctr->maxK, nkeys);
  if (jb < L) atomicAdd(&a.ctr->nchain, 1);
  unsigned long long idx = atomicAdd(&a.ctr->nfeas, 1ull);
  a.feas[idx] = (uint32_t)q;
  atomicAdd(&a.ctr->outstanding, 1ull);
}

// ---------------------------------------------------------------------------
// path enumeration
// ---------------------------------------------------------------------------

__device__ __forceinline__ unsigned long long vload(const unsigned long long *p) {
  return *reinterpret_cast<const volatile unsigned long long *>(p);
}

// Per-lane state of the DFS, all in the warp's shared memory:
//   vals  value bytes of the levels (slot 0 = constant zero, level j = slot j + 1),
//         lane-interleaved by word (lofp_slot_off): the prefix handed to other lanes/warps;
//   keys  one word per attached factor: the variable bytes (a, b, c, y) of its inputs,
//         written when a level's value is set (scatter list of the plan), read with one
//         32-bit load per factor and turned into the table index with two dp4a;
//   stack ring of LOFP_STK branch entries [bot, top) (product before the level, level,
//         last value), a local-memory overflow below it for rare deep stacks.
struct WarpSmem {
  unsigned char *plan;  // staged plan of the current output
  unsigned char *vcol;  // vals words [slots/4][32]
  unsigned char *kcol;  // key words [nfac][32]
  double2 *stkP;        // [LOFP_STK][32]
  uint32_t *stkM;       // [LOFP_STK][32]
};

// Scatter entries of a level to write: all of them; none while the chain engine is on
// (then every factor's key is gathered from the value bytes and no key words exist).
template <bool CHAIN>
__device__ __forceinline__ int scatter_count(const PlanLevel &lv) {
  return CHAIN ? 0 : (int)(lv.send & 0xfff) - (int)lv.sbeg;
}

// Write value v of level j: the vals byte and every key byte that holds it.  (Used off
// the hot step; the step writes with a warp-uniform trip count, see below.)
template <bool CHAIN>
__device__ __forceinline__ void set_level(unsigned char *lb, unsigned char *kb, const PlanLevel &lvref,
                                          const uint16_t *scat, int j, int v) {
  const PlanLevel lv = lvref;
  const int sbeg = lv.sbeg, n = scatter_count<CHAIN>(lv);
  lb[lofp_level_off(j)] = (unsigned char)v;
  for (int s = 0; s < n; ++s) kb[scat[sbeg + s]] = (unsigned char)v;
}

// A factor's key gathered from value bytes (slot 0xff: constant -> 0).
__device__ __forceinline__ int gather_key(const PlanFactor &fd, const unsigned char *lb) {
  uint32_t k = 0;
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const int sl = fd.slot[p];
    const uint32_t b = sl == 0xff ? 0u : (uint32_t)lb[lofp_level_off(sl)];
    k |= b << (8 * p);
  }
  return (int)k;
}

// Product of the factors attached to level lv, times P.  The trip count is the warp's
// largest factor count (nmax, warp-uniform) so that every lane runs the same instruction
// stream; a lane past its own count multiplies by table entry 0, which is exactly 1 (the
// vacuum element of BS 0, R16).
template <bool COUNTED, bool CHAIN>
__device__ __forceinline__ int factor_entry(const PlanFactor *fp, const unsigned char *kp, int i, int fcnt,
                                            const int32_t *s_off, const unsigned char *lb, unsigned long long &ncm) {
  // past the lane's own count: re-read its last factor (always a valid descriptor, key
  // and table row) and use entry 0 (= 1)
  const bool on = i < fcnt;
  const int fi = on ? i : max(fcnt - 1, 0);
  const int2 fd = *reinterpret_cast<const int2 *>(fp + fi);  // crow, base
  // engine on: no key words, the key is gathered from the lane's value bytes
  const int key = CHAIN ? gather_key(fp[fi], lb) : *reinterpret_cast<const int *>(kp + fi * 128);
  const int row = __dp4a(key, fd.x, fd.y);
  const int o = s_off[on ? row : 0] + __dp4a(key, 0x010000ff, (int)fp[fi].dy);  // + y - a
  if (COUNTED) ncm += (on && __dp4a(key, 0x000100ff, (int)fp[fi].dx) > 0);  // x1 + x2 = c - a
  return on ? o : 0;
}

// Product of the factors attached to a level, times P.  The trip count is the warp's
// largest factor count (nmax, warp-uniform) so that every lane runs the same instruction
// stream; a lane past its own count multiplies by table entry 0, which is exactly 1 (the
// vacuum element of BS 0, R16).  Factors are taken in pairs: e_i e_{i+1} does not depend on P,
// so the dependent fp64 chain is one complex multiplication per pair.
template <bool COUNTED, bool CHAIN>
__device__ __forceinline__ double2 level_product(double2 P, int fbeg, int fcnt, int nmax, const PlanFactor *fac,
                                                 const unsigned char *kb, const int32_t *s_off,
                                                 const double2 *s_ent, const unsigned char *lb,
                                                 unsigned long long &ncm) {
  const PlanFactor *fp = fac + fbeg;
  const unsigned char *kp = kb + fbeg * 128;
  int i = 0;
#pragma unroll 1
  for (; i + 1 < nmax; i += 2) {
    const int o0 = factor_entry<COUNTED, CHAIN>(fp, kp, i, fcnt, s_off, lb, ncm);
    const int o1 = factor_entry<COUNTED, CHAIN>(fp, kp, i + 1, fcnt, s_off, lb, ncm);
    P = cmul(P, cmul(s_ent[o0], s_ent[o1]));
  }
  if (i < nmax) P = cmul(P, s_ent[factor_entry<COUNTED, CHAIN>(fp, kp, i, fcnt, s_off, lb, ncm)]);
  return P;
}

template <bool COUNTED, bool CHAIN, bool SMALL>
__global__ void __launch_bounds__(LOFP_ENUM_MAX_THREADS, 1) lofp_enum_kernel(CallArgs a) {
  // branch-stack entries kept in shared memory: fewer with the chain engine (the walk
  // above the chains is short; the overflow below the ring catches the rest)
  constexpr unsigned STK = CHAIN ? LOFP_STK_CHAIN : LOFP_STK;
  extern __shared__ __align__(16) unsigned char smem[];
  double2 *s_ent = reinterpret_cast<double2 *>(smem);
  int32_t *s_off = reinterpret_cast<int32_t *>(s_ent + a.nentries);
  for (int i = threadIdx.x; i < a.nentries; i += blockDim.x)
    reinterpret_cast<int4 *>(s_ent)[i] = reinterpret_cast<const int4 *>(a.entries)[i];
  for (int i = threadIdx.x; i < a.noffsets; i += blockDim.x) s_off[i] = a.offsets[i];
  __syncthreads();

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned char *wb = smem + a.table_bytes + (size_t)warp * a.warp_bytes;
  unsigned char *s_plan = wb;
  const PlanLevel *s_lev = reinterpret_cast<const PlanLevel *>(s_plan + sizeof(PlanHead));
  unsigned char *vcol = wb + a.plan_smem;                                   // [slots/4][32] words
  unsigned char *kcol = vcol + a.vals_slots * 32;                           // [maxfac][32] words
  double2 *stkP = reinterpret_cast<double2 *>(kcol + (size_t)a.maxfac * 128);  // [LOFP_STK][32]
  uint32_t *stkM = reinterpret_cast<uint32_t *>(stkP + STK * 32);         // [LOFP_STK][32]
  double2 *mbP = reinterpret_cast<double2 *>(stkM + STK * 32);             // hand-over mailbox
  uint32_t *mbM = reinterpret_cast<uint32_t *>(mbP + 1);
  // chain engine scratch: pair table W, per-lane suffix products, per-digit arrays
  double2 *cW = mbP + 2;                                     // [LOFP_W_MAX]
  double2 *cPs = cW + LOFP_W_MAX;                            // [LOFP_SUF_ENTRIES] suffix table
  // per chain level m: (range r_m, low end / digit m of the stride 32, pair-table block base, 1 / r_m)
  int4 *c_lv = reinterpret_cast<int4 *>(cPs + LOFP_SUF_ENTRIES);  // [33]
  int *c_wb = reinterpret_cast<int *>(c_lv + 33);            // [33] block bases (binary search)
  int *c_pv = c_wb + 33;                                     // [32] 1 / prefix place values
  unsigned char *c_dig = reinterpret_cast<unsigned char *>(c_pv + 32);  // [32 digits][32 lanes]
  // small-chain batch: per emitting lane (column) its chain's ranges and table offsets
  double2 *sc_proot = reinterpret_cast<double2 *>(
      (reinterpret_cast<uintptr_t>(c_dig + 32 * 32) + 15) & ~uintptr_t(15));  // [32] root products
  int *sc_wbase = reinterpret_cast<int *>(sc_proot + 32);                // [33] pair-table bases
  int *sc_pbase = sc_wbase + 33;                                         // [33] path bases
  uint16_t *sc_wb = reinterpret_cast<uint16_t *>(sc_pbase + 33);        // [16 levels][32]
  unsigned char *sc_lo = reinterpret_cast<unsigned char *>(sc_wb + LOFP_SMALL_LEVELS * 32);  // [16][32]
  unsigned char *sc_r = sc_lo + LOFP_SMALL_LEVELS * 32;                  // [16][32]
  unsigned char *lb = vcol + 4 * lane;  // this lane's vals byte base
  unsigned char *kb = kcol + 4 * lane;  // this lane's key byte base
  lb[LOFP_ZERO_OFF] = 0;
  const uint16_t dummy_off = lofp_slot_off(a.vals_slots - 1);  // scratch byte for idle lanes
  const unsigned nfeas = (unsigned)a.ctr->nfeas;

  // local-memory overflow below the shared ring: entries [obot, otop) (ring indices mod
  // LOFP_OVF), all shallower than the shared-memory entries
  double2 ovfP[LOFP_OVF];
  uint32_t ovfM[LOFP_OVF];

  unsigned cur_out = 0xffffffffu;
  const PlanFactor *s_fac = nullptr;
  const uint16_t *s_scat = nullptr;
  int L = 0, NF = 0;
  unsigned long long spills = 0, ovfc = 0, dons = 0, items = 0, nchains = 0, nchainfb = 0;
  unsigned long long ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long tph = COUNTED ? clock64() : 0;
#define LOFP_PHASE(k)                        \
  do {                                       \
    if (COUNTED) {                           \
      const long long _t = clock64();        \
      ph[k] += (unsigned long long)(_t - tph); \
      tph = _t;                              \
    }                                        \
  } while (0)
  uint32_t *const mySM = stkM + lane;    // this lane's stack metas, entry e at [e * 32]
  double2 *const mySP = stkP + lane;     // this lane's stack products
  const int dummy_rel = (int)dummy_off - a.vals_slots * 32;  // kb + dummy_rel = scratch byte

  // spill a branch (level jd = m & 0xff, last value m >> 8) of this lane to the global queue
  auto spill = [&](unsigned long long slot, unsigned out, uint32_t m, double2 Pe) {
    Item *it = a.ring + (slot & a.ring_mask);
    while (*reinterpret_cast<volatile unsigned *>(&it->seq) != 0u) __nanosleep(64);
    int jd = m & 0xff, hh = (m >> 8) & 0xff;
    if (COUNTED) atomicAdd(&a.ctr->spill_hist[min(L - 1 - jd, 63)], 1ull);
    it->out = out;
    it->j0 = (unsigned short)jd;
    it->vs = (unsigned char)(lb[lofp_level_off(jd)] + 1);
    it->ve = (unsigned char)hh;
    it->P[0] = Pe.x;
    it->P[1] = Pe.y;
    uint32_t *pw = reinterpret_cast<uint32_t *>(it->prefix);
    for (int w = 0; w < (jd + 4) / 4; ++w) pw[w] = *reinterpret_cast<const uint32_t *>(vcol + w * 128 + 4 * lane);
    __threadfence();
    *reinterpret_cast<volatile unsigned *>(&it->seq) = (unsigned)(slot + 1);
  };

  while (true) {
    // ---------------- acquire a work item (lane 0) ----------------
    int kind = 0;  // 0 done, 1 fresh output, 2 queued subtree
    unsigned out = 0;
    unsigned long long tk = 0;
    if (lane == 0) {
      unsigned long long idx = atomicAdd(&a.ctr->fresh_next, 1ull);
      if (idx < nfeas) {
        kind = 1;
        out = a.feas[idx];
      } else {
        tk = atomicAdd(&a.ctr->ticket, 1ull);
        const Item *it = a.ring + (tk & a.ring_mask);
        unsigned ns = 32;
        while (true) {
          unsigned seq = *reinterpret_cast<const volatile unsigned *>(&it->seq);
          if (seq == (unsigned)(tk + 1)) {
            __threadfence();
            kind = 2;
            out = __ldcg(&it->out);
            break;
          }
          if (vload(&a.ctr->outstanding) == 0ull) break;
          __nanosleep(ns);
          if (ns < 8192) ns <<= 1;
        }
      }
    }
    kind = __shfl_sync(FULL, kind, 0);
    if (kind == 0) break;
    out = __shfl_sync(FULL, out, 0);
    tk = __shfl_sync(FULL, tk, 0);
    ++items;

    LOFP_PHASE(6);
    // ---------------- stage the output's plan ----------------
    if (out != cur_out) {
      const unsigned char *gp = a.plans + (size_t)out * a.plan_stride;
      const PlanHead *gh = reinterpret_cast<const PlanHead *>(gp);
      int Lq = gh->L, nf = gh->nfac, ns = gh->nscat;
      for (int i = lane; i < 2 + Lq; i += 32)
        reinterpret_cast<int4 *>(s_plan)[i] = reinterpret_cast<const int4 *>(gp)[i];
      const unsigned char *gf = gp + sizeof(PlanHead) + (size_t)a.Lg * sizeof(PlanLevel);
      unsigned char *sf = s_plan + sizeof(PlanHead) + (size_t)Lq * sizeof(PlanLevel);
      for (int i = lane; i < nf; i += 32) reinterpret_cast<int4 *>(sf)[i] = reinterpret_cast<const int4 *>(gf)[i];
      const uint16_t *gs = reinterpret_cast<const uint16_t *>(gf + (size_t)a.nbs * sizeof(PlanFactor));
      uint16_t *ss = reinterpret_cast<uint16_t *>(sf + (size_t)nf * sizeof(PlanFactor));
      for (int i = lane; i < ns; i += 32) ss[i] = gs[i];
      s_fac = reinterpret_cast<const PlanFactor *>(sf);
      s_scat = ss;
      L = Lq;
      NF = nf;
      cur_out = out;
      __syncwarp();
    }
    const PlanHead *sh = reinterpret_cast<const PlanHead *>(s_plan);
    const int Lm1 = L - 1;
    const int jbq = CHAIN ? (int)sh->jb : L;  // first chain level (== L: no chain)
    bool chain_pending = false;
    const int NK = CHAIN ? 0 : NF;  // key words of this output (none while the engine is on)

    // ---------------- lane 0 begins the item ----------------
    // Lane state: j = current level, v = its value, Pb = product before level j's
    // factors, leafhi = last sibling when j is the leaf level, stack [bot, top) of open
    // branches (meta = level | last value << 8, product before that level), overflow
    // [obot, otop) below it.
    bool working = false;
    int j = 0, v = 0, leafhi = 0;
    unsigned bot = 0, top = 0, obot = 0, otop = 0;
    double2 Pb = make_double2(0.0, 0.0), acc = make_double2(0.0, 0.0);
    unsigned long long npaths = 0, ncm = 0;
    {
      // all key words of this warp start at zero (constant inputs contribute 0)
      for (int f = 0; f < NK; ++f) *reinterpret_cast<uint32_t *>(kb + f * 128) = 0u;
      int j0 = 0, vs = 0, ve = 0;
      double2 P0;
      if (kind == 1) {
        PlanLevel l0 = s_lev[0];
        vs = max((int)lb[l0.ol] + l0.cl, (int)l0.lo);
        ve = min((int)lb[l0.or_] + l0.cr, (int)l0.hi);
        P0 = make_double2(sh->root[0], sh->root[1]);
      } else {
        Item *it = a.ring + (tk & a.ring_mask);
        // the slot was written by another SM: read around L1
        uint32_t w2 = __ldcg(reinterpret_cast<const uint32_t *>(it) + 2);
        j0 = w2 & 0xffff;
        vs = (w2 >> 16) & 0xff;
        ve = w2 >> 24;
        P0 = __ldcg(reinterpret_cast<const double2 *>(it->P));
        int nw = (j0 + 4) >> 2;  // slots [0, j0]: the zero slot and levels < j0
        const uint32_t *pw = reinterpret_cast<const uint32_t *>(it->prefix);
        for (int w = lane; w < nw; w += 32) *reinterpret_cast<uint32_t *>(vcol + w * 128) = __ldcg(pw + w);
        __syncwarp();
        if (lane == 0) {
          __threadfence();
          *reinterpret_cast<volatile unsigned *>(&it->seq) = 0u;  // slot free again
          for (int jj = 0; jj < j0; ++jj)  // rebuild the keys of the prefix levels
            set_level<CHAIN>(lb, kb, s_lev[jj], s_scat, jj, lb[lofp_level_off(jj)]);
        }
      }
      if (lane == 0 && kind == 1 && jbq == 0) {  // the whole tree is one chain
        working = true;
        chain_pending = true;
        Pb = P0;
      } else if (lane == 0) {
        working = true;
        j = j0;
        v = vs;
        set_level<CHAIN>(lb, kb, s_lev[j0], s_scat, j0, vs);
        if (j0 == Lm1) {
          leafhi = ve;
        } else if (ve > vs) {
          mySM[0] = (uint32_t)j0 | ((uint32_t)ve << 8);
          mySP[0] = P0;
          top = 1;
        }
        Pb = P0;
      }
    }
    __syncwarp();

    // after a chain's subtree is done: pop the deepest open branch (or become idle)
    auto resume_walk = [&]() {
      if (top != bot) {
        const unsigned e2 = ((top - 1u) & (STK - 1)) * 32;
        const uint32_t m2 = mySM[e2];
        const int jj = m2 & 0xff;
        const int nv2 = (int)lb[lofp_level_off(jj)] + 1;
        Pb = mySP[e2];
        if (nv2 == (int)((m2 >> 8) & 0xff)) --top;
        j = jj;
        v = nv2;
        set_level<CHAIN>(lb, kb, s_lev[jj], s_scat, jj, nv2);
      } else if (otop != obot) {
        const unsigned e2 = (otop - 1u) & (LOFP_OVF - 1);
        const uint32_t m2 = ovfM[e2];
        const int jj = m2 & 0xff;
        const int nv2 = (int)lb[lofp_level_off(jj)] + 1;
        Pb = ovfP[e2];
        if (nv2 == (int)((m2 >> 8) & 0xff)) --otop;
        j = jj;
        v = nv2;
        set_level<CHAIN>(lb, kb, s_lev[jj], s_scat, jj, nv2);
      } else {
        working = false;
      }
    };

    unsigned iter = 0;
    while (true) {
      // ---------------- intra-warp hand-over ----------------
      // One per step: the lane holding the shallowest open branch of the warp gives it
      // (all its remaining siblings) to the lowest idle lane.
      const unsigned idle = __ballot_sync(FULL, !working);
      if (idle) {
        int myshal = 0x7fffffff;
        if (working) {
          if (otop != obot)
            myshal = (int)(ovfM[obot & (LOFP_OVF - 1)] & 0xff);
          else if (top != bot)
            myshal = (int)(mySM[(bot & (STK - 1)) * 32] & 0xff);
        }
        const int shal = __reduce_min_sync(FULL, myshal);
        if (shal == 0x7fffffff) {
          if (idle == FULL) break;  // item finished
        } else {
          const int donor = __ffs(__ballot_sync(FULL, myshal == shal)) - 1;
          const int recv = __ffs(idle) - 1;
          if (lane == donor) {  // publish the shallowest open branch
            uint32_t m;
            double2 P;
            if (otop != obot) {
              m = ovfM[obot & (LOFP_OVF - 1)];
              P = ovfP[obot & (LOFP_OVF - 1)];
              ++obot;
            } else {
              const unsigned e = (bot & (STK - 1)) * 32;
              m = mySM[e];
              P = mySP[e];
              ++bot;
            }
            mbM[0] = m;
            mbP[0] = P;
          }
          __syncwarp();
          if (lane == recv) {
            const uint32_t m = mbM[0];
            const double2 P = mbP[0];
            const int jd = m & 0xff, hh = (m >> 8) & 0xff;
            const int nw = ((jd + 1) >> 2) + 1;  // words holding slots [0, jd + 1]
            for (int w = 0; w < nw; ++w)
              *reinterpret_cast<uint32_t *>(vcol + w * 128 + 4 * lane) =
                  *reinterpret_cast<const uint32_t *>(vcol + w * 128 + 4 * donor);
            // the donor's keys hold the prefix values (deeper bytes are rewritten on descent)
            for (int f = 0; f < NK; ++f)
              *reinterpret_cast<uint32_t *>(kcol + f * 128 + 4 * lane) =
                  *reinterpret_cast<const uint32_t *>(kcol + f * 128 + 4 * donor);
            const int nv = (int)lb[lofp_level_off(jd)] + 1;
            set_level<CHAIN>(lb, kb, s_lev[jd], s_scat, jd, nv);
            bot = top = obot = otop = 0;
            leafhi = 0;
            if (jd == Lm1) {
              leafhi = hh;
            } else if (hh > nv) {
              mySM[0] = (uint32_t)jd | ((uint32_t)hh << 8);
              mySP[0] = P;
              top = 1;
            }
            Pb = P;
            j = jd;
            v = nv;
            working = true;
            ++dons;
            if (COUNTED) atomicAdd(&a.ctr->don_hist[min(Lm1 - jd, 63)], 1ull);
          }
          __syncwarp();
        }
      }

      // ---------------- one DFS node per lane ----------------
      // Every lane runs the same instruction stream: the product of its current level's
      // factors (warp-uniform trip count), one move -- next leaf sibling, pop of the
      // deepest open branch, or descent -- chosen by predicates, and one write of the new
      // value into the vals byte and the key bytes (warp-uniform trip count; a lane with
      // nothing to write writes a scratch byte).
      {
        const bool stepping = working && !chain_pending;  // a pending lane waits for the engine
        const PlanLevel lv = s_lev[stepping ? j : 0];
        const int fcnt = stepping ? (int)lv.fend - (int)lv.fbeg : 0;
        const int nmax = __reduce_max_sync(FULL, fcnt);
        const double2 P = level_product<COUNTED, CHAIN>(Pb, lv.fbeg, fcnt, nmax, s_fac, kb, s_off, s_ent, lb, ncm);
        const bool isleaf = stepping && j == Lm1;
        if (isleaf) {
          acc.x += P.x;
          acc.y += P.y;
          if (COUNTED) ++npaths;
        }
        const bool sib = isleaf && v < leafhi;
        const bool desc = stepping && !isleaf;
        const bool popsm = isleaf && !sib && top != bot;
        const unsigned te = ((top - 1u) & (STK - 1)) * 32;
        uint32_t m = mySM[te];
        double2 Ps = mySP[te];
        bool popov = false;
        if (isleaf && !sib && !popsm && otop != obot) {  // rare: the local overflow
          popov = true;
          const unsigned e = (otop - 1u) & (LOFP_OVF - 1);
          m = ovfM[e];
          Ps = ovfP[e];
        }
        const bool pop = popsm || popov;
        const bool moves = desc || sib || pop;
        const int nj = desc ? j + 1 : (sib ? j : (pop ? (int)(m & 0xff) : 0));
        const PlanLevel nl = s_lev[nj];
        const uint16_t noff = lofp_level_off(nj);
        const int dlo = max((int)lb[nl.ol] + nl.cl, (int)nl.lo);
        const int dhi = min((int)lb[nl.or_] + nl.cr, (int)nl.hi);
        const int pv = (int)lb[noff] + 1;
        const int nv = desc ? dlo : (sib ? v + 1 : pv);
        if (pop) {
          Pb = Ps;
          if (pv == (int)((m >> 8) & 0xff)) {
            if (popsm) --top; else --otop;
          }
        }
        const bool tochain = desc && nj == jbq;
        if (tochain) {
          Pb = P;  // product through level jb - 1: the chain's root product
          chain_pending = true;
        } else if (desc) {
          Pb = P;
          if (nj == Lm1) {
            leafhi = dhi;  // leaf siblings are walked one per step
          } else if (dhi > dlo) {
            if (top - bot == STK) {  // full: the shallowest entry goes to the overflow
              const unsigned e = (bot & (STK - 1)) * 32, o = otop & (LOFP_OVF - 1);
              ovfM[o] = mySM[e];
              ovfP[o] = mySP[e];
              ++otop;
              ++bot;
              ++ovfc;
            }
            const unsigned e = (top & (STK - 1)) * 32;
            mySM[e] = (uint32_t)nj | ((uint32_t)dhi << 8);
            mySP[e] = P;
            ++top;
          }
        }
        const bool wr = moves && !tochain;
        if (stepping) working = moves;
        if (wr) {
          j = nj;
          v = nv;
        }
        // the new value: vals byte and key bytes
        lb[wr ? (int)noff : (int)dummy_off] = (unsigned char)nv;
        const int scnt = wr ? scatter_count<CHAIN>(nl) : 0;
        const int smax = __reduce_max_sync(FULL, scnt);
        const uint16_t *sp = s_scat + nl.sbeg;  // reads past the list stay in the warp's smem
#pragma unroll 1
        for (int i = 0; i < smax; i += 4) {  // four loads in flight, then four stores
          const uint2 w = make_uint2(sp[i] | ((uint32_t)sp[i + 1] << 16), sp[i + 2] | ((uint32_t)sp[i + 3] << 16));
          kb[i < scnt ? (int)(w.x & 0xffff) : dummy_rel] = (unsigned char)nv;
          kb[i + 1 < scnt ? (int)(w.x >> 16) : dummy_rel] = (unsigned char)nv;
          kb[i + 2 < scnt ? (int)(w.y & 0xffff) : dummy_rel] = (unsigned char)nv;
          kb[i + 3 < scnt ? (int)(w.y >> 16) : dummy_rel] = (unsigned char)nv;
        }
      }

      LOFP_PHASE(0);
      // ---------------- chain engine (lockstep, whole warp) ----------------
      // Each lane that reached the first chain level hands its chain -- the Cartesian
      // product of the chain levels' ranges, fixed by its levels < jb -- to the whole warp:
      // (1) lane m computes chain level m's range; (2) the pair table
      // W_m(v_{m-1}, v_m) = product of level m's factors is built (one entry per lane per
      // round); (3) every path of the chain is enumerated: the leading digits are split
      // over the lanes, the remaining digits run one odometer shared by all lanes (warp-
      // uniform control), each path's product = root * prod_m W_m formed with prefix
      // sharing and added to the lane's accumulator.  Then the emitting lane pops its
      // stack as after a finished subtree.
      {
        unsigned pend = CHAIN ? __ballot_sync(FULL, chain_pending) : 0u;
        if (pend) {
          // Every pending lane sizes its own chain; short chains (few paths) are
          // enumerated together below, the others get a warp pass each.
          const int Mb = L - jbq;
          bool small = false;
          int myE = 0, myR = 0;
          if (SMALL && chain_pending && Mb <= LOFP_SMALL_LEVELS) {
            int rprev = 1, E = 0;
            float R = 1.f;
            for (int m = 0; m < Mb; ++m) {
              const PlanLevel cl = s_lev[jbq + m];
              const int lo = max((int)lb[cl.ol] + cl.cl, (int)cl.lo);
              const int r = min((int)lb[cl.or_] + cl.cr, (int)cl.hi) - lo + 1;
              sc_lo[m * 32 + lane] = (unsigned char)lo;
              sc_r[m * 32 + lane] = (unsigned char)r;
              sc_wb[m * 32 + lane] = (uint16_t)min(E, 65535);
              E += rprev * r;
              rprev = r;
              R *= (float)r;
            }
            small = R < (float)a.small_paths && E <= LOFP_W_MAX;
            myE = E;
            myR = (int)R;
          }
          unsigned smask = SMALL ? __ballot_sync(FULL, small) : 0u;
          pend &= ~smask;
          // ---- short chains, batched: all their pair tables, then all their paths ----
          while (smask) {
            const bool cand = (smask >> lane) & 1u;
            int incE = cand ? myE : 0;
            for (int o = 1; o < 32; o <<= 1) {
              const int tv = __shfl_up_sync(FULL, incE, o);
              if (lane >= o) incE += tv;
            }
            const bool ing = cand && incE <= LOFP_W_MAX;  // a prefix of the candidates
            const unsigned gmask = __ballot_sync(FULL, ing);
            smask &= ~gmask;
            const int eg = ing ? myE : 0, rg = ing ? myR : 0;
            int ie = eg, ir = rg;
            for (int o = 1; o < 32; o <<= 1) {
              const int te = __shfl_up_sync(FULL, ie, o), tr = __shfl_up_sync(FULL, ir, o);
              if (lane >= o) {
                ie += te;
                ir += tr;
              }
            }
            const int Eg = __shfl_sync(FULL, ie, 31), Rg = __shfl_sync(FULL, ir, 31);
            sc_wbase[lane] = ie - eg;
            sc_pbase[lane] = ir - rg;
            if (lane == 0) {
              sc_wbase[32] = Eg;
              sc_pbase[32] = Rg;
            }
            sc_proot[lane] = Pb;
            __syncwarp();
            if (lane == 0) nchains += __popc(gmask);
            for (int w = lane; w < Eg; w += 32) {  // pair tables W of every chain of the group
              int c = 0;
              for (int st = 16; st > 0; st >>= 1)
                if (sc_wbase[c + st] <= w) c += st;
              const int loc = w - sc_wbase[c];
              int m = 0;
              for (int st = LOFP_SMALL_LEVELS / 2; st > 0; st >>= 1)
                if (m + st < Mb && sc_wb[(m + st) * 32 + c] <= loc) m += st;
              const int rm = sc_r[m * 32 + c], rel = loc - sc_wb[m * 32 + c];
              const int ii = (int)(((float)rel + 0.5f) * __frcp_rn((float)rm)), kk = rel - ii * rm;
              const int vm = sc_lo[m * 32 + c] + kk, vp = m > 0 ? sc_lo[(m - 1) * 32 + c] + ii : 0;
              const PlanLevel lv = s_lev[jbq + m];
              double2 Q = make_double2(1.0, 0.0);
              for (int f = lv.fbeg; f < lv.fend; ++f) {
                const PlanFactor fd = s_fac[f];
                const int key = (int)__byte_perm((uint32_t)gather_key(fd, vcol + 4 * c),
                                                 (uint32_t)vm | ((uint32_t)vp << 8), fd.chain);
                const int row = __dp4a(key, fd.crow, fd.base);
                const int o = s_off[row] + __dp4a(key, 0x010000ff, (int)fd.dy);
                Q = cmul(Q, s_ent[o]);
                if (COUNTED) ncm += __dp4a(key, 0x000100ff, (int)fd.dx) > 0;
              }
              cW[w] = Q;
            }
            __syncwarp();
            for (int p = lane; p < Rg; p += 32) {  // every path: root * prod_m W_m
              int c = 0;
              for (int st = 16; st > 0; st >>= 1)
                if (sc_pbase[c + st] <= p) c += st;
              int rem = p - sc_pbase[c];
              const double2 *wc = cW + sc_wbase[c];
              double2 P = sc_proot[c];
              int m = Mb - 1, rm = sc_r[m * 32 + c];
              int q = (int)(((float)rem + 0.5f) * __frcp_rn((float)rm));
              int cur = rem - q * rm;
              rem = q;
              for (; m > 0; --m) {  // digits from the last level; W_m(v_{m-1}, v_m)
                const int rp = sc_r[(m - 1) * 32 + c];
                const int q2 = (int)(((float)rem + 0.5f) * __frcp_rn((float)rp));
                const int nxt = rem - q2 * rp;
                rem = q2;
                P = cmul(P, wc[sc_wb[m * 32 + c] + nxt * rm + cur]);
                cur = nxt;
                rm = rp;
              }
              P = cmul(P, wc[cur]);  // W_0(v_0)
              acc.x += P.x;
              acc.y += P.y;
              if (COUNTED) {
                ++npaths;
                ncm += Mb;
              }
            }
            __syncwarp();
            if (ing) {
              chain_pending = false;
              resume_walk();
            }
          }
        }
        LOFP_PHASE(1);
        while (pend) {
          const int em = __ffs(pend) - 1;
          pend &= pend - 1;
          const unsigned char *lbe = vcol + 4 * em;
          const double2 Proot = make_double2(__shfl_sync(FULL, Pb.x, em), __shfl_sync(FULL, Pb.y, em));
          const int Mb = L - jbq;
          int clo = 0, crr = 1;
          if (lane < Mb) {
            const PlanLevel cl = s_lev[jbq + lane];
            clo = max((int)lbe[cl.ol] + cl.cl, (int)cl.lo);
            crr = min((int)lbe[cl.or_] + cl.cr, (int)cl.hi) - clo + 1;
          }
          int rprev = __shfl_up_sync(FULL, crr, 1);
          if (lane == 0) rprev = 1;
          const int sz = lane < Mb ? rprev * crr : 0;
          int inc = sz;
          for (int o = 1; o < 32; o <<= 1) {
            const int tv = __shfl_up_sync(FULL, inc, o);
            if (lane >= o) inc += tv;
          }
          const int E = __shfl_sync(FULL, inc, 31);
          // lane m: product of the ranges of levels <= m (exact in double); lane 31: paths
          double pinc = (double)crr;
          for (int o = 1; o < 32; o <<= 1) {
            const double tv = __shfl_up_sync(FULL, pinc, o);
            if (lane >= o) pinc *= tv;
          }
          const double Rd = __shfl_sync(FULL, pinc, 31);
          const bool fb = E > LOFP_W_MAX || Rd > 2.0e9 || Rd < (double)a.chain_rmin;
          if (lane == 0) {
            if (fb) ++nchainfb; else ++nchains;
          }
          if (fb) {  // too few paths (or too many pairs/paths): the emitting lane walks the chain itself
            if (lane == em) {
              chain_pending = false;
              j = jbq;
              v = clo;  // lane em's own range of level jb (it is lane 0's value: broadcast)
            }
            const int lo0 = __shfl_sync(FULL, clo, 0), r0 = __shfl_sync(FULL, crr, 0);
            if (lane == em) {
              v = lo0;
              set_level<CHAIN>(lb, kb, s_lev[jbq], s_scat, jbq, lo0);
              if (jbq == Lm1) {
                leafhi = lo0 + r0 - 1;
              } else if (r0 > 1) {
                if (top - bot == STK) {
                  const unsigned e2 = (bot & (STK - 1)) * 32, o2 = otop & (LOFP_OVF - 1);
                  ovfM[o2] = mySM[e2];
                  ovfP[o2] = mySP[e2];
                  ++otop;
                  ++bot;
                  ++ovfc;
                }
                const unsigned e2 = (top & (STK - 1)) * 32;
                mySM[e2] = (uint32_t)jbq | ((uint32_t)(lo0 + r0 - 1) << 8);
                mySP[e2] = Pb;
                ++top;
              }
            }
            continue;
          }
          LOFP_PHASE(1);
          // reciprocal of the range: floor(n / r) = (int)((n + 0.5) * inv) exactly for n < 2^12
          c_lv[lane] = make_int4(crr, clo, inc - sz, __float_as_int(__fdividef(1.0f, (float)crr)));  // (.y: low end until the split)
          c_wb[lane] = inc - sz;
          if (lane == 0) c_wb[32] = E;
          __syncwarp();
          // (2) pair table.  First the chain factors' keys (gathered once per chain from the
          // emitter's value bytes; the chain bytes are replaced below), then one entry per
          // lane per round: W_m(v_{m-1}, v_m) = product of level m's factors.
          const int fc0 = s_lev[jbq].fbeg, nfc = NF - fc0;  // chain factors come last
          uint32_t *ckey = reinterpret_cast<uint32_t *>(cPs);  // (the suffix table comes later)
          const bool pre = nfc <= 2 * LOFP_SUF_ENTRIES;
          if (pre) {
            for (int f = lane; f < nfc; f += 32) {
              ckey[f] = (uint32_t)gather_key(s_fac[fc0 + f], lbe);
            }
            __syncwarp();
          }
          for (int w = lane; w < E; w += 32) {
            int m = 0;
            for (int st = 16; st > 0; st >>= 1)
              if (m + st < Mb && c_wb[m + st] <= w) m += st;
            const int4 lvm = c_lv[m];
            const int rm = lvm.x, rel = w - lvm.z;
            const int ii = (int)(((float)rel + 0.5f) * __int_as_float(lvm.w)), kk = rel - ii * rm;
            const uint32_t vmp = (uint32_t)(lvm.y + kk) | ((uint32_t)(m > 0 ? c_lv[m - 1].y + ii : 0) << 8);
            const PlanLevel lv = s_lev[jbq + m];
            double2 Q = make_double2(1.0, 0.0);
#pragma unroll 1
            for (int f = lv.fbeg; f < lv.fend; ++f) {
              const PlanFactor fd = s_fac[f];
              // the chain bytes of the key: v_m and v_{m-1} put in by one byte permutation
              const uint32_t base = pre ? ckey[f - fc0] : (uint32_t)gather_key(fd, lbe);
              const int key = (int)__byte_perm(base, vmp, fd.chain);
              const int row = __dp4a(key, fd.crow, fd.base);
              const int o = s_off[row] + __dp4a(key, 0x010000ff, (int)fd.dy);
              Q = cmul(Q, s_ent[o]);
              if (COUNTED) ncm += __dp4a(key, 0x000100ff, (int)fd.dx) > 0;
            }
            cW[w] = Q;
          }
          __syncwarp();  // the key scratch is reused by the suffix table below
          LOFP_PHASE(2);
          // (3) enumeration.  Digits [0, t) (prefix) are split over the lanes, digits
          // [t, Mb) (suffix) form a table Suf[s] = prod_{m > t} W_m shared by all lanes
          // (one lane per entry).  Every path of the chain is then formed as
          //   (root * prod_{m < t} W_m * W_t) * Suf[s]
          // -- one complex multiplication per path in a warp-uniform inner loop -- and
          // added to the lane's accumulator.  t maximises lane use with |Suf| <= 64.
          __syncwarp();
          // split: the shortest prefix with >= 32 combinations (every lane busy), then
          // lengthened until the suffix table has <= 64 entries (pinc: see the ranges).
          const double Rdd = Rd;
          const double thr = fmax(32.0, Rdd * (1.0 / LOFP_SUF_ENTRIES));
          const unsigned okm = __ballot_sync(FULL, lane < Mb && pinc >= thr);
          const int t = okm ? __ffs(okm) : Mb;  // prefix digits [0, t)
          const double Ctd = t > 0 ? __shfl_sync(FULL, pinc, t - 1) : 1.0;
          const long long Ct = (long long)Ctd;
          // R / C_t: an exact integer <= 64 (float quotient error ~1e-7 of it: rounding is safe)
          const int Rsi = __float2int_rn(__fdividef((float)Rdd, (float)Ctd));
          // per-lane prefix digits (digit t-1 least significant) of the lane's first prefix
          // index (= lane), and the digits of the stride 32, for an incremental add per round:
          // digit m of c = floor(c / pv_m) mod r_m, pv_m = Ct / pinc_m (place value)
          if (lane < t) {  // lane m: 1 / pv_m and digit m of the stride 32
            const float ipv = __fdividef((float)pinc, (float)Ctd), ir = __fdividef(1.0f, (float)crr);
            c_pv[lane] = __float_as_int(ipv);
            const int q32 = (int)((32.0f + 0.5f) * ipv);
            reinterpret_cast<int *>(c_lv + lane)[1] = q32 - (int)(((float)q32 + 0.5f) * ir) * crr;
          }
          __syncwarp();
#pragma unroll 4
          for (int m = 0; m < t; ++m) {
            const int4 lvm = c_lv[m];
            const float ipv = __int_as_float(c_pv[m]), ir = __int_as_float(lvm.w);
            const int rm = lvm.x;
            const int q = (int)(((float)lane + 0.5f) * ipv);
            const int d = q - (int)(((float)q + 0.5f) * ir) * rm;
            c_dig[m * 32 + lane] = (unsigned char)d;
          }
          LOFP_PHASE(3);
          // suffix table: entry s (digit t most significant) = prod_{m = t+1}^{Mb-1} W_m;
          // entries lane and lane + 32 are built together (two independent chains)
          if (Rsi <= 32) {  // one entry per lane
            const int s0 = lane;
            int rem0 = s0;
            double2 Q0 = make_double2(1.0, 0.0);
            int4 lvm = c_lv[Mb - 1];
            for (int m = Mb - 1; m > t; --m) {  // decode from the last digit
              const int4 lvp = c_lv[m - 1];
              const int rm = lvm.x, rp = lvp.x;
              const float im = __int_as_float(lvm.w), ip = __int_as_float(lvp.w);
              const int q0 = (int)(((float)rem0 + 0.5f) * im);
              const int cur0 = rem0 - q0 * rm;
              rem0 = q0;
              const int nx0 = rem0 - (int)(((float)rem0 + 0.5f) * ip) * rp;  // digit m-1
              const int blk_m = rp * rm;  // the level's pair-table block (m >= 1)
              const double2 w0 = cW[lvm.z + min(nx0 * rm + cur0, blk_m - 1)];
              lvm = lvp;
              Q0 = cmul(Q0, w0);
              if (COUNTED) ncm += (s0 < Rsi);
            }
            if (s0 < Rsi) cPs[s0] = Q0;
          } else {
            const int s0 = lane, s1 = lane + 32;
            int rem0 = s0, rem1 = s1;
            double2 Q0 = make_double2(1.0, 0.0), Q1 = Q0;
            int4 lvm = c_lv[Mb - 1];
            for (int m = Mb - 1; m > t; --m) {  // decode from the last digit
              const int4 lvp = c_lv[m - 1];
              const int rm = lvm.x, rp = lvp.x;
              const float im = __int_as_float(lvm.w), ip = __int_as_float(lvp.w);
              const int q0 = (int)(((float)rem0 + 0.5f) * im), q1 = (int)(((float)rem1 + 0.5f) * im);
              const int cur0 = rem0 - q0 * rm, cur1 = rem1 - q1 * rm;
              rem0 = q0;
              rem1 = q1;
              const int nx0 = rem0 - (int)(((float)rem0 + 0.5f) * ip) * rp;  // digit m-1
              const int nx1 = rem1 - (int)(((float)rem1 + 0.5f) * ip) * rp;
              const int blk_m = rp * rm;  // the level's pair-table block (m >= 1)
              const double2 w0 = cW[lvm.z + min(nx0 * rm + cur0, blk_m - 1)];
              const double2 w1 = cW[lvm.z + min(nx1 * rm + cur1, blk_m - 1)];
              lvm = lvp;
              Q0 = cmul(Q0, w0);
              Q1 = cmul(Q1, w1);
              if (COUNTED) ncm += (s0 < Rsi) + (s1 < Rsi);
            }
            if (s0 < Rsi) cPs[s0] = Q0;
            if (s1 < Rsi) cPs[s1] = Q1;
          }
          __syncwarp();
          LOFP_PHASE(7);
          const int4 lvt = c_lv[min(t, Mb - 1)];
          const int rt = t < Mb ? lvt.x : 1;
          const int blk = Rsi / rt;  // suffix entries per value of digit t
          for (long long c0 = 0; c0 < Ct; c0 += 32) {
            const long long cc = c0 + lane;
            const bool act = cc < Ct;
            if (c0 > 0) {  // advance this lane's prefix index by 32 (mixed-radix add)
              int carry = 0;
#pragma unroll 1
              for (int m = t - 1; m >= 0; --m) {
                const int2 rd = *reinterpret_cast<const int2 *>(c_lv + m);  // (r_m, digit of 32)
                int d = c_dig[m * 32 + lane] + rd.y + carry;
                carry = d >= rd.x;
                d -= carry ? rd.x : 0;
                c_dig[m * 32 + lane] = (unsigned char)d;
              }
            }
            double2 P = Proot;
            int vprev = 0;
#pragma unroll 4
            for (int m = 0; m < t; ++m) {
              const int d = c_dig[m * 32 + lane];
              const int4 lv = c_lv[m];
              const int idx = lv.z + (m > 0 ? vprev * lv.x : 0) + d;
              P = cmul(P, cW[idx]);
              if (COUNTED) ncm += act;
              vprev = d;  // digit (offset from the level's low end)
            }
            if (t == Mb) {  // no suffix: the prefix is the whole path
              if (act) {
                acc.x += P.x;
                acc.y += P.y;
                if (COUNTED) ++npaths;
              }
              continue;
            }
            for (int dt = 0; dt < rt; ++dt) {
              const double2 Q = cmul(P, cW[lvt.z + (t > 0 ? vprev * rt : 0) + dt]);
              if (COUNTED) ncm += act;
              const double2 *sf = cPs + dt * blk;
              double2 a0 = make_double2(0.0, 0.0), a1 = make_double2(0.0, 0.0);
              int k = 0;
              for (; k + 1 < blk; k += 2) {
                const double2 l0 = cmul(Q, sf[k]), l1 = cmul(Q, sf[k + 1]);
                a0.x += l0.x;
                a0.y += l0.y;
                a1.x += l1.x;
                a1.y += l1.y;
              }
              if (k < blk) {
                const double2 l0 = cmul(Q, sf[k]);
                a0.x += l0.x;
                a0.y += l0.y;
              }
              if (act) {
                acc.x += a0.x + a1.x;
                acc.y += a0.y + a1.y;
                if (COUNTED) {
                  npaths += blk;
                  ncm += blk;
                }
              }
            }
          }
          __syncwarp();
          LOFP_PHASE(4);
          // the emitting lane continues its depth-first walk after the chain's subtree
          if (lane == em) {
            chain_pending = false;
            resume_walk();
          }
        }
      }

      LOFP_PHASE(5);
      // ---------------- feed idle warps through the global queue ----------------
      // At most one subtree per warp per check: the warp's shallowest open branch, and
      // only when it is far from the leaves (a large subtree) and some warp is waiting.
      if (((++iter) & (CHAIN ? 0u : 31u)) == 0u) {  // (a chain step is long: check often)
        long long waiting = 0;
        if (lane == 0) waiting = (long long)(vload(&a.ctr->ticket) - vload(&a.ctr->tail));
        waiting = __shfl_sync(FULL, waiting, 0);
        if (waiting > 0) {
          int myshal = 0x7fffffff;
          if (working) {
            if (otop != obot)
              myshal = (int)(ovfM[obot & (LOFP_OVF - 1)] & 0xff);
            else if (top != bot)
              myshal = (int)(mySM[(bot & (STK - 1)) * 32] & 0xff);
          }
          const int shal = __reduce_min_sync(FULL, myshal);
          if (shal != 0x7fffffff && Lm1 - shal >= LOFP_SPILL_MIN_DIST) {
            const int giver = __ffs(__ballot_sync(FULL, myshal == shal)) - 1;
            if (lane == giver) {
              atomicAdd(&a.ctr->outstanding, 1ull);
              const unsigned long long slot = atomicAdd(&a.ctr->tail, 1ull);
              if (otop != obot) {
                const unsigned e = obot & (LOFP_OVF - 1);
                spill(slot, out, ovfM[e], ovfP[e]);
                ++obot;
              } else {
                const unsigned e = (bot & (STK - 1)) * 32;
                spill(slot, out, mySM[e], mySP[e]);
                ++bot;
              }
              ++spills;
            }
          }
        }
      }
    }

    LOFP_PHASE(6);
    // ---------------- item finished: warp reduction, one atomic per item ----------------
    for (int s = 16; s > 0; s >>= 1) {
      acc.x += __shfl_xor_sync(FULL, acc.x, s);
      acc.y += __shfl_xor_sync(FULL, acc.y, s);
      if (COUNTED) {
        npaths += __shfl_xor_sync(FULL, npaths, s);
        ncm += __shfl_xor_sync(FULL, ncm, s);
      }
    }
    if (lane == 0) {
      atomicAdd(&a.amps[2 * out], acc.x);
      atomicAdd(&a.amps[2 * out + 1], acc.y);
      if (COUNTED) {
        atomicAdd(&a.counts[out], npaths);
        atomicAdd(&a.ctr->leaves, npaths);
        atomicAdd(&a.ctr->cmuls, ncm);
      }
      __threadfence();
      atomicAdd(&a.ctr->outstanding, ~0ull);  // -1
    }
    __syncwarp();
  }
  // statistics
  for (int s = 16; s > 0; s >>= 1) {
    spills += __shfl_xor_sync(FULL, spills, s);
    ovfc += __shfl_xor_sync(FULL, ovfc, s);
    dons += __shfl_xor_sync(FULL, dons, s);
  }
  if (COUNTED && lane == 0)
    for (int k = 0; k < 8; ++k) atomicAdd(&a.ctr->phase_cyc[k], ph[k]);
  if (lane == 0) {
    atomicAdd(&a.ctr->chains, nchains);
    atomicAdd(&a.ctr->chain_fb, nchainfb);
    atomicAdd(&a.ctr->items, items);
    atomicAdd(&a.ctr->spills, spills);
    atomicAdd(&a.ctr->ovf, ovfc);
    atomicAdd(&a.ctr->donations, dons);
  }
}

}  // namespace

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
cudaError_t lofp_launch_prep(const CallArgs &a, cudaStream_t s) {
  if (a.B == 0) return cudaSuccess;
  int bs = 256;
  lofp_prep_kernel<<<(unsigned)((a.B + bs - 1) / bs), bs, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t lofp_launch_tables(const CallArgs &a, cudaStream_t s) {
  if (a.nentries == 0) return cudaSuccess;
  int bs = 128;
  lofp_table_kernel<<<(a.nentries + bs - 1) / bs, bs, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t lofp_launch_plan(const CallArgs &a, cudaStream_t s) {
  if (a.B == 0) return cudaSuccess;
  int bs = 64;
  lofp_plan_kernel<<<(unsigned)((a.B + bs - 1) / bs), bs, 0, s>>>(a);
  return cudaGetLastError();
}

// The enumeration kernel variants: validation counters, chain engine, batched short chains
// (the last only on request; it enlarges the engine's code).
static const void *pick_enum(bool counted, bool chain, bool small) {
  if (counted) {
    if (!chain) return (const void *)lofp_enum_kernel<true, false, false>;
    return small ? (const void *)lofp_enum_kernel<true, true, true> : (const void *)lofp_enum_kernel<true, true, false>;
  }
  if (!chain) return (const void *)lofp_enum_kernel<false, false, false>;
  return small ? (const void *)lofp_enum_kernel<false, true, true> : (const void *)lofp_enum_kernel<false, true, false>;
}

cudaError_t lofp_enum_config(const CallArgs &a, bool counted, int *grid, int *block, size_t *smem) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  int sms = 0, maxblk = 0, maxsm = 0;
  e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return e;
  e = cudaDeviceGetAttribute(&maxblk, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (e != cudaSuccess) return e;
  e = cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
  if (e != cudaSuccess) return e;
  const void *fn = pick_enum(counted, a.chain_on != 0, a.small_paths > 0);
  cudaFuncAttributes fa;
  e = cudaFuncGetAttributes(&fa, fn);
  if (e != cudaSuccess) return e;
  // Pick warps per block W and blocks per SM n to maximise resident warps: the staged
  // tables are paid once per block, the per-warp state once per warp.
  const size_t tb = (size_t)a.table_bytes, wbytes = (size_t)a.warp_bytes;
  const int max_w = LOFP_ENUM_MAX_THREADS / 32;
  int regs_warps = fa.numRegs > 0 ? 65536 / (fa.numRegs * 32) : 64;
  int best_w = 0, best_n = 0;
  for (int w = 1; w <= max_w; ++w) {
    size_t per_block = tb + (size_t)w * wbytes + 1024;  // + the per-block reservation
    if (per_block - 1024 > (size_t)maxblk) break;
    int n = (int)((size_t)maxsm / per_block);
    int nw = regs_warps / w;
    if (nw < n) n = nw;
    if (n > 32) n = 32;
    if (n < 1) continue;
    if (n * w > best_n * best_w || (n * w == best_n * best_w && w > best_w)) {
      best_w = w;
      best_n = n;
    }
  }
  if (best_w == 0) return cudaErrorInvalidConfiguration;
  size_t sm = tb + (size_t)best_w * wbytes;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, best_w * 32, sm);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  *grid = per_sm * sms;
  *block = best_w * 32;
  *smem = sm;
  return cudaSuccess;
}

cudaError_t lofp_launch_enum(const CallArgs &a, bool counted, int grid, int block, size_t smem,
                             cudaStream_t s) {
  void *args[] = {const_cast<CallArgs *>(&a)};
  cudaError_t e = cudaLaunchKernel(pick_enum(counted, a.chain_on != 0, a.small_paths > 0), dim3(grid), dim3(block),
                                   args, smem, s);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}
