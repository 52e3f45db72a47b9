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
  PlanFactor *fac = reinterpret_cast<PlanFactor *>(plan + sizeof(PlanHead) + (size_t)a.Lg * sizeof(PlanLevel));
  PlanFactor *tmp = fac + a.nbs;                            // unsorted factors
  uint16_t *att = reinterpret_cast<uint16_t *>(tmp + a.nbs);  // their levels
  const uint16_t zero_off = LOFP_ZERO_OFF;
  const double2 *ent = reinterpret_cast<const double2 *>(a.entries);

  Ref cur[LOFP_MAX_CUTS];
  for (int k = 0; k <= M; ++k) cur[k] = Ref{-1, (int)a.cumS[k]};
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
      pl.pad = 0;
      lev[L] = pl;
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
    PlanFactor pf;
    pf.oa = A.slot < 0 ? zero_off : lofp_level_off(A.slot);
    pf.ob = Bv.slot < 0 ? zero_off : lofp_level_off(Bv.slot);
    pf.oc = C.slot < 0 ? zero_off : lofp_level_off(C.slot);
    pf.oy = Y.slot < 0 ? zero_off : lofp_level_off(Y.slot);
    pf.base = a.bs_base[b] + stride * (cb - ca) + (cc - cb);
    pf.stride = (int16_t)stride;
    pf.dy = (int8_t)(cy - ca);
    pf.dx = (int8_t)(cc - ca);
    tmp[nf] = pf;
    att[nf] = (uint16_t)at;
    ++nf;
  }
  // counting sort of the factors by level
  uint16_t cnt[LOFP_MAX_LEVELS + 1];
  for (int j = 0; j <= L; ++j) cnt[j] = 0;
  for (int f = 0; f < nf; ++f) cnt[att[f] + 1]++;
  for (int j = 0; j < L; ++j) cnt[j + 1] += cnt[j];
  for (int j = 0; j < L; ++j) {
    lev[j].fbeg = cnt[j];
    lev[j].fend = cnt[j + 1];
  }
  for (int f = 0; f < nf; ++f) fac[cnt[att[f]]++] = tmp[f];
  PlanHead h;
  h.root[0] = root.x;
  h.root[1] = root.y;
  h.L = (uint16_t)L;
  h.nfac = (uint16_t)nf;
  h.pad0 = 0;
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
  unsigned long long idx = atomicAdd(&a.ctr->nfeas, 1ull);
  a.feas[idx] = (uint32_t)q;
  atomicAdd(&a.ctr->outstanding, 1ull);
}

// ---------------------------------------------------------------------------
// path enumeration
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ unsigned long long vload(const unsigned long long *p) {
  return *reinterpret_cast<const volatile unsigned long long *>(p);
}

// Per-lane state of the DFS.  vals bytes live in the warp's shared-memory column (lb);
// the branch stack is a ring of LOFP_STK shared-memory entries [bot, top) plus a
// local-memory overflow below it for rare deep stacks.
template <bool COUNTED>
__global__ void __launch_bounds__(LOFP_ENUM_MAX_THREADS, 1) lofp_enum_kernel(CallArgs a) {
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
  unsigned char *vcol = wb + a.plan_smem;                 // vals words [slots/4][32]
  unsigned char *lb = vcol + 4 * lane;                    // this lane's byte base
  double2 *stkP = reinterpret_cast<double2 *>(vcol + a.vals_slots * 32);  // [LOFP_STK][32]
  uint32_t *stkM = reinterpret_cast<uint32_t *>(stkP + LOFP_STK * 32);     // [LOFP_STK][32]
  lb[LOFP_ZERO_OFF] = 0;
  const unsigned nfeas = (unsigned)a.ctr->nfeas;

  double2 ovfP[LOFP_OVF];
  uint32_t ovfM[LOFP_OVF];
  int novf = 0;

  unsigned cur_out = 0xffffffffu;
  const PlanFactor *s_fac = nullptr;
  int L = 0;
  unsigned long long spills = 0, ovfc = 0, dons = 0, items = 0;

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
          if (ns < 1024) ns <<= 1;
        }
      }
    }
    kind = __shfl_sync(FULL, kind, 0);
    if (kind == 0) break;
    out = __shfl_sync(FULL, out, 0);
    tk = __shfl_sync(FULL, tk, 0);
    ++items;

    // ---------------- stage the output's plan ----------------
    if (out != cur_out) {
      const unsigned char *gp = a.plans + (size_t)out * a.plan_stride;
      const PlanHead *gh = reinterpret_cast<const PlanHead *>(gp);
      int Lq = gh->L, nf = gh->nfac;
      // head + levels
      int n16 = 2 + Lq;
      for (int i = lane; i < n16; i += 32)
        reinterpret_cast<int4 *>(s_plan)[i] = reinterpret_cast<const int4 *>(gp)[i];
      // factors (stored after Lg levels in global, after Lq levels in shared)
      const int4 *gf = reinterpret_cast<const int4 *>(gp + sizeof(PlanHead) + (size_t)a.Lg * sizeof(PlanLevel));
      int4 *sf = reinterpret_cast<int4 *>(s_plan + sizeof(PlanHead) + (size_t)Lq * sizeof(PlanLevel));
      for (int i = lane; i < nf; i += 32) sf[i] = gf[i];
      s_fac = reinterpret_cast<const PlanFactor *>(sf);
      L = Lq;
      cur_out = out;
      __syncwarp();
    }
    const PlanHead *sh = reinterpret_cast<const PlanHead *>(s_plan);

    // ---------------- lane 0 begins the item ----------------
    bool working = false;
    int j = 0, bot = 0, top = 0;
    novf = 0;
    double2 Pb = make_double2(0.0, 0.0), acc = make_double2(0.0, 0.0);
    unsigned long long npaths = 0, ncm = 0;
    {
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
        // prefix bytes -> lane 0's column (one word per lane)
        int nw = (j0 + 4) >> 2;  // slots [0, j0]: the zero slot and levels < j0
        const uint32_t *pw = reinterpret_cast<const uint32_t *>(it->prefix);
        for (int w = lane; w < nw; w += 32) *reinterpret_cast<uint32_t *>(vcol + w * 128) = __ldcg(pw + w);
        __syncwarp();
        if (lane == 0) {
          __threadfence();
          *reinterpret_cast<volatile unsigned *>(&it->seq) = 0u;  // slot free again
        }
      }
      if (lane == 0) {
        working = true;
        j = j0;
        lb[lofp_level_off(j0)] = (unsigned char)vs;
        if (ve > vs) {
          stkM[0 * 32 + lane] = (uint32_t)j0 | ((uint32_t)ve << 8);
          stkP[0 * 32 + lane] = P0;
          top = 1;
        }
        Pb = P0;
      }
    }
    __syncwarp();

    unsigned iter = 0;
    while (true) {
      // ---------------- intra-warp hand-over ----------------
      unsigned idle = __ballot_sync(FULL, !working);
      if (idle) {
        unsigned donors = __ballot_sync(FULL, working && (top > bot));
        if (donors == 0) {
          if (idle == FULL) break;  // item finished
        } else {
          int ni = __popc(idle), nd = __popc(donors);
          int n = ni < nd ? ni : nd;
          unsigned lt = lanemask_lt();
          int partner = lane;
          bool recv = false, give = false;
          if (!working) {
            int r = __popc(idle & lt);
            if (r < n) {
              partner = __fns(donors, 0, r + 1);
              recv = true;
            }
          } else if (top > bot) {
            int r = __popc(donors & lt);
            if (r < n) {
              partner = __fns(idle, 0, r + 1);
              give = true;
            }
          }
          int pbot = __shfl_sync(FULL, bot, partner);
          if (recv) {
            int e = pbot % LOFP_STK;
            uint32_t m = stkM[e * 32 + partner];
            double2 P = stkP[e * 32 + partner];
            int jd = m & 0xff, hh = (m >> 8) & 0xff;
            int nw = ((jd + 1) >> 2) + 1;  // words holding slots [0, jd + 1]
            for (int w = 0; w < nw; ++w)
              *reinterpret_cast<uint32_t *>(vcol + w * 128 + 4 * lane) =
                  *reinterpret_cast<const uint32_t *>(vcol + w * 128 + 4 * partner);
            int v = (int)lb[lofp_level_off(jd)] + 1;
            lb[lofp_level_off(jd)] = (unsigned char)v;
            bot = top = 0;
            if (hh > v) {
              stkM[lane] = (uint32_t)jd | ((uint32_t)hh << 8);
              stkP[lane] = P;
              top = 1;
            }
            Pb = P;
            j = jd;
            working = true;
            ++dons;
          }
          __syncwarp();
          if (give) ++bot;
        }
      }

      // ---------------- one DFS node per working lane ----------------
      if (working) {
        PlanLevel lv = s_lev[j];
        double2 P = Pb;
        for (int f = lv.fbeg; f < lv.fend; ++f) {
          PlanFactor fd = s_fac[f];
          int va = lb[fd.oa], vb = lb[fd.ob], vc = lb[fd.oc], vy = lb[fd.oy];
          int row = fd.base + fd.stride * (vb - va) + (vc - vb);
          int o = s_off[row] + (vy - va) + fd.dy;
          P = cmul(P, s_ent[o]);
          if (COUNTED) ncm += (vc - va + fd.dx) > 0;
        }
        if (j == L - 1) {  // a leaf: one valid path of eq. (1)
          acc.x += P.x;
          acc.y += P.y;
          if (COUNTED) ++npaths;
          if (top > bot) {
            int e = (top - 1) % LOFP_STK;
            uint32_t m = stkM[e * 32 + lane];
            int jj = m & 0xff, hh = (m >> 8) & 0xff;
            int v = (int)lb[lofp_level_off(jj)] + 1;
            lb[lofp_level_off(jj)] = (unsigned char)v;
            Pb = stkP[e * 32 + lane];
            if (v == hh) --top;
            j = jj;
          } else if (novf > 0) {
            uint32_t m = ovfM[novf - 1];
            int jj = m & 0xff, hh = (m >> 8) & 0xff;
            int v = (int)lb[lofp_level_off(jj)] + 1;
            lb[lofp_level_off(jj)] = (unsigned char)v;
            Pb = ovfP[novf - 1];
            if (v == hh) --novf;
            j = jj;
          } else {
            working = false;
          }
        } else {  // descend: the next level's exact range (never empty, reading R5)
          int jn = j + 1;
          PlanLevel nl = s_lev[jn];
          int lo = max((int)lb[nl.ol] + nl.cl, (int)nl.lo);
          int hi = min((int)lb[nl.or_] + nl.cr, (int)nl.hi);
          lb[lofp_level_off(jn)] = (unsigned char)lo;
          if (hi > lo) {
            if (top - bot == LOFP_STK) {  // full: move the shallowest entry away
              int e = bot % LOFP_STK;
              uint32_t m = stkM[e * 32 + lane];
              double2 Pe = stkP[e * 32 + lane];
              int jd = m & 0xff, hh = (m >> 8) & 0xff;
              bool pushed = false;
              unsigned long long tl = vload(&a.ctr->tail), tkc = vload(&a.ctr->ticket);
              if (tl < tkc + (a.ring_mask >> 1)) {  // room in the global queue
                atomicAdd(&a.ctr->outstanding, 1ull);
                unsigned long long slot = atomicAdd(&a.ctr->tail, 1ull);
                Item *it = a.ring + (slot & a.ring_mask);
                while (*reinterpret_cast<volatile unsigned *>(&it->seq) != 0u) __nanosleep(64);
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
                pushed = true;
                ++spills;
              }
              if (!pushed) {
                // shift the overflow stack: entries there are shallower than the ring's
                ovfM[novf] = m;
                ovfP[novf] = Pe;
                // keep LIFO order inside overflow: the new entry is deeper than older
                // overflow entries, so it belongs on top
                ++novf;
                ++ovfc;
              }
              ++bot;
            }
            int e = top % LOFP_STK;
            stkM[e * 32 + lane] = (uint32_t)jn | ((uint32_t)hi << 8);
            stkP[e * 32 + lane] = P;
            ++top;
          }
          Pb = P;
          j = jn;
        }
      }

      // ---------------- feed idle warps through the global queue ----------------
      if (((++iter) & 31u) == 0u) {
        long long waiting = 0;
        if (lane == 0) waiting = (long long)(vload(&a.ctr->ticket) - vload(&a.ctr->tail));
        waiting = __shfl_sync(FULL, waiting, 0);
        if (waiting > 0) {
          bool can = working && (top > bot);
          unsigned cands = __ballot_sync(FULL, can);
          int r = __popc(cands & lanemask_lt());
          bool give = can && r < waiting;
          unsigned givers = __ballot_sync(FULL, give);
          if (givers) {
            int leader = __ffs(givers) - 1;
            unsigned long long base = 0;
            if (lane == leader) {
              atomicAdd(&a.ctr->outstanding, (unsigned long long)__popc(givers));
              base = atomicAdd(&a.ctr->tail, (unsigned long long)__popc(givers));
            }
            base = __shfl_sync(FULL, base, leader);
            if (give) {
              unsigned long long slot = base + __popc(givers & lanemask_lt());
              Item *it = a.ring + (slot & a.ring_mask);
              while (*reinterpret_cast<volatile unsigned *>(&it->seq) != 0u) __nanosleep(64);
              int e = bot % LOFP_STK;
              uint32_t m = stkM[e * 32 + lane];
              int jd = m & 0xff, hh = (m >> 8) & 0xff;
              double2 Pe = stkP[e * 32 + lane];
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
              ++bot;
              ++spills;
            }
          }
        }
      }
    }

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
  if (lane == 0) {
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
  const void *fn = counted ? (const void *)lofp_enum_kernel<true> : (const void *)lofp_enum_kernel<false>;
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
  if (counted)
    lofp_enum_kernel<true><<<grid, block, smem, s>>>(a);
  else
    lofp_enum_kernel<false><<<grid, block, smem, s>>>(a);
  return cudaGetLastError();
}
