// lofp_kernels.cu — sm_100a kernels of the LOFP path sum (arXiv 2510.26408).
//
//   lofp_prep_kernel      per output row: validity, photon number, per-mode max of T.
//   lofp_table_kernel     Appendix-A BS elements for every (x1, x2, y1)
//                         inside the paper's light-cone caps, fp64.
//   lofp_feasible_kernel  per output: G = cum(T), exact light-cone reachability
//                         (reading R5), product of the constant factors, compaction.
//   lofp_enum_kernel      persistent path enumeration: each lane runs an iterative DFS
//                         over the free BS outputs (the "green" waveguides),
//                         multiplying fp64 complex Appendix-A factors staged in shared
//                         memory and summing leaves (eq. (1)); subtrees are
//                         balanced through a global atomic work queue.
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
  a.amps[2 * q] = bad ? __longlong_as_double(0x7ff8000000000000ll) : 0.0;
  a.amps[2 * q + 1] = bad ? __longlong_as_double(0x7ff8000000000000ll) : 0.0;
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
// feasibility: G row, exact box at time 0, root product, compaction
// ---------------------------------------------------------------------------
__device__ double2 table_lookup(const int32_t *offsets, const double2 *entries, const FactorDesc &fd,
                                int x1, int x2, int y1) {
  int o = offsets[fd.offbase + x1 * fd.stride + x2] + y1;
  return entries[o];
}

__global__ void lofp_feasible_kernel(CallArgs a) {
  int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= a.B) return;
  if (a.flags[q] != 1) return;  // amps already 0 (photon number) or NaN (bad row)
  const int32_t *t = a.T + q * a.M;
  uint8_t G[LOFP_VALS / 2];
  int g = 0;
  for (int k = 0; k <= a.M; ++k) {
    G[k] = (uint8_t)g;
    if (k < a.M) g += t[k];
  }
  bool ok = true;
  for (int k = 0; k <= a.M; ++k) {
    int f = a.cumS[k];
    if (f < G[a.rho0[k]] || f > G[a.sigma0[k]]) ok = false;
  }
  uint8_t *grow = a.G + q * a.grow;
  for (int k = 0; k <= a.M; ++k) grow[k] = G[k];
  if (!ok) return;  // structurally unreachable: exact zero
  // product of the factors whose inputs are all fixed by S and T
  double2 P = make_double2(1.0, 0.0);
  const double2 *ent = reinterpret_cast<const double2 *>(a.entries);
  for (int f = 0; f < a.nroot; ++f) {
    FactorDesc fd = a.factors[f];
    auto val = [&](uint16_t r) -> int {
      // root factors only reference G (L .. L+M) and cumS (L+M+1 .. L+2M+1)
      int c = r - a.L;
      return c <= a.M ? (int)G[c] : (int)a.cumS[c - a.M - 1];
    };
    int l = val(fd.xl), m = val(fd.xm), r = val(fd.xr), y = val(fd.y);
    int x1 = m - l, x2 = r - m, y1 = y - l;
    if (x1 + x2 == 0) continue;
    P = cmul(P, table_lookup(a.offsets, ent, fd, x1, x2, y1));
  }
  if (a.L == 0) {  // a single valid path (eq. (10))
    a.amps[2 * q] = P.x;
    a.amps[2 * q + 1] = P.y;
    if (a.counts) a.counts[q] = 1;
    return;
  }
  a.root[2 * q] = P.x;
  a.root[2 * q + 1] = P.y;
  unsigned long long idx = atomicAdd(&a.ctr->nfeas, 1ull);
  a.feas[idx] = (uint32_t)q;
  atomicAdd(&a.ctr->outstanding, 1ull);
}

// ---------------------------------------------------------------------------
// path enumeration
// ---------------------------------------------------------------------------
// Lane states
enum : int { ST_NEED = 0, ST_WAIT = 1, ST_WORK = 2, ST_DONE = 3 };

template <bool COUNTED>
__global__ void __launch_bounds__(256) lofp_enum_kernel(CallArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  // shared layout: entries | offsets | levels | factors | cumS
  double2 *s_ent = reinterpret_cast<double2 *>(smem);
  int32_t *s_off = reinterpret_cast<int32_t *>(s_ent + a.nentries);
  LevelDesc *s_lev = reinterpret_cast<LevelDesc *>(
      (reinterpret_cast<uintptr_t>(s_off + a.noffsets) + 15) & ~uintptr_t(15));
  FactorDesc *s_fac = reinterpret_cast<FactorDesc *>(s_lev + a.L);
  uint8_t *s_cumS = reinterpret_cast<uint8_t *>(s_fac + a.nfactors);

  {  // stage the tables (the per-call Appendix-A elements) into shared memory
    const int4 *src = reinterpret_cast<const int4 *>(a.entries);
    int4 *dst = reinterpret_cast<int4 *>(s_ent);
    for (int i = threadIdx.x; i < a.nentries; i += blockDim.x) dst[i] = src[i];
    for (int i = threadIdx.x; i < a.noffsets; i += blockDim.x) s_off[i] = a.offsets[i];
    for (int i = threadIdx.x; i < a.L; i += blockDim.x) s_lev[i] = a.levels[i];
    for (int i = threadIdx.x; i < a.nfactors; i += blockDim.x) s_fac[i] = a.factors[i];
    for (int i = threadIdx.x; i <= a.M; i += blockDim.x) s_cumS[i] = a.cumS[i];
  }
  __syncthreads();

  const int L = a.L, M = a.M;
  const int lane = threadIdx.x & 31;
  const unsigned nfeas = (unsigned)a.ctr->nfeas;
  const double2 *g_root = reinterpret_cast<const double2 *>(a.root);

  // per-lane DFS state (local memory; stack accesses stay near the top)
  uint32_t valw[LOFP_VALS / 4];
  uint8_t *vals = reinterpret_cast<uint8_t *>(valw);
  uint8_t stk_lv[LOFP_STACK];
  uint8_t stk_hi[LOFP_STACK];
  double2 stk_P[LOFP_STACK];
  int sb = 0, sp = 0;  // branch stack [sb, sp)

  int state = ST_NEED;
  unsigned long long ticket = 0;
  unsigned out = 0;
  int j = 0;
  double2 Pcur = make_double2(0.0, 0.0);
  double2 acc = make_double2(0.0, 0.0);
  unsigned long long npaths = 0;
  unsigned iter = 0;

  auto load_g_and_s = [&](unsigned o) {
    // G(0..M) -> vals[L .. L+M]; cumS(0..M) -> vals[L+M+1 .. L+2M+1]
    const uint8_t *g = a.G + (size_t)o * a.grow;
    for (int k = 0; k <= M; ++k) vals[L + k] = g[k];
    for (int k = 0; k <= M; ++k) vals[L + M + 1 + k] = s_cumS[k];
  };

  // Begin a subtree at level j0 with level value range [vs, ve] and product P0.
  auto begin = [&](int j0, int vs, int ve, double2 P0) {
    j = j0;
    vals[j0] = (uint8_t)vs;
    sb = sp = 0;
    if (ve > vs) {
      stk_lv[0] = (uint8_t)j0;
      stk_hi[0] = (uint8_t)ve;
      stk_P[0] = P0;
      sp = 1;
    }
    Pcur = P0;
    acc = make_double2(0.0, 0.0);
    npaths = 0;
  };

  while (true) {
    // ---------------- acquire work ----------------
    unsigned need = __ballot_sync(FULL, state == ST_NEED);
    if (need) {
      unsigned long long base = 0;
      int leader = __ffs(need) - 1;
      int rank = __popc(need & ((1u << lane) - 1));
      if (lane == leader) base = atomicAdd(&a.ctr->fresh_next, (unsigned long long)__popc(need));
      base = __shfl_sync(FULL, base, leader);
      if (state == ST_NEED) {
        unsigned long long idx = base + rank;
        if (idx < nfeas) {
          out = a.feas[idx];
          load_g_and_s(out);
          LevelDesc ld = s_lev[0];
          int lo = max((int)vals[ld.refL], (int)vals[ld.gLo]);
          int hi = min((int)vals[ld.refR], (int)vals[ld.gHi]);
          begin(0, lo, hi, g_root[out]);
          state = ST_WORK;
          atomicAdd(&a.ctr->items, 1ull);
        } else {
          state = ST_WAIT;
        }
      }
    }
    // tickets for lanes that found no fresh output (second ballot: lanes just switched)
    unsigned tk = __ballot_sync(FULL, state == ST_WAIT && ticket == 0);
    if (tk) {
      int leader = __ffs(tk) - 1;
      int rank = __popc(tk & ((1u << lane) - 1));
      unsigned long long base = 0;
      if (lane == leader) base = atomicAdd(&a.ctr->ticket, (unsigned long long)__popc(tk));
      base = __shfl_sync(FULL, base, leader);
      if (state == ST_WAIT && ticket == 0) ticket = base + rank + 1;  // stored +1 (0 = none)
    }
    if (state == ST_WAIT) {
      unsigned long long t = ticket - 1;
      Item *it = a.ring + (t & a.ring_mask);
      unsigned seq = *reinterpret_cast<volatile unsigned *>(&it->seq);
      if (seq == (unsigned)(t + 1)) {
        __threadfence();
        out = it->out;
        int j0 = it->j0;
        const uint32_t *pw = reinterpret_cast<const uint32_t *>(it->prefix);
        for (int w = 0; w < (j0 + 3) / 4; ++w) valw[w] = pw[w];
        load_g_and_s(out);  // after the prefix: its last word may spill past j0
        double2 P0 = make_double2(it->P[0], it->P[1]);
        int vs = it->vs, ve = it->ve;
        __threadfence();
        *reinterpret_cast<volatile unsigned *>(&it->seq) = 0u;  // slot free again
        begin(j0, vs, ve, P0);
        ticket = 0;
        state = ST_WORK;
        atomicAdd(&a.ctr->items, 1ull);
      } else if (*reinterpret_cast<volatile unsigned long long *>(&a.ctr->outstanding) == 0ull) {
        state = ST_DONE;
      }
    }
    if (__all_sync(FULL, state == ST_DONE)) break;

    // ---------------- one DFS node per working lane ----------------
    if (state == ST_WORK) {
      LevelDesc ld = s_lev[j];
      double2 P = Pcur;
      for (int f = ld.fbeg; f < ld.fend; ++f) {
        FactorDesc fd = s_fac[f];
        int vl = vals[fd.xl], vm = vals[fd.xm], vr = vals[fd.xr], vy = vals[fd.y];
        int x1 = vm - vl, x2 = vr - vm, y1 = vy - vl;
        if (x1 + x2 != 0) {
          int o = s_off[fd.offbase + x1 * fd.stride + x2] + y1;
          P = cmul(P, s_ent[o]);
        }
      }
      bool finished = false;
      if (j == L - 1) {  // a leaf: one valid path of eq. (1)
        acc.x += P.x;
        acc.y += P.y;
        if (COUNTED) ++npaths;
        if (sp == sb) {
          finished = true;
        } else {
          int top = sp - 1;
          j = stk_lv[top];
          int v = vals[j] + 1;
          vals[j] = (uint8_t)v;
          Pcur = stk_P[top];
          if (v == stk_hi[top]) sp = top;
        }
      } else {  // descend: next level's exact range (never empty, reading R5)
        ++j;
        LevelDesc nd = s_lev[j];
        int lo = max((int)vals[nd.refL], (int)vals[nd.gLo]);
        int hi = min((int)vals[nd.refR], (int)vals[nd.gHi]);
        vals[j] = (uint8_t)lo;
        if (hi > lo) {
          stk_lv[sp] = (uint8_t)j;
          stk_hi[sp] = (uint8_t)hi;
          stk_P[sp] = P;
          ++sp;
        }
        Pcur = P;
      }
      if (finished) {
        atomicAdd(&a.amps[2 * out], acc.x);
        atomicAdd(&a.amps[2 * out + 1], acc.y);
        if (COUNTED) atomicAdd(&a.counts[out], npaths);
        __threadfence();
        atomicAdd(&a.ctr->outstanding, ~0ull);  // -1
        state = ST_NEED;
      }
    }

    // ---------------- donation: split the shallowest open branch ----------------
    if (((++iter) & 63u) == 0u) {
      long long waiting = 0;
      if (lane == 0) {
        unsigned long long tkc = *reinterpret_cast<volatile unsigned long long *>(&a.ctr->ticket);
        unsigned long long tl = *reinterpret_cast<volatile unsigned long long *>(&a.ctr->tail);
        waiting = (long long)(tkc - tl);
      }
      waiting = __shfl_sync(FULL, waiting, 0);
      if (waiting > 0) {
        bool can = (state == ST_WORK) && (sp > sb);
        unsigned donors = __ballot_sync(FULL, can);
        int rank = __popc(donors & ((1u << lane) - 1));
        bool give = can && rank < waiting;
        unsigned givers = __ballot_sync(FULL, give);
        if (givers) {
          int leader = __ffs(givers) - 1;
          unsigned long long base = 0;
          if (lane == leader) {
            atomicAdd(&a.ctr->outstanding, (unsigned long long)__popc(givers));
            atomicAdd(&a.ctr->donations, (unsigned long long)__popc(givers));
            base = atomicAdd(&a.ctr->tail, (unsigned long long)__popc(givers));
          }
          base = __shfl_sync(FULL, base, leader);
          if (give) {
            unsigned long long t = base + __popc(givers & ((1u << lane) - 1));
            Item *it = a.ring + (t & a.ring_mask);
            while (*reinterpret_cast<volatile unsigned *>(&it->seq) != 0u) {
            }  // previous occupant not consumed yet (cannot happen within the ring bound)
            int jd = stk_lv[sb];
            it->out = out;
            it->j0 = (unsigned short)jd;
            it->vs = (unsigned char)(vals[jd] + 1);
            it->ve = stk_hi[sb];
            it->P[0] = stk_P[sb].x;
            it->P[1] = stk_P[sb].y;
            uint32_t *pw = reinterpret_cast<uint32_t *>(it->prefix);
            for (int w = 0; w < (jd + 3) / 4; ++w) pw[w] = valw[w];
            ++sb;  // this lane no longer owns the rest of that level
            __threadfence();
            *reinterpret_cast<volatile unsigned *>(&it->seq) = (unsigned)(t + 1);
          }
        }
      }
    }
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

cudaError_t lofp_launch_feasible(const CallArgs &a, cudaStream_t s) {
  if (a.B == 0) return cudaSuccess;
  int bs = 128;
  lofp_feasible_kernel<<<(unsigned)((a.B + bs - 1) / bs), bs, 0, s>>>(a);
  return cudaGetLastError();
}

static size_t enum_smem(const CallArgs &a) {
  size_t b = (size_t)a.nentries * 16 + (size_t)a.noffsets * 4;
  b = (b + 15) & ~size_t(15);
  b += (size_t)a.L * sizeof(LevelDesc) + (size_t)a.nfactors * sizeof(FactorDesc) + (size_t)(a.M + 1);
  return (b + 15) & ~size_t(15);
}

cudaError_t lofp_enum_config(const CallArgs &a, bool counted, int *grid, int *block, size_t *smem) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  int sms = 0;
  e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return e;
  size_t sm = enum_smem(a);
  const void *fn = counted ? (const void *)lofp_enum_kernel<true> : (const void *)lofp_enum_kernel<false>;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  int bt = 256, per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, bt, sm);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  *grid = per_sm * sms;
  *block = bt;
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
