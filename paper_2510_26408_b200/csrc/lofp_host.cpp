// lofp_host.cpp — host side of liblofp: the C ABI of include/lofp.h, circuit
// canonicalisation, the column / light-cone topology tables, per-call buffer sizing and
// the kernel launches.  See DESIGN.md for the derivations (readings R1-R20) and the paper
// passages each step follows.  No call here waits for the device except lofp_create
// (one upload), lofp_stats, lofp_amplitudes_host and lofp_destroy.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>  // tracing: one NVTX range per API call (header-only NVTX v3)

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "../../include/lofp.h"
#include "lofp_internal.h"

using namespace lofp;

namespace {

constexpr double kPi = 3.14159265358979323846;

struct DevBuf {
  void *p = nullptr;
  size_t n = 0;
  cudaError_t ensure(size_t bytes) {
    if (bytes <= n && p) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    cudaError_t e = cudaMalloc(&p, bytes ? bytes : 16);
    if (e == cudaSuccess) n = bytes;
    return e;
  }
  // stream-ordered growth: the old block is freed after the work already queued on the
  // stream, the new one allocated before the work that follows (no host synchronisation)
  cudaError_t ensure_async(size_t bytes, cudaStream_t st) {
    if (bytes <= n && p) return cudaSuccess;
    if (p) cudaFreeAsync(p, st);
    p = nullptr;
    n = 0;
    cudaError_t e = cudaMallocAsync(&p, bytes ? bytes : 16, st);
    if (e == cudaSuccess) n = bytes;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
};

struct HostPinned {
  void *p = nullptr;
  size_t n = 0;
  cudaError_t ensure(size_t bytes) {
    if (bytes <= n && p) return cudaSuccess;
    if (p) cudaFreeHost(p);
    p = nullptr;
    n = 0;
    cudaError_t e = cudaMallocHost(&p, bytes ? bytes : 16);
    if (e == cudaSuccess) n = bytes;
    return e;
  }
  void release() {
    if (p) cudaFreeHost(p);
    p = nullptr;
    n = 0;
  }
};

// A beam splitter after canonicalisation: port 1 = mode cut-1, port 2 = mode cut.
struct CanonBS {
  int layer;  // 1-based
  int cut;    // k = max(mode_a, mode_b): the upper mode
  int lo;     // min(mode_a, mode_b): the lower mode (port 1 after canonicalisation)
  double theta, phi;
};

struct Mask {  // a set of modes (M <= 128)
  uint64_t w[2] = {0, 0};
  void set(int m) { w[m >> 6] |= 1ull << (m & 63); }
  bool has(int m) const { return (w[m >> 6] >> (m & 63)) & 1ull; }
};

long long env_ll(const char *name, long long dflt) {
  const char *v = std::getenv(name);
  if (!v || !*v) return dflt;
  char *end = nullptr;
  long long x = std::strtoll(v, &end, 10);
  return (end && *end == 0 && x > 0) ? x : dflt;
}

}  // namespace

struct lofp_ctx {
  int device = 0;
  int M = 0, D = 0, nbs = 0, ngate = 0;
  std::vector<CanonBS> bs;
  // topology (lofp_internal.h)
  std::vector<ColInfo> col;
  std::vector<SegInfo> seg;
  std::vector<CmpPair> cmp;
  std::vector<FacInfo> fac;
  std::vector<GateInfo> gat;
  std::vector<BSInfo> bsi;
  std::vector<EqCon> eqc;
  std::vector<BoundInfo> bnd;
  bool general = false;  // non-local pairs (NEXT-4)
  std::vector<SeqBS> seq;      // generic engine: layer-major BS order
  std::vector<uint64_t> cone;  // generic engine: past / future cone masks per waveguide
  int seq_gl0 = 0;
  std::vector<double> gate_ab;
  std::vector<int16_t> gate_mode, gate_after;
  DevBuf d_topo;
  size_t off_col = 0, off_seg = 0, off_cmp = 0, off_fac = 0, off_gat = 0, off_bsi = 0, off_gab = 0, off_gm = 0,
         off_gl = 0, off_eqc = 0, off_bnd = 0, off_seq = 0, off_cone = 0;
  // per-call device buffers
  DevBuf d_tableA, d_tabAoff;  // contraction: the x1-linear copy of the tables (lofp_tableA_kernel)
  DevBuf d_table, d_taboff, d_gatetab, d_units, d_sched, d_nunits, d_ubase, d_status, d_pexp, d_pdone, d_partial, d_slab,
      d_ctr, d_hostT, d_hostA;
  HostPinned h_ctr;
  long long table_entries = 0, tableA_entries = 0;
  int grid = 0;
  long long slab_bytes = 0;
  unsigned long long path_budget = 0;  // lofp_set_path_budget
  cudaEvent_t ev_start = nullptr, ev_u0 = nullptr, ev_u1 = nullptr, ev_end = nullptr;
  bool have_call = false, timed = false;
  lofp_run_stats stats{};
  std::string err;
  cudaStream_t own_stream = nullptr;
};

namespace {

lofp_status fail(lofp_ctx *ctx, lofp_status s, const std::string &msg) {
  if (ctx) ctx->err = msg;
  return s;
}

#define CK(call, what)                                                                          \
  do {                                                                                          \
    cudaError_t e_ = (call);                                                                    \
    if (e_ != cudaSuccess)                                                                      \
      return fail(ctx, e_ == cudaErrorMemoryAllocation ? LOFP_E_OOM : LOFP_E_CUDA,             \
                  std::string(what) + ": " + cudaGetErrorString(e_));                          \
  } while (0)

struct DeviceGuard {  // restores the caller's current device
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

// Column / light-cone topology of the circuit (readings R5, R15, R20).
lofp_status build_topology(lofp_ctx *ctx, const std::vector<lofp_gate> &gates) {
  const int M = ctx->M, D = ctx->D, W = M + 1;
  std::vector<int> act((size_t)(D + 1) * W, -1);  // act[l][k] = BS index or -1
  for (int i = 0; i < ctx->nbs; ++i) act[(size_t)ctx->bs[i].layer * W + ctx->bs[i].cut] = i;
  auto A = [&](int l, int k) { return act[(size_t)l * W + k] >= 0; };
  // backward maps (from T): F_l(k) in [G(rho_l(k)), G(sig_l(k))]   (reading R5)
  std::vector<int> rho((size_t)(D + 1) * W), sig((size_t)(D + 1) * W);
  // forward maps (from S): F_l(k) in [cumS(rhop_l(k)), cumS(sigp_l(k))]  (reading R15)
  std::vector<int> rhop((size_t)(D + 1) * W), sigp((size_t)(D + 1) * W);
  for (int k = 0; k <= M; ++k) {
    rho[(size_t)D * W + k] = sig[(size_t)D * W + k] = k;
    rhop[k] = sigp[k] = k;
  }
  for (int l = D; l >= 1; --l)
    for (int k = 0; k <= M; ++k) {
      const bool a = A(l, k);
      rho[(size_t)(l - 1) * W + k] = a ? rho[(size_t)l * W + k - 1] : rho[(size_t)l * W + k];
      sig[(size_t)(l - 1) * W + k] = a ? sig[(size_t)l * W + k + 1] : sig[(size_t)l * W + k];
    }
  for (int l = 1; l <= D; ++l)
    for (int k = 0; k <= M; ++k) {
      const bool a = A(l, k);
      rhop[(size_t)l * W + k] = a ? rhop[(size_t)(l - 1) * W + k - 1] : rhop[(size_t)(l - 1) * W + k];
      sigp[(size_t)l * W + k] = a ? sigp[(size_t)(l - 1) * W + k + 1] : sigp[(size_t)(l - 1) * W + k];
    }
  // segments of every column: F(k) is constant between consecutive active layers of cut k
  std::vector<std::vector<int>> al(W);         // active layers of cut k
  std::vector<std::vector<int>> segof(W);      // time t -> segment index
  for (int k = 0; k <= M; ++k) {
    for (int l = 1; l <= D; ++l)
      if (A(l, k)) al[k].push_back(l);
    segof[k].assign(D + 1, 0);
    int s = 0;
    for (int t = 0; t <= D; ++t) {
      if (s < (int)al[k].size() && al[k][s] == t) ++s;
      segof[k][t] = s;
    }
  }
  ctx->col.assign(W, ColInfo{});
  ctx->seg.clear();
  ctx->cmp.clear();
  ctx->fac.clear();
  ctx->gat.clear();
  // gates by cut: a gate on mode m reads columns m and m+1 -> folded into cut m+1
  // (or cut M-1 for the last mode); M == 1 has no cut: the kernels multiply those in.
  std::vector<std::vector<GateInfo>> gates_of(W);
  for (size_t g = 0; g < gates.size(); ++g) {
    const int m = gates[g].mode, j = gates[g].after_layer;
    if (M == 1) continue;
    const int c = (m + 1 <= M - 1) ? m + 1 : m;
    GateInfo gi{};
    gi.gate = (int32_t)g;
    gi.col_off = (uint8_t)(m - (c - 1));
    gi.seg_lo = (uint8_t)segof[m][j];
    gi.seg_hi = (uint8_t)segof[m + 1][j];
    gates_of[c].push_back(gi);
  }
  for (int k = 0; k <= M; ++k) {
    ColInfo &ci = ctx->col[k];
    const int nseg = (int)al[k].size() + 1;
    if (ctx->seg.size() + nseg > 8192 || nseg > 255) return LOFP_E_UNSUPPORTED;
    ci.seg_base = (uint16_t)ctx->seg.size();
    ci.nseg = (uint8_t)nseg;
    ci.nvar = (uint8_t)nseg;
    for (int i = 0; i < nseg; ++i) {
      const int t0 = i == 0 ? 0 : al[k][i - 1];
      SegInfo si;
      si.rho = (uint8_t)rho[(size_t)t0 * W + k];
      si.sig = (uint8_t)sig[(size_t)t0 * W + k];
      si.rhop = (uint8_t)rhop[(size_t)t0 * W + k];
      si.sigp = (uint8_t)sigp[(size_t)t0 * W + k];
      ctx->seg.push_back(si);
    }
    // adjacent-column constraints F_t(k-1) <= F_t(k), one check per time interval
    ci.cmp_base = (uint16_t)ctx->cmp.size();
    int ncmp = 0;
    if (k >= 1) {
      int la = -1, lb = -1;
      for (int t = 0; t <= D; ++t) {
        const int sa = segof[k - 1][t], sb = segof[k][t];
        if (sa == la && sb == lb) continue;
        ctx->cmp.push_back(CmpPair{(uint8_t)sa, (uint8_t)sb});
        la = sa;
        lb = sb;
        ++ncmp;
      }
    }
    if (ncmp > 255 || ctx->cmp.size() > 65535) return LOFP_E_UNSUPPORTED;
    ci.ncmp = (uint8_t)ncmp;
    // the BS of cut k, in layer order (its cut factor, eq. (1))
    ci.fac_base = (uint16_t)ctx->fac.size();
    int nfac = 0;
    if (k >= 1 && k <= M - 1) {
      for (int i = 0; i < (int)al[k].size(); ++i) {
        const int l = al[k][i];
        FacInfo fi{};
        fi.bs = act[(size_t)l * W + k];
        fi.sA = (uint8_t)segof[k - 1][l - 1];
        fi.i = (uint8_t)i;
        fi.sC = (uint8_t)segof[k + 1][l - 1];
        ctx->fac.push_back(fi);
        ++nfac;
      }
    }
    if (nfac > 255 || ctx->fac.size() > 65535) return LOFP_E_UNSUPPORTED;
    ci.nfac = (uint8_t)nfac;
    ci.gate_base = (uint16_t)ctx->gat.size();
    ci.ngate = (uint8_t)std::min<size_t>(gates_of[k].size(), 255);
    if (gates_of[k].size() > 255 || ctx->gat.size() + gates_of[k].size() > 65535) return LOFP_E_UNSUPPORTED;
    for (const GateInfo &g : gates_of[k]) ctx->gat.push_back(g);
  }
  // BS parameters and the past-cone photon bound that sizes their Appendix-A blocks
  ctx->bsi.assign(std::max(ctx->nbs, 1), BSInfo{});
  for (int i = 0; i < ctx->nbs; ++i) {
    const CanonBS &b = ctx->bs[i];
    BSInfo &bi = ctx->bsi[i];
    bi.c = std::cos(b.theta);
    bi.s = std::sin(b.theta);
    bi.phi = b.phi;
    bi.cap_lo = (uint8_t)rhop[(size_t)(b.layer - 1) * W + b.cut - 1];
    bi.cap_hi = (uint8_t)sigp[(size_t)(b.layer - 1) * W + b.cut + 1];
  }
  ctx->ngate = (int)gates.size();
  ctx->gate_ab.assign(2 * std::max<size_t>(gates.size(), 1), 0.0);
  ctx->gate_mode.assign(std::max<size_t>(gates.size(), 1), 0);
  ctx->gate_after.assign(std::max<size_t>(gates.size(), 1), 0);
  for (size_t g = 0; g < gates.size(); ++g) {
    ctx->gate_ab[2 * g] = gates[g].a;
    ctx->gate_ab[2 * g + 1] = gates[g].b;
    ctx->gate_mode[g] = (int16_t)gates[g].mode;
    ctx->gate_after[g] = (int16_t)gates[g].after_layer;
  }
  return LOFP_OK;
}

// Column topology of a circuit with non-local pairs (NEXT-4, reading R21).  A BS
// on modes (a, b) changes F(k) for every cut k in (a, b] by y1 - x1; columns in its span get
// a segment break.  A BS whose span covers more than one cut, or whose cut another BS of the
// same layer also spans, is "carried": its (x1, y1) are state variables of the columns
// a+1..b, defined from columns (a, a+1), passed on unchanged, and consumed at cut b by its
// factor and by the conservation check of mode b.  Idle modes inside a span keep their
// occupation.  All checks are between adjacent columns (EqCon), so the column machinery
// (counts, lists, contraction) is unchanged.  The light-cone bounds become sums over mode
// sets (P:153-164 cones of a set of modes).
lofp_status build_topology_general(lofp_ctx *ctx, const std::vector<lofp_gate> &gates) {
  const int M = ctx->M, D = ctx->D, W = M + 1, nb = ctx->nbs;
  std::vector<std::vector<int>> layer_bs(D + 1);
  std::vector<int> owner((size_t)(D + 1) * std::max(M, 1), -1);
  std::vector<int> nspan((size_t)(D + 1) * W, 0);
  for (int i = 0; i < nb; ++i) {
    const CanonBS &b = ctx->bs[i];
    layer_bs[b.layer].push_back(i);
    owner[(size_t)b.layer * M + b.lo] = i;
    owner[(size_t)b.layer * M + b.cut] = i;
    for (int k = b.lo + 1; k <= b.cut; ++k) nspan[(size_t)b.layer * W + k]++;
  }
  auto spanned = [&](int l, int k) { return nspan[(size_t)l * W + k] > 0; };
  std::vector<char> carried(nb, 0);
  for (int i = 0; i < nb; ++i) {
    const CanonBS &b = ctx->bs[i];
    carried[i] = (b.cut - b.lo > 1) || nspan[(size_t)b.layer * W + b.cut] > 1;
  }
  std::vector<std::vector<int>> al(W), segof(W);
  for (int k = 0; k <= M; ++k) {
    for (int l = 1; l <= D; ++l)
      if (spanned(l, k)) al[k].push_back(l);
    segof[k].assign(D + 1, 0);
    int s = 0;
    for (int t = 0; t <= D; ++t) {
      if (s < (int)al[k].size() && al[k][s] == t) ++s;
      segof[k][t] = s;
    }
  }
  auto past = [&](int t, Mask X) {  // input modes that can reach X by time t
    for (int l = t; l >= 1; --l)
      for (int i : layer_bs[l]) {
        const CanonBS &b = ctx->bs[i];
        if (X.has(b.lo) || X.has(b.cut)) {
          X.set(b.lo);
          X.set(b.cut);
        }
      }
    return X;
  };
  auto fut = [&](int t, Mask X) {  // output modes reachable from X after time t
    for (int l = t + 1; l <= D; ++l)
      for (int i : layer_bs[l]) {
        const CanonBS &b = ctx->bs[i];
        if (X.has(b.lo) || X.has(b.cut)) {
          X.set(b.lo);
          X.set(b.cut);
        }
      }
    return X;
  };
  Mask all;
  for (int m = 0; m < M; ++m) all.set(m);
  auto range_mask = [&](int a, int e) {
    Mask X;
    for (int m = a; m < e; ++m) X.set(m);
    return X;
  };
  auto bound = [&](Mask m0, Mask m1, Mask m2, Mask m3) {
    BoundInfo bi{};
    const Mask ms[4] = {m0, m1, m2, m3};
    for (int w = 0; w < 4; ++w)
      for (int h = 0; h < 2; ++h) bi.m[w][h] = ms[w].w[h];
    return bi;
  };
  // variables: the segments of each column, then (x1, y1) of every carried BS spanning it
  std::vector<std::vector<int>> cvar(nb);  // cvar[i][k - lo - 1] = x1's variable index in column k
  std::vector<int> nvar(W, 0);
  for (int k = 0; k <= M; ++k) nvar[k] = (int)al[k].size() + 1;
  for (int i = 0; i < nb; ++i) {
    if (!carried[i]) continue;
    const CanonBS &b = ctx->bs[i];
    for (int k = b.lo + 1; k <= b.cut; ++k) {
      cvar[i].push_back(nvar[k]);
      nvar[k] += 2;
    }
  }
  ctx->col.assign(W, ColInfo{});
  ctx->seg.clear();
  ctx->bnd.clear();
  ctx->cmp.clear();
  ctx->eqc.clear();
  ctx->fac.clear();
  ctx->gat.clear();
  std::vector<std::vector<GateInfo>> gates_of(W);
  for (size_t g = 0; g < gates.size(); ++g) {
    const int m = gates[g].mode, j = gates[g].after_layer;
    if (M == 1) continue;
    const int c = (m + 1 <= M - 1) ? m + 1 : m;
    GateInfo gi{};
    gi.gate = (int32_t)g;
    gi.col_off = (uint8_t)(m - (c - 1));
    gi.seg_lo = (uint8_t)segof[m][j];
    gi.seg_hi = (uint8_t)segof[m + 1][j];
    gates_of[c].push_back(gi);
  }
  for (int k = 0; k <= M; ++k) {
    ColInfo &ci = ctx->col[k];
    const int nseg = (int)al[k].size() + 1;
    if (ctx->seg.size() + nvar[k] > 8192 || nvar[k] > 127) return LOFP_E_UNSUPPORTED;
    ci.seg_base = (uint16_t)ctx->seg.size();
    ci.nseg = (uint8_t)nseg;
    ci.nvar = (uint8_t)nvar[k];
    for (int i = 0; i < nseg; ++i) {
      const int t0 = i == 0 ? 0 : al[k][i - 1];
      const Mask lo = range_mask(0, k), hi = range_mask(k, M);
      ctx->seg.push_back(SegInfo{});
      ctx->bnd.push_back(bound(past(t0, lo), past(t0, hi), fut(t0, lo), fut(t0, hi)));
    }
    std::vector<BoundInfo> extra(nvar[k] - nseg);
    for (int i = 0; i < nb; ++i) {
      if (!carried[i]) continue;
      const CanonBS &b = ctx->bs[i];
      if (k <= b.lo || k > b.cut) continue;
      Mask a;
      a.set(b.lo);
      const int v = cvar[i][k - b.lo - 1] - nseg;
      extra[v] = bound(past(b.layer - 1, a), all, fut(b.layer - 1, a), all);      // x1: mode a before
      extra[v + 1] = bound(past(b.layer, a), all, fut(b.layer, a), all);          // y1: mode a after
    }
    for (const BoundInfo &e : extra) {
      ctx->seg.push_back(SegInfo{});
      ctx->bnd.push_back(e);
    }
    // F_t(k-1) <= F_t(k) at every time
    ci.cmp_base = (uint16_t)ctx->cmp.size();
    int ncmp = 0;
    if (k >= 1) {
      int la = -1, lb = -1;
      for (int t = 0; t <= D; ++t) {
        const int sa = segof[k - 1][t], sb = segof[k][t];
        if (sa == la && sb == lb) continue;
        ctx->cmp.push_back(CmpPair{(uint8_t)sa, (uint8_t)sb});
        la = sa;
        lb = sb;
        ++ncmp;
      }
    }
    if (ncmp > 255 || ctx->cmp.size() > 65535) return LOFP_E_UNSUPPORTED;
    ci.ncmp = (uint8_t)ncmp;
    // equalities between columns k-1 and k (mode m = k-1 and the carried variables)
    int neq = 0;
    auto add_eq = [&](std::vector<std::pair<int, int>> terms) {  // (coef, side<<7 | var)
      std::vector<std::pair<int, int>> merged;
      for (auto &t : terms) {
        bool found = false;
        for (auto &u : merged)
          if (u.second == t.second) {
            u.first += t.first;
            found = true;
          }
        if (!found) merged.push_back(t);
      }
      EqCon e{};
      int n = 0;
      for (auto &u : merged)
        if (u.first != 0 && n < 11) {
          e.coef[n] = (int8_t)u.first;
          e.var[n] = (uint8_t)u.second;
          ++n;
        }
      if (n == 0) return;
      e.nterm = (uint8_t)n;
      ctx->eqc.push_back(e);
      ++neq;
    };
    // inside column k: at every layer whose spanning BSs are carried, the jump of F(k) is
    // the sum of their y1 - x1 (photon conservation of the BSs crossing cut k)
    ci.intra_base = (uint16_t)ctx->eqc.size();
    int nintra = 0;
    for (int l = 1; l <= D; ++l) {
      if (!spanned(l, k)) continue;
      std::vector<std::pair<int, int>> terms{{1, 0x80 | segof[k][l]}, {-1, 0x80 | segof[k][l - 1]}};
      bool any_carried = false;
      for (int i : layer_bs[l]) {
        const CanonBS &b = ctx->bs[i];
        if (k <= b.lo || k > b.cut || !carried[i]) continue;
        any_carried = true;
        const int xv = 0x80 | cvar[i][k - b.lo - 1];
        terms.push_back({-1, xv + 1});
        terms.push_back({1, xv});
      }
      if (!any_carried) continue;
      if (terms.size() > 11) return LOFP_E_UNSUPPORTED;
      const size_t before = ctx->eqc.size();
      const int save = neq;
      add_eq(terms);
      if (ctx->eqc.size() > before) ++nintra;
      neq = save;
    }
    ci.nintra = (uint8_t)nintra;
    ci.eq_base = (uint16_t)ctx->eqc.size();
    neq = 0;
    if (k >= 1) {
      const int m = k - 1;
      for (int l = 1; l <= D; ++l) {
        const int a0 = segof[k - 1][l - 1], a1 = segof[k - 1][l];
        const int b0 = 0x80 | segof[k][l - 1], b1 = 0x80 | segof[k][l];
        const int o = owner[(size_t)l * M + m];
        if (o < 0) {  // idle mode: its occupation is unchanged
          if (spanned(l, k)) add_eq({{1, b1}, {-1, b0}, {-1, a1}, {1, a0}});
        } else if (carried[o]) {
          const CanonBS &b = ctx->bs[o];
          if (b.lo == m) {  // x1 = n_m before, y1 = n_m after
            const int xv = 0x80 | cvar[o][0];
            add_eq({{1, xv}, {-1, b0}, {1, a0}});
            add_eq({{1, xv + 1}, {-1, b1}, {1, a1}});
          } else {  // upper mode: n_m changes by -(y1 - x1)
            const int xv = cvar[o][b.cut - b.lo - 1];
            add_eq({{1, b1}, {-1, a1}, {-1, b0}, {1, a0}, {1, xv + 1}, {-1, xv}});
          }
        }
      }
      for (int i = 0; i < nb; ++i) {  // carried variables pass through the span unchanged
        if (!carried[i]) continue;
        const CanonBS &b = ctx->bs[i];
        if (k - 1 > b.lo && k <= b.cut) {
          const int xa = cvar[i][k - 1 - b.lo - 1], xb = 0x80 | cvar[i][k - b.lo - 1];
          add_eq({{1, xa}, {-1, xb}});
          add_eq({{1, xa + 1}, {-1, xb + 1}});
        }
      }
    }
    if (neq > 255 || ctx->eqc.size() > 65535) return LOFP_E_UNSUPPORTED;
    ci.neq = (uint8_t)neq;
    // factors carried by cut k: NN BS on (k-1, k), carried BS ending at mode k
    ci.fac_base = (uint16_t)ctx->fac.size();
    int nfac = 0;
    if (k >= 1 && k <= M - 1) {
      for (int i = 0; i < nb; ++i) {
        const CanonBS &b = ctx->bs[i];
        if (b.cut != k) continue;
        const int l = b.layer;
        FacInfo fi{};
        fi.bs = i;
        fi.sC = (uint8_t)segof[k + 1][l - 1];
        if (!carried[i]) {
          fi.kind = 0;
          fi.sA = (uint8_t)segof[k - 1][l - 1];
          fi.i = (uint8_t)segof[k][l - 1];
        } else {
          const int xv = cvar[i][k - b.lo - 1];
          fi.kind = 1;
          fi.i = (uint8_t)xv;
          fi.sA = (uint8_t)(xv + 1);
          fi.sB = (uint8_t)segof[k][l - 1];
        }
        ctx->fac.push_back(fi);
        ++nfac;
      }
    }
    if (nfac > 255 || ctx->fac.size() > 65535) return LOFP_E_UNSUPPORTED;
    ci.nfac = (uint8_t)nfac;
    ci.gate_base = (uint16_t)ctx->gat.size();
    if (gates_of[k].size() > 255 || ctx->gat.size() + gates_of[k].size() > 65535) return LOFP_E_UNSUPPORTED;
    ci.ngate = (uint8_t)gates_of[k].size();
    for (const GateInfo &g : gates_of[k]) ctx->gat.push_back(g);
  }
  ctx->bsi.assign(std::max(nb, 1), BSInfo{});
  for (int i = 0; i < nb; ++i) {
    const CanonBS &b = ctx->bs[i];
    BSInfo &bi = ctx->bsi[i];
    bi.c = std::cos(b.theta);
    bi.s = std::sin(b.theta);
    bi.phi = b.phi;
    Mask ab;
    ab.set(b.lo);
    ab.set(b.cut);
    const Mask pc = past(b.layer - 1, ab);
    bi.capmask[0] = pc.w[0];
    bi.capmask[1] = pc.w[1];
  }
  ctx->ngate = (int)gates.size();
  ctx->gate_ab.assign(2 * std::max<size_t>(gates.size(), 1), 0.0);
  ctx->gate_mode.assign(std::max<size_t>(gates.size(), 1), 0);
  ctx->gate_after.assign(std::max<size_t>(gates.size(), 1), 0);
  for (size_t g = 0; g < gates.size(); ++g) {
    ctx->gate_ab[2 * g] = gates[g].a;
    ctx->gate_ab[2 * g + 1] = gates[g].b;
    ctx->gate_mode[g] = (int16_t)gates[g].mode;
    ctx->gate_after[g] = (int16_t)gates[g].after_layer;
  }
  return LOFP_OK;
}

// Tables of the generic engine (the paper's layer-major recursion, with the
// per-waveguide light-cone bounds of P:164): the BS order, the layers whose gates follow
// each BS, and the past / future cone of every waveguide (mode m after layer t).
void build_generic(lofp_ctx *ctx) {
  const int M = ctx->M, D = ctx->D, nb = ctx->nbs;
  ctx->seq.clear();
  for (int i = 0; i < nb; ++i) {
    const CanonBS &b = ctx->bs[i];
    SeqBS q{};
    q.bs = i;
    q.lo = (uint8_t)b.lo;
    q.hi = (uint8_t)b.cut;
    q.layer = (uint8_t)b.layer;
    const bool last_of_layer = (i + 1 == nb) || ctx->bs[i + 1].layer != b.layer;
    if (last_of_layer) {
      q.gl0 = (uint8_t)b.layer;
      q.gl1 = (uint8_t)((i + 1 == nb) ? D + 1 : ctx->bs[i + 1].layer);
    }
    ctx->seq.push_back(q);
  }
  ctx->seq_gl0 = nb > 0 ? ctx->bs[0].layer : D + 1;
  ctx->cone.assign((size_t)(D + 1) * std::max(M, 1) * 4, 0);
  std::vector<std::vector<int>> layer_bs(D + 1);
  for (int i = 0; i < nb; ++i) layer_bs[ctx->bs[i].layer].push_back(i);
  auto grow = [&](Mask X, int l) {
    for (int i : layer_bs[l]) {
      const CanonBS &b = ctx->bs[i];
      if (X.has(b.lo) || X.has(b.cut)) {
        X.set(b.lo);
        X.set(b.cut);
      }
    }
    return X;
  };
  for (int t = 0; t <= D; ++t)
    for (int m = 0; m < M; ++m) {
      Mask pa, fu;
      pa.set(m);
      fu.set(m);
      for (int l = t; l >= 1; --l) pa = grow(pa, l);
      for (int l = t + 1; l <= D; ++l) fu = grow(fu, l);
      uint64_t *c = &ctx->cone[((size_t)t * M + m) * 4];
      c[0] = pa.w[0];
      c[1] = pa.w[1];
      c[2] = fu.w[0];
      c[3] = fu.w[1];
    }
}

template <class T>
size_t append(std::vector<char> &blob, const std::vector<T> &v) {
  size_t off = (blob.size() + 15) & ~size_t(15);
  blob.resize(off + std::max<size_t>(v.size(), 1) * sizeof(T), 0);
  if (!v.empty()) std::memcpy(blob.data() + off, v.data(), v.size() * sizeof(T));
  return off;
}

lofp_status upload_topology(lofp_ctx *ctx) {
  std::vector<char> blob;
  ctx->off_col = append(blob, ctx->col);
  ctx->off_seg = append(blob, ctx->seg);
  ctx->off_cmp = append(blob, ctx->cmp);
  ctx->off_fac = append(blob, ctx->fac);
  ctx->off_gat = append(blob, ctx->gat);
  ctx->off_bsi = append(blob, ctx->bsi);
  ctx->off_gab = append(blob, ctx->gate_ab);
  ctx->off_gm = append(blob, ctx->gate_mode);
  ctx->off_gl = append(blob, ctx->gate_after);
  ctx->off_eqc = append(blob, ctx->eqc);
  ctx->off_bnd = append(blob, ctx->bnd);
  ctx->off_seq = append(blob, ctx->seq);
  ctx->off_cone = append(blob, ctx->cone);
  CK(ctx->d_topo.ensure(blob.size()), "alloc topology");
  CK(cudaMemcpy(ctx->d_topo.p, blob.data(), blob.size(), cudaMemcpyHostToDevice), "upload topology");
  return LOFP_OK;
}

lofp_status create_impl(int32_t modes, int32_t n_layers, const int32_t *bs_per_layer, const lofp_bs *bs,
                        int32_t n_gates, const lofp_gate *gates, lofp_ctx **out) {
  if (!out) return LOFP_E_INVALID_ARG;
  *out = nullptr;
  if (modes < 1 || n_layers < 0 || n_gates < 0) return LOFP_E_INVALID_ARG;
  if (modes > LOFP_MAX_MODES || n_layers > LOFP_MAX_LAYERS || n_gates > LOFP_MAX_GATES) return LOFP_E_UNSUPPORTED;
  if (n_layers > 0 && !bs_per_layer) return LOFP_E_INVALID_ARG;
  if (n_gates > 0 && !gates) return LOFP_E_INVALID_ARG;
  int64_t total = 0;
  for (int l = 0; l < n_layers; ++l) {
    if (bs_per_layer[l] < 0) return LOFP_E_INVALID_ARG;
    total += bs_per_layer[l];
  }
  if (total > 0 && !bs) return LOFP_E_INVALID_ARG;
  if (total > 65535) return LOFP_E_UNSUPPORTED;
  std::vector<lofp_gate> gv;
  for (int g = 0; g < n_gates; ++g) {
    const lofp_gate &x = gates[g];
    if (x.mode < 0 || x.mode >= modes || x.after_layer < 0 || x.after_layer > n_layers || !std::isfinite(x.a) ||
        !std::isfinite(x.b))
      return LOFP_E_INVALID_ARG;
    gv.push_back(x);
  }
  lofp_ctx *ctx = new (std::nothrow) lofp_ctx();
  if (!ctx) return LOFP_E_OOM;
  ctx->M = modes;
  ctx->D = n_layers;
  ctx->nbs = (int)total;
  lofp_status st = LOFP_OK;
  int idx = 0;
  for (int l = 0; l < n_layers && st == LOFP_OK; ++l) {
    std::vector<uint8_t> used(modes, 0);
    for (int i = 0; i < bs_per_layer[l]; ++i, ++idx) {
      const lofp_bs &b = bs[idx];
      if (b.mode_a < 0 || b.mode_b < 0 || b.mode_a >= modes || b.mode_b >= modes || b.mode_a == b.mode_b ||
          !std::isfinite(b.theta) || !std::isfinite(b.phi)) {
        st = LOFP_E_INVALID_ARG;
        break;
      }
      if (used[b.mode_a] || used[b.mode_b]) {
        st = LOFP_E_INVALID_ARG;
        break;
      }
      used[b.mode_a] = used[b.mode_b] = 1;
      if (std::abs(b.mode_a - b.mode_b) != 1) ctx->general = true;  // non-local pair (NEXT-4)
      CanonBS c;
      c.layer = l + 1;
      c.cut = std::max(b.mode_a, b.mode_b);
      c.lo = std::min(b.mode_a, b.mode_b);
      c.theta = b.theta;
      // port swap: (b, a, theta, phi) == (a, b, theta, pi - phi) (reading R4)
      c.phi = b.mode_a < b.mode_b ? b.phi : kPi - b.phi;
      ctx->bs.push_back(c);
    }
  }
  std::stable_sort(ctx->bs.begin(), ctx->bs.end(),
                   [](const CanonBS &x, const CanonBS &y) { return x.layer != y.layer ? x.layer < y.layer : x.cut < y.cut; });
  if (st == LOFP_OK) st = ctx->general ? build_topology_general(ctx, gv) : build_topology(ctx, gv);
  if (st == LOFP_OK) build_generic(ctx);
  if (st != LOFP_OK) {
    delete ctx;
    return st;
  }
  cudaError_t e = cudaGetDevice(&ctx->device);
  if (e == cudaSuccess) {
    lofp_status s2 = upload_topology(ctx);
    if (s2 != LOFP_OK) {
      lofp_destroy(ctx);
      return s2;
    }
  }
  for (cudaEvent_t *ev : {&ctx->ev_start, &ctx->ev_u0, &ctx->ev_u1, &ctx->ev_end})
    if (e == cudaSuccess) e = cudaEventCreate(ev);
  if (e == cudaSuccess) e = ctx->h_ctr.ensure(sizeof(Counters));
  if (e == cudaSuccess) {
    ctx->grid = lofp_units_grid(ctx->device);
    if (ctx->grid <= 0) e = cudaErrorInvalidDevice;
  }
  // per-block scratch: at least the fixed part of the column engine's layout (1.36 MiB)
  ctx->slab_bytes = std::max(2ll, env_ll("LOFP_SLAB_MB", 16)) << 20;
  if (e != cudaSuccess) {
    lofp_status s = e == cudaErrorMemoryAllocation ? LOFP_E_OOM : LOFP_E_CUDA;
    lofp_destroy(ctx);
    return s;
  }
  *out = ctx;
  return LOFP_OK;
}

// Validated per-call setup shared by the path-sum and contraction entries.
lofp_status prepare(lofp_ctx *ctx, const int32_t *input_occ, int64_t batch, const int32_t *output_occ,
                    double *amps, cudaStream_t stream, CallParams &P, bool &capturing) {
  if (!input_occ || batch < 0) return fail(ctx, LOFP_E_INVALID_ARG, "null input_occ or negative batch");
  if (batch > 0 && (!output_occ || !amps)) return fail(ctx, LOFP_E_INVALID_ARG, "null output_occ or amps");
  if (batch > (int64_t)0x7fffffff) return fail(ctx, LOFP_E_UNSUPPORTED, "batch too large");
  const int M = ctx->M;
  int N = 0;
  for (int i = 0; i < M; ++i) {
    if (input_occ[i] < 0) return fail(ctx, LOFP_E_INVALID_ARG, "negative input occupation");
    N += input_occ[i];
    if (N > LOFP_MAX_PHOTONS) return fail(ctx, LOFP_E_UNSUPPORTED, "too many photons");
  }
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  CK(cudaStreamIsCapturing(stream, &cs), "cudaStreamIsCapturing");
  capturing = cs != cudaStreamCaptureStatusNone;
  // order after the previous call on this context (its buffers are reused or freed)
  if (!capturing && ctx->have_call) CK(cudaStreamWaitEvent(stream, ctx->ev_end, 0), "cudaStreamWaitEvent");
  std::memset(&P, 0, sizeof(P));
  P.M = M;
  P.D = ctx->D;
  P.N = N;
  P.B = (int)batch;
  P.nbs = ctx->nbs;
  P.ngate = ctx->ngate;
  P.cumS[0] = 0;
  for (int i = 0; i < M; ++i) P.cumS[i + 1] = (uint8_t)(P.cumS[i] + input_occ[i]);
  char *topo = (char *)ctx->d_topo.p;
  P.col = (const ColInfo *)(topo + ctx->off_col);
  P.seg = (const SegInfo *)(topo + ctx->off_seg);
  P.cmp = (const CmpPair *)(topo + ctx->off_cmp);
  P.fac = (const FacInfo *)(topo + ctx->off_fac);
  P.gat = (const GateInfo *)(topo + ctx->off_gat);
  P.bsi = (const BSInfo *)(topo + ctx->off_bsi);
  P.gate_ab = (const double *)(topo + ctx->off_gab);
  P.gate_mode = (const int16_t *)(topo + ctx->off_gm);
  P.gate_after = (const int16_t *)(topo + ctx->off_gl);
  P.eqc = (const EqCon *)(topo + ctx->off_eqc);
  P.bnd = (const BoundInfo *)(topo + ctx->off_bnd);
  P.general = ctx->general ? 1 : 0;
  P.seq = (const SeqBS *)(topo + ctx->off_seq);
  P.cone = (const uint64_t *)(topo + ctx->off_cone);
  P.seq_gl0 = ctx->seq_gl0;
  // Appendix-A table: per BS all (x1, x2, y1) with x1 + x2 <= its past-cone photon bound
  long long entries = 0, entriesA = 0;
  for (int i = 0; i < ctx->nbs; ++i) {
    const BSInfo &bi = ctx->bsi[i];
    int c = 0;
    if (!ctx->general) {
      c = (int)P.cumS[bi.cap_hi] - (int)P.cumS[bi.cap_lo];
    } else {
      for (int m = 0; m < ctx->M; ++m)
        if ((bi.capmask[m >> 6] >> (m & 63)) & 1ull) c += input_occ[m];
    }
    entries += tri_entries(std::min(N, c));
    entriesA += lin_entries(std::min(N, c));
  }
  ctx->table_entries = entries;
  ctx->tableA_entries = entriesA;
  CK(ctx->d_table.ensure_async((size_t)std::max(entries, 1ll) * 16, stream), "alloc table");
  CK(ctx->d_taboff.ensure_async((size_t)(ctx->nbs + 1) * 8, stream), "alloc table offsets");
  CK(ctx->d_gatetab.ensure_async((size_t)std::max(ctx->ngate, 1) * (N + 1) * 16, stream), "alloc gate table");
  P.table = (double2 *)ctx->d_table.p;
  P.tab_off = (long long *)ctx->d_taboff.p;
  P.gate_tab = (double2 *)ctx->d_gatetab.p;
  P.table_cap = (long long)(ctx->d_table.n / 16);
  // units: per-output slots; partial sums; per-output status/counters
  const long long B = std::max<long long>(batch, 1);
  long long budget = (1ll << 21) / B;
  budget = std::max(8ll, std::min(budget, 1ll << 17));
  P.budget = (int)budget;
  P.thr = (unsigned long long)env_ll("LOFP_UNIT_PATHS", 1ll << 24);
  P.slab_bytes = ctx->slab_bytes;
  P.units_per_block = (int)env_ll("LOFP_UNITS_PER_BLOCK", 2);
  P.force_generic = env_ll("LOFP_FORCE_GENERIC", 0) > 0 ? 1 : 0;
  P.contract_block_only = env_ll("LOFP_CONTRACT_BLOCK", 0) > 0 ? 1 : 0;
  P.contract_group = (int)env_ll("LOFP_CONTRACT_GROUP", 0);
  P.contract_nosort = env_ll("LOFP_CONTRACT_NOSORT", 0) > 0 ? 1 : 0;
  P.max_nfac = 0;
  for (const ColInfo &ci : ctx->col) P.max_nfac = std::max(P.max_nfac, (int)ci.nfac);
  P.path_budget = ctx->path_budget;
  CK(ctx->d_units.ensure_async((size_t)(B * budget) * sizeof(Unit), stream), "alloc units");
  CK(ctx->d_partial.ensure_async((size_t)(B * budget) * 16, stream), "alloc partials");
  CK(ctx->d_sched.ensure_async((size_t)(B * budget) * 4, stream), "alloc schedule");
  CK(ctx->d_nunits.ensure_async((size_t)B * 4, stream), "alloc nunits");
  CK(ctx->d_ubase.ensure_async((size_t)(B + 1) * 4, stream), "alloc ubase");
  CK(ctx->d_status.ensure_async((size_t)B, stream), "alloc status");
  CK(ctx->d_pexp.ensure_async((size_t)B * 8, stream), "alloc pexp");
  CK(ctx->d_pdone.ensure_async((size_t)B * 8, stream), "alloc pdone");
  CK(ctx->d_slab.ensure_async((size_t)ctx->grid * (size_t)ctx->slab_bytes, stream), "alloc scratch");
  CK(ctx->d_ctr.ensure_async(sizeof(Counters), stream), "alloc counters");
  P.units = (Unit *)ctx->d_units.p;
  P.partial = (double2 *)ctx->d_partial.p;
  P.sched = (int *)ctx->d_sched.p;
  P.nunits = (int *)ctx->d_nunits.p;
  P.ubase = (int *)ctx->d_ubase.p;
  P.status = (uint8_t *)ctx->d_status.p;
  P.pexp = (unsigned long long *)ctx->d_pexp.p;
  P.pdone = (unsigned long long *)ctx->d_pdone.p;
  P.slab = (char *)ctx->d_slab.p;
  P.ctr = (Counters *)ctx->d_ctr.p;
  P.T = output_occ;
  P.amps = (double2 *)amps;
  return LOFP_OK;
}

struct NvtxRange {  // shows each call (and its kernels) as one range in Nsight Systems
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

lofp_status run(lofp_ctx *ctx, const int32_t *input_occ, int64_t batch, const int32_t *output_occ, double *amps,
                unsigned long long *counts, cudaStream_t stream, int mode) {
  if (!ctx) return LOFP_E_INVALID_ARG;
  NvtxRange range(mode == 0 ? (counts ? "lofp_amplitudes_counted" : "lofp_amplitudes") : "lofp_amplitudes_contract");
  ctx->err.clear();
  DeviceGuard guard(ctx->device);
  CallParams P;
  bool capturing = false;
  lofp_status s = prepare(ctx, input_occ, batch, output_occ, amps, stream, P, capturing);
  if (s != LOFP_OK) return s;
  ctx->stats = lofp_run_stats{};
  ctx->stats.batch = batch;
  if (batch == 0) return LOFP_OK;
  P.counts = counts;
  P.mode = mode;
  if (mode == 1) {  // the contraction's x1-linear copy of the tables
    CK(ctx->d_tableA.ensure_async((size_t)std::max(ctx->tableA_entries, 1ll) * 16, stream), "alloc table (x1-linear)");
    CK(ctx->d_tabAoff.ensure_async((size_t)(ctx->nbs + 1) * 8, stream), "alloc table offsets (x1-linear)");
    P.tableA = (double2 *)ctx->d_tableA.p;
    P.tabA_off = (long long *)ctx->d_tabAoff.p;
    P.tableA_cap = (long long)(ctx->d_tableA.n / 16);
  }
  ctx->timed = !capturing;
  if (ctx->timed) CK(cudaEventRecord(ctx->ev_start, stream), "cudaEventRecord");
  CK(cudaMemsetAsync(P.ctr, 0, sizeof(Counters), stream), "clear counters");
  int launches = 0;
  // the Appendix-A tables depend on S only through their size; rebuilt every call (a few
  // microseconds) so that each call, and each graph replay, is self-contained
  CK((cudaError_t)lofp_launch_tables(&P, stream), "table kernels");
  launches += ctx->nbs > 0 ? 2 : 1;
  if (mode == 0) {
    CK((cudaError_t)lofp_launch_paths(&P, ctx->grid, stream, ctx->timed ? ctx->ev_u0 : nullptr,
                                      ctx->timed ? ctx->ev_u1 : nullptr),
       "path-sum kernels");
    launches += 7;
  } else {
    CK((cudaError_t)lofp_launch_contract(&P, ctx->grid, stream), "contraction kernels");
    launches += ctx->general ? 2 : 4;  // (x1-linear tables, warp kernel,) block kernel, generic kernel
  }
  if (!capturing) {  // statistics of calls replayed from a graph are not read back
    CK(cudaMemcpyAsync(ctx->h_ctr.p, P.ctr, sizeof(Counters), cudaMemcpyDeviceToHost, stream), "read counters");
    CK(cudaEventRecord(ctx->ev_end, stream), "cudaEventRecord");
    ctx->have_call = true;
  }
  ctx->stats.launches = launches;
  ctx->stats.mode = mode;
  ctx->stats.grid_blocks = ctx->grid;
  ctx->stats.block_threads = kThreads;
  ctx->stats.table_entries = ctx->table_entries;
  return LOFP_OK;
}

}  // namespace

extern "C" {

const char *lofp_status_string(lofp_status s) {
  switch (s) {
    case LOFP_OK: return "ok";
    case LOFP_E_INVALID_ARG: return "invalid argument";
    case LOFP_E_UNSUPPORTED: return "unsupported";
    case LOFP_E_CUDA: return "CUDA error";
    case LOFP_E_OOM: return "out of device memory";
    case LOFP_E_BAD_OUTPUT: return "bad output row";
  }
  return "unknown status";
}

const char *lofp_last_error(const lofp_ctx *ctx) { return ctx ? ctx->err.c_str() : ""; }

lofp_status lofp_create(int32_t modes, int32_t n_layers, const int32_t *bs_per_layer, const lofp_bs *bs,
                        lofp_ctx **out) {
  return create_impl(modes, n_layers, bs_per_layer, bs, 0, nullptr, out);
}

lofp_status lofp_create_ex(int32_t modes, int32_t n_layers, const int32_t *bs_per_layer, const lofp_bs *bs,
                           int32_t n_gates, const lofp_gate *gates, lofp_ctx **out) {
  return create_impl(modes, n_layers, bs_per_layer, bs, n_gates, gates, out);
}

lofp_status lofp_amplitudes(lofp_ctx *ctx, const int32_t *input_occ, int64_t batch, const int32_t *output_occ,
                            double *amps, void *cuda_stream) {
  return run(ctx, input_occ, batch, output_occ, amps, nullptr, (cudaStream_t)cuda_stream, 0);
}

lofp_status lofp_amplitudes_counted(lofp_ctx *ctx, const int32_t *input_occ, int64_t batch,
                                    const int32_t *output_occ, double *amps, uint64_t *path_counts,
                                    void *cuda_stream) {
  if (!ctx) return LOFP_E_INVALID_ARG;
  if (batch > 0 && !path_counts) return fail(ctx, LOFP_E_INVALID_ARG, "null path_counts");
  return run(ctx, input_occ, batch, output_occ, amps, (unsigned long long *)path_counts, (cudaStream_t)cuda_stream,
             0);
}

lofp_status lofp_amplitudes_contract(lofp_ctx *ctx, const int32_t *input_occ, int64_t batch,
                                     const int32_t *output_occ, double *amps, uint64_t *path_counts,
                                     void *cuda_stream) {
  return run(ctx, input_occ, batch, output_occ, amps, (unsigned long long *)path_counts,
             (cudaStream_t)cuda_stream, 1);
}

lofp_status lofp_distribution(lofp_ctx *ctx, const int32_t *input_occ, int64_t max_outputs, int32_t *outputs,
                              double *amps, int64_t *n_outputs, int32_t method, void *cuda_stream) {
  if (!ctx) return LOFP_E_INVALID_ARG;
  ctx->err.clear();
  if (!input_occ || !n_outputs || max_outputs < 0 || (method != 0 && method != 1))
    return fail(ctx, LOFP_E_INVALID_ARG, "bad arguments");
  int N = 0;
  for (int i = 0; i < ctx->M; ++i) {
    if (input_occ[i] < 0) return fail(ctx, LOFP_E_INVALID_ARG, "negative input occupation");
    N += input_occ[i];
    if (N > LOFP_MAX_PHOTONS) return fail(ctx, LOFP_E_UNSUPPORTED, "too many photons");
  }
  // C(N + M - 1, M - 1) patterns, computed exactly with an overflow guard
  const int n = N + ctx->M - 1, k = std::min(ctx->M - 1, N);
  unsigned long long c = 1;
  for (int i = 1; i <= k; ++i) {
    const unsigned long long num = (unsigned long long)(n - k + i);
    if (c > (~0ull >> 1) / num) return fail(ctx, LOFP_E_UNSUPPORTED, "too many output patterns");
    c = c * num / (unsigned long long)i;
  }
  if (c > (unsigned long long)0x7fffffff) return fail(ctx, LOFP_E_UNSUPPORTED, "too many output patterns");
  *n_outputs = (int64_t)c;
  if ((int64_t)c > max_outputs) return fail(ctx, LOFP_E_INVALID_ARG, "max_outputs is smaller than the pattern count");
  if (!outputs || !amps) return fail(ctx, LOFP_E_INVALID_ARG, "null outputs or amps");
  DeviceGuard guard(ctx->device);
  CK((cudaError_t)lofp_launch_outputs(ctx->M, N, (long long)c, outputs, cuda_stream), "output patterns");
  return run(ctx, input_occ, (int64_t)c, outputs, amps, nullptr, (cudaStream_t)cuda_stream, method == 0 ? 1 : 0);
}

lofp_status lofp_set_path_budget(lofp_ctx *ctx, uint64_t max_paths_per_output) {
  if (!ctx) return LOFP_E_INVALID_ARG;
  ctx->path_budget = max_paths_per_output;
  return LOFP_OK;
}

lofp_status lofp_amplitudes_host(lofp_ctx *ctx, const int32_t *input_occ, int64_t batch, const int32_t *output_occ,
                                 double *amps) {
  if (!ctx) return LOFP_E_INVALID_ARG;
  if (batch < 0 || !input_occ) return fail(ctx, LOFP_E_INVALID_ARG, "bad arguments");
  if (batch == 0) return LOFP_OK;
  if (!output_occ || !amps) return fail(ctx, LOFP_E_INVALID_ARG, "null output_occ or amps");
  DeviceGuard guard(ctx->device);
  if (!ctx->own_stream) CK(cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking), "stream");
  size_t tb = (size_t)batch * ctx->M * 4, ab = (size_t)batch * 16;
  if (ctx->have_call) CK(cudaEventSynchronize(ctx->ev_end), "cudaEventSynchronize");
  CK(ctx->d_hostT.ensure(tb), "alloc T");
  CK(ctx->d_hostA.ensure(ab), "alloc amps");
  CK(cudaMemcpyAsync(ctx->d_hostT.p, output_occ, tb, cudaMemcpyHostToDevice, ctx->own_stream), "copy T");
  lofp_status s = run(ctx, input_occ, batch, (const int32_t *)ctx->d_hostT.p, (double *)ctx->d_hostA.p, nullptr,
                      ctx->own_stream, 0);
  if (s != LOFP_OK) return s;
  CK(cudaMemcpyAsync(amps, ctx->d_hostA.p, ab, cudaMemcpyDeviceToHost, ctx->own_stream), "copy amps");
  CK(cudaStreamSynchronize(ctx->own_stream), "cudaStreamSynchronize");
  return LOFP_OK;
}

lofp_status lofp_stats(lofp_ctx *ctx, lofp_run_stats *out) {
  if (!ctx || !out) return LOFP_E_INVALID_ARG;
  DeviceGuard guard(ctx->device);
  if (ctx->have_call) {
    CK(cudaEventSynchronize(ctx->ev_end), "cudaEventSynchronize");
    const Counters *hc = (const Counters *)ctx->h_ctr.p;
    lofp_run_stats &st = ctx->stats;
    st.feasible = (int64_t)hc->feasible;
    st.paths = (int64_t)hc->paths;
    st.cmuls = (int64_t)hc->cmuls;
    st.units = (int64_t)hc->units;
    st.subsplits = (int64_t)hc->subsplits;
    st.pairs = (int64_t)hc->pairs;
    st.elements = (int64_t)hc->elements;
    st.unsupported = (int64_t)hc->unsupported;
    st.bad_rows = (int64_t)hc->bad_rows;
    st.check_errors = (int64_t)hc->table_error;
    st.max_states = (int64_t)hc->max_states;
    st.max_list = (int64_t)hc->max_list;
    st.terms = (int64_t)hc->contractions;
    st.generic = (int64_t)hc->generic;
    st.over_budget = (int64_t)hc->over_budget;
    st.contract_deferred = (int64_t)hc->cdeferred;
    st.tile_cycles[0] = (int64_t)hc->tile_stage;
    st.tile_cycles[1] = (int64_t)hc->tile_fma;
    for (int i = 0; i < 8; ++i) st.phase_cycles[i] = (int64_t)hc->phase[i];
    if (ctx->timed) {
      float ms = 0.f;
      if (st.mode == 0 && cudaEventElapsedTime(&ms, ctx->ev_u0, ctx->ev_u1) == cudaSuccess) st.units_ms = ms;
      if (cudaEventElapsedTime(&ms, ctx->ev_start, ctx->ev_end) == cudaSuccess) st.total_ms = ms;
      if (st.mode == 1) st.units_ms = st.total_ms;
    }
  }
  *out = ctx->stats;
  if (ctx->stats.bad_rows) return LOFP_E_BAD_OUTPUT;
  return LOFP_OK;
}

void lofp_destroy(lofp_ctx *ctx) {
  if (!ctx) return;
  DeviceGuard guard(ctx->device);
  if (ctx->have_call && ctx->ev_end) cudaEventSynchronize(ctx->ev_end);
  for (DevBuf *b : {&ctx->d_topo, &ctx->d_tableA, &ctx->d_tabAoff, &ctx->d_table, &ctx->d_taboff, &ctx->d_gatetab, &ctx->d_units, &ctx->d_sched, &ctx->d_nunits,
                    &ctx->d_ubase, &ctx->d_status, &ctx->d_pexp, &ctx->d_pdone, &ctx->d_partial, &ctx->d_slab,
                    &ctx->d_ctr, &ctx->d_hostT, &ctx->d_hostA})
    b->release();
  ctx->h_ctr.release();
  for (cudaEvent_t ev : {ctx->ev_start, ctx->ev_u0, ctx->ev_u1, ctx->ev_end})
    if (ev) cudaEventDestroy(ev);
  if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
  delete ctx;
}

}  // extern "C"
