// lofp_host.cpp — host side of liblofp: the C ABI of include/lofp.h, circuit
// canonicalisation, the column / light-cone topology tables, per-call buffer sizing and
// the kernel launches.  See DESIGN.md for the derivations (readings R1-R20) and the paper
// passages each step follows.  No call here waits for the device except lofp_create
// (one upload), lofp_stats, lofp_amplitudes_host and lofp_destroy.
#include <cuda_runtime.h>

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
  int cut;    // k = max(mode_a, mode_b)
  double theta, phi;
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
  std::vector<double> gate_ab;
  std::vector<int16_t> gate_mode, gate_after;
  DevBuf d_topo;
  size_t off_col = 0, off_seg = 0, off_cmp = 0, off_fac = 0, off_gat = 0, off_bsi = 0, off_gab = 0, off_gm = 0,
         off_gl = 0;
  // per-call device buffers
  DevBuf d_table, d_taboff, d_gatetab, d_units, d_sched, d_nunits, d_ubase, d_status, d_pexp, d_pdone, d_partial, d_slab,
      d_ctr, d_hostT, d_hostA;
  HostPinned h_ctr;
  long long table_entries = 0;
  int grid = 0;
  long long slab_bytes = 0;
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
      if (std::abs(b.mode_a - b.mode_b) != 1) {
        st = LOFP_E_UNSUPPORTED;
        break;
      }
      CanonBS c;
      c.layer = l + 1;
      c.cut = std::max(b.mode_a, b.mode_b);
      c.theta = b.theta;
      // port swap: (b, a, theta, phi) == (a, b, theta, pi - phi) (reading R4)
      c.phi = b.mode_a < b.mode_b ? b.phi : kPi - b.phi;
      ctx->bs.push_back(c);
    }
  }
  std::stable_sort(ctx->bs.begin(), ctx->bs.end(),
                   [](const CanonBS &x, const CanonBS &y) { return x.layer != y.layer ? x.layer < y.layer : x.cut < y.cut; });
  if (st == LOFP_OK) st = build_topology(ctx, gv);
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
  ctx->slab_bytes = env_ll("LOFP_SLAB_MB", 16) << 20;
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
  // Appendix-A table: per BS all (x1, x2, y1) with x1 + x2 <= its past-cone photon bound
  long long entries = 0;
  for (int i = 0; i < ctx->nbs; ++i) {
    const BSInfo &bi = ctx->bsi[i];
    const int cap = std::min(N, (int)P.cumS[bi.cap_hi] - (int)P.cumS[bi.cap_lo]);
    entries += tri_entries(cap);
  }
  ctx->table_entries = entries;
  CK(ctx->d_table.ensure((size_t)std::max(entries, 1ll) * 16), "alloc table");
  CK(ctx->d_taboff.ensure((size_t)(ctx->nbs + 1) * 8), "alloc table offsets");
  CK(ctx->d_gatetab.ensure((size_t)std::max(ctx->ngate, 1) * (N + 1) * 16), "alloc gate table");
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
  CK(ctx->d_units.ensure((size_t)(B * budget) * sizeof(Unit)), "alloc units");
  CK(ctx->d_partial.ensure((size_t)(B * budget) * 16), "alloc partials");
  CK(ctx->d_sched.ensure((size_t)(B * budget) * 4), "alloc schedule");
  CK(ctx->d_nunits.ensure((size_t)B * 4), "alloc nunits");
  CK(ctx->d_ubase.ensure((size_t)(B + 1) * 4), "alloc ubase");
  CK(ctx->d_status.ensure((size_t)B), "alloc status");
  CK(ctx->d_pexp.ensure((size_t)B * 8), "alloc pexp");
  CK(ctx->d_pdone.ensure((size_t)B * 8), "alloc pdone");
  CK(ctx->d_slab.ensure((size_t)ctx->grid * (size_t)ctx->slab_bytes), "alloc scratch");
  CK(ctx->d_ctr.ensure(sizeof(Counters)), "alloc counters");
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
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  CK(cudaStreamIsCapturing(stream, &cs), "cudaStreamIsCapturing");
  capturing = cs != cudaStreamCaptureStatusNone;
  // order after the previous call on this context (its buffers are reused)
  if (!capturing && ctx->have_call) CK(cudaStreamWaitEvent(stream, ctx->ev_end, 0), "cudaStreamWaitEvent");
  return LOFP_OK;
}

lofp_status run(lofp_ctx *ctx, const int32_t *input_occ, int64_t batch, const int32_t *output_occ, double *amps,
                unsigned long long *counts, cudaStream_t stream, int mode) {
  if (!ctx) return LOFP_E_INVALID_ARG;
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
    launches += 6;
  } else {
    CK((cudaError_t)lofp_launch_contract(&P, ctx->grid, stream), "contraction kernels");
    launches += 1;
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
  for (DevBuf *b : {&ctx->d_topo, &ctx->d_table, &ctx->d_taboff, &ctx->d_gatetab, &ctx->d_units, &ctx->d_sched, &ctx->d_nunits,
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
