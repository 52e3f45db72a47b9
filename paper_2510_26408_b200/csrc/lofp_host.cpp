// lofp_host.cpp — host side of liblofp: the C ABI of include/lofp.h, circuit
// canonicalisation, light-cone topology maps, per-call Appendix-A table layout and the
// kernel launches.  See DESIGN.md for the derivations (readings R1-R9) and the paper
// passages each step follows.
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

namespace {

constexpr double kPi = 3.14159265358979323846;

struct DevBuf {
  void *p = nullptr;
  size_t n = 0;
  cudaError_t ensure(size_t bytes) {
    if (bytes <= n) return cudaSuccess;
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
    if (bytes <= n) return cudaSuccess;
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

// A beam splitter after canonicalisation: port 1 = mode k-1, port 2 = mode k.
struct CanonBS {
  int layer;  // 1-based
  int cut;    // k = max(mode_a, mode_b)
  double theta, phi;
};

}  // namespace

struct lofp_ctx {
  int M = 0, D = 0, nbs = 0, Lg = 0;
  std::vector<CanonBS> bs;                  // layer-major, by cut inside a layer
  std::vector<std::vector<uint8_t>> act;    // [D+1][M+1]
  std::vector<uint8_t> maps;                // [4][D+1][M+1]: rho, sigma, rho', sigma'
  // static device data
  DevBuf d_maps, d_bs_lk, d_bs_cs;
  // per-call device data
  DevBuf d_flags, d_plans, d_feas, d_ctr, d_ring, d_edesc, d_offsets, d_entries, d_cumS, d_bsrow;
  DevBuf d_hostT, d_hostA;
  HostPinned h_stage, h_ctr;
  unsigned ring_cap = 0;
  cudaEvent_t ev_start = nullptr, ev_enum0 = nullptr, ev_enum1 = nullptr, ev_end = nullptr;
  cudaStream_t own_stream = nullptr;
  bool have_call = false;
  lofp_run_stats stats{};
  std::string err;
  int device = 0;
};

namespace {

lofp_status fail(lofp_ctx *c, lofp_status s, const std::string &msg) {
  if (c) c->err = msg;
  return s;
}

lofp_status cuda_fail(lofp_ctx *c, cudaError_t e, const char *where) {
  std::string m = std::string(where) + ": " + cudaGetErrorString(e);
  return fail(c, e == cudaErrorMemoryAllocation ? LOFP_E_OOM : LOFP_E_CUDA, m);
}

#define CK(expr, where)                                      \
  do {                                                       \
    cudaError_t _e = (expr);                                 \
    if (_e != cudaSuccess) return cuda_fail(ctx, _e, where); \
  } while (0)

// Topology-only light-cone maps (reading R5).  Backward: rho_D(k) = sigma_D(k) = k and,
// going back through layer l, an active cut k takes rho_{l-1}(k) = rho_l(k-1),
// sigma_{l-1}(k) = sigma_l(k+1); then F_l(k) lies in [G(rho_l(k)), G(sigma_l(k))].
// Forward (the same construction from the input side): rho'_0(k) = sigma'_0(k) = k,
// rho'_l(k) = rho'_{l-1}(k-1), sigma'_l(k) = sigma'_{l-1}(k+1) at active cuts; then
// F_l(k) lies in [cumS(rho'_l(k)), cumS(sigma'_l(k))] (P:153-164 cones, cumulative form).
lofp_status plan_circuit(lofp_ctx *c) {
  const int M = c->M, D = c->D, W = M + 1;
  c->act.assign(D + 1, std::vector<uint8_t>(M + 1, 0));
  for (const CanonBS &b : c->bs) c->act[b.layer][b.cut] = 1;
  c->maps.assign(4 * (D + 1) * W, 0);
  uint8_t *rho = c->maps.data(), *sig = rho + (D + 1) * W, *frho = sig + (D + 1) * W, *fsig = frho + (D + 1) * W;
  for (int k = 0; k <= M; ++k) rho[D * W + k] = sig[D * W + k] = (uint8_t)k;
  for (int l = D; l >= 1; --l)
    for (int k = 0; k <= M; ++k) {
      rho[(l - 1) * W + k] = c->act[l][k] ? rho[l * W + k - 1] : rho[l * W + k];
      sig[(l - 1) * W + k] = c->act[l][k] ? sig[l * W + k + 1] : sig[l * W + k];
    }
  for (int k = 0; k <= M; ++k) frho[k] = fsig[k] = (uint8_t)k;
  for (int l = 1; l <= D; ++l)
    for (int k = 0; k <= M; ++k) {
      frho[l * W + k] = c->act[l][k] ? frho[(l - 1) * W + k - 1] : frho[(l - 1) * W + k];
      fsig[l * W + k] = c->act[l][k] ? fsig[(l - 1) * W + k + 1] : fsig[(l - 1) * W + k];
    }
  // global bound on DFS levels: BS outputs whose backward box is not a single cut
  int L = 0;
  for (const CanonBS &b : c->bs)
    if (rho[b.layer * W + b.cut] != sig[b.layer * W + b.cut]) ++L;
  if (L > LOFP_MAX_LEVELS) return fail(c, LOFP_E_UNSUPPORTED, "too many free BS outputs (DFS levels)");
  c->Lg = L;
  return LOFP_OK;
}

// Per-segment occupation caps: min(photons of S in the past light cone, photons of
// max-over-batch T in the future light cone).  cap[j][m] for the segment of
// mode m after layer j.
std::vector<std::vector<int>> segment_caps(const lofp_ctx *c, const std::vector<int> &S, const int32_t *tmax) {
  const int M = c->M, D = c->D;
  std::vector<std::vector<int>> cap(D + 1, std::vector<int>(M, 0));
  std::vector<std::vector<const CanonBS *>> byl(D + 1);
  for (const CanonBS &b : c->bs) byl[b.layer].push_back(&b);
  std::vector<uint8_t> in(M);
  for (int j = 0; j <= D; ++j)
    for (int m = 0; m < M; ++m) {
      std::fill(in.begin(), in.end(), 0);
      in[m] = 1;
      for (int l = j; l >= 1; --l)
        for (const CanonBS *b : byl[l])
          if (in[b->cut - 1] || in[b->cut]) in[b->cut - 1] = in[b->cut] = 1;
      int past = 0;
      for (int i = 0; i < M; ++i)
        if (in[i]) past += S[i];
      std::fill(in.begin(), in.end(), 0);
      in[m] = 1;
      for (int l = j + 1; l <= D; ++l)
        for (const CanonBS *b : byl[l])
          if (in[b->cut - 1] || in[b->cut]) in[b->cut - 1] = in[b->cut] = 1;
      int fut = 0;
      for (int i = 0; i < M; ++i)
        if (in[i]) fut += tmax[i];
      cap[j][m] = std::min(past, fut);
    }
  return cap;
}

inline size_t round16(size_t x) { return (x + 15) & ~size_t(15); }

lofp_status run(lofp_ctx *ctx, const int32_t *input_occ, int64_t batch, const int32_t *output_occ, double *amps,
                unsigned long long *counts, cudaStream_t stream) {
  if (!ctx) return LOFP_E_INVALID_ARG;
  ctx->err.clear();
  if (!input_occ || batch < 0) return fail(ctx, LOFP_E_INVALID_ARG, "null input_occ or negative batch");
  if (batch > 0 && (!output_occ || !amps)) return fail(ctx, LOFP_E_INVALID_ARG, "null output_occ or amps");
  if (batch > (int64_t)0x7fffffff) return fail(ctx, LOFP_E_UNSUPPORTED, "batch too large");
  const int M = ctx->M;
  std::vector<int> S(M);
  int N = 0;
  for (int m = 0; m < M; ++m) {
    if (input_occ[m] < 0) return fail(ctx, LOFP_E_INVALID_ARG, "negative input occupation");
    S[m] = input_occ[m];
    N += S[m];
    if (N > LOFP_MAX_PHOTONS) return fail(ctx, LOFP_E_UNSUPPORTED, "too many photons");
  }
  CK(cudaSetDevice(ctx->device), "cudaSetDevice");
  ctx->stats = lofp_run_stats{};
  ctx->stats.batch = batch;
  ctx->have_call = false;
  if (batch == 0) return LOFP_OK;
  // serialise with this context's previous call (its buffers are reused)
  CK(cudaEventSynchronize(ctx->ev_end), "cudaEventSynchronize");

  const int64_t B = batch;
  CallArgs a{};
  a.M = M;
  a.D = ctx->D;
  a.N = N;
  a.nbs = ctx->nbs;
  a.Lg = ctx->Lg;
  a.vals_slots = (int)((ctx->Lg + 1 + 3) & ~3);
  a.B = B;
  // head | levels [Lg] | factors [nbs] | scatter u16 [4 nbs] | pad | scratch factors [nbs] |
  // scratch scatter u32 [4 nbs]  (see lofp_plan_kernel)
  a.plan_stride = (int)round16(sizeof(PlanHead) + (size_t)ctx->Lg * sizeof(PlanLevel) +
                               2 * (size_t)ctx->nbs * sizeof(PlanFactor) + 8 * (size_t)ctx->nbs + 16 +
                               16 * (size_t)ctx->nbs);
  // chain-engine thresholds (env overrides exist for the tests, which exercise the
  // engine on small circuits)
  a.chain_rbox = LOFP_CHAIN_RBOX;
  a.chain_rmin = LOFP_CHAIN_RMIN;
  if (const char *e = std::getenv("LOFP_CHAIN_RBOX")) a.chain_rbox = std::atof(e);
  if (const char *e = std::getenv("LOFP_CHAIN_RMIN")) a.chain_rmin = std::atoi(e);
  a.small_paths = LOFP_SMALL_PATHS;
  if (const char *e = std::getenv("LOFP_SMALL_PATHS")) a.small_paths = std::min(std::atoi(e), 256);
  a.T = output_occ;
  a.amps = amps;
  a.counts = counts;
  CK(ctx->d_flags.ensure((size_t)B), "alloc flags");
  CK(ctx->d_plans.ensure((size_t)B * a.plan_stride), "alloc plans");
  CK(ctx->d_feas.ensure((size_t)B * 4), "alloc feas");
  CK(ctx->d_ctr.ensure(sizeof(Counters)), "alloc counters");
  CK(ctx->d_cumS.ensure(256), "alloc cumS");
  a.flags = (uint8_t *)ctx->d_flags.p;
  a.plans = (unsigned char *)ctx->d_plans.p;
  a.feas = (uint32_t *)ctx->d_feas.p;
  a.ctr = (Counters *)ctx->d_ctr.p;
  a.cumS = (const uint8_t *)ctx->d_cumS.p;
  a.maps = (const uint8_t *)ctx->d_maps.p;
  a.bs_lk = (const int16_t *)ctx->d_bs_lk.p;
  a.bs_cs = (const double *)ctx->d_bs_cs.p;

  CK(cudaEventRecord(ctx->ev_start, stream), "cudaEventRecord");
  // cum(S) to the device (pinned staging; the previous call has completed)
  CK(ctx->h_stage.ensure(4096), "alloc staging");
  uint8_t *cs = (uint8_t *)ctx->h_stage.p;
  {
    int f = 0;
    for (int k = 0; k <= M; ++k) {
      cs[k] = (uint8_t)f;
      if (k < M) f += S[k];
    }
  }
  CK(cudaMemcpyAsync(ctx->d_cumS.p, cs, M + 1, cudaMemcpyHostToDevice, stream), "upload cumS");
  CK(cudaMemsetAsync(a.ctr, 0, sizeof(Counters), stream), "reset counters");
  CK(lofp_launch_prep(a, stream), "prep kernel");
  ctx->stats.launches += a.B > 0 ? 1 : 0;
  // (sync 1) the batch's per-mode maximum sizes the tables
  CK(ctx->h_ctr.ensure(sizeof(Counters)), "alloc pinned counters");
  CK(cudaMemcpyAsync(ctx->h_ctr.p, a.ctr, sizeof(Counters), cudaMemcpyDeviceToHost, stream), "read tmax");
  CK(cudaStreamSynchronize(stream), "cudaStreamSynchronize");
  const Counters *hc = (const Counters *)ctx->h_ctr.p;
  int32_t tmax[LOFP_MAX_MODES];
  for (int m = 0; m < M; ++m) tmax[m] = hc->tmax[m];

  // Appendix-A table layout inside the light-cone caps
  std::vector<std::vector<int>> cap = segment_caps(ctx, S, tmax);
  std::vector<int32_t> offsets;
  std::vector<EntryDesc> edesc;
  std::vector<int32_t> bsrow(2 * std::max(ctx->nbs, 1));  // [base | stride]
  for (int i = 0; i < ctx->nbs; ++i) {
    const CanonBS &b = ctx->bs[i];
    int X1 = cap[b.layer - 1][b.cut - 1], X2 = cap[b.layer - 1][b.cut];
    int Y1 = cap[b.layer][b.cut - 1], Y2 = cap[b.layer][b.cut];
    bsrow[i] = (int32_t)offsets.size();
    bsrow[ctx->nbs + i] = X2 + 1;
    for (int x1 = 0; x1 <= X1; ++x1)
      for (int x2 = 0; x2 <= X2; ++x2) {
        int n = x1 + x2;
        int ylo = std::max(0, n - Y2), yhi = std::min(Y1, n);
        offsets.push_back((int32_t)edesc.size() - ylo);
        for (int y1 = ylo; y1 <= yhi; ++y1) {
          EntryDesc e{};
          e.bs = (uint16_t)i;
          e.x1 = (uint8_t)x1;
          e.x2 = (uint8_t)x2;
          e.y1 = (uint8_t)y1;
          edesc.push_back(e);
        }
      }
  }
  if (edesc.empty()) edesc.push_back(EntryDesc{});  // keep pointers valid
  if (offsets.empty()) offsets.push_back(0);
  a.nentries = (int)edesc.size();
  a.noffsets = (int)offsets.size();
  a.table_bytes = (int)round16((size_t)a.nentries * 16 + (size_t)a.noffsets * 4);
  CK(ctx->d_edesc.ensure(edesc.size() * sizeof(EntryDesc)), "alloc edesc");
  CK(ctx->d_offsets.ensure(offsets.size() * 4), "alloc offsets");
  CK(ctx->d_entries.ensure(edesc.size() * 16), "alloc entries");
  CK(ctx->d_bsrow.ensure(bsrow.size() * 4), "alloc bs rows");
  size_t need = edesc.size() * sizeof(EntryDesc) + offsets.size() * 4 + bsrow.size() * 4 + 64;
  CK(ctx->h_stage.ensure(need), "alloc staging");
  {
    uint8_t *st = (uint8_t *)ctx->h_stage.p;
    size_t o = 0;
    memcpy(st + o, edesc.data(), edesc.size() * sizeof(EntryDesc));
    CK(cudaMemcpyAsync(ctx->d_edesc.p, st + o, edesc.size() * sizeof(EntryDesc), cudaMemcpyHostToDevice, stream),
       "upload edesc");
    o += edesc.size() * sizeof(EntryDesc);
    memcpy(st + o, offsets.data(), offsets.size() * 4);
    CK(cudaMemcpyAsync(ctx->d_offsets.p, st + o, offsets.size() * 4, cudaMemcpyHostToDevice, stream),
       "upload offsets");
    o += offsets.size() * 4;
    memcpy(st + o, bsrow.data(), bsrow.size() * 4);
    CK(cudaMemcpyAsync(ctx->d_bsrow.p, st + o, bsrow.size() * 4, cudaMemcpyHostToDevice, stream), "upload bs rows");
  }
  a.edesc = (const EntryDesc *)ctx->d_edesc.p;
  a.offsets = (const int32_t *)ctx->d_offsets.p;
  a.entries = (double *)ctx->d_entries.p;
  a.bs_base = (const int32_t *)ctx->d_bsrow.p;
  a.bs_stride = (const int32_t *)ctx->d_bsrow.p + ctx->nbs;
  ctx->stats.table_entries = a.nentries;

  CK(lofp_launch_tables(a, stream), "table kernel");
  CK(lofp_launch_plan(a, stream), "plan kernel");
  ctx->stats.launches += (a.nentries > 0 ? 1 : 0) + (a.B > 0 ? 1 : 0);
  // (sync 2) the largest per-output plan sizes the enumeration kernel's shared memory
  CK(cudaMemcpyAsync(ctx->h_ctr.p, a.ctr, sizeof(Counters), cudaMemcpyDeviceToHost, stream), "read plan sizes");
  CK(cudaStreamSynchronize(stream), "cudaStreamSynchronize");
  const int maxL = hc->maxL, maxF = hc->maxF, maxS = hc->maxS, maxK = hc->maxK;
  ctx->stats.levels = maxL;
  CK(cudaEventRecord(ctx->ev_enum0, stream), "cudaEventRecord");
  if (hc->nfeas > 0) {
    a.vals_slots = (maxL + 2 + 3) & ~3;  // zero slot, levels, a scratch slot
    // plans were written with the zero slot of the global bound; re-base is not needed
    // because the kernel only dereferences slots < maxL and the zero slot below
    // (the step's uniform loops read up to maxF descriptors / key words and maxS + 3
    // scatter entries past a level's own list: vals, keys and stack follow inside the
    // warp's region, so those reads never leave it)
    a.plan_smem = (int)round16(sizeof(PlanHead) + (size_t)(maxL + maxF) * 16 + 2 * (size_t)maxS);
    // Chain engine (R17): on when most outputs have chains of >= LOFP_CHAIN_MODE_RBOX box
    // paths (then every output whose chain box is >= LOFP_CHAIN_RBOX gets its chain).
    // Otherwise, if most outputs have the chain structure with chains of moderate size
    // (geometric-mean box >= 2^LOFP_SHORT_CHAIN_LOG2 paths), every such output gets the
    // engine with the short chains batched (R20; the plans are rebuilt with those
    // thresholds).  Environment overrides (tests) disable this choice.
    const bool env_chain = std::getenv("LOFP_NO_CHAIN") || std::getenv("LOFP_FORCE_CHAIN") ||
                           std::getenv("LOFP_CHAIN_RBOX") || std::getenv("LOFP_CHAIN_RMIN") ||
                           std::getenv("LOFP_SMALL_PATHS");
    const double mlog = hc->nchain_ok > 0 ? (double)hc->rbox_log16 / 16.0 / hc->nchain_ok : 0.0;
    bool short_chains = false;
    if (!env_chain && 2ull * (unsigned long long)hc->nchain_big < hc->nfeas &&
        2ull * (unsigned long long)hc->nchain_ok >= hc->nfeas && mlog >= LOFP_SHORT_CHAIN_LOG2) {
      a.chain_rbox = 1.0;
      a.chain_rmin = 1;
      a.small_paths = 256;
      // the plan kernel counts the feasible outputs and the outstanding work: reset those
      CK(cudaMemsetAsync(reinterpret_cast<char *>(a.ctr) + offsetof(Counters, nfeas), 0, sizeof(unsigned long long),
                         stream), "reset counters");
      CK(cudaMemsetAsync(reinterpret_cast<char *>(a.ctr) + offsetof(Counters, outstanding), 0,
                         sizeof(unsigned long long), stream), "reset counters");
      CK(lofp_launch_plan(a, stream), "plan kernel (short chains)");
      ++ctx->stats.launches;
      short_chains = true;
    }
    a.chain_on = short_chains ||
                 (hc->nchain > 0 && !std::getenv("LOFP_NO_CHAIN") &&
                  (2ull * (unsigned long long)hc->nchain_big >= hc->nfeas || std::getenv("LOFP_FORCE_CHAIN")));
    // key words per lane: every attached factor (none while the engine is on)
    a.maxfac = a.chain_on ? 0 : maxF;
    (void)maxK;
    a.warp_bytes = (int)round16((size_t)a.plan_smem + (size_t)a.vals_slots * 32 + (size_t)a.maxfac * 128 +
                                (size_t)(a.chain_on ? LOFP_STK_CHAIN : LOFP_STK) * 32 * 20 + 32 +
                                (a.chain_on ? (size_t)LOFP_W_MAX * 16 + (size_t)LOFP_SUF_ENTRIES * 16 + 33 * 16 + 65 * 4 + 1024 +
                                                  (a.small_paths > 0 ? 512 + 264 + 4 * 32 * LOFP_SMALL_LEVELS + 16 : 0)
                                            : 0));
    int grid = 0, block = 0;
    size_t smem = 0;
    cudaError_t e = lofp_enum_config(a, counts != nullptr, &grid, &block, &smem);
    if (e == cudaErrorInvalidConfiguration)
      return fail(ctx, LOFP_E_UNSUPPORTED, "BS tables do not fit in shared memory");
    CK(e, "enumeration config");
    unsigned lanes = (unsigned)grid * (unsigned)block;
    // Queue capacity: spills are accepted while fewer than cap/2 are waiting, which
    // keeps every reused slot's previous item already claimed (see the kernel).
    unsigned cap_items = 1u << 20;
    while (cap_items < 8u * lanes) cap_items <<= 1;
    if (cap_items > ctx->ring_cap) {
      CK(ctx->d_ring.ensure((size_t)cap_items * sizeof(Item)), "alloc work queue");
      CK(cudaMemsetAsync(ctx->d_ring.p, 0, (size_t)cap_items * sizeof(Item), stream), "clear work queue");
      ctx->ring_cap = cap_items;
    }
    a.ring = (Item *)ctx->d_ring.p;
    a.ring_mask = ctx->ring_cap - 1;
    ctx->stats.smem_bytes = (int32_t)smem;
    ctx->stats.max_factors = maxF;
    ctx->stats.max_scatter = maxS;
    ctx->stats.engine = a.chain_on ? (a.small_paths > 0 ? 2 : 1) : 0;
    ctx->stats.grid_blocks = grid;
    ctx->stats.block_threads = block;
    CK(lofp_launch_enum(a, counts != nullptr, grid, block, smem, stream), "enumeration kernel");
    ++ctx->stats.launches;
  }
  CK(cudaEventRecord(ctx->ev_enum1, stream), "cudaEventRecord");
  CK(cudaMemcpyAsync(ctx->h_ctr.p, a.ctr, sizeof(Counters), cudaMemcpyDeviceToHost, stream), "read counters");
  CK(cudaEventRecord(ctx->ev_end, stream), "cudaEventRecord");
  ctx->have_call = true;
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
  if (!out) return LOFP_E_INVALID_ARG;
  *out = nullptr;
  if (modes < 1 || n_layers < 0) return LOFP_E_INVALID_ARG;
  if (modes > LOFP_MAX_MODES || n_layers > LOFP_MAX_LAYERS) return LOFP_E_UNSUPPORTED;
  if (n_layers > 0 && !bs_per_layer) return LOFP_E_INVALID_ARG;
  int64_t total = 0;
  for (int l = 0; l < n_layers; ++l) {
    if (bs_per_layer[l] < 0) return LOFP_E_INVALID_ARG;
    total += bs_per_layer[l];
  }
  if (total > 0 && !bs) return LOFP_E_INVALID_ARG;
  if (total > 65535) return LOFP_E_UNSUPPORTED;
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
  // layer-major, top to bottom inside a layer: the DFS level order ("systematic way")
  std::stable_sort(ctx->bs.begin(), ctx->bs.end(),
                   [](const CanonBS &x, const CanonBS &y) { return x.layer != y.layer ? x.layer < y.layer : x.cut < y.cut; });
  if (st == LOFP_OK) st = plan_circuit(ctx);
  if (st != LOFP_OK) {
    delete ctx;
    return st;
  }
  cudaError_t e = cudaGetDevice(&ctx->device);
  std::vector<int16_t> lk(2 * std::max(ctx->nbs, 1));
  std::vector<double> csv(4 * std::max(ctx->nbs, 1));
  for (int i = 0; i < ctx->nbs; ++i) {
    lk[2 * i] = (int16_t)ctx->bs[i].layer;
    lk[2 * i + 1] = (int16_t)ctx->bs[i].cut;
    csv[4 * i] = std::cos(ctx->bs[i].theta);
    csv[4 * i + 1] = std::sin(ctx->bs[i].theta);
    csv[4 * i + 2] = std::cos(ctx->bs[i].phi);
    csv[4 * i + 3] = std::sin(ctx->bs[i].phi);
  }
  if (e == cudaSuccess) e = ctx->d_maps.ensure(ctx->maps.size());
  if (e == cudaSuccess) e = cudaMemcpy(ctx->d_maps.p, ctx->maps.data(), ctx->maps.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = ctx->d_bs_lk.ensure(lk.size() * 2);
  if (e == cudaSuccess) e = cudaMemcpy(ctx->d_bs_lk.p, lk.data(), lk.size() * 2, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = ctx->d_bs_cs.ensure(csv.size() * 8);
  if (e == cudaSuccess) e = cudaMemcpy(ctx->d_bs_cs.p, csv.data(), csv.size() * 8, cudaMemcpyHostToDevice);
  for (cudaEvent_t *ev : {&ctx->ev_start, &ctx->ev_enum0, &ctx->ev_enum1, &ctx->ev_end})
    if (e == cudaSuccess) e = cudaEventCreate(ev);
  if (e == cudaSuccess) e = cudaEventRecord(ctx->ev_end, 0);
  if (e == cudaSuccess) e = cudaEventSynchronize(ctx->ev_end);
  if (e != cudaSuccess) {
    lofp_status s = e == cudaErrorMemoryAllocation ? LOFP_E_OOM : LOFP_E_CUDA;
    lofp_destroy(ctx);
    return s;
  }
  *out = ctx;
  return LOFP_OK;
}

lofp_status lofp_amplitudes(lofp_ctx *ctx, const int32_t *input_occ, int64_t batch, const int32_t *output_occ,
                            double *amps, void *cuda_stream) {
  return run(ctx, input_occ, batch, output_occ, amps, nullptr, (cudaStream_t)cuda_stream);
}

lofp_status lofp_amplitudes_counted(lofp_ctx *ctx, const int32_t *input_occ, int64_t batch,
                                    const int32_t *output_occ, double *amps, uint64_t *path_counts,
                                    void *cuda_stream) {
  if (!ctx) return LOFP_E_INVALID_ARG;
  if (batch > 0 && !path_counts) return fail(ctx, LOFP_E_INVALID_ARG, "null path_counts");
  return run(ctx, input_occ, batch, output_occ, amps, (unsigned long long *)path_counts, (cudaStream_t)cuda_stream);
}

lofp_status lofp_amplitudes_host(lofp_ctx *ctx, const int32_t *input_occ, int64_t batch, const int32_t *output_occ,
                                 double *amps) {
  if (!ctx) return LOFP_E_INVALID_ARG;
  if (batch < 0 || !input_occ) return fail(ctx, LOFP_E_INVALID_ARG, "bad arguments");
  if (batch == 0) return LOFP_OK;
  if (!output_occ || !amps) return fail(ctx, LOFP_E_INVALID_ARG, "null output_occ or amps");
  CK(cudaSetDevice(ctx->device), "cudaSetDevice");
  if (!ctx->own_stream) CK(cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking), "stream");
  size_t tb = (size_t)batch * ctx->M * 4, ab = (size_t)batch * 16;
  CK(cudaEventSynchronize(ctx->ev_end), "cudaEventSynchronize");
  CK(ctx->d_hostT.ensure(tb), "alloc T");
  CK(ctx->d_hostA.ensure(ab), "alloc amps");
  CK(cudaMemcpyAsync(ctx->d_hostT.p, output_occ, tb, cudaMemcpyHostToDevice, ctx->own_stream), "copy T");
  lofp_status s =
      run(ctx, input_occ, batch, (const int32_t *)ctx->d_hostT.p, (double *)ctx->d_hostA.p, nullptr, ctx->own_stream);
  if (s != LOFP_OK) return s;
  CK(cudaMemcpyAsync(amps, ctx->d_hostA.p, ab, cudaMemcpyDeviceToHost, ctx->own_stream), "copy amps");
  CK(cudaStreamSynchronize(ctx->own_stream), "cudaStreamSynchronize");
  return LOFP_OK;
}

lofp_status lofp_stats(lofp_ctx *ctx, lofp_run_stats *out) {
  if (!ctx || !out) return LOFP_E_INVALID_ARG;
  if (ctx->have_call) {
    CK(cudaEventSynchronize(ctx->ev_end), "cudaEventSynchronize");
    const Counters *hc = (const Counters *)ctx->h_ctr.p;
    ctx->stats.feasible = (int64_t)hc->nfeas;
    ctx->stats.items = (int64_t)hc->items;
    ctx->stats.spills = (int64_t)hc->spills;
    ctx->stats.donations = (int64_t)hc->donations;
    ctx->stats.overflows = (int64_t)hc->ovf;
    ctx->stats.paths = (int64_t)hc->leaves;
    ctx->stats.cmuls = (int64_t)hc->cmuls;
    ctx->stats.chains = (int64_t)hc->chains;
    ctx->stats.chain_fallbacks = (int64_t)hc->chain_fb;
    ctx->stats.bad_rows = (int32_t)hc->bad_rows;
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, ctx->ev_enum0, ctx->ev_enum1) == cudaSuccess) ctx->stats.enum_ms = ms;
    if (cudaEventElapsedTime(&ms, ctx->ev_start, ctx->ev_end) == cudaSuccess) ctx->stats.total_ms = ms;
    ctx->have_call = false;
  }
  *out = ctx->stats;
  return ctx->stats.bad_rows ? LOFP_E_BAD_OUTPUT : LOFP_OK;
}

lofp_status lofp_work_histograms(lofp_ctx *ctx, uint64_t *handover, uint64_t *spill) {
  if (!ctx || !handover || !spill) return LOFP_E_INVALID_ARG;
  if (ctx->h_ctr.p == nullptr) {
    for (int i = 0; i < 64; ++i) handover[i] = spill[i] = 0;
    return LOFP_OK;
  }
  CK(cudaEventSynchronize(ctx->ev_end), "cudaEventSynchronize");
  const Counters *hc = (const Counters *)ctx->h_ctr.p;
  for (int i = 0; i < 64; ++i) {
    handover[i] = hc->don_hist[i];
    spill[i] = hc->spill_hist[i];
  }
  return LOFP_OK;
}

lofp_status lofp_phase_cycles(lofp_ctx *ctx, uint64_t *cycles) {
  if (!ctx || !cycles) return LOFP_E_INVALID_ARG;
  for (int i = 0; i < 8; ++i) cycles[i] = 0;
  if (ctx->h_ctr.p == nullptr) return LOFP_OK;
  CK(cudaEventSynchronize(ctx->ev_end), "cudaEventSynchronize");
  const Counters *hc = (const Counters *)ctx->h_ctr.p;
  for (int i = 0; i < 8; ++i) cycles[i] = hc->phase_cyc[i];
  return LOFP_OK;
}

void lofp_destroy(lofp_ctx *ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->ev_end) cudaEventSynchronize(ctx->ev_end);
  for (DevBuf *b : {&ctx->d_maps, &ctx->d_bs_lk, &ctx->d_bs_cs, &ctx->d_flags, &ctx->d_plans, &ctx->d_feas,
                    &ctx->d_ctr, &ctx->d_ring, &ctx->d_edesc, &ctx->d_offsets, &ctx->d_entries, &ctx->d_cumS,
                    &ctx->d_bsrow, &ctx->d_hostT, &ctx->d_hostA})
    b->release();
  ctx->h_stage.release();
  ctx->h_ctr.release();
  for (cudaEvent_t ev : {ctx->ev_start, ctx->ev_enum0, ctx->ev_enum1, ctx->ev_end})
    if (ev) cudaEventDestroy(ev);
  if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
  delete ctx;
}

}  // extern "C"
