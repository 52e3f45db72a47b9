// lofp_internal.h — data layout shared by the host planner (lofp_host.cpp) and the
// sm_100a kernels (lofp_kernels.cu).  Nothing here is part of the public ABI.
//
// Vocabulary.  Cut k (0..M) sits between modes k-1 and k; F_l(k) is the
// number of photons in modes < k after layer l (F_0 = cum(S), F_D = G = cum(T)).  A BS
// of layer l on modes {k-1, k} is "active at cut k" and sets F_l(k); its Appendix-A
// element depends on a = F_{l-1}(k-1), b = F_{l-1}(k), c = F_{l-1}(k+1), y = F_l(k):
// x1 = b - a, x2 = c - b, y1 = y - a.
//
// Per output the plan kernel intersects the backward light-cone box [G(rho_l(k)),
// G(sigma_l(k))] (exact, reading R5) with the forward one [cumS(rho'_l(k)),
// cumS(sigma'_l(k))]; a BS output whose box is a single value is a constant (a "red"
// waveguide of P:130 for this output), the others are the DFS levels ("green")
// in layer-major order.  Every BS element is attached to the deepest level among its
// inputs; elements with constant inputs are folded into the output's root product.
#pragma once
#include <stdint.h>

#define LOFP_MAX_LEVELS 128   // DFS levels (free BS outputs) per circuit
#define LOFP_STK 4            // per-lane branch-stack entries kept in shared memory
#define LOFP_STK_CHAIN 2      // the same with the chain engine on
#define LOFP_OVF 128           // per-lane local-memory overflow entries (>= LOFP_MAX_LEVELS)
#define LOFP_ITEM_BYTES 256   // one global work-queue slot
#define LOFP_ITEM_PREFIX 224  // prefix bytes an item can carry (>= LOFP_MAX_LEVELS)
#define LOFP_SPILL_MIN_DIST 6  // global-queue spills only for branches >= this many levels above the leaf level
#define LOFP_CHAIN_MIN 4       // shortest chain handed to the chain engine
#define LOFP_CHAIN_RBOX 256    // smallest box product (paths bound) of an output's chain
#define LOFP_CHAIN_MODE_RBOX 1024.0  // batch mode: chain engine if most outputs' chain box >= this
#define LOFP_SMALL_LEVELS 16   // chains with <= this many levels and
#define LOFP_SMALL_PATHS 0     // < this many paths are enumerated in batches (0: off; the
                               // batched mode is slower than the walk on the configs measured)
#define LOFP_W_MAX 128         // chain pair-table entries per warp (else: plain DFS)
#ifndef LOFP_CHAIN_RMIN
#define LOFP_CHAIN_RMIN 8      // fewest paths of a chain enumerated by the engine (else: plain DFS)
#define LOFP_SHORT_CHAIN_LOG2 7.0  // short-chain mode: geometric-mean chain box >= 2^this paths
#endif
#define LOFP_SUF_ENTRIES 64     // chain suffix-table entries per warp
#define LOFP_ENUM_MAX_THREADS 640  // largest block of the enumeration kernel
#define LOFP_MAX_CUTS 130     // M + 1 for M <= LOFP_MAX_MODES (128)

// Per-lane value array ("vals") lives in shared memory, lane-interleaved by 32-bit word:
// byte s of lane i is at  warp_vals + ((s >> 2) * 32 + i) * 4 + (s & 3), so any 32 lanes
// reading any slots hit 32 distinct banks.  Plans store slots as the byte offset
// slot_off(s) relative to the lane's base (warp_vals + 4 * lane).
// Slot 0 is the lane's constant zero; DFS level j is slot j + 1.
__host__ __device__ inline uint16_t lofp_slot_off(int s) { return (uint16_t)(((s >> 2) << 7) | (s & 3)); }
__host__ __device__ inline uint16_t lofp_level_off(int j) { return lofp_slot_off(j + 1); }
#define LOFP_ZERO_OFF 0

// A DFS level j (a free F_l(k)).  Range at run time:
//   [max(vals[ol] + cl, lo), min(vals[or_] + cr, hi)]  with vals[ol] + cl = F_{l-1}(k-1),
//   vals[or_] + cr = F_{l-1}(k+1) (a constant uses the lane's zero slot), lo/hi the
//   output's box.  Factors [fbeg, fend) are the elements attached to this level;
//   scatter entries [sbeg, send & 0xfff) are the key bytes that hold this level's value;
//   the last (send >> 12) of them belong to chain factors (skipped while the engine is on).
struct __align__(16) PlanLevel {
  uint16_t ol, or_;
  uint8_t cl, cr, lo, hi;
  uint16_t fbeg, fend;
  uint16_t sbeg, send;
};

// One attached BS element.  Its per-lane key word holds the variable parts of its four
// inputs as bytes (a, b, c, y) = (F_{l-1}(k-1), F_{l-1}(k), F_{l-1}(k+1), F_l(k)); a
// constant input contributes 0 and is folded into base / dy / dx.  Then
//   row   = dp4a(key, crow, base)      = off_b + stride (x1) + x2
//   entry = offsets[row] + dp4a(key, (-1, 0, 0, 1), dy)   (+ y1)
//   x1 + x2 = dp4a(key, (-1, 0, 1, 0), dx)                 (counted mode only)
// with crow = (-stride, stride - 1, 1, 0) as signed bytes.
struct __align__(16) PlanFactor {
  int32_t crow;
  int32_t base;
  int8_t dy, dx;
  uint16_t chain;   // byte selector of the chain engine's pair-table key:
                    // key = __byte_perm(gathered key, v_m | v_{m-1} << 8, chain), nibble p =
                    // p (keep), 4 (v_m: the factor's own chain level) or 5 (v_{m-1})
  uint8_t slot[4];  // levels of (a, b, c, y) (0xff: constant), to gather a key from the
                    // value bytes (chain factors have no key word while the engine is on)
};

// The chain of an output (R17): the suffix of levels [jb, L) (the last
// free layer) whose ranges depend only on levels < jb and whose factors depend, among
// chain levels, only on their own level and the previous one.  Given levels < jb its
// subtree is a Cartesian product of fixed ranges, enumerated by a whole warp in lockstep.
struct PlanHead {
  double root[2];   // product of the elements with constant inputs
  uint16_t L, nfac; // levels and attached factors of this output
  uint16_t nscat;   // scatter entries (u16 key-byte offsets, after the factors)
  uint16_t jb;      // first chain level (L = no chain)
  uint64_t pad1;
};
static_assert(sizeof(PlanLevel) == 16 && sizeof(PlanFactor) == 16 && sizeof(PlanHead) == 32, "plan layout");

// One Appendix-A table entry to build: BS b, (x1, x2) -> (y1, x1 + x2 - y1).
struct EntryDesc {
  uint16_t bs;
  uint8_t x1, x2, y1, pad0, pad1, pad2;
};

// Per-call device counters (reset by the host before every call).
struct Counters {
  unsigned long long fresh_next;   // next feasible output to start
  unsigned long long ticket;       // next queue ticket (consumer side)
  unsigned long long tail;         // next queue slot (producer side)
  unsigned long long outstanding;  // work items not yet finished
  unsigned long long items;        // items started (stats)
  unsigned long long spills;       // items pushed to the global queue (stats)
  unsigned long long nfeas;        // outputs with a non-trivial tree
  unsigned long long bad_rows;     // rows with a negative entry
  unsigned long long cmuls;        // non-vacuum complex multiplications (counted mode)
  unsigned long long leaves;       // valid paths summed (counted mode)
  unsigned long long ovf;          // pushes that went to the local overflow stack
  unsigned long long donations;    // intra-warp hand-overs (stats)
  unsigned long long chains;       // chain subtrees enumerated by the chain engine
  unsigned long long phase_cyc[8]; // counted mode: SM cycles per phase (lane 0 of each warp)
  unsigned long long chain_fb;     // chains handed back to the plain walk (pair table too big)
  unsigned long long don_hist[64]; // counted mode: hand-overs by (leaf level - level)
  unsigned long long spill_hist[64];  // counted mode: queue spills by (leaf level - level)
  int32_t tmax[128];               // per-mode maximum of T over the batch
  int32_t maxL;                    // largest per-output level count
  int32_t maxF;                    // largest per-output attached-factor count
  int32_t maxS;                    // largest per-output scatter-list length
  int32_t maxK;                    // largest per-output count of non-chain factors
  int32_t nchain;                  // outputs whose plan has a chain
  int32_t nchain_ok;               // outputs whose last free layer has the chain structure
  int32_t nchain_big;              // those whose chain box >= LOFP_CHAIN_MODE_RBOX
  unsigned long long rbox_log16;   // sum over those of 16 log2(chain box product)
};

// A queued subtree: output `out`, levels [0, j0) fixed to prefix[], level j0 ranging
// over [vs, ve], product P of every factor attached to levels < j0 (and the root).
struct __align__(16) Item {
  unsigned int seq;   // = ticket + 1 once published, 0 when free
  unsigned int out;
  unsigned short j0;
  unsigned char vs, ve;
  unsigned int pad;
  double P[2];
  unsigned char prefix[LOFP_ITEM_PREFIX];
};
static_assert(sizeof(Item) == LOFP_ITEM_BYTES, "item size");

// Everything the kernels need for one call.
struct CallArgs {
  int M, D, N, nbs;
  int Lg;                             // global level bound (sizes the vals array)
  int vals_slots;                     // slots per lane (multiple of 4; slot 0 = zero)
  int nentries, noffsets;
  int64_t B;
  int plan_stride;                    // bytes per output plan (multiple of 16)
  int plan_smem;                      // bytes reserved per warp for a staged plan
  int maxfac;                         // attached factors per output (max; key words per lane)
  int warp_bytes;                     // per-warp shared memory (plan + vals + stack)
  int chain_on;                       // some output has a chain: engine scratch present
  int chain_rmin;                     // fewest paths of a chain run by the engine
  int small_paths;                    // chains with fewer paths are batched (0: off)
  double chain_rbox;                  // smallest box product of an output's chain
  int table_bytes;                    // shared memory of the staged tables (16-aligned)
  const int32_t *T;                   // [B][M] device
  double *amps;                       // [B][2] device
  unsigned long long *counts;         // [B] device or null
  uint8_t *flags;                     // [B] 1 = photon number matches, 2 = bad row
  unsigned char *plans;               // [B][plan_stride]
  uint32_t *feas;                     // [B] outputs with a non-trivial tree
  const uint8_t *cumS;                // [M+1]
  const uint8_t *maps;                // [4][D+1][M+1]: rho, sigma, rho', sigma'
  const int16_t *bs_lk;               // [nbs][2]: layer (1-based), cut; layer-major, by cut
  const int32_t *bs_base;             // [nbs]: offsets-table row of (x1, x2) = (0, 0)
  const int32_t *bs_stride;           // [nbs]: X2 cap + 1
  const EntryDesc *edesc;             // [nentries]
  const int32_t *offsets;             // [noffsets]
  double *entries;                    // [nentries][2]
  const double *bs_cs;                // [nbs][4]: cos theta, sin theta, cos phi, sin phi
  Counters *ctr;
  Item *ring;
  unsigned int ring_mask;             // capacity - 1 (power of two)
};

// Launchers (lofp_kernels.cu).
#include <cuda_runtime.h>
cudaError_t lofp_launch_prep(const CallArgs &a, cudaStream_t s);
cudaError_t lofp_launch_tables(const CallArgs &a, cudaStream_t s);
cudaError_t lofp_launch_plan(const CallArgs &a, cudaStream_t s);
cudaError_t lofp_enum_config(const CallArgs &a, bool counted, int *grid, int *block, size_t *smem);
cudaError_t lofp_launch_enum(const CallArgs &a, bool counted, int grid, int block, size_t smem,
                             cudaStream_t s);
