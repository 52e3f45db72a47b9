// lofp_internal.h — data layout shared by the host planner (lofp_host.cpp) and the
// sm_100a kernels (lofp_kernels.cu).  Nothing here is part of the public ABI.
//
// Vocabulary.  Cut k (0..M) sits between modes k-1 and k; F_l(k) is the
// number of photons in modes < k after layer l (F_0 = cum(S), F_D = G = cum(T)).  A BS
// of layer l on modes {k-1, k} is "active at cut k" and sets F_l(k); its Appendix-A
// element depends on x1 = F_{l-1}(k) - F_{l-1}(k-1), x2 = F_{l-1}(k+1) - F_{l-1}(k),
// y1 = F_l(k) - F_{l-1}(k-1).  The exact light-cone box (reading R5) confines F_l(k) to
// [G(rho_l(k)), G(sigma_l(k))]; a BS output with rho == sigma is forced (a "red"
// waveguide of P:130), the others are the DFS levels ("green" waveguides).
#pragma once
#include <stdint.h>

#define LOFP_MAX_LEVELS 224   // DFS levels (free BS outputs) per circuit
#define LOFP_VALS 512         // per-lane value array: [levels | G(0..M) | cumS(0..M)]
#define LOFP_STACK 64         // branch stack depth (>= log2 of any subtree's path count)
#define LOFP_ITEM_BYTES 256   // one work-queue slot
#define LOFP_ITEM_PREFIX 224  // prefix bytes an item can carry (= LOFP_MAX_LEVELS)

// A DFS level: the free output F_l(k) of one BS, in layer-major order (top to bottom
// inside a layer).  Its range is [max(v[refL], v[gLo]), min(v[refR], v[gHi])] where
// refL/refR are F_{l-1}(k-1), F_{l-1}(k+1) and gLo/gHi are G(rho_l(k)), G(sigma_l(k)).
// Factors [fbeg, fend) are the BS elements whose last unknown input is this level.
struct LevelDesc {
  uint16_t refL, refR, gLo, gHi;
  uint16_t fbeg, fend;
  uint16_t pad0, pad1;
};

// One BS element factor: value references of F_{l-1}(k-1), F_{l-1}(k), F_{l-1}(k+1)
// and F_l(k) into the per-lane value array, and the BS's table coordinates.
struct FactorDesc {
  uint16_t xl, xm, xr, y;
  int32_t offbase;  // index of (x1 = 0, x2 = 0) in the offsets table
  uint16_t stride;  // X2 cap + 1
  uint16_t bs;      // canonical BS index
};

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
  unsigned long long donations;    // items pushed by donation (stats)
  unsigned long long nfeas;        // feasible outputs (written by the feasibility kernel)
  unsigned long long bad_rows;     // rows with a negative entry
  int32_t tmax[128];               // per-mode maximum of T over the batch
  int32_t sum_mismatch;            // unused padding / diagnostics
  int32_t pad;
};

// A queued subtree: output `out`, levels [0, j0) fixed to prefix[], level j0 ranging
// over [vs, ve], product P of every factor attached to levels < j0 (and the root).
struct __align__(16) Item {
  unsigned int seq;   // = ticket + 1 once published
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
  int M, D, N, L, nfactors, nroot;    // nroot: factors attached to no level (constants)
  int nentries, noffsets;
  int64_t B;
  int grow;                           // bytes per G row (M+1 rounded up to 16)
  const int32_t *T;                   // [B][M] device
  double *amps;                       // [B][2] device
  unsigned long long *counts;         // [B] device or null
  uint8_t *flags;                     // [B] 1 = photon number matches, 2 = bad row
  uint8_t *G;                         // [B][grow]
  double *root;                       // [B][2]
  uint32_t *feas;                     // [B] feasible output ids
  const uint8_t *rho0, *sigma0;       // [M+1] box maps at time 0
  const uint8_t *cumS;                // [M+1]
  const LevelDesc *levels;            // [L]
  const FactorDesc *factors;          // [nfactors]; the first nroot are root factors
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
cudaError_t lofp_launch_feasible(const CallArgs &a, cudaStream_t s);
cudaError_t lofp_launch_finalize_counts(const CallArgs &a, cudaStream_t s);
cudaError_t lofp_enum_config(const CallArgs &a, bool counted, int *grid, int *block, size_t *smem);
cudaError_t lofp_launch_enum(const CallArgs &a, bool counted, int grid, int block, size_t smem,
                             cudaStream_t s);
