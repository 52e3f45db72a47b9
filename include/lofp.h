/*
 * lofp.h — C ABI of liblofp, a B200 (sm_100a) implementation of the Linear-Optical
 * Feynman Path sum of arXiv 2510.26408 ("Feynman path sum approach for simulation of
 * linear optics").  Citations "P:n" are lines of the paper's text.
 *
 * What is computed.  For a mesh of two-mode beam splitters (BS) arranged in layers
 * with BS matrix (eq. bs_matrix)
 *     BS(theta, phi) = [[cos theta, -e^{-i phi} sin theta], [e^{i phi} sin theta, cos theta]],
 * an input Fock state |S> and a batch of output Fock states |T_b>, every call returns
 *     <T_b| U_P |S> = sum over valid paths p of prod_{BS i} <y1_i, y2_i| BS_i |x1_i, x2_i>
 * (eq. (1)): a valid path assigns photon numbers to every waveguide segment,
 * conserving x1+x2 = y1+y2 at every BS, with the input segments equal to S and the
 * output segments equal to T.  The BS elements are those of Appendix A
 * (P:354-408).  The sum is enumerated on the GPU path by path; no permanent is used.
 *
 * Conventions.
 *   - Modes are 0-based.  A BS is given as (mode_a, mode_b, theta, phi); mode_a is BS
 *     port 1, the "upper" waveguide of P:92 and P:363 (x1 = photons entering mode_a,
 *     y1 = photons leaving it).  A pair listed in reverse order is accepted and is the
 *     same element as (mode_b, mode_a, theta, pi - phi) (port swap).
 *   - Layers are applied in the order given (layer 0 first); BS inside one layer must
 *     act on disjoint modes (P:65 planar mesh).  Modes not covered by a layer pass
 *     through unchanged.  This version requires nearest-neighbour pairs
 *     (|mode_a - mode_b| = 1), the locally connected meshes of P:105 and P:144.
 *   - theta and phi may be any finite doubles (P:80 states theta in [0, pi/2] and phi in
 *     [0, pi]; the benchmark configurations draw phi in [0, 2 pi)).
 *   - An output whose photon number differs from the input's gets exactly 0; so does an
 *     output that no path reaches.
 *
 * Threading and ownership.  A context owns its device memory and must not be used from
 * two host threads at once; separate contexts are independent.  The library never frees
 * caller memory and never throws or aborts across this boundary.
 */
#ifndef LOFP_H
#define LOFP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct lofp_ctx lofp_ctx;

/* One beam splitter: modes (mode_a, mode_b), angles (theta, phi) of eq. bs_matrix. */
typedef struct {
  int32_t mode_a;
  int32_t mode_b;
  double theta;
  double phi;
} lofp_bs;

typedef enum {
  LOFP_OK = 0,
  LOFP_E_INVALID_ARG = 1, /* null pointer, bad count, mode out of range, overlapping
                             pairs in one layer, non-finite angle, negative input */
  LOFP_E_UNSUPPORTED = 2, /* non-adjacent pair, too many modes/photons/levels */
  LOFP_E_CUDA = 3,        /* a CUDA runtime error; text in lofp_last_error() */
  LOFP_E_OOM = 4,         /* device allocation failed */
  LOFP_E_BAD_OUTPUT = 5   /* an output row had a negative entry; its amplitude is NaN */
} lofp_status;

/* Limits of this build (uint8 photon numbers; bounded DFS metadata). */
#define LOFP_MAX_MODES 128
#define LOFP_MAX_PHOTONS 120
#define LOFP_MAX_LAYERS 64

/* Create a context for one circuit.
 *   modes         M >= 1, M <= LOFP_MAX_MODES.
 *   n_layers      D >= 0 (D = 0 is the identity circuit), D <= LOFP_MAX_LAYERS.
 *   bs_per_layer  host array [n_layers], each >= 0 (NULL allowed when n_layers == 0).
 *   bs            host array [sum bs_per_layer], layer-major (NULL allowed when empty).
 *   out           receives the new context (set to NULL on failure).
 * Copies everything it is given; allocates only small device buffers.  Uses the
 * current CUDA device.  Errors: LOFP_E_INVALID_ARG, LOFP_E_UNSUPPORTED, LOFP_E_CUDA,
 * LOFP_E_OOM. */
lofp_status lofp_create(int32_t modes, int32_t n_layers, const int32_t *bs_per_layer,
                        const lofp_bs *bs, lofp_ctx **out);

/* Amplitudes <T_b|U_P|S> for a batch of outputs (eq. (1)).
 *   input_occ     host int32 [modes]: S (entries >= 0, sum <= LOFP_MAX_PHOTONS).
 *   batch         B >= 0 (B = 0 is a no-op).
 *   output_occ    DEVICE int32 [B][modes], row-major: T_b.
 *   amps          DEVICE double [B][2]: complex128 results (re, im interleaved).
 *   cuda_stream   cudaStream_t to run on (NULL = legacy default stream).
 * Host arguments are validated before any device work.  The call enqueues its kernels
 * on cuda_stream; it synchronises that stream once, after the first (feasibility)
 * kernel, to size the shared-memory BS tables from the batch's per-mode maximum, and
 * returns with the enumeration still running: the caller synchronises the stream before
 * reading amps.  output_occ and amps must stay valid until then.  A row with a negative
 * entry gets NaN and LOFP_E_BAD_OUTPUT is returned by lofp_stats() after completion.
 * Errors: LOFP_E_INVALID_ARG, LOFP_E_UNSUPPORTED, LOFP_E_CUDA, LOFP_E_OOM. */
lofp_status lofp_amplitudes(lofp_ctx *ctx, const int32_t *input_occ, int64_t batch,
                            const int32_t *output_occ, double *amps, void *cuda_stream);

/* Same as lofp_amplitudes, and also the exact number of valid paths summed for every
 * output: path_counts is a DEVICE uint64 [B] (written, not accumulated).  Slightly
 * slower (one integer add per path); used by the parity tests to check that every path
 * of eq. (1) is enumerated exactly once. */
lofp_status lofp_amplitudes_counted(lofp_ctx *ctx, const int32_t *input_occ, int64_t batch,
                                    const int32_t *output_occ, double *amps,
                                    uint64_t *path_counts, void *cuda_stream);

/* End-to-end convenience: HOST buffers in and out.  Copies output_occ (host int32
 * [B][modes]) to the device, runs lofp_amplitudes on an internal stream, copies the
 * amplitudes back into amps (host double [B][2]) and returns when they are there. */
lofp_status lofp_amplitudes_host(lofp_ctx *ctx, const int32_t *input_occ, int64_t batch,
                                 const int32_t *output_occ, double *amps);

/* Synchronises the context's work and frees everything it owns.  NULL is a no-op. */
void lofp_destroy(lofp_ctx *ctx);

/* Static description of a status code. */
const char *lofp_status_string(lofp_status s);

/* Message for the last failing call on ctx ("" if none); valid until the next call. */
const char *lofp_last_error(const lofp_ctx *ctx);

/* Measurement / validation counters of the last lofp_amplitudes* call.  Reading them
 * synchronises the call's stream. */
typedef struct {
  int64_t batch;          /* B of the last call */
  int64_t feasible;       /* outputs whose path tree has at least one free level */
  int64_t items;          /* work items (subtrees) processed by the enumeration kernel */
  int64_t spills;         /* subtrees pushed to the global work queue */
  int64_t donations;      /* subtrees handed between lanes of one warp */
  int64_t overflows;      /* branch-stack entries that went to the local overflow */
  int64_t paths;          /* valid paths summed (lofp_amplitudes_counted only, else 0) */
  int64_t cmuls;          /* complex multiplications executed (counted only, else 0): DFS
                             factors with x1 + x2 > 0, chain pair-table factors, chain products */
  int64_t chains;         /* chain subtrees enumerated by the lockstep chain engine */
  int64_t chain_fallbacks;/* chains walked depth-first instead (pair table over capacity) */
  int32_t levels;         /* largest number of free DFS levels of one output */
  int32_t table_entries;  /* Appendix-A elements staged in shared memory */
  int32_t smem_bytes;     /* dynamic shared memory per block of the enumeration kernel */
  int32_t grid_blocks;    /* persistent grid size */
  int32_t block_threads;  /* threads per block */
  int32_t bad_rows;       /* rows with a negative entry (their amplitude is NaN) */
  int32_t max_factors;    /* largest number of attached BS elements of one output */
  int32_t max_scatter;    /* largest number of key bytes written per level value, one output */
  int32_t engine;         /* 0: depth-first walk only; 1: chain engine (R17); 2: chain engine
                             with the short chains batched (short-chain mode) */
  int32_t launches;       /* kernels launched by the call (prep, tables, plan(s), enumeration) */
  float enum_ms;          /* device time of the enumeration kernel (CUDA events) */
  float total_ms;         /* device time from the first to the last kernel */
} lofp_run_stats;

lofp_status lofp_stats(lofp_ctx *ctx, lofp_run_stats *out);

/* Work-distribution histograms of the last lofp_amplitudes_counted call (zeros after an
 * uncounted call): subtrees handed between lanes of a warp (handover) and pushed to the
 * global queue (spill), indexed by (deepest level - level of the handed-over branch),
 * clamped to 63.  handover and spill are host uint64 [64].  Synchronises the call. */
lofp_status lofp_work_histograms(lofp_ctx *ctx, uint64_t *handover, uint64_t *spill);

/* Enumeration-kernel time split of the last lofp_amplitudes_counted call (zeros after an
 * uncounted call): SM clock cycles summed over warps (lane 0's clock) in 8 phases --
 * 0 depth-first step and hand-over, 1 chain ranges, 2 chain pair table, 3 chain split and
 * prefix digits, 4 chain path products, 5 return to the walk and global-queue feeding,
 * 6 work acquisition, plan staging and item reduction, 7 chain suffix table.  cycles is a host uint64 [8].  Synchronises the call. */
lofp_status lofp_phase_cycles(lofp_ctx *ctx, uint64_t *cycles);

#ifdef __cplusplus
}
#endif

#endif /* LOFP_H */
