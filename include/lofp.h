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
 * (P:354-408).  lofp_amplitudes forms the product of every valid path on the GPU and
 * adds it (no permanent is used); lofp_amplitudes_contract evaluates the same sum by the
 * paper's strip tensor contraction instead.
 *
 * Conventions.
 *   - Modes are 0-based.  A BS is given as (mode_a, mode_b, theta, phi); mode_a is BS
 *     port 1, the "upper" waveguide of P:92 and P:363 (x1 = photons entering mode_a,
 *     y1 = photons leaving it).  A pair listed in reverse order is accepted and is the
 *     same element as (mode_b, mode_a, theta, pi - phi) (port swap).
 *   - Layers are applied in the order given (layer 0 first); BS inside one layer must
 *     act on disjoint modes (P:65 planar mesh).  Modes not covered by a layer pass
 *     through unchanged.  Pairs may be non-adjacent and may cross ("non-local
 *     connections"); nearest-neighbour meshes are the fast case.
 *   - theta and phi may be any finite doubles (P:80 states theta in [0, pi/2] and phi in
 *     [0, pi]; the benchmark configurations draw phi in [0, 2 pi)).
 *   - An output whose photon number differs from the input's gets exactly 0; so does an
 *     output that no path reaches.
 *   - Results are bitwise reproducible run to run (fixed summation order; no floating-
 *     point atomics).
 *
 * Threading, streams and ownership.  A context owns its device memory and must not be
 * used from two host threads at once; separate contexts are independent.  Every device
 * call enqueues its work on the stream it is given and returns without waiting for it
 * (no host synchronisation, no device-to-host read); buffers that must grow (a bigger
 * batch or input than before) are reallocated stream-ordered (cudaFreeAsync /
 * cudaMallocAsync on the call's stream).  A call can be captured in a CUDA graph once a
 * call of the same sizes has run outside capture (no buffer grows during capture).
 * Consecutive calls on one context are ordered after each other even on different
 * streams (outside capture).  The library never frees caller memory and never throws or
 * aborts across this boundary.
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

/* A photon-number-preserving phase gate ("nonlinear phase gates are also photon-
 * number preserving"): on mode `mode` after layer `after_layer` (0 = on the input, D =
 * on the output) it multiplies the state |n> of that mode by exp(i (a n + b n^2)).
 * b = 0 is a linear phase shifter; b != 0 a Kerr-type nonlinear phase. */
typedef struct {
  int32_t mode;
  int32_t after_layer;
  double a;
  double b;
} lofp_gate;

typedef enum {
  LOFP_OK = 0,
  LOFP_E_INVALID_ARG = 1, /* null pointer, bad count, mode out of range, overlapping
                             pairs in one layer, non-finite angle, negative input */
  LOFP_E_UNSUPPORTED = 2, /* too many modes/photons/layers/gates, or a circuit whose
                             column description exceeds the topology limits */
  LOFP_E_CUDA = 3,        /* a CUDA runtime error; text in lofp_last_error() */
  LOFP_E_OOM = 4,         /* device allocation failed */
  LOFP_E_BAD_OUTPUT = 5   /* an output row had a negative entry; its amplitude is NaN */
} lofp_status;

/* Limits of this build.  Photon numbers are uint8 segment values; a column of the path
 * tree (the photon counts left of one cut over all layers) may take at
 * most 4096 values inside the light-cone box, 65536 summed over the columns of one
 * output; an output over these limits is evaluated by the generic engine (the paper's
 * layer-major recursion, lofp_run_stats.generic) and gets NaN only if that exceeds its
 * node budget (lofp_run_stats.unsupported). */
#define LOFP_MAX_MODES 128
#define LOFP_MAX_PHOTONS 120
#define LOFP_MAX_LAYERS 64
#define LOFP_MAX_GATES 4096

/* Create a context for one circuit.
 *   modes         M >= 1, M <= LOFP_MAX_MODES.
 *   n_layers      D >= 0 (D = 0 is the identity circuit), D <= LOFP_MAX_LAYERS.
 *   bs_per_layer  host array [n_layers], each >= 0 (NULL allowed when n_layers == 0).
 *   bs            host array [sum bs_per_layer], layer-major (NULL allowed when empty).
 *   out           receives the new context (set to NULL on failure).
 * Copies everything it is given; uploads the circuit's topology tables (synchronously,
 * once).  Uses the current CUDA device.  Errors: LOFP_E_INVALID_ARG, LOFP_E_UNSUPPORTED,
 * LOFP_E_CUDA, LOFP_E_OOM. */
lofp_status lofp_create(int32_t modes, int32_t n_layers, const int32_t *bs_per_layer,
                        const lofp_bs *bs, lofp_ctx **out);

/* lofp_create plus phase gates.  gates: host array [n_gates] (NULL when 0),
 * 0 <= mode < modes, 0 <= after_layer <= n_layers, finite a and b, n_gates <=
 * LOFP_MAX_GATES.  Several gates on one (mode, layer) multiply. */
lofp_status lofp_create_ex(int32_t modes, int32_t n_layers, const int32_t *bs_per_layer,
                           const lofp_bs *bs, int32_t n_gates, const lofp_gate *gates,
                           lofp_ctx **out);

/* Amplitudes <T_b|U_P|S> for a batch of outputs by the path sum (eq. (1)):
 * every valid path's product is formed and added on the GPU.
 *   input_occ     host int32 [modes]: S (entries >= 0, sum <= LOFP_MAX_PHOTONS).
 *   batch         B >= 0 (B = 0 is a no-op).
 *   output_occ    DEVICE int32 [B][modes], row-major: T_b.
 *   amps          DEVICE double [B][2]: complex128 results (re, im interleaved).
 *   cuda_stream   cudaStream_t to run on (NULL = legacy default stream).
 * Host arguments are validated before any device work; the kernels are enqueued on
 * cuda_stream and the call returns (see "Threading, streams and ownership").
 * output_occ and amps must stay valid until the stream has run the work.  A row with a
 * negative entry gets NaN (lofp_stats() then returns LOFP_E_BAD_OUTPUT).
 * Errors: LOFP_E_INVALID_ARG, LOFP_E_UNSUPPORTED, LOFP_E_CUDA, LOFP_E_OOM. */
lofp_status lofp_amplitudes(lofp_ctx *ctx, const int32_t *input_occ, int64_t batch,
                            const int32_t *output_occ, double *amps, void *cuda_stream);

/* Same as lofp_amplitudes, and also the number of path products formed for every
 * output: path_counts is a DEVICE uint64 [B] (written, not accumulated).  Equal to the
 * exact number of valid paths of eq. (1) (the kernel checks it against an independent
 * count; lofp_stats() reports a mismatch).  Same cost as lofp_amplitudes. */
lofp_status lofp_amplitudes_counted(lofp_ctx *ctx, const int32_t *input_occ, int64_t batch,
                                    const int32_t *output_occ, double *amps,
                                    uint64_t *path_counts, void *cuda_stream);

/* The same amplitudes by the paper's strip tensor contraction (its code path
 * for every D > 2): the circuit is contracted cut by cut from the top mode to the
 * bottom one; the state crossing cut k is the pair of light-cone-live columns (photon
 * counts left of cuts k-1 and k over all layers, the tuples l_{k,j} of P:183-185), each
 * with its partial amplitude.  Work per output is the number of (column, column, column)
 * triples instead of the number of paths, so outputs with 1e15+ paths (configs[3] as
 * drawn) take microseconds; no path products are formed.  Arguments, asynchrony, errors
 * and NaN/zero rules as lofp_amplitudes.  path_counts: optional DEVICE uint64 [B]
 * (NULL allowed) receiving the exact number of valid paths of each output (the column
 * count, saturating at 2^64-1).  An output whose column-pair level exceeds the scratch
 * gets NaN and is counted as unsupported. */
lofp_status lofp_amplitudes_contract(lofp_ctx *ctx, const int32_t *input_occ, int64_t batch,
                                     const int32_t *output_occ, double *amps,
                                     uint64_t *path_counts, void *cuda_stream);

/* All output amplitudes for one input ("simultaneously calculate and store the
 * amplitudes of all possible output states for a given input").  Writes the
 * C(N+M-1, M-1) patterns of N = sum(S) photons in M modes to outputs (DEVICE int32
 * [count][modes], ordered by decreasing T_0, then decreasing T_1, ...) and their
 * amplitudes to amps (DEVICE double [count][2]) in one stream-ordered call.
 *   max_outputs   capacity of outputs / amps in rows.
 *   n_outputs     HOST int64: receives the pattern count (also when it exceeds
 *                 max_outputs, which returns LOFP_E_INVALID_ARG without device work).
 *   method        0 = strip contraction (lofp_amplitudes_contract), 1 = path sum
 *                 (lofp_amplitudes).
 * Errors: LOFP_E_INVALID_ARG, LOFP_E_UNSUPPORTED (more than 2^31 - 1 patterns),
 * LOFP_E_CUDA, LOFP_E_OOM. */
lofp_status lofp_distribution(lofp_ctx *ctx, const int32_t *input_occ, int64_t max_outputs,
                              int32_t *outputs, double *amps, int64_t *n_outputs,
                              int32_t method, void *cuda_stream);

/* Guard against unexpectedly large path trees (SURVEY §5 "failure detection"): path-sum
 * calls on ctx skip every output with more than max_paths_per_output valid paths (counted
 * exactly by the plan kernel before any enumeration) and give it NaN; lofp_stats() reports
 * how many (over_budget).  0 (the default) = no limit.  The contraction and the
 * distribution are not limited (their cost does not grow with the path count). */
lofp_status lofp_set_path_budget(lofp_ctx *ctx, uint64_t max_paths_per_output);

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

/* Measurement / validation counters of the last device call.  Reading them synchronises
 * that call's work (the only synchronising entry besides _host and destroy). */
typedef struct {
  int64_t batch;          /* B of the last call */
  int64_t feasible;       /* outputs with at least one valid path */
  int64_t paths;          /* path products formed (sum over the batch) */
  int64_t cmuls;          /* other complex multiplications: half-path list products, the
                             per-pair scalings of the lists */
  int64_t units;          /* work units (subtrees) processed */
  int64_t subsplits;      /* units split again inside the kernel (lists over capacity) */
  int64_t pairs;          /* column-pair states multiplied out */
  int64_t elements;       /* half-path list elements built */
  int64_t unsupported;    /* outputs over a state limit (their amplitude is NaN) */
  int64_t bad_rows;       /* rows with a negative entry (their amplitude is NaN) */
  int64_t check_errors;   /* internal consistency failures (must be 0): a path-count
                             mismatch or a table index outside its block */
  int64_t max_states;     /* largest number of column states of one output */
  int64_t max_list;       /* largest half-path list */
  int64_t table_entries;  /* Appendix-A elements in the table */
  int64_t terms;          /* contraction mode: (state, state, state) terms summed */
  int64_t over_budget;    /* outputs skipped by lofp_set_path_budget (their amplitude is NaN) */
  int64_t generic;        /* outputs evaluated by the generic engine (the paper's layer-major
                             recursion with its cone bounds) because their
                             columns exceed the column engine's limits */
  int64_t phase_cycles[8];/* unit kernel, SM clock cycles of each block's thread 0 summed over
                             blocks: 0 kernel tail, 1 path counts and split choice, 2 left
                             lists, 3 right lists, 4 pair list and scaling tables, 5 warp tiles
                             (path products), 6 waiting for the block's other warps after the
                             tiles, 7 unit fetch, output setup, stack pops and reduction */
  int64_t tile_cycles[2]; /* unit kernel, warp clocks (lane 0, summed over warps) in the path-
                             product tiles: [0] staging the tile's X and Y values, [1] the FMA
                             loop */
  int32_t grid_blocks;    /* persistent grid of the unit kernel */
  int32_t block_threads;  /* threads per block */
  int32_t launches;       /* kernels launched by the call */
  int32_t mode;           /* 0 path sum, 1 strip contraction */
  float units_ms;         /* device time of the unit (enumeration) kernel, CUDA events;
                             contraction mode: of the contraction kernel */
  float total_ms;         /* device time from the first to the last kernel */
  int64_t contract_deferred; /* contraction mode: outputs whose state space exceeded the
                             warp-per-output kernel's limits and went to the block kernel */
} lofp_run_stats;

lofp_status lofp_stats(lofp_ctx *ctx, lofp_run_stats *out);

#ifdef __cplusplus
}
#endif

#endif /* LOFP_H */
