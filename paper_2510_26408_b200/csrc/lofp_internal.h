// lofp_internal.h — data shared by the host runtime (lofp_host.cpp) and the sm_100a
// kernels (lofp_kernels.cu) of liblofp.  Nothing here is part of the C ABI.
//
// The path sum of eq. (1) is organised by *columns*: column k (k = 0..M) is the
// history F_0(k), ..., F_D(k) of the cumulative photon number F_t(k) = photons in modes
// < k after layer t (reading R5).  F_t(k) changes only at the layers whose BS
// sits on modes (k-1, k) ("cut k active"), so a column is a short tuple of *segment*
// values; a valid path is a sequence of columns with F_t(k-1) <= F_t(k) for every t
// (non-negative occupations) between the fixed columns 0 (all 0) and M (all N),
// whose first segment is cum(S) and last is cum(T).  A BS on cut c reads columns
// c-1, c, c+1 only (x1 = F(c) - F(c-1), x2 = F(c+1) - F(c), y1 = F'(c) - F(c-1)),
// so the product of eq. (1) factorises into one *cut factor* per cut c = 1..M-1
// (reading R20).
#ifndef LOFP_INTERNAL_H
#define LOFP_INTERNAL_H

#include <cstdint>

namespace lofp {

constexpr int kMaxModes = 128;     // LOFP_MAX_MODES
constexpr int kMaxLayers = 64;     // LOFP_MAX_LAYERS
constexpr int kMaxPhotons = 120;   // LOFP_MAX_PHOTONS (uint8 segment values)
constexpr int kMaxStates = 4096;   // states of one column (uint16 indices)
constexpr int kMaxStatesTotal = 1 << 16;  // sum over the columns of one output
constexpr int kMaxSegments = 1 << 16;     // (state, predecessor) pairs of one BFS level
constexpr int kThreads = 256;      // threads per block of the plan / unit / contraction kernels
constexpr int kKX = 8;             // X values held in registers per lane (outer product)
constexpr int kXT = 32 * kKX;      // X values per warp tile
constexpr int kYT = 256;           // Y values per warp tile (staged in the warp's shared slice)
constexpr int kCY = kYT * (kThreads / 32);  // shared memory: one Y slice per warp
constexpr int kStackMax = 4096;    // sub-split stack entries per block
constexpr int kMaxRawStates = 1 << 18;  // non-local circuits: raw variable product per column

// ---- topology (lofp_create; constant per circuit) --------------------------------
struct ColInfo {         // column k = 0..M
  uint16_t seg_base;     // first SegInfo / variable slot of the column
  uint8_t nseg;          // number of segments (1 + number of active layers of cut k)
  uint8_t ncmp;          // CmpPair checks against column k-1 (k >= 1)
  uint16_t cmp_base;
  uint16_t fac_base;     // FacInfo of the BS whose factor cut k carries, in layer order
  uint8_t nfac;
  uint8_t ngate;         // phase gates folded into cut k's factor
  uint16_t gate_base;
  uint8_t nvar;          // state variables: the nseg segments, then carried BS variables
  uint8_t neq;           // EqCon checks against column k-1 (non-local circuits only)
  uint16_t eq_base;
  uint8_t nintra;        // EqCon checks inside column k (non-local circuits only)
  uint8_t pad;
  uint16_t intra_base;
};

// Non-local circuits (NEXT-4): a BS on modes (a, b), b > a + 1, shifts every cut in
// (a, b]; its photon numbers (x1, y1) on mode a are carried as state variables through the
// columns a+1..b, so that every constraint stays between adjacent columns (R21).
struct EqCon {           // sum_t coef[t] * var[t] == 0 over variables of columns k-1 and k
  int8_t coef[11];
  uint8_t var[11];       // bit 7: column k (else k-1); bits 0..6: variable index
  uint8_t nterm;
  uint8_t pad;
};

struct SeqBS {           // generic engine: BS in layer-major order
  int32_t bs;            // table block
  uint8_t lo, hi;        // port-1 (lower) and port-2 modes
  uint8_t layer;         // 1-based
  uint8_t gl0, gl1;      // gates of layers gl0..gl1-1 apply after this BS (layer ends)
  uint8_t pad[3];
};

struct BoundInfo {       // non-local circuits: light-cone bounds of a variable as mode sets
  uint64_t m[4][2];      // hi <= sum S over m[0] and sum T over m[2];
};                       // lo >= N - sum S over m[1] and N - sum T over m[3]

struct SegInfo {         // light-cone box of a segment (readings R5, R15)
  uint8_t rho, sig;      // backward maps: F in [G(rho), G(sig)]
  uint8_t rhop, sigp;    // forward maps:  F in [cumS(rhop), cumS(sigp)]
};

struct CmpPair {         // F(k-1) on segment sa <= F(k) on segment sb (one time interval)
  uint8_t sa, sb;
};

struct FacInfo {         // a BS whose factor cut c carries (layer l)
  int32_t bs;            // canonical BS index (table block)
  uint8_t sA;            // kind 0: segment of column c-1 holding F_{l-1}(c-1);
                         // kind 1: variable of column c holding y1 (carried)
  uint8_t i;             // kind 0: segments i (F_{l-1}(c)) and i+1 (F_l(c)) of column c;
                         // kind 1: variable of column c holding x1 (carried)
  uint8_t sC;            // segment of column c+1 holding F_{l-1}(c+1)
  uint8_t kind;          // 0 nearest-neighbour BS on (c-1, c); 1 carried BS ending at mode c
  uint8_t sB;            // kind 1: segment of column c holding F_{l-1}(c)
  uint8_t pad[3];
};

struct GateInfo {        // gate on mode m after layer j, folded into cut c's factor
  int32_t gate;          // row of the phase table
  uint8_t col_off;       // mode m's lower column is c-1+col_off (its upper is c+col_off)
  uint8_t seg_lo, seg_hi;  // segments of those columns holding time j
  uint8_t pad;
};

struct BSInfo {          // canonical BS (port 1 = the lower mode), eq. bs_matrix
  double c, s, phi;      // cos theta, sin theta, phi (port swap applied, reading R4)
  uint8_t cap_lo, cap_hi;  // photons through it <= cumS(cap_hi) - cumS(cap_lo) (past cone)
  uint8_t pad[6];
  uint64_t capmask[2];   // non-local circuits: photons through it <= sum S over this mode set
};

// ---- per-call data -----------------------------------------------------------------
struct Unit {            // a subtree of one output: columns 0..j fixed
  int32_t q;             // output row
  int16_t j;             // last fixed column
  uint16_t sjm1, sj;     // states of columns j-1 and j
  uint16_t pad;
  double re, im;         // product of the cut factors of cuts 1..j-1 along the prefix
  uint64_t paths;        // exact number of paths below the prefix
};

struct Counters {        // device counters of one call (zeroed by the host)
  unsigned long long paths;      // path products formed (units kernel)
  unsigned long long cmuls;      // other complex multiplications (lists, scalings)
  unsigned long long units;      // units processed
  unsigned long long subsplits;  // units split inside the units kernel (lists over capacity)
  unsigned long long pairs;      // column-pair states multiplied out
  unsigned long long elements;   // half-path list elements built
  unsigned long long feasible;   // outputs with >= 1 path
  unsigned long long unsupported;// outputs over a state limit (NaN)
  unsigned long long bad_rows;   // outputs with a negative entry (NaN)
  unsigned long long ticket;     // unit work queue
  unsigned long long total_units;
  unsigned long long table_error;// a factor index outside its table block (must stay 0)
  unsigned long long max_states; // largest column state count seen
  unsigned long long max_list;   // largest half-path list built
  unsigned long long contractions; // contraction mode: column-pair states carried
  unsigned long long thr;        // unit size of the call (paths)
  unsigned long long phase[8];   // unit kernel, thread 0's SM clocks per phase
  unsigned long long generic;    // outputs evaluated by the generic (layer-major) engine
  unsigned long long over_budget;// outputs above the caller's path budget (NaN, not evaluated)
  unsigned long long tile_stage; // warp clocks staging X / Y of the path-product tiles
  unsigned long long tile_fma;   // warp clocks in the path-product FMA loop
  unsigned long long cticket;    // contraction: output queue of the warp kernel
  unsigned long long cdeferred;  // contraction: outputs the warp kernel left to the block kernel
};

enum : uint8_t { kStatusOk = 0, kStatusZero = 1, kStatusBad = 2, kStatusUnsupported = 3, kStatusOverBudget = 4,
                 kStatusDeferred = 5 /* contraction: left by the warp kernel to the block kernel */ };

struct CallParams {
  int M, D, N, B, nbs, ngate;
  int budget;            // unit slots per output
  int mode;              // 0 path sum, 1 contraction
  int units_per_block;   // unit size = max(thr, total paths / (units_per_block * grid))
  unsigned long long thr;  // smallest unit size (paths); the call's is in Counters::thr
  long long slab_bytes;  // per-block scratch in global memory
  long long cw_bytes;    // contraction warp kernel: scratch per warp (carved from the slab)
  int deferred_only;     // contraction block kernel: only outputs with kStatusDeferred
  int max_nfac;          // most BS a cut carries (contraction warp kernel instantiation)
  int contract_block_only;  // test hook (LOFP_CONTRACT_BLOCK): contraction by the block kernel only
  int contract_group;    // test hook (LOFP_CONTRACT_GROUP = 8 or 32): lanes per output of the warp kernel
  int contract_nosort;   // test hook (LOFP_CONTRACT_NOSORT): entries taken in storage order, not by row length
  long long table_cap;   // entries allocated for the Appendix-A table
  const ColInfo *col;
  const SegInfo *seg;
  const CmpPair *cmp;
  const FacInfo *fac;
  const GateInfo *gat;
  const BSInfo *bsi;
  const EqCon *eqc;
  const BoundInfo *bnd;      // [variables] non-local circuits only
  int general;               // 1: non-local circuit (mask bounds, carried variables)
  const SeqBS *seq;          // generic engine: the BS in layer-major order
  const uint64_t *cone;      // generic engine: [D+1][M][2][2] past / future cone masks of (t, m)
  int seq_gl0;               // gates of layers 0..seq_gl0-1 apply before the first BS
  int force_generic;         // test hook (LOFP_FORCE_GENERIC): every output by the generic engine
  unsigned long long path_budget;  // outputs with more paths are not evaluated (0 = no limit)
  const double *gate_ab;     // [ngate][2] (a, b)
  const int16_t *gate_mode;  // [ngate] mode, for M == 1 (no cut to fold into)
  const int16_t *gate_after; // [ngate] layer
  double2 *table;            // Appendix-A elements, per BS: tri(n) + x1 (n+1) + y1
  long long *tab_off;        // [nbs + 1]
  double2 *tableA;           // contraction only: the same elements, per BS [x2][y2][x1] (x1 <= cap - x2),
  long long *tabA_off;       //   so that for fixed (x2, y2) the index is linear in x1; [nbs + 1]
  long long tableA_cap;      //   entries allocated (0: not built)
  double2 *gate_tab;         // [ngate][N+1] exp(i (a n + b n^2))
  const int32_t *T;          // [B][M] device
  double2 *amps;             // [B]
  unsigned long long *counts;  // [B] or null: path products formed per output
  Unit *units;               // [B][budget]
  int *nunits;               // [B]
  int *ubase;                // [B+1] (exclusive scan of nunits)
  int *sched;                // [B][budget]: unit indices, largest size class first
  uint8_t *status;           // [B]
  unsigned long long *pexp;  // [B] exact number of paths (column count, reading R6)
  unsigned long long *pdone; // [B] path products formed
  double2 *partial;          // [sum nunits]
  char *slab;                // [grid][slab_bytes]
  Counters *ctr;
  uint8_t cumS[kMaxModes + 1];
};

// host-side size of the Appendix-A block of a BS that carries up to cap photons
inline long long tri_entries(int cap) {  // sum_{n=0}^{cap} (n+1)^2
  long long n = cap + 1;
  return n * (n + 1) * (2 * n + 1) / 6;
}

// host-side size of the contraction's x1-linear block ([x2][y2][x1], x1 + x2 <= cap)
inline long long lin_entries(int cap) {  // (cap+1) * sum_{x2=0}^{cap} (cap+1-x2)
  const long long c = cap + 1;
  return c * c * (c + 1) / 2;
}

}  // namespace lofp

// kernel launchers (lofp_kernels.cu)
extern "C" {
int lofp_launch_tables(const lofp::CallParams *p, void *stream);
int lofp_launch_paths(const lofp::CallParams *p, int grid, void *stream, void *ev_units0, void *ev_units1);
int lofp_launch_contract(const lofp::CallParams *p, int grid, void *stream);
int lofp_launch_contract_warp(const lofp::CallParams *p, int grid, void *stream);  // lofp_contract.cu
int lofp_units_grid(int device);
int lofp_launch_outputs(int M, int N, long long count, int32_t *T, void *stream);
int lofp_launch_generic(const lofp::CallParams *p, int grid, void *stream);
}

#endif  // LOFP_INTERNAL_H
