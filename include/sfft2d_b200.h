/*
 * sfft2d_b200 — C ABI of the B200-native 2D sparse FFT (SFFT, Algorithm 1) and
 * adaptive-sparsity ATSFFT (Algorithm 2) of arXiv 1908.02461.
 *
 * The reference (`/root/reference/pkg/src/sfft2d`) is a pure-Python package
 * with no FFI; its drop-in boundary is its Python API.  Each entry point below
 * replaces one reference function (cited) and is what a binding of that API
 * calls (see INTEGRATION.md for the ctypes stub the Python mirror uses).
 *
 * Conventions
 *  - Images are square N x N, N a power of two, row-major complex64
 *    (SFFT2D_C64) or complex128 (SFFT2D_C128), i.e. numpy's memory layout.
 *    `x_on_host` = 1: `x` is a host pointer (pinned or pageable) and the
 *    library performs the host->device copy on `stream`.
 *  - Arithmetic precision is selected per call: SFFT2D_FP64 reproduces the
 *    reference's float64 arithmetic (verification mode, 1e-10 parity);
 *    SFFT2D_FP32 is the fast path (1e-4 parity on values).
 *  - Permutations are drawn by the caller (numpy Generator, reference draw
 *    order, hashing.py:72-80) and passed in; the library never draws random
 *    numbers, so results are bit-reproducible for a given permutation list.
 *  - Window and twiddle tables are built by the caller on the host with the
 *    reference's formulas (hashing.py:138-246) and registered once per
 *    (N, delta_pass, delta_stop) with sfft2d_ctx_set_tables.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  Every call is
 *    stream-ordered; the transform entry points synchronise `stream` at the
 *    data-dependent decision points of the algorithm (tuner counts).
 *  - Return value: SFFT2D_OK or a negative status; nothing throws across the
 *    ABI.  sfft2d_ctx_last_error returns the message of the last failure.
 *  - Device workspace: by default a context grows named buffers stream-
 *    ordered from its OWN memory pool (never the device's default pool, whose
 *    attributes are left untouched).  A caller that owns all device memory
 *    (e.g. torch's caching allocator) hands the context one arena with
 *    sfft2d_ctx_set_workspace; the library then never allocates device memory
 *    and reports SFFT2D_ERR_NOMEM when the arena is too small.  The size a
 *    workload needs is sfft2d_ctx_workspace_size's `peak` after running it
 *    once.  Small pinned host buffers (count publication, result staging)
 *    stay library-owned.  A context is bound to one device and must not be
 *    used concurrently from two host threads.
 */
#ifndef SFFT2D_B200_H
#define SFFT2D_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SFFT2D_ABI_VERSION 3
#define SFFT2D_MAX_HISTORY 256

enum sfft2d_status {
  SFFT2D_OK = 0,
  SFFT2D_ERR_VALUE = -1,       /* maps to ValueError (corefft.py:45-50, hashing.py:306-311) */
  SFFT2D_ERR_CONFIG = -2,      /* maps to ConfigurationError (engine.py:45-109) */
  SFFT2D_ERR_CUDA = -3,
  SFFT2D_ERR_NOMEM = -4,
  SFFT2D_ERR_UNSUPPORTED = -5,
  SFFT2D_ERR_STATE = -6        /* missing tables / nothing to fetch */
};

enum sfft2d_dtype { SFFT2D_C64 = 0, SFFT2D_C128 = 1 };
enum sfft2d_precision { SFFT2D_FP32 = 0, SFFT2D_FP64 = 1 };

typedef struct sfft2d_ctx sfft2d_ctx;

/* PermutationParams (hashing.py:45-69) */
typedef struct {
  int64_t sigma1, sigma2, tau1, tau2, sigma1_inv, sigma2_inv;
} sfft2d_perm;

/* SfftConfig after __post_init__ defaults (engine.py:69-113) */
typedef struct {
  int32_t n, k, loops, d_factor, vote_threshold, b_bins;
  double window_delta_pass, window_delta_stop, gain_floor, prune_rel;
} sfft2d_sfft_config;

/* TunerConfig (tuner.py:47-78); max_tuning_iters < 0 means 2*log2(n) */
typedef struct {
  int32_t b0, max_tuning_iters;
  double eps1, eps2, delta1, delta2, mag_floor;
  double window_delta_pass, window_delta_stop, gain_floor, prune_rel;
} sfft2d_tuner_config;

/* TunerState (tuner.py:81-94) plus bookkeeping */
typedef struct {
  int32_t passes;
  int32_t hist_bins[SFFT2D_MAX_HISTORY];
  int64_t hist_count[SFFT2D_MAX_HISTORY];
  double hist_ratio[SFFT2D_MAX_HISTORY];
  int32_t hist_has_ratio[SFFT2D_MAX_HISTORY];
  double hist_us[SFFT2D_MAX_HISTORY];   /* host wall time of each pass (diagnostic) */
  int32_t converged;
  int64_t detected_k;
  int32_t b_detect, b_estimate, vote_passes;
  int32_t perms_used;       /* permutations consumed from the caller's list   */
  int64_t n_votes;          /* distinct voted coordinates (detect_sparsity)   */
  int64_t n_candidates;     /* coordinates at or above the vote threshold     */
  int32_t perms_drawn;      /* permutations drawn from the caller's generator:
                               the speculative fold draws the next pass's one
                               early, so when no estimation loop follows it
                               can exceed perms_used by one — a caller sharing
                               the generator with the reference restores its
                               state and redraws perms_used permutations    */
  int32_t pad_;
} sfft2d_tuner_state;

typedef struct {
  int64_t count;                 /* recovered coefficients available to fetch  */
  int32_t ordered_by_magnitude;  /* 1: reference dict order is lexsort(-|v|, i, j)
                                    (top-k cut happened, engine.py:245-248);
                                    0: row-major (i, j) order                  */
  int32_t precision;             /* element type of fetched values            */
  int64_t n_candidates;          /* voted coordinates that were estimated      */
  int32_t perms_used;
  int32_t gpu_launches;          /* kernels launched by this call             */
} sfft2d_result;

int sfft2d_abi_version(void);
int sfft2d_ctx_create(int device, sfft2d_ctx** out);
void sfft2d_ctx_destroy(sfft2d_ctx* ctx);
const char* sfft2d_ctx_last_error(const sfft2d_ctx* ctx);
/* host time the last transform spent blocked in stream synchronisation (us) */
double sfft2d_ctx_sync_us(const sfft2d_ctx* ctx);

/* Register host-built tables for side n and window tolerances
 * (WindowCache.get, hashing.py:249-261):
 *   space/freq: float64[(log2(n)+1) * n], row log2(B) = FlatWindow.space_1d /
 *               freq_1d for B bins (rows for B < 4 ignored; row log2(n) is the
 *               all-pass window, hashing.py:228-246);
 *   twiddle:    float64[2n] interleaved exp(-2*pi*i*k/n), k < n.             */
int sfft2d_ctx_set_tables(sfft2d_ctx* ctx, int n, double delta_pass, double delta_stop,
                          const double* space, const double* freq, const double* twiddle);

/* Algorithm 1 — replaces sfft2d(x, cfg, rng) (engine.py:256-284).
 * perms: 2*loops permutations; [0, loops) location loops, [loops, 2 loops)
 * estimation loops (the per-loop child streams of engine.py:268).          */
int sfft2d_sfft(sfft2d_ctx* ctx, const void* x, int x_dtype, int x_on_host,
                const sfft2d_sfft_config* cfg, const sfft2d_perm* perms, int precision,
                void* stream, sfft2d_result* res);

/* Algorithm 1's stream derivation (engine.py:266-280) done natively: from the
 * caller's numpy Generator (`Generator.bit_generator.ctypes.bit_generator`,
 * a bitgen_t*), 2*loops child seeds rng.integers(2**63), each child
 * np.random.default_rng(seed) (numpy's SeedSequence + PCG64, restated in
 * csrc/npyrng.h) and one draw_permutation per child (hashing.py:72-80):
 * out[0..loops) location loops, out[loops..2 loops) estimation loops.
 * Host only (no device work); the caller's Generator advances exactly as
 * under the reference.                                                     */
int sfft2d_sfft_draw_perms(void* numpy_bitgen, int n, int loops, sfft2d_perm* out);

/* sfft2d with the permutations derived natively from the caller's Generator
 * (sfft2d_sfft_draw_perms then sfft2d_sfft).                               */
int sfft2d_sfft_bitgen(sfft2d_ctx* ctx, const void* x, int x_dtype, int x_on_host,
                       const sfft2d_sfft_config* cfg, void* numpy_bitgen, int precision,
                       void* stream, sfft2d_result* res);

/* Loop split across devices: the location phase of
 * sfft2d for a SUBSET of the location loops (engine.py:130-145, per-loop
 * dedup).  counts: device uint8[n*n rounded up to a multiple of 32], set to the
 * number of these loops that voted each coordinate.  Summing the ranks'
 * counts (an allreduce) gives the full vote histogram of engine.py:148-160.  */
int sfft2d_sfft_votes(sfft2d_ctx* ctx, const void* x, int x_dtype, int x_on_host,
                      const sfft2d_sfft_config* cfg, const sfft2d_perm* perms, int nloops,
                      int precision, void* stream, void* counts);

/* Vote threshold + estimation loops + median/top-k/prune from a summed count
 * histogram (engine.py:148-160, 163-284); est_perms: cfg->loops permutations. */
int sfft2d_sfft_from_votes(sfft2d_ctx* ctx, const void* x, int x_dtype, int x_on_host,
                           const sfft2d_sfft_config* cfg, const void* counts,
                           const sfft2d_perm* est_perms, int precision, void* stream,
                           sfft2d_result* res);

/* Algorithm 2 — replaces atsfft2d(x, cfg, est_loops, rng) (tuner.py:244-282).
 * perms: the shared Generator's draws in order; at least
 * iters(n) + 2 + max(est_loops, 1) of them (tuner passes, confirmation passes,
 * estimation loops).  state->perms_used reports how many were consumed.   */
/* The two halves of the estimation phase (engine.py:163-195 and 228-253) as
 * separate calls, so ranks can split the estimation loops
 * (paper_1908_02461_b200/distributed.py).  All pointers but perms are device
 * pointers.  keys: candidate coordinates i*n + j (int32, ascending), m of them.
 * sfft2d_estimate_loops: vals[l*m + e] = complex estimate of loop l (the
 *   precision's complex type), usable[l*m + e] = 1 where the window gain is at
 *   least gain_floor; B x B hash passes with perms[0..nloops).
 * sfft2d_median_select: componentwise median over the usable loops (any loop
 *   order), top-k cut (ties -> lowest index), prune below prune_rel * max;
 *   results through sfft2d_fetch_result.                                   */
int sfft2d_estimate_loops(sfft2d_ctx* ctx, const void* x, int x_dtype, int x_on_host, int n, int b,
                          double delta_pass, double delta_stop, double gain_floor,
                          const int32_t* keys, int64_t m, const sfft2d_perm* perms, int nloops,
                          int precision, void* stream, void* vals, uint8_t* usable);
int sfft2d_median_select(sfft2d_ctx* ctx, int n, const int32_t* keys, int64_t m, const void* vals,
                         const uint8_t* usable, int nloops, int64_t k, double prune_rel,
                         int precision, void* stream, sfft2d_result* res);

int sfft2d_atsfft(sfft2d_ctx* ctx, const void* x, int x_dtype, int x_on_host, int n,
                  const sfft2d_tuner_config* cfg, int est_loops, const sfft2d_perm* perms,
                  int n_perms, int precision, void* stream, sfft2d_result* res,
                  sfft2d_tuner_state* state);

/* Same as sfft2d_atsfft, but each permutation is drawn on demand from a numpy
 * Generator's bit generator (`numpy.random.Generator.bit_generator.ctypes.
 * bit_generator`, a bitgen_t*) with numpy's own bounded-integer routine
 * (libnpyrandom random_bounded_uint64_fill), consuming the stream exactly like
 * the reference's draw_permutation calls (hashing.py:72-80, tuner.py:170,277):
 * the caller's Generator ends in the same state as after the reference.     */
int sfft2d_atsfft_bitgen(sfft2d_ctx* ctx, const void* x, int x_dtype, int x_on_host, int n,
                         const sfft2d_tuner_config* cfg, int est_loops, void* numpy_bitgen,
                         int precision, void* stream, sfft2d_result* res,
                         sfft2d_tuner_state* state);

/* detect_sparsity (tuner.py:142-241): tuning loop + votes only; fetch the
 * (coordinate, tally) pairs with sfft2d_fetch_votes.                      */
int sfft2d_detect_sparsity(sfft2d_ctx* ctx, const void* x, int x_dtype, int x_on_host, int n,
                           const sfft2d_tuner_config* cfg, const sfft2d_perm* perms,
                           int n_perms, int precision, void* stream,
                           sfft2d_tuner_state* state);

int sfft2d_detect_sparsity_bitgen(sfft2d_ctx* ctx, const void* x, int x_dtype, int x_on_host,
                                  int n, const sfft2d_tuner_config* cfg, void* numpy_bitgen,
                                  int precision, void* stream, sfft2d_tuner_state* state);

/* Copy the last transform's recovered spectrum: ij int64[count][2], values
 * complex (float2 for FP32, double2 for FP64)[count], row-major (i, j) order. */
int sfft2d_fetch_result(sfft2d_ctx* ctx, int64_t* ij, void* values, int dst_on_host,
                        void* stream);

/* Copy the last detection's votes: keys int32[n_votes] (i*n + j, ascending)
 * and tallies int32[n_votes].                                             */
int sfft2d_fetch_votes(sfft2d_ctx* ctx, int32_t* keys, int32_t* tallies, int dst_on_host,
                       void* stream);

/* Kernel-level profiling: when enabled, every kernel launch is bracketed by
 * a CUDA event pair on its launching stream and tagged with its algorithmic
 * bytes.  The report synchronises the device and returns
 * lines "name launches total_ms total_bytes" (then clears the records); the
 * return value is the report length (negative status on error).          */
int sfft2d_ctx_set_profiling(sfft2d_ctx* ctx, int enable);
int64_t sfft2d_ctx_profile_report(sfft2d_ctx* ctx, char* buf, int64_t buflen);

/* ---- building blocks (device pointers, stream-ordered, no host sync) ---- */

/* binned_spectrum (hashing.py:308-337) for `nloops` permutations sharing one
 * read of x: out = complex[nloops][b][b] of `precision`.                  */
int sfft2d_binned_spectrum(sfft2d_ctx* ctx, const void* x, int x_dtype, int n, int b,
                           const sfft2d_perm* perms, int nloops, double delta_pass,
                           double delta_stop, int precision, void* out, void* stream);

/* fft2d (corefft.py:101-109): unscaled forward 2D DFT of `count` b x b grids
 * in place; uses the twiddle table registered for side n_table >= b.      */
int sfft2d_fft2d(sfft2d_ctx* ctx, void* grids, int b, int count, int n_table, int precision,
                 void* stream);

/* count_local_maxima (tuner.py:97-118) of one b x b grid; *count is written
 * to host memory (this call synchronises `stream`); the first min(count,
 * capacity) flat indices (row-major) are written to out_flat (device).    */
int sfft2d_local_maxima(sfft2d_ctx* ctx, const void* grid, int b, double mag_floor,
                        int precision, int64_t* count, int32_t* out_flat, int64_t capacity,
                        void* stream);

/* _top_bins (engine.py:122-127) for `nseg` b x b grids: the `num` largest
 * |Z| per grid, ties to the lowest flat index, written in ascending flat
 * index order to out_flat[nseg][num] (device).                            */
int sfft2d_top_bins(sfft2d_ctx* ctx, const void* grids, int b, int nseg, int64_t num,
                    int precision, int32_t* out_flat, void* stream);

/* Caller-owned device workspace: `base` (device, at
 * least `bytes`) replaces the context's pool for every later call; NULL / 0
 * returns to the pool.  Synchronises the device (buffers are dropped).      */
int sfft2d_ctx_set_workspace(sfft2d_ctx* ctx, void* base, int64_t bytes);
/* Workspace bytes currently held and the high-water mark since the last
 * sfft2d_ctx_set_workspace (or context creation).                          */
int sfft2d_ctx_workspace_size(const sfft2d_ctx* ctx, int64_t* in_use, int64_t* peak);

/* ---- workload generator (no reference counterpart:
 * the reference generates on the host, signals.py:42-65) ----
 * out (device, n x n, SFFT2D_C64 or SFFT2D_C128) = ifft2(S) + noise_sd * (n1 + i n2)
 * where S holds coeffs[i] (interleaved re/im doubles, host) at (rows[i],
 * cols[i]) (host int64) and n1, n2 are standard normals from Philox4x32-10
 * keyed by noise_seed, counter = flat element index (Box-Muller in double;
 * paper_1908_02461_b200/csrc/generate.cuh).  The inverse DFT runs through the
 * library's own forward FFT (fp32 for C64, fp64 for C128); needs the twiddle
 * table of side n (sfft2d_ctx_set_tables).  Stream-ordered, no host sync.  */
int sfft2d_generate(sfft2d_ctx* ctx, int n, int64_t k, const int64_t* rows, const int64_t* cols,
                    const double* coeffs, double noise_sd, uint64_t noise_seed, int out_dtype,
                    void* out, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SFFT2D_B200_H */
