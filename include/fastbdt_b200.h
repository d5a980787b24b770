/*
 * fastbdt_b200.h — C ABI of the B200-native FastBDT hot path
 * (libfastbdt_b200.so).  Plain pointers and sizes; no torch types.
 *
 * The reference (/root/reference/pkg, "binboost") is pure Python with no FFI,
 * so its plugin surface is the Python signatures these entry points sit
 * behind (INTEGRATION.md shows the ctypes binding):
 *
 *   bb_fit      replaces binboost.boosting.fit_forest
 *               (pkg/src/binboost/boosting.py:117-173), reached from
 *               binboost_bridge.fit (pkg/bridge/src/binboost_bridge/__init__.py:146-171)
 *   bb_predict  replaces binboost.boosting.predict_batch
 *               (boosting.py:196-219), reached from BoundModel.predict
 *               (bridge __init__.py:85-93)
 *   bb_bin      fit_binning + bin_values (pkg/src/binboost/binning.py:52-79)
 *   bb_layer_hist / bb_split
 *               accumulate_layer_histograms / find_best_cuts
 *               (pkg/src/binboost/trees.py:139-204), exposed for parity tests
 *   bb_subsample_masks
 *               subsample (pkg/src/binboost/sample.py:120-132) driven by
 *               numpy Generator(PCG64(seed)) (boosting.py:162); host only
 *   bb_pairwise_sum
 *               numpy's pairwise float64 sum used by prior (boosting.py:76-83);
 *               host only
 *   bb_roc_auc  replaces binboost.analysis.roc_auc (pkg/src/binboost/analysis.py:45-70)
 *   bb_elim_create / bb_elim_fit / bb_elim_destroy
 *               the refits of binboost.analysis.elimination_importance
 *               (analysis.py:104-173, fit loop :136-142): training rows binned
 *               once, each refit on a feature subset returns its validation AUC
 *
 * Conventions: every function returns BB_OK (0) or an error code and sets a
 * thread-local message readable with bb_last_error().  BB_EINVAL maps to the
 * reference's ValueError, everything else to RuntimeError.  No host pointer
 * is retained after a call returns.  Calls on one context are serialised by
 * a mutex (one CUDA stream per context); use one context per thread for
 * concurrency.
 */
#ifndef FASTBDT_B200_H
#define FASTBDT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BB_ABI_VERSION 1

enum { BB_OK = 0, BB_EINVAL = 1, BB_ECUDA = 2, BB_ESTATE = 3 };
enum { BB_F32 = 0, BB_F64 = 1 };

typedef struct bb_ctx bb_ctx;

const char* bb_last_error(void);
int bb_abi_version(void);
int bb_device_count(int32_t* out);

/* One context per device: owns a CUDA stream and, for multi-process row
 * sharding, the rank's position in the job (rank, world). */
int bb_ctx_create(int32_t device, bb_ctx** out);
int bb_ctx_destroy(bb_ctx* ctx);

/* Row-sharded fits: join an NCCL communicator of `world`
 * ranks (unique_id: the 128-byte ncclUniqueId of rank 0, e.g. from
 * torch.cuda.nccl.unique_id()).  Afterwards bb_fit on this context takes the
 * rank's shard of rows: the contiguous rank-th slice of the signal block and
 * of the background block (input order = class-block order), ranks in order.
 * Histograms and node sums are all-reduced (int64) per layer, so every rank
 * takes the same cuts; binning statistics are all-reduced too. */
int bb_ctx_init_comm(bb_ctx* ctx, int32_t rank, int32_t world, const uint8_t* unique_id);

/* FitConfig (boosting.py:36-57) plus the numpy PCG64(seed) state the
 * subsample draws from (PCG64(seed).state["state"]: 128-bit state and
 * increment split into hi/lo words, has_uint32, uinteger). */
typedef struct {
  int32_t n_trees;
  int32_t depth;
  int32_t binning_levels;
  int32_t flags;        /* bit 0: time every histogram launch with CUDA events */
  double shrinkage;
  double subsample;
  uint64_t pcg_state_hi, pcg_state_lo;
  uint64_t pcg_inc_hi, pcg_inc_lo;
  int32_t pcg_has_uint32;
  uint32_t pcg_uinteger;
  double f0_override;  /* NaN: compute the prior here; required (from all rows,
                        * numpy pairwise sums) when the context is sharded */
} bb_fit_config;

/* Teacher-forced parity protocol: at (tree, heap node)
 * take this cut instead of the argmax. */
typedef struct {
  int32_t tree, node, valid, feature, cut_bin;
} bb_forced_cut;

/* Caller-allocated host outputs.  I = 2^depth - 1, N = 2^(depth+1) - 1,
 * B = 2^binning_levels. */
typedef struct {
  double* boundaries;   /* [d][B-1]                                     */
  int32_t* feature;     /* [T][I]  -1 where invalid (trees.py:64)       */
  int32_t* cut_bin;     /* [T][I]                                       */
  uint8_t* valid;       /* [T][I]                                       */
  double* threshold;    /* [T][I]  NaN where invalid                    */
  double* gain;         /* [T][I]                                       */
  double* node_weight;  /* [T][N]  shrinkage applied (boosting.py:168)  */
  double* node_purity;  /* [T][N]                                       */
  double* f0;           /* [1]                                          */
  int32_t* fixed_shift; /* [1]  S of the int64 fixed-point sums         */
  int64_t* n_sig;       /* [1]  rows in the signal block                */
  uint16_t* leaves;     /* optional [T][n] final node per row, class-block order */
  double* scores;       /* optional [n] final F per row, class-block order */
  double* timing_ms;    /* optional [16]: [0] upload [1] binning [2] trees [3] download
                         * [4] host total (ms); [5] device total (CUDA events, ms);
                         * [6] histogram kernels (ms, flags bit 0); [7] histogram
                         * launches; [8] all kernel launches; [9] mask generation (host ms) */
} bb_fit_out;

/* X: row-major (n, d) float32 (BB_F32) or float64 (BB_F64); y01: int8, > 0
 * is signal; w: float64 or NULL (unit weights).  *_on_device != 0 means the
 * pointer is CUDA device memory on the context's device. */
int bb_fit(bb_ctx* ctx, const void* X, int32_t x_dtype, int32_t x_on_device, int64_t n, int32_t d,
           const int8_t* y01, int32_t y_on_device, const double* w, int32_t w_on_device,
           const bb_fit_config* cfg, const bb_forced_cut* forced, int32_t n_forced, bb_fit_out* out);

/* A fitted forest (Forest, boosting.py:60-73), host arrays laid out as in
 * bb_fit_out. */
typedef struct {
  int32_t n_trees;
  int32_t depth;
  int32_t n_features;
  int32_t reserved0;
  double f0;
  const int32_t* feature;
  const uint8_t* valid;
  const double* threshold;
  const double* node_weight;
} bb_forest;

/* Signal probabilities sigmoid(2F) (and optionally F) per row. */
int bb_predict(bb_ctx* ctx, const bb_forest* forest, const void* X, int32_t x_dtype, int32_t x_on_device,
               int64_t n, int32_t d, double* out_prob, double* out_score, int32_t out_on_device);

/* Parity entry points ------------------------------------------------ */

/* Boundaries [d][B-1] and codes [d][n] (int16, input row order; out_codes
 * may be NULL: boundaries only). */
int bb_bin(bb_ctx* ctx, const void* X, int32_t x_dtype, int64_t n, int32_t d, int32_t levels,
           double* out_boundaries, int16_t* out_codes);

/* One layer's integer histograms from host inputs in class-block order:
 * codes [d][n] (uint16, 0 = missing), node [n] (uint16 heap ids), q [n]
 * int64 fixed-point weights.  out_hist [2][2^(layer-1)][d][B] int64, slot
 * b holds code b+1. */
int bb_layer_hist(bb_ctx* ctx, const uint16_t* codes, const uint16_t* node, const int64_t* q, int64_t n,
                  int64_t n_sig, int32_t d, int32_t levels, int32_t layer, int64_t* out_hist);

/* Best cuts of one layer from integer histograms [2][nodes][d][B] (as
 * produced by bb_layer_hist), fixed-point scale 2^-shift. */
int bb_split(bb_ctx* ctx, const int64_t* hist, int32_t d, int32_t levels, int32_t layer, int32_t final_layer,
             int32_t shift, const double* boundaries, uint8_t* out_valid, int32_t* out_feature,
             int32_t* out_cut, double* out_gain, double* out_threshold);

/* GPU generator (the fit's default path), same output as bb_subsample_masks. */
int bb_subsample_masks_gpu(bb_ctx* ctx, int64_t n_sig, int64_t n_bkg, double rate, int32_t n_trees,
                           const bb_fit_config* rng, uint32_t* out_bits);

/* Host only (no GPU needed): active bits [T][ceil((n_sig+n_bkg)/32)]. */
int bb_subsample_masks(int64_t n_sig, int64_t n_bkg, double rate, int32_t n_trees, const bb_fit_config* rng,
                       uint32_t* out_bits);
double bb_pairwise_sum(const double* a, int64_t n);

/* Virtual shards: a group of `world` contexts of this process whose
 * all-reduces go through host memory (rank-order sums) instead of NCCL, so
 * the row-sharded fit runs with several shards on one GPU (parity tests;
 * one thread per shard).  Bind each context with bb_ctx_init_virtual. */
typedef struct bb_vgroup bb_vgroup;
int bb_vgroup_create(int32_t world, bb_vgroup** out);
int bb_vgroup_destroy(bb_vgroup* group);
int bb_ctx_init_virtual(bb_ctx* ctx, int32_t rank, bb_vgroup* group);

/* CSV ingestion (replaces the csv/float() loop of binboost.dataset.load_csv
 * / load_matrix, pkg/src/binboost/dataset.py:31-137): host-side, threaded.
 * bb_csv_open reads the file and delimits its records (excel dialect);
 * bb_csv_parse parses the chosen columns of every data record as float64
 * (Python float() grammar) into out[records][n_cols]; finite_col (or -1)
 * must hold finite values.  On BB_EINVAL bb_csv_error gives the first error
 * in record order: kind 1 = cell count, 2 = not a number, 3 = non-finite. */
typedef struct bb_csv bb_csv;
int bb_csv_open(const char* path, bb_csv** out);
int32_t bb_csv_n_header(const bb_csv* h);
int64_t bb_csv_n_records(const bb_csv* h);
const char* bb_csv_header(const bb_csv* h, int32_t j, int64_t* len);
int bb_csv_parse(bb_csv* h, const int32_t* cols, int32_t n_cols, int32_t finite_col, int32_t n_threads, double* out);
int bb_csv_error(const bb_csv* h, int64_t* row, int32_t* kind, int32_t* col, int32_t* cells, const char** cell,
                 int64_t* cell_len, double* value);
int bb_csv_close(bb_csv* h);

/* Analysis ------------------------------------------------------------ */

/* Weighted ROC AUC of host scores (labels y01 > 0 = signal; w may be NULL).
 * BB_EINVAL if either class has non-positive total weight. */
int bb_roc_auc(bb_ctx* ctx, const double* scores, const int8_t* y01, const double* w, int64_t n, double* out_auc);

/* Elimination session: training rows X[n][d] (row-major, x_dtype), y01, w
 * (NULL = unit) binned once with `levels`; validation rows Xv[n_val][d]
 * binned with the training boundaries.  Read-only after creation: refits may
 * run concurrently from several contexts on the session's device. */
typedef struct bb_elim bb_elim;
int bb_elim_create(bb_ctx* ctx, const void* X, int32_t x_dtype, int64_t n, int32_t d, const int8_t* y01,
                   const double* w, int32_t levels, const void* Xv, int64_t n_val, const int8_t* y01_val,
                   const double* w_val, bb_elim** out);
/* Refit on feature columns cols[n_cols] (the forest's feature j is column
 * cols[j]); out_auc (may be NULL) = validation AUC; out (may be NULL)
 * receives the forest arrays like bb_fit (boundaries, leaves, scores and
 * timing are not written). */
int bb_elim_fit(bb_ctx* ctx, const bb_elim* session, const int32_t* cols, int32_t n_cols, const bb_fit_config* cfg,
                double* out_auc, bb_fit_out* out);
int bb_elim_destroy(bb_elim* session);

#ifdef __cplusplus
}
#endif

#endif /* FASTBDT_B200_H */
