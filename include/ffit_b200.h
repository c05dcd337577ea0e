/* C ABI of the B200-native likelihood engine (libffit_b200.so).
 *
 * Drop-in boundary for the reference engine `ffit` (arXiv 2003.12875 artifact):
 * the `ffit_*` entry points below carry the SAME names, argument meaning, status
 * codes and ownership rules as the reference's include/ffit.h
 * (/root/reference/proj/include/ffit.h:1-110), so a caller that links the
 * reference's libffit.so can relink against this library.  The computation
 * behind ffit_nll / ffit_probabilities / ffit_fit runs on the GPU (sm_100a):
 * datasets are SoA fp64 columns resident in HBM and the whole PDF graph plus the
 * -log / compensated-sum reduction is one fused kernel.  There is no CPU
 * fallback: without a usable CUDA device the evaluation calls fail with
 * FFIT_ERR_NUMERIC and a CUDA error message.
 *
 * Conventions (reference include/ffit.h:1-9, src/capi.cpp:28-50): every function
 * returns a status code; handles are opaque, caller-owned and released by the
 * matching *_free (free(NULL) is a no-op); on failure out-parameters are left
 * untouched and ffit_last_error() describes the failure (thread-local).
 *
 * The `ffcu_*` entry points are the device-level layer the north star asks for
 * (SURVEY.md §8(b2)): multi-point launches, device-resident results for the
 * multi-GPU exchange, zero-copy device datasets, per-PDF batch evaluation.
 */
#ifndef FFIT_B200_H
#define FFIT_B200_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes -- reference include/ffit.h:20-25 */
enum {
  FFIT_OK = 0,
  FFIT_ERR_USAGE = 1,
  FFIT_ERR_DATA = 2,
  FFIT_ERR_NUMERIC = 3,
};

/* Evaluation modes -- reference include/ffit.h:27-31, plus FFIT_MODE_GPU.
 * Every mode runs the fused sm_100a kernel.  The reference's SCALAR is bitwise equal
 * to its BATCH_PRECISE (proj/tests/test_eval.cpp:113-157), and here SCALAR, BATCH_PRECISE,
 * BATCH_FAST and GPU return the same bits, so the reference CLI's mode comparisons
 * (tools/ffit_main.cpp bench / parity) relink unchanged. */
typedef enum {
  FFIT_MODE_SCALAR = 0,
  FFIT_MODE_BATCH_PRECISE = 1,
  FFIT_MODE_BATCH_FAST = 2,
  FFIT_MODE_GPU = 3,
} ffit_mode;

typedef struct ffit_model ffit_model;
typedef struct ffit_dataset ffit_dataset;
typedef struct ffit_fit_result ffit_fit_result;

/* reference include/ffit.h:37 */
const char* ffit_last_error(void);

/* ---- models: reference include/ffit.h:39-53 --------------------------------
 * Model-file grammar of the reference (proj/docs/model-file.md) plus, on the
 * GPU path: ArgusBG(x, m0, c, p), Chebychev(x, a1..an), Polynomial(x, a1..an),
 * ProdPdf(p1, ..., pk) over distinct observables, AddPdf(c1, f1, ..., cn) (=
 * WeightedSum) and AddPdf(c1, y1, ..., cn, yn) (extended), several
 * `observable` lines.  Expression("formula", vars...) pdfs run on the device
 * (formula-specialised builds, else the device interpreter). */
int ffit_model_load(const char* path, ffit_model** out);
int ffit_model_parse(const char* text, ffit_model** out);
void ffit_model_free(ffit_model* m);
const char* ffit_model_observable(const ffit_model* m); /* the first observable */
int ffit_model_observable_range(const ffit_model* m, double* lo, double* hi);
int ffit_model_param_count(const ffit_model* m);
const char* ffit_model_param_name(const ffit_model* m, int i);
int ffit_model_param_is_constant(const ffit_model* m, const char* name, int* constant);
int ffit_model_get_param(const ffit_model* m, const char* name, double* value,
                         double* uncertainty);
int ffit_model_set_param(ffit_model* m, const char* name, double value);

/* ---- datasets: reference include/ffit.h:55-66 ------------------------------
 * Datasets live in HBM on the CUDA device current at creation time. */
int ffit_dataset_read_csv(const ffit_model* m, const char* path, ffit_dataset** out,
                          long* dropped);
int ffit_dataset_write_csv(const ffit_dataset* ds, const char* path);
long ffit_dataset_rows(const ffit_dataset* ds);
void ffit_dataset_free(ffit_dataset* ds);

/* ---- sampling: reference include/ffit.h:68-73 ------------------------------ */
int ffit_sample(ffit_model* m, long n, unsigned long long seed, ffit_dataset** out,
                double* efficiency);

/* ---- evaluation: reference include/ffit.h:75-85 ----------------------------
 * *n_evaluations = kernels launched (independent of the number of events, as
 * the reference's batch-mode call accounting). */
int ffit_nll(ffit_model* m, const ffit_dataset* ds, ffit_mode mode, double* value,
             unsigned long long* n_evaluations);
int ffit_probabilities(ffit_model* m, const ffit_dataset* ds, ffit_mode mode, double* out);

/* ---- fitting: reference include/ffit.h:87-104 ------------------------------
 * The reference's Nelder-Mead (proj/src/fit.cpp:86-251) with batched GPU points. */
int ffit_fit(ffit_model* m, const ffit_dataset* ds, ffit_mode mode, double tolerance,
             long max_iterations, ffit_fit_result** out);
int ffit_result_converged(const ffit_fit_result* r);
double ffit_result_nll(const ffit_fit_result* r);
unsigned long long ffit_result_nll_calls(const ffit_fit_result* r);
double ffit_result_wall_seconds(const ffit_fit_result* r);
int ffit_result_uncertainties_valid(const ffit_fit_result* r);
int ffit_result_param_count(const ffit_fit_result* r);
const char* ffit_result_param_name(const ffit_fit_result* r, int i);
double ffit_result_param_value(const ffit_fit_result* r, int i);
double ffit_result_param_uncertainty(const ffit_fit_result* r, int i);
void ffit_result_free(ffit_fit_result* r);

/* ======================= device-level layer (ffcu_*) ======================= */

/* Dataset from host columns (uploaded once to HBM; replaces the reference's
 * DataSet(names, columns) constructor, proj/include/ffit/dataset.hpp:25). */
int ffcu_dataset_from_host(const char* const* names, const double* const* cols, int ncols,
                           long long n, ffit_dataset** out);
/* Zero-copy view over caller-owned device columns (e.g. torch tensors) on
 * `device`; the memory must outlive the view. */
int ffcu_dataset_from_device(const char* const* names, const double* const* dev_cols, int ncols,
                             long long n, int device, ffit_dataset** out);
/* Refill an owned dataset from host columns of the same shape. */
int ffcu_dataset_copy_from_host(ffit_dataset* ds, const double* const* cols);
/* The same, asynchronous on `stream` (a cudaStream_t): with pinned host columns the copy
 * overlaps other work (double-buffered input pipelines); the caller orders it against
 * the launches that read the dataset (events) and keeps the host columns alive. */
int ffcu_dataset_copy_from_host_async(ffit_dataset* ds, const double* const* cols, void* stream);
/* Rows [begin, end) as a zero-copy view (event sharding). */
int ffcu_dataset_slice(const ffit_dataset* ds, long long begin, long long end, ffit_dataset** out);
/* Columns: count, names, a column copied to host memory, a column's device pointer. */
int ffcu_dataset_ncols(const ffit_dataset* ds);
const char* ffcu_dataset_column_name(const ffit_dataset* ds, int i);
int ffcu_dataset_download(const ffit_dataset* ds, int col, double* host_out);
int ffcu_dataset_device_column(const ffit_dataset* ds, int col, const double** dev_ptr);

/* Binary SoA dataset files (the reference's only on-disk format is
 * CSV, proj/src/dataset.cpp:61-146).  `.ffsoa` = the HBM layout on disk: a 4 KiB-aligned
 * header (magic, column names, per-column checksums) then each fp64 column contiguous and
 * 4 KiB-aligned (csrc/soa_io.hpp).  Loading reads chunks into two pinned staging buffers,
 * each chunk's host-to-device copy overlapping the read of the next; checksums are
 * verified (FFIT_ERR_DATA on mismatch, truncation or a bad header). */
int ffcu_soa_write(const char* path, const char* const* names, const double* const* cols, int ncols,
                   long long n);
int ffcu_dataset_save_soa(const ffit_dataset* ds, const char* path);
int ffcu_dataset_load_soa(const char* path, ffit_dataset** out, double* seconds);
int ffcu_soa_info(const char* path, int* ncols, long long* nrows);
int ffcu_soa_column_name(const char* path, int col, char* buf, int cap);
/* Host read of every column (cols[i]: nrows doubles each), checksums verified. */
int ffcu_soa_read_host(const char* path, double* const* cols);

/* NLL at P parameter points in ONE launch.  points: P x ffit_model_param_count
 * doubles, row-major, parameters in ffit_model_param_name order.  values[p]
 * = NLL (+inf if an event has p <= 0 or non-finite; first_invalid[p] = its
 * index, else -1).  first_invalid and n_evaluations may be NULL. */
int ffcu_nll_points(ffit_model* m, const ffit_dataset* ds, const double* points, int P,
                    double* values, long long* first_invalid, unsigned long long* n_evaluations);
/* Same, returning the uncombined Neumaier pairs (sc[2p], sc[2p+1]) of the event
 * sum only (no extended term) -- the per-rank partials of the multi-GPU path. */
int ffcu_nll_points_partial(ffit_model* m, const ffit_dataset* ds, const double* points, int P,
                            double* sc, long long* first_invalid,
                            unsigned long long* n_evaluations);
/* Asynchronous on `stream` (cudaStream_t; NULL = the model's stream): writes P
 * pairs to device d_sc (2P doubles) and P indices to device d_bad
 * (0xFFFFFFFFFFFFFFFF = none).  P <= 512. */
int ffcu_nll_points_device(ffit_model* m, const ffit_dataset* ds, const double* points, int P,
                           double* d_sc, unsigned long long* d_bad, void* stream,
                           unsigned long long* n_evaluations);
/* The same with the constant rows copied on `upload_stream` (a pipeline's copy stream, next
 * to its input uploads; the launch on `stream` waits for them): a caller can queue the next
 * step while the current one runs without its H2D copies queueing behind the kernels. */
int ffcu_nll_points_device_upload(ffit_model* m, const ffit_dataset* ds, const double* points, int P,
                                  double* d_sc, unsigned long long* d_bad, void* stream, void* upload_stream,
                                  unsigned long long* n_evaluations);
/* NLL and its analytic gradient in ONE fused pass over the events (SURVEY.md
 * §8(f) f1; replaces the finite-difference gradients a Minuit-style driver builds
 * from 2d+1 proj/src/eval.cpp:119-163 evaluations).  grads: P x param_count,
 * dNLL/dtheta_j in ffit_model_param_name order, 0 for constant parameters, NaN
 * where values[p] is +inf.  FFIT_ERR_USAGE if the model's gradient layout exceeds
 * the device pass (more than 48 accumulators). */
int ffcu_nll_grad(ffit_model* m, const ffit_dataset* ds, const double* points, int P,
                  double* values, double* grads, long long* first_invalid,
                  unsigned long long* n_evaluations);
/* Accumulators per point of the gradient pass (slot 0 = the event NLL sum). */
int ffcu_grad_slot_count(ffit_model* m, int* nslots);
/* Multi-GPU split of ffcu_nll_grad: the per-shard uncombined Neumaier pairs
 * (sc: P x nslots x 2), then the host finish from the rank-combined slot sums
 * (P x nslots) with the global event count. */
int ffcu_nll_grad_partial(ffit_model* m, const ffit_dataset* ds, const double* points, int P,
                          double* sc, long long* first_invalid, unsigned long long* n_evaluations);
int ffcu_nll_grad_finish(ffit_model* m, const double* points, int P, const double* slot_sums,
                         double n_events, double* values, double* grads);
/* Fixed-rank-order compensated combine of R x P device pairs into P pairs. */
int ffcu_combine_pairs_device(const double* d_in, int R, int P, double* d_out, void* stream);
/* The sharded exchange's combine (csrc/shard.hpp) for callers doing their own collective:
 * d_in = R gathered rank blocks of 2*rows + P 8-byte words ([rows Neumaier pairs | P local
 * first-invalid indices]); d_out = rows pairs combined in rank order, d_bad = P global
 * indices (d_offsets[r] = rank r's first global row; 0xFFFFFFFFFFFFFFFF = none). */
int ffcu_combine_shards_device(const double* d_in, int R, int rows, int P, const long long* d_offsets,
                               double* d_out, unsigned long long* d_bad, void* stream);
/* Extended term nu - N log nu per point (0 for non-extended models). */
int ffcu_extended_terms(const ffit_model* m, const double* points, int P, double n_events,
                        double* out);
/* probabilities() at an explicit point (NULL = current parameter values). */
int ffcu_probabilities_at(ffit_model* m, const ffit_dataset* ds, const double* point,
                          double* out);
/* PdfSpec::eval_batch (proj/include/ffit/pdfs.hpp:59-60): unnormalised values of
 * the named (sub-)pdf over the dataset at the current parameter values. */
int ffcu_eval_batch(ffit_model* m, const char* pdf, const ffit_dataset* ds, double* out);
int ffcu_eval_batch_device(ffit_model* m, const char* pdf, const ffit_dataset* ds, double* d_out,
                           void* stream);
/* normalization(spec, lo, hi, graph) (proj/include/ffit/eval.hpp:26) of a named
 * pdf at a point (NULL = current values). */
int ffcu_normalization(const ffit_model* m, const char* pdf, const double* point, double* out);
/* Device-side numeric normalisation (replaces the host's
 * integrate_adaptive_simpson, proj/src/eval.cpp:40-69, for the nodes without a closed form).
 * Off by default: the host's quadrature is bit-identical to the reference's.  On (per model, or
 * FFB_DEVICE_NORM=1 for the process): every likelihood / probabilities / eval_batch call
 * integrates those nodes on the GPU for all its points at once -- the reference's own adaptive
 * rule, one warp per point, one lane per pre-panel -- and agrees with the host's value to
 * <= 1e-13 relative. */
int ffcu_model_set_device_normalization(ffit_model* m, int on);
int ffcu_model_device_normalization(const ffit_model* m);
/* The normalisation integral of a named pdf (NULL = the model's top pdf) at P points (P rows of
 * all model parameters, declaration order; NULL with P = 1 = current values) by the device
 * quadrature, whatever the model's switch says; closed forms stay closed forms. */
int ffcu_device_normalization(ffit_model* m, const char* pdf, const double* points, int P, double* out);
/* Quadrature kernels this model's engine has launched. */
unsigned long long ffcu_device_normalization_launches(const ffit_model* m);
/* The flattened plan and one point's constant row (host logic, no GPU needed). */
int ffcu_plan_info(const ffit_model* m, int* nterms, int* ncols, int* stride);
int ffcu_plan_term(const ffit_model* m, int i, int* kind, int* col, int* order, int* flags,
                   int* coff);
int ffcu_point_constants(const ffit_model* m, const double* point, double* row);
/* d coef_c / d theta_param for each plan term c (the row's coefficient entries;
 * host logic of the gradient pass, no GPU needed). */
int ffcu_coef_derivatives(const ffit_model* m, const double* point, int param, double* out);
/* The Expression formula language (proj/docs/expression-grammar.md):
 * compile `text` over `nvars` variable names and evaluate it on the host at npts rows
 * of values (row-major npts x nvars).  FFIT_ERR_USAGE with the reference's messages on
 * syntax / unknown identifier / unknown function / arity errors. */
int ffcu_expr_eval(const char* text, const char* const* vars, int nvars, const double* values, int npts,
                   double* out);
/* Formula-specialised likelihood builds for models with Expression pdfs: each formula
 * becomes straight-line device code and the fused kernels are compiled around it at run
 * time with NVRTC (csrc/jit.cpp), else the device interpreter runs.  enable: 1 on, 0 off,
 * -1 query; returns the previous setting (default on; FFB_NO_EXPR_JIT=1 turns it off). */
int ffcu_expression_jit(int enable);
const char* ffcu_expression_jit_status(void);
/* The generated formula source of a model (compile = 1: also NVRTC-compile the kernels
 * around it, no GPU needed); at most cap-1 characters into buf. */
int ffcu_expression_jit_source(const ffit_model* m, int compile, char* buf, int cap);
/* The same for a launch over P points: formula subtrees whose inputs (x, constants,
 * parameters) are identical over all the points are computed once per staged tile
 * (launch-constant cache) and the generated source shows them (ffb_expr_hoist). */
int ffcu_expression_jit_source_points(ffit_model* m, const double* points, int P, int compile, char* buf, int cap);
/* The build the model's last likelihood launch ran: 0 the static kernels, 1 the
 * formula-specialised build, 2 the plan-specialised build (below). */
int ffcu_last_launch_jit(const ffit_model* m);
/* Plan-specialised likelihood builds: launches of at least FFB_PLAN_SPEC_MIN (default 5e7)
 * event-points of models without Expression pdfs run the tile kernel (or, for <= 8 points
 * of a single-column single-sum model, the streaming kernel) compiled at run time (NVRTC)
 * around the launch's term list; values as the static build's; FFB_NO_PLAN_SPEC=1 (or ffcu_expression_jit(0)) turns it off.  The
 * generated source for P points (points may be null: the model's plan as is); compile = 1
 * also NVRTC-compiles it (no GPU needed); at most cap-1 characters into buf. */
int ffcu_plan_spec_source(ffit_model* m, const double* points, int P, int compile, char* buf, int cap);
/* The event-point threshold of the plan-specialised builds: v >= 0 sets it, -1 turns the
 * builds off, -2 only queries; returns the previous value (-1: off). */
double ffcu_plan_spec_min_work(double v);
/* The plan-specialised gradient pass (one point per launch: a fit's iteration) for
 * single-column single-sum models: the generated term list / slot layout (compile_ks >=
 * 0: also NVRTC-compile the kernel for that leaf-kind set, no GPU needed), and whether
 * the model's last gradient launch ran it. */
int ffcu_grad_spec_source(ffit_model* m, int compile_ks, char* buf, int cap);
int ffcu_last_grad_jit(ffit_model* m);
/* Model introspection: the named pdfs and the observables, in model-file order. */
int ffcu_model_pdf_count(const ffit_model* m);
const char* ffcu_model_pdf_name(const ffit_model* m, int i);
int ffcu_model_observable_count(const ffit_model* m);
const char* ffcu_model_observable_name(const ffit_model* m, int i);

/* Minuit-style batched fit: BFGS on central finite differences, 2d+1 points per
 * launch per iteration; Hessian uncertainties from one launch. */
int ffcu_fit_gradient(ffit_model* m, const ffit_dataset* ds, double tolerance,
                      long max_iterations, ffit_fit_result** out);
/* analytic = 1: gradients from the fused NLL + gradient pass when the model's
 * layout fits it, 0: central finite differences, -1 (ffcu_fit_gradient's default):
 * analytic except for models with Expression pdfs while their formula-specialised
 * likelihood builds are on (their normalisation derivatives are host quadratures, and
 * 2d+1 points of the specialised build are faster). */
int ffcu_fit_gradient_opts(ffit_model* m, const ffit_dataset* ds, double tolerance,
                           long max_iterations, int analytic, ffit_fit_result** out);
/* 1 if the fit's gradients came from the fused pass. */
int ffcu_result_analytic_gradient(const ffit_fit_result* r);
/* fit_gradient: BFGS iterations taken. */
int ffcu_result_iterations(const ffit_fit_result* r);
/* fit_gradient: the last estimated distance to the minimum, g^T H^-1 g / 2. */
double ffcu_result_edm(const ffit_fit_result* r);
/* fit_gradient: likelihood / gradient launches, and the per-iteration NLL trace. */
unsigned long long ffcu_result_launches(const ffit_fit_result* r);
int ffcu_result_trace(const ffit_fit_result* r, double* out, int cap);

/* ---- event-sharded likelihood over several GPUs (csrc/shard.hpp) ----
 * Every rank owns a contiguous range of the events of every column, resident in its HBM.
 * A batch of P points is one fused launch per rank plus ONE collective: an NCCL all-gather
 * of the rank's [P Neumaier pairs | P first-invalid indices] (24P bytes), then a fixed
 * rank-order combine on the device -- the values are bitwise independent of NCCL's
 * algorithm and identical on every rank; the extended term uses the global event count.
 * NCCL is loaded at run time (the copy already in the process, e.g. PyTorch's, else
 * libnccl.so.2); without it these calls fail with FFIT_ERR_NUMERIC. */
typedef struct ffcu_shard_group ffcu_shard_group;
#define FFCU_NCCL_ID_BYTES 128
/* A fresh ncclUniqueId (FFCU_NCCL_ID_BYTES bytes) for create_rank: rank 0 makes it, the
 * caller hands it to every rank (torch.distributed, MPI, a file...). */
int ffcu_nccl_unique_id(void* id);
/* "major.minor.patch" of the NCCL the library bound ("" when none is loadable). */
const char* ffcu_nccl_version(void);
/* One process per GPU: this process is global rank `rank` of `world`; `shard` (a dataset
 * on this process's device) holds rows [offset, offset + rows) of the n_total events.  The
 * ranks' shards must tile [0, n_total) in rank order (checked once, collectively). */
int ffcu_shard_group_create_rank(ffit_model* m, const ffit_dataset* shard, long long n_total, long long offset,
                                 const void* nccl_id, int world, int rank, ffcu_shard_group** out);
/* One process, ndev distinct devices (ncclCommInitAll): host columns of n_total rows cut
 * into ndev contiguous shards, one uploaded to each device. */
int ffcu_shard_group_create_local(ffit_model* m, const char* const* names, const double* const* host_cols,
                                  int ncols, long long n_total, const int* devices, int ndev,
                                  ffcu_shard_group** out);
void ffcu_shard_group_free(ffcu_shard_group* g);
/* world size, local devices, n_total, and the first local device's rows / first row */
int ffcu_shard_group_info(const ffcu_shard_group* g, int* world, int* local_devices, long long* n_total,
                          long long* local_rows, long long* local_offset);
/* ffcu_nll_points over all ranks' events (collective: every rank calls it with the same
 * points; values identical on every rank). */
int ffcu_shard_group_nll_points(ffcu_shard_group* g, const double* points, int P, double* values,
                                long long* first_invalid, unsigned long long* n_evaluations);
/* Asynchronous on `stream` (groups with one local device): the combined event pairs (2P
 * doubles, no extended term) and global first-invalid indices stay on the device;
 * upload_stream (may be NULL) as in ffcu_nll_points_device_upload. */
int ffcu_shard_group_nll_points_device(ffcu_shard_group* g, const double* points, int P, double* d_sc,
                                       unsigned long long* d_bad, void* stream, void* upload_stream,
                                       unsigned long long* n_evaluations);
/* ffcu_nll_grad over all ranks: per-rank slot pairs of the fused gradient pass, one
 * all-gather, rank-order combine, host finish with the global event count. */
int ffcu_shard_group_nll_grad(ffcu_shard_group* g, const double* points, int P, double* values, double* grads,
                              long long* first_invalid, unsigned long long* n_evaluations);
/* The fit drivers on the sharded likelihood (collective; the fitted values are written
 * into the group's model on every rank): the reference's Nelder-Mead (ffit_fit) and the
 * Minuit-style BFGS (ffcu_fit_gradient_opts; analytic as there). */
int ffcu_shard_group_fit(ffcu_shard_group* g, double tolerance, long max_iterations, ffit_fit_result** out);
int ffcu_shard_group_fit_gradient(ffcu_shard_group* g, double tolerance, long max_iterations, int analytic,
                                  ffit_fit_result** out);

/* Last fused-NLL launch shape: threads, events/thread, tile, tiles, chunks, grid. */
int ffcu_last_launch(const ffit_model* m, int* info6);
/* Terms of the model's last likelihood launch served by the launch-constant branch cache
 * (ArgusBG with m0 and p = 1/2 fixed over the launch's points: its data-only part computed
 * once per staged tile; values bit-identical; FFB_NO_CONST_CACHE=1 turns it off). */
int ffcu_last_launch_cached(const ffit_model* m);
/* CUDA-event timing of every fused NLL kernel launch while enabled (on the
 * launching stream); _read synchronises, returns the summed ms and the launch
 * count, and clears. */
int ffcu_kernel_timer(int enable);
int ffcu_kernel_timer_read(double* total_ms, unsigned long long* count);
/* Kernels this library has launched in this process. */
unsigned long long ffcu_kernel_launches(void);
/* Test hook: the fused kernel's device exp (0), log (1), sqrt (2) or rsqrt seed (3) over n host doubles. */
int ffcu_math_probe(int which, const double* in, double* out, long long n);
/* Measured FP64 FMA instructions per second on the current device. */
int ffcu_fp64_peak(double* fma_per_s, float* ms);
/* Issue-slot probe: FP64 FMA instructions per second with `others_per_8` (0, 2, 4, 5, 6, 8 or 16)
 * independent integer multiply-adds issued per eight DFMAs. */
int ffcu_fp64_issue_probe(int others_per_8, double* fma_per_s);
/* Seeded generator into host columns (one per observable, each n doubles). */
int ffcu_sample_host(ffit_model* m, long long n, unsigned long long seed, double* const* cols,
                     double* efficiency);

#ifdef __cplusplus
}
#endif

#endif /* FFIT_B200_H */
