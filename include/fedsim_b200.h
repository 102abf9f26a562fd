/*
 * fedsim_b200.h -- C ABI of the B200 (sm_100a) central-iteration kernels.
 *
 * One shared library, libfedsim_b200.so, loaded by the Python host side
 * with ctypes (paper_2404_06430_b200/native.py).  Every entry point is a
 * batched-cohort replacement for a per-user reference function; the
 * reference function each one replaces is cited beside it
 * (paths relative to /root/reference/pkg/src/).
 *
 * Conventions
 *   - Every pointer argument is a caller-owned, contiguous DEVICE buffer
 *     (fp32 unless the type says otherwise) except where marked [host].
 *   - Every call is asynchronous on the given stream (a cudaStream_t passed
 *     as void*; NULL = legacy default stream) and never synchronises.
 *   - No hidden allocations: scratch comes from the caller, sized with the
 *     matching *_workspace_bytes query.
 *   - Return 0 (FB_OK) or a negative FB_ERR_* code; fb_last_error() returns
 *     a thread-local message describing the last failure on this thread.
 *   - Parameter vectors are flat in the model's entry order
 *     (paper_2404_06430_b200/models.py), the payload order of the
 *     reference's Statistics (fedsim/core/statistics.py:97-101).
 *   - A cohort is described by per-client arrays over a packed dataset:
 *       row_start[c] (int64)  first row of client c in X / y
 *       num_rows[c]  (int32)  n_c >= 1
 *       perm_off[c]  (int64)  first entry of client c in perms
 *       perms        (int32)  epochs * n_c local row indices per client,
 *                             epoch-major: batch j of epoch e is
 *                             perms[perm_off[c] + e*n_c + j*B ...]
 *                             (fedsim/models/kernels.py:46-50)
 *   - Local SGD writes delta_out[c*ld + i] = theta_t[i] - theta_c[i]
 *     (unweighted; fedsim/models/params.py:32-45 before weighting).
 */
#ifndef FEDSIM_B200_H
#define FEDSIM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FB_OK 0
#define FB_ERR_ARG (-1)         /* invalid argument (reference: ValueError)   */
#define FB_ERR_CUDA (-2)        /* CUDA runtime / launch failure              */
#define FB_ERR_UNSUPPORTED (-3) /* shape outside what the kernels implement   */

#define FB_ABI_VERSION 1

int fb_abi_version(void);
const char* fb_last_error(void);
/* [host] writes the device's SM count and L2 bytes; 0 on success. */
int fb_device_info(int device, int* sm_count, int64_t* l2_bytes);

/* [host] Launch accounting (bench/profiling).  fb_launch_count: kernels
 * launched by this library since load.  fb_timing_enable(1) clears and starts
 * bracketing every launch with CUDA events on its own stream;
 * fb_timing_report synchronises on them and writes, per kernel name,
 * the summed device milliseconds and launch count (names '\n'-separated);
 * returns the number of entries (or < 0 on error).                          */
int64_t fb_launch_count(void);
void fb_timing_enable(int on);
int fb_timing_report(char* names, int names_len, double* ms, int64_t* counts, int max_entries);

/* [host] Per-user minibatch orders, bit-exact with the reference's
 * default_rng(derive_seed(ctx, "user", uid)).permutation(n) per epoch
 * (fedsim/core/seeds.py:18-33, fedsim/models/models.py:252-255): SHA-256,
 * numpy SeedSequence + PCG64 and Generator.permutation restated natively.
 * id_reprs holds repr(uid).encode() of every user back to back, user u at
 * [id_off[u], id_off[u+1]).  Writes epochs * num_rows[u] int32 at
 * perms_out + perm_off[u].  fb_derive_seed: the 63-bit seed of a message.  */
int fb_user_permutations(uint64_t context_seed, const uint8_t* id_reprs, const int64_t* id_off, int num_users,
                         const int32_t* num_rows, int epochs, int32_t* perms_out, const int64_t* perm_off);
int fb_derive_seed(const uint8_t* data, int64_t len, uint64_t* out);

/* ---------------------------------------------------------------- a4 eval
 * Per-client summed cross-entropy and correct count at the shared theta,
 * over all of the client's rows.  Replaces fedsim/models/kernels.py:70-83
 * (_logistic_eval) and :123-136 (_mlp_eval) via evaluate_model
 * (fedsim/models/models.py:275-296), batched over the cohort.
 * loss_sum[c] += ..., correct[c] += ... are OVERWRITTEN (not accumulated).
 * Argmax takes the first maximal logit (numpy.argmax).                     */
int fb_eval_linear_f32(const float* theta, int dim, int num_classes,
                       const float* X, const int32_t* y,
                       const int64_t* row_start, const int32_t* num_rows, int num_clients,
                       double* loss_sum, int32_t* correct, void* stream);
int fb_eval_mlp_f32(const float* theta, int dim, int hidden, int num_classes,
                    const float* X, const int32_t* y,
                    const int64_t* row_start, const int32_t* num_rows, int num_clients,
                    double* loss_sum, int32_t* correct, void* stream);

/* --------------------------------------------------------- a5 local SGD
 * E epochs of minibatch SGD from theta_t for every client at once; batch
 * gradients are means over the ACTUAL batch size (tail batch kept), update
 * theta <- theta - lr*(g + prox_mu*(theta - theta_t) + control).
 * control may be NULL (zero) or [num_clients, ld_control] (ld 0 = one
 * vector shared by all clients).  nonfinite[c] is set to 1 if client c's
 * delta contains a non-finite value, else 0.
 * Replaces fedsim/models/kernels.py:38-67 (_logistic_fit) and :86-120
 * (_mlp_fit) driven by local_train_sgd (fedsim/models/models.py:231-264).  */
int fb_local_sgd_linear_f32(const float* theta_t, int dim, int num_classes,
                            const float* X, const int32_t* y,
                            const int64_t* row_start, const int32_t* num_rows,
                            const int32_t* perms, const int64_t* perm_off, int num_clients,
                            int epochs, int batch_size, float lr, float prox_mu,
                            const float* control, int64_t ld_control,
                            float* delta_out, int64_t ld_delta, int32_t* nonfinite,
                            void* stream);
int fb_local_sgd_mlp_f32(const float* theta_t, int dim, int hidden, int num_classes,
                         const float* X, const int32_t* y,
                         const int64_t* row_start, const int32_t* num_rows,
                         const int32_t* perms, const int64_t* perm_off, int num_clients,
                         int epochs, int batch_size, float lr, float prox_mu,
                         const float* control, int64_t ld_control,
                         float* delta_out, int64_t ld_delta, int32_t* nonfinite,
                         void* stream);

/* ----------------------------------------------------------------- CNN
 * The BASELINE "small CIFAR-10 CNN" (paper_2404_06430_b200/models.py:CNN):
 * conv3x3(3->32)+ReLU, conv3x3(32->64)+ReLU, maxpool2, fc(12544->128)+ReLU,
 * fc(128->10), valid convolutions, CHW input rows of 3072, D = 1,626,442.
 * The reference has no CNN; these replace the generic Model.fit_local loop
 * (fedsim/models/models.py:53-79) and evaluate_model (:275-296) for a Model
 * with that layout, batched over the cohort (one SGD step of every client
 * per sequence of layer kernels).
 * max_slots = samples processed per layer launch (>= batch_size; clients
 * are trained in waves of max_slots / batch_size); the workspace for a
 * given max_slots and client count comes from fb_cnn_workspace_bytes.
 * max_steps = max over clients of epochs * ceil(n_c / batch_size).
 * batch_size <= 16.  nonfinite[] is zeroed (non-finite deltas are caught by
 * fb_delta_norm_clip_f32).
 * hist_steps selects the fc1 update form: 0 = every step reads and rewrites
 * each client's fc1 delta (6.4 MB); >= max_steps (with hist_steps *
 * batch_size <= 64) = factored: fc1 runs at theta_t plus a low-rank history
 * correction and each client's fc1 delta is written once at the end (same
 * arithmetic, see csrc/cnn.cu "fc1 in factored form").  The workspace must
 * be sized with the same hist_steps.  fc1_sumsq (nullable, [num_clients],
 * factored form only) receives each client's sum of squares of its fc1
 * weight delta block [O_F1, O_BF1), for fb_delta_norm_clip_ex_f32.          */
int64_t fb_cnn_workspace_bytes(int max_slots, int max_clients, int hist_steps);
/* Validation knob: 1 (default) = the convolutions on tcgen05; 2 = tcgen05
 * with the conv2 forward on 2-CTA clusters (cta_group::2, M = 256; correct,
 * measured slower); 3 = tcgen05 with the conv1 forward on the im2col-staged
 * kernel instead of the implicit GEMM; 4 = the conv1 weight gradient on a
 * register-blocked FP32 kernel (faster, not the default: see DESIGN.md); 0 =
 * the FP32 CUDA-core kernels kept as an independent check.                  */
int fb_cnn_set_conv_impl(int impl);
/* perms / perm_off nullable: when given, client c's evaluated rows are epoch 0's
 * perms[perm_off[c] + min(skip, n_c) ..] (the rows past the first local batch, whose
 * theta_t loss / hits fb_local_sgd_cnn_f32 adds through eval_loss / eval_correct) and
 * total_rows counts only those.                                                   */
int fb_eval_cnn_f32(const float* theta, const float* X, const int32_t* y,
                    const int64_t* row_start, const int32_t* num_rows, int num_clients,
                    int64_t total_rows, double* loss_sum, int32_t* correct,
                    int max_slots, void* workspace, int64_t workspace_bytes,
                    const int32_t* perms, const int64_t* perm_off, int skip, void* stream);
int fb_local_sgd_cnn_f32(const float* theta_t, const float* X, const int32_t* y,
                         const int64_t* row_start, const int32_t* num_rows,
                         const int32_t* perms, const int64_t* perm_off, int num_clients,
                         int epochs, int batch_size, int max_steps, float lr, float prox_mu,
                         float* delta_out, int64_t ld_delta, int32_t* nonfinite,
                         int max_slots, int hist_steps, void* workspace, int64_t workspace_bytes,
                         double* fc1_sumsq, const float* control /* nullable [C, ld_control]: c - c_i */,
                         int64_t ld_control,
                         const int32_t* h_client_steps /* nullable HOST [C]: local steps per client */,
                         int fc1_store,
                         double* eval_loss /* nullable [C]: += the first batch's theta_t loss */,
                         int32_t* eval_correct /* nullable [C]: += its first-argmax hits */, void* stream);
/* fc1_store = 0 (factored tcgen05 form, one wave of clients, fc1_sumsq set):
 * the clients' fc1 weight-delta blocks [O_F1, O_BF1) are NOT materialised --
 * fc1_sumsq still receives their sums of squares (for the clip norms) and
 * fb_cnn_fc1_aggregate_f32 then forms sum_c coef[c] * delta_c over that block
 * straight from the low-rank history left in the workspace (K3 for the fc1
 * block; replaces the fc1 part of SumAggregator.accumulate,
 * fedsim/engine/aggregator.py:39-44).  Call it after this function with the
 * same workspace and arguments, before the workspace is reused; agg_fc1 is
 * the [12544 x 128] fc1 block of the aggregate (overwritten).                */
int fb_cnn_fc1_aggregate_f32(const float* coef, int num_clients, int batch_size, int max_steps, float lr,
                             float prox_mu, int max_slots, int hist_steps, void* workspace,
                             int64_t workspace_bytes, float* agg_fc1, void* stream);

/* ------------------------------------------------------- data movement
 * Copy each cohort client's contiguous rows (num_rows[c] rows of row_bytes
 * starting at row row_start[c] of src) to row dst_start[c] of dst.  src may
 * be device memory or pinned host memory (UVA); one launch per context.
 * max_rows_per_client sizes the grid.  Used by the host-resident-dataset
 * (end-to-end) path in place of per-user host arrays
 * (fedsim/feddata/datasets.py:12-40).                                     */
int fb_gather_rows(const void* src, int64_t row_bytes, const int64_t* row_start,
                   const int32_t* num_rows, int num_clients, const int64_t* dst_start,
                   void* dst, int64_t max_rows_per_client, void* stream);
/* The same copy with at most num_blocks thread blocks, each copying whole
 * clients: for a copy stream running beside the compute kernels (the
 * engine's prefetch of iteration t+1's cohort rows during iteration t). */
int fb_gather_rows_lite(const void* src, int64_t row_bytes, const int64_t* row_start,
                        const int32_t* num_rows, int num_clients, const int64_t* dst_start,
                        void* dst, int num_blocks, void* stream);
/* Upload `bytes` (multiple of 16, 16-byte aligned pointers) from pinned host
 * memory to the device with a kernel reading the host buffer over UVA, not a
 * copy-engine memcpy: the engine's per-context descriptors (row offsets,
 * permutations, weights) then never queue behind the copy engines' prefetch
 * of the next iteration's cohort rows. */
int fb_upload_pinned(const void* host_src, void* dst, int64_t bytes, void* stream);

/* ------------------------------------- config C: transformer LM (a4 + a5)
 * models.TransformerLM, the StackOverflow-shaped next-word model of BASELINE
 * configs[2].  dims (host int32[6])
 * = {vocab, d_model, heads, ff, layers, seq}.  X rows are sentences of seq+1
 * token ids stored as floats (0 = pad); h_num_rows is the host copy of
 * num_rows.  Eval: per-client summed CE over non-pad targets and correct
 * (first-argmax) targets, processed in chunks of eval_groups x batch_size
 * sentences.  Local SGD: the generic update rule of fedsim/models/models.py:
 * 53-79 with the batch loss the mean CE over the batch's non-pad targets,
 * clients trained clients_per_wave at a time; delta / nonfinite as in
 * fb_local_sgd_mlp_f32.  Shapes: d <= 256, d % heads == 0, d / heads <= 32,
 * seq <= 32 (FB_ERR_UNSUPPORTED otherwise).                                */
int64_t fb_lm_num_params(const int32_t* dims);
/* [host] GEMM implementation of the LM entry points (process-wide): 1 =
 * tcgen05 3xTF32 (default: TMA-fed persistent kernel, split products on the
 * tensor cores, TMEM accumulation in 2-slice windows folded into fp32), 0 =
 * the SIMT FP32 tiled GEMM (validation).                                    */
int fb_lm_set_gemm_impl(int impl);
int64_t fb_lm_workspace_bytes(const int32_t* dims, int batch_size, int clients_per_wave, int eval_groups);
/* perms / perm_off nullable, as in fb_eval_cnn_f32: when given, client c's evaluated
 * sentences are epoch 0's perms[perm_off[c] + min(skip, n_c) ..], the first batch's
 * theta_t loss / hits being added by fb_local_sgd_lm_f32 through eval_loss / eval_correct. */
int fb_eval_lm_f32(const float* theta, const int32_t* dims, const float* X, const int64_t* row_start,
                   const int32_t* num_rows, const int32_t* h_num_rows, int num_clients, double* loss_sum,
                   int32_t* correct, int batch_size, int eval_groups, void* workspace, int64_t workspace_bytes,
                   const int32_t* perms, const int64_t* perm_off, int skip, void* stream);
int fb_local_sgd_lm_f32(const float* theta_t, const int32_t* dims, const float* X, const int64_t* row_start,
                        const int32_t* num_rows, const int32_t* h_num_rows, const int32_t* perms,
                        const int64_t* perm_off, int num_clients, int epochs, int batch_size, float lr,
                        float prox_mu, const float* control, int64_t ld_control, float* delta_out, int64_t ld_delta,
                        int32_t* nonfinite, int clients_per_wave, void* workspace, int64_t workspace_bytes,
                        double* eval_loss /* nullable [C]: += the first batch's theta_t loss */,
                        int32_t* eval_correct /* nullable [C] */, void* stream);

/* ------------------------------- config D: ResNet-18, multi-label (a4 + a5)
 * models.ResNet18, the FLAIR-shaped image model of BASELINE configs[3]
 * (/root/reference/PAPER.md:1104-1138): torchvision's ResNet-18 layout with
 * GroupNorm, dims (host int32[4]) = {num_classes, width, groups, image side}.
 * X rows (ldx floats, >= 3 S^2 + K) hold an image's CHW pixels followed by its K
 * label indicators; h_num_rows is the host copy of num_rows.  Loss per image: the
 * mean sigmoid BCE over its K labels; eval: per-client summed per-image loss and
 * exact-match images, in chunks of groups x batch_size images.  Local SGD: the
 * generic update rule of fedsim/models/models.py:53-79 (batch loss = mean over
 * the batch's images), clients trained clients_per_wave at a time, largest
 * first; delta / nonfinite / perms / eval_loss as in fb_local_sgd_lm_f32.
 * Shapes: width a power of two in [4, 64], groups dividing it, S in [32, 1024],
 * K <= 256 (FB_ERR_UNSUPPORTED otherwise).                                  */
int64_t fb_resnet_num_params(const int32_t* dims);
int64_t fb_resnet_workspace_bytes(const int32_t* dims, int batch_size, int clients_per_wave);
int fb_eval_resnet_f32(const float* theta, const int32_t* dims, const float* X, int64_t ldx, const int64_t* row_start,
                       const int32_t* num_rows, const int32_t* h_num_rows, int num_clients, double* loss_sum,
                       int32_t* correct, int batch_size, int groups, void* workspace, int64_t workspace_bytes,
                       const int32_t* perms, const int64_t* perm_off, int skip, void* stream);
int fb_local_sgd_resnet_f32(const float* theta_t, const int32_t* dims, const float* X, int64_t ldx,
                            const int64_t* row_start, const int32_t* num_rows, const int32_t* h_num_rows,
                            const int32_t* perms, const int64_t* perm_off, int num_clients, int epochs,
                            int batch_size, float lr, float prox_mu, const float* control, int64_t ld_control,
                            float* delta_out, int64_t ld_delta, int32_t* nonfinite, int clients_per_wave,
                            void* workspace, int64_t workspace_bytes, double* eval_loss, int32_t* eval_correct,
                            void* stream);

/* ------------------------------------------------- a6 + a7 (kernel K2)
 * For every client c: norm[c] = || w[c] * delta[c, :D] ||_2 (fp64
 * accumulation), clipped[c] = norm[c] > bound (strict), coef[c] =
 * w[c] * (clipped ? bound / norm : 1), nonfinite[c] = !isfinite(norm).
 * Replaces model_update_delta -> weighted (fedsim/models/params.py:32-45,
 * fedsim/core/statistics.py:124-136) followed by clip_norm
 * (fedsim/privacy/clipping.py:37-56) over the payload entries.
 * bound <= 0 disables clipping (coef = w, clipped = 0).                   */
int64_t fb_clip_workspace_bytes(int num_clients, int64_t D);
int fb_delta_norm_clip_f32(const float* delta, int64_t ld_delta, int num_clients, int64_t D,
                           const float* w, double bound,
                           double* norm, float* coef, int32_t* clipped, int32_t* nonfinite,
                           void* workspace, int64_t workspace_bytes, void* stream);
/* K2 with the columns [skip_lo, skip_hi) excluded from the scan and their
 * per-client sum of squares supplied in extra_sumsq[C] (nullable = 0): the
 * CNN's factored fc1 block, whose squares fb_local_sgd_cnn_f32 sums while it
 * materialises the block (same values, fp64, fixed order).  skip_hi must be
 * a multiple of 4; workspace >= fb_clip_workspace_bytes(C, D) + 16 * C bytes. */
int fb_delta_norm_clip_ex_f32(const float* delta, int64_t ld_delta, int num_clients, int64_t D,
                              int64_t skip_lo, int64_t skip_hi, const double* extra_sumsq,
                              const float* w, double bound, double* norm, float* coef,
                              int32_t* clipped, int32_t* nonfinite, void* workspace,
                              int64_t workspace_bytes, void* stream);

/* ------------------------------------------------------- a8 (kernel K3)
 * agg[i] (+)= sum_c coef[c] * delta[c*ld + i], fp64 accumulation per
 * element; accumulate = 0 overwrites agg, 1 adds into it.
 * Replaces SumAggregator.accumulate (fedsim/engine/aggregator.py:39-44,
 * fedsim/core/statistics.py:96-102) over a worker's queue.                 */
int64_t fb_weighted_sum_workspace_bytes(int num_clients, int64_t D);
int fb_weighted_sum_f32(const float* delta, int64_t ld_delta, int num_clients, int64_t D,
                        const float* coef, float* agg, int accumulate,
                        void* workspace, int64_t workspace_bytes, void* stream);

/* ------------------------------------------ a6 + a7 + a8 fused (K2 + K3)
 * One HBM pass: the outputs of fb_delta_norm_clip_f32 (norm, coef, clipped,
 * nonfinite) AND of fb_weighted_sum_f32 (agg (+)= sum_c coef[c] delta[c])
 * from a single persistent cooperative kernel that keeps each SM's column
 * slice of the aggregate on chip and re-reads client c-1 from L2 while it
 * streams client c from HBM.  Same reference semantics as K2 and K3
 * (fedsim/privacy/clipping.py:37-56, fedsim/engine/aggregator.py:39-44);
 * fp32 accumulation in blocks of 64 clients, fp64 across blocks.
 * Requires D <= fb_clip_aggregate_max_columns() (FB_ERR_UNSUPPORTED
 * otherwise: use K2 + K3), ld_delta % 4 == 0 and a 16-byte aligned delta. */
int64_t fb_clip_aggregate_max_columns(void);
int64_t fb_clip_aggregate_workspace_bytes(int num_clients, int64_t D);
int fb_clip_aggregate_f32(const float* delta, int64_t ld_delta, int num_clients, int64_t D,
                          const float* w, double bound, double* norm, float* coef,
                          int32_t* clipped, int32_t* nonfinite, float* agg, int accumulate,
                          void* workspace, int64_t workspace_bytes, void* stream);
/* The same with client c's update at delta row rows[c] (int32 device array): a
 * queue order that differs from the storage order, or one pool of rows reused
 * (the configs[4] microbench) -- all C clients in one launch.               */
int fb_clip_aggregate_rows_f32(const float* delta, const int32_t* rows, int64_t ld_delta, int num_clients,
                               int64_t D, const float* w, double bound, double* norm, float* coef,
                               int32_t* clipped, int32_t* nonfinite, float* agg, int accumulate,
                               void* workspace, int64_t workspace_bytes, void* stream);

/* ------------------------------------------------ a9 (worker_reduce)
 * Per-context sums over the C clients of this rank, fp64 in a fixed order,
 * written as fp32 (hi, lo) pairs: tail[2f] + tail[2f+1] == sum f (hi alone
 * exact for integer-valued sums < 2^24).  The tail sits behind the payload in
 * one flat fp32 buffer so a single all-reduce replaces the reference's
 * worker_reduce of payload + bookkeeping (fedsim/engine/aggregator.py:55-62)
 * and the metric merge (fedsim/engine/runtime.py:148-153).  Fields:        */
#define FB_SUM_LOSS 0      /* sum eval loss            (fedsim/algorithms/fedavg.py:127-139) */
#define FB_SUM_CORRECT 1   /* sum correct predictions                                      */
#define FB_SUM_POINTS 2    /* sum n_c                                                      */
#define FB_SUM_USER_ACC 3  /* sum correct_c / n_c      (fedsim/core/metrics.py:52-53)      */
#define FB_SUM_USERS 4     /* number of clients                                            */
#define FB_SUM_CLIPPED 5   /* sum clip indicators      (fedsim/privacy/clipping.py:113-116)  */
#define FB_SUM_COUNT 6     /* training clients                                             */
#define FB_SUM_NORM 7      /* sum pre-clip norms                                           */
#define FB_SUM_WEIGHT 8    /* sum w_c                  (fedsim/core/statistics.py:96-102)  */
#define FB_SUM_NONFINITE 9 /* clients with a non-finite update (fedsim/engine/runtime.py:202-208) */
#define FB_NUM_SUMS 10
/* train = 0 (evaluation context): norm / clipped / nonfinite / w may be NULL and
 * fields 5..9 are 0.  tail: 2 * FB_NUM_SUMS floats (OVERWRITTEN).           */
int fb_context_sums(const double* loss, const int32_t* correct, const int32_t* num_rows, const double* norm,
                    const int32_t* clipped, const int32_t* nonfinite, const float* w, int num_clients, int train,
                    float* tail, void* stream);

/* ------------------------------------------------- a10 helpers (K4 SNR)
 * out[0] = sum_i x[i]^2 in fp64 (OVERWRITTEN).  workspace >= 8 KiB.         */
int fb_sumsq_f32(const float* x, int64_t n, double* out, void* workspace,
                 int64_t workspace_bytes, void* stream);

/* Counter-based Gaussian: out[i] (+)= std * N(0,1) from Philox4x32-10 keyed
 * by seed, counter = offset + i.  accumulate = 0 overwrites.               */
int fb_gaussian_f32(float* out, int64_t n, double std, uint64_t seed, uint64_t offset,
                    int accumulate, void* stream);

/* ------------------------------------------ a10 + a12 (kernels K4 + K5)
 * theta[i] -= lr * inv_weight * (agg[i] + noise_i) where noise_i is
 *   injected[i]                          if injected != NULL (parity runs),
 *   noise_std * Philox-normal(seed, i)   otherwise (0 if noise_std == 0).
 * Replaces _add_noise (fedsim/privacy/mechanisms.py:58-75) + average
 * (fedsim/core/statistics.py:105-113) + SGDOptimizer.step / apply_delta
 * (fedsim/models/optimizers.py:13-21, fedsim/models/params.py:48-53).
 * If agg_out != NULL the noised aggregate is also written there.           */
int fb_noise_avg_sgd_f32(float* theta, const float* agg, int64_t D,
                         double noise_std, uint64_t seed, const float* injected,
                         double inv_weight, double lr, float* agg_out, void* stream);

/* ------------------------------------------ a10 + a12 with central Adam
 * a = (agg + noise) * inv_weight (noise as in fb_noise_avg_sgd_f32), then
 * one bias-corrected Adam step at step count `step` (>= 1):
 *   m1 = b1*m1 + (1-b1)*a,  m2 = b2*m2 + (1-b2)*a^2   (in place)
 *   theta -= lr * (m1/(1-b1^step)) / (sqrt(m2/(1-b2^step)) + eps)
 * Replaces AdamOptimizer.step (fedsim/models/optimizers.py:24-68) after
 * average (fedsim/core/statistics.py:105-113).  eps = adaptivity_degree.   */
int fb_noise_avg_adam_f32(float* theta, float* m1, float* m2, const float* agg, int64_t D,
                          double noise_std, uint64_t seed, const float* injected,
                          double inv_weight, double lr, double beta1, double beta2, double eps,
                          int64_t step, float* agg_out, void* stream);

/* ------------------------------------------ SCAFFOLD control variates
 * (fedsim/algorithms/scaffold.py:46-79).  Per-user controls live in a
 * device store [rows, ld_store]; rows[c] = store row of client c, -1 = zero
 * control (first participation).
 * correction[c] = server - store[rows[c]]       -> the local-SGD control term
 * payload[c]    = [delta_c | delta_c*scale_c - server]   (model/, control/)
 * new_control[c] = store[rows[c]] - server + delta_c*scale_c
 * with scale_c = 1 / (steps_c * lr).  fb_scatter_rows_f32 writes
 * store[rows[c]] = src[c] (the user updates of process_aggregated_...). */
int fb_scaffold_correction_f32(const float* server, const float* store, int64_t ld_store,
                               const int32_t* rows, int num_clients, int64_t D, float* out,
                               int64_t ld_out, void* stream);
int fb_scaffold_payload_f32(const float* delta, int64_t ld_delta, const float* server,
                            const float* store, int64_t ld_store, const int32_t* rows,
                            const float* scale, int num_clients, int64_t D, float* payload,
                            int64_t ld_payload, float* new_control, int64_t ld_new, void* stream);
int fb_scatter_rows_f32(float* store, int64_t ld_store, const int32_t* rows, const float* src,
                        int64_t ld_src, int num_rows, int64_t D, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* FEDSIM_B200_H */
