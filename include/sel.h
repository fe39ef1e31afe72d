/*
 * sel.h -- C ABI of the B200-native SZ-vs-ZFP rate-distortion estimator.
 *
 * Implements the hot path of Tao et al., "Optimizing Lossy Compression
 * Rate-Distortion from Automatic Online Selection between SZ and ZFP"
 * (arXiv 1806.08901): Algorithm 1 lines 1-10 for one
 * float32 field resident in GPU memory:
 *   - value range VR and eb = eb_abs or eb_rel*VR            (Alg.1 line 2)
 *   - block sampling with per-axis stride                      (Alg.1 line 3)
 *   - SZ: Lorenzo residual on original values, linear
 *     quantisation with bin width 2*eb, histogram of codes with
 *     65,535 bins, Shannon-entropy bit-rate (Eq. entropy P:326,
 *     Eq. bitrate-sz) + 0.5 bit offset, PSNR Eq. psnr-sz
 *   - ZFP: per 4^d block exponent, block floating point, decorrelating lift,
 *     sequency reorder, negabinary, exact group-testing EC bit count at the
 *     fixed-accuracy cut and truncation-error PSNR
 *
 *   - selection at equal PSNR (Alg.1 lines 7-10)
 * DESIGN.md section 3 lists every reading taken where the paper is silent.
 *
 * Conventions
 *   - dims are C order: dims[0] slowest, dims[ndims-1] fastest (contiguous).
 *   - All entry points are extern "C", never throw, never abort; they return a
 *     sel_status (0 = OK, < 0 = error) and leave *out untouched on error.
 *   - A plan is not reentrant: at most one estimate call in flight per plan.
 *     Distinct plans are independent.  The plan owns all device workspace.
 *   - Device pointers must be CUDA device (or managed) memory of the current
 *     device, float32, C-contiguous; 16-byte alignment enables the vector path
 *     (torch's allocator guarantees 256 B).  The field must stay valid and
 *     unmodified until the call returns.
 *   - stream: a cudaStream_t passed as void* (NULL = legacy default stream).
 *     Estimate calls enqueue on that stream and synchronise it before
 *     returning the host-side result.
 */
#ifndef SEL_H
#define SEL_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SEL_OK = 0,
  SEL_EINVAL = -1,      /* bad argument: ndims not in {1,2,3}, dims < 1, prod(dims) overflow,
                           eb not finite or <= 0, 1/(2 eb_abs) not finite in float, stride < 1,
                           block != 4, NULL pointer, unknown option key */
  SEL_ENOMEM = -2,      /* device or host allocation failed */
  SEL_ECUDA = -3,       /* any CUDA runtime error; sel_strerror(SEL_ECUDA) has the message */
  SEL_ENONFINITE = -4,  /* the field contains NaN or +-Inf (detected on the device) */
  SEL_EDEGENERATE = -5, /* relative eb with VR == 0, or no SZ point besides the origin */
  SEL_ENOTIMPL = -6
} sel_status;

typedef enum { SEL_EB_ABS = 0, SEL_EB_REL = 1 } sel_eb_mode;

typedef struct sel_plan_st *sel_plan_t;

/* Per-field result.  The first six members are north_star's result tuple. */
typedef struct {
  double sz_bits_per_value;  /* H + offset + 32*p_ovf  (bins of width 2*eb_abs)               */
  double sz_psnr;            /* 20 log10(VR/eb_abs) + 10 log10 3              (Eq. psnr-sz)  */
  double zfp_bits_per_value; /* exact fixed-accuracy EC bits / values in processed blocks     */
  double zfp_psnr;           /* 20 log10 VR - 10 log10 MSE; +INF if MSE == 0                  */
  int32_t choice;            /* Alg.1 selection bit s_i: 0 = SZ, 1 = ZFP                      */
  int32_t matched;           /* 1 if compared at equal PSNR; 0 = fallback at the user's eb    */
  /* diagnostics (parity tests compare these too) */
  double value_range;        /* (double)max - (double)min over the whole field                */
  double eb_abs;             /* absolute error bound used                                     */
  double sz_entropy;         /* H in bits/value                                               */
  double sz_overflow_frac;   /* fraction of SZ points in the overflow ("unpredictable") slot */
  double sz_bits_matched;    /* BR_sz at the PSNR-matched bin delta* (Alg.1 line 9)          */
  double sz_eb_matched;      /* delta_star / 2: SZ bound giving PSNR_zfp (Alg.1 line 11 reading) */
  double zfp_mse;            /* sum_b E_b / n_values                                          */
  uint64_t n_sz_points;      /* SZ residuals histogrammed (processed points minus the origin) */
  uint64_t n_values;         /* real values in processed blocks                               */
  uint64_t n_blocks;         /* processed 4^d blocks                                          */
  uint64_t zfp_total_bits;   /* sum of per-block EC bits incl. headers                        */
  double zfp_err_sum;        /* sum_b E_b                                                     */
  int32_t minexp;            /* floor(log2 eb_abs)                                            */
  float r_f;                 /* float(1/(2 eb_abs)), the quantiser scale                      */
  int32_t status;            /* sel_status of this field (batch calls)                        */
  int32_t choice_eb;         /* selection based on the error bound (Lu et al.): the  */
                             /* lower bit-rate at the user's eb, 0 = SZ iff BR_sz < BR_zfp    */
  uint64_t hist_total;       /* sum of the 65,536 histogram counts as the finalize read them  */
                             /* on the device (== n_sz_points unless a count was lost)        */
  uint64_t hist_ovf;         /* count in the overflow slot 65,535, device-counted              */
} sel_result;

/* the paper's own estimator as printed (Alg. 1 lines 3-10),
 * reported next to the exact estimate of sel_estimate (which counts every coefficient's
 * EC bits and gain-weights the error, R13/R14). */
typedef struct {
  double zfp_nsb_bits;       /* BR_zfp: average n_sb, 3/9/16 sampled coefficients per block     */
                             /* linearly interpolated over the block          */
  double zfp_mse_sp;         /* MSE_sp: mean (dropped-plane value x 2^(emax-30))^2 of the samples */
                             /* (unit weights)                                        */
  double zfp_psnr_sp;        /* -10 log10 MSE_sp + 20 log10 VR; +INF if MSE_sp == 0              */
  double sz_delta;           /* delta = VR sqrt(12) 10^(-PSNR_sp/20) (Alg.1 line 7); 2 eb_abs if  */
                             /* matched == 0                                                     */
  double sz_bits;            /* BR_sz: entropy of the residuals at bin width delta + 0.5 + 32 p_ovf */
  double sz_entropy;
  double sz_overflow_frac;
  double value_range, eb_abs;
  uint64_t nsb2_total;       /* 2 x sum of the interpolated n_sb (exact integer)                 */
  uint64_t n_samples;        /* sampled coefficients (m x processed blocks)                      */
  uint64_t n_values;         /* real values in processed blocks                                  */
  uint64_t hist_total, hist_ovf;
  float r_star;              /* float(1 / delta), the quantiser scale of the re-quantisation      */
  int32_t choice;            /* Alg.1 line 10: 0 = SZ iff sz_bits < zfp_nsb_bits, else 1 = ZFP    */
  int32_t matched;           /* 0: MSE_sp == 0 or VR == 0, compared at the user's bound           */
  int32_t status;
} sel_paper_result;

/* the variant quantisers of the paper's Section 5.1.4 evaluated with its
 * general Stage-II estimators -- BR = -sum_i P_i log2 P_i (Eq. bit-rate-pdf), MSE
 * = (1/12) sum_i delta_i^2 P_i, PSNR = 20 log10 VR - 10 log10 MSE (Eq. psnr-pdf,
 * P:377-380) -- on the PDF the selector stores, the field's 65,535-bin code histogram
 * (P:637): cell q = [(q - 1/2) delta, (q + 1/2) delta), delta = 2 eb_abs, uniform inside
 * (reading R21; codes in the overflow slot are outside the PDF). */
typedef struct {
  double lin_bits, lin_psnr; /* linear: entropy of the in-range codes, Eq. psnr-pdf-linear */
  double log_bits, log_psnr; /* log-scale, integer base b: central bin |q| < b, bin +-i  */
  double log_mse;            /* holds b^i <= |q| < b^(i+1) (widths 2b - 1 and b^(i+1) - b^i cells)   */
  double eqp_bits, eqp_psnr; /* equal-probability, 2n - 1 bins: BR = 1 + log2 n,  */
  double eqp_mse;            /* edges at the quantiles k / (2n - 1) of the piecewise-linear CDF,      */
                             /* MSE = delta^2 sum_k w_k^2 / (12 (2n - 1))                             */
  double eqp_width_sum;      /* sum_k w_k (cells) = occupied support                                  */
  double value_range, eb_abs;
  uint64_t n_in;             /* in-range codes (the PDF's mass)                                       */
  uint64_t hist_ovf;         /* codes in the overflow slot                                            */
  int32_t log_base, log_bins;/* b; occupied log-scale bins                                            */
  int32_t eqp_n;             /* n                                                                     */
  int32_t status;
} sel_variant_result;

/* Create a plan for fields of shape dims[0..ndims-1].
 *   mode, eb : SEL_EB_ABS -> eb_abs = eb; SEL_EB_REL -> eb_abs = eb * VR (Alg.1 line 2)
 *   stride   : ndims entries >= 1, block b is processed iff b_a % stride[a] == 0 for
 *              every axis a; NULL = all 1 (every block)
 *   block    : ZFP block edge, must be 4
 * Allocates the device workspace on the current device.  Errors: SEL_EINVAL,
 * SEL_ENOMEM, SEL_ECUDA. */
int sel_plan(sel_plan_t *out, int ndims, const int64_t *dims, sel_eb_mode mode, double eb,
             const int32_t *stride, int32_t block);

/* Options:
 *   "sz_offset_bits"  SZ bit-rate offset beta (default 0.5)
 *   "debug"           1 = dump intermediates for sel_debug_copy (per-field kernels;
 *                     test sizes only)
 *   "kernel_timing"   1 = record CUDA events around every launch (sel_kernel_times)
 *   "batch_kernel"    1 (default) = one persistent k_batch launch per call where the
 *                     shape allows (2D/3D, fastest extent % 4 == 0, 16-byte aligned
 *                     fields); 0 = per-field kernels
 *   "pipeline"        1 (default) = per-field kernels of a batch on three streams
 *   "groups"          k_batch CTA groups, 0 (default) = automatic, else 1..148
 *   "lag"             k_batch phases between a field's range pass and its tiles, 1..4
 *                     (default 2)
 *   "range_warps"     1 (default) = k_batch streams the value range of full-field stacks on
 *                     dedicated warps; 0 = as range tasks through the tile stage ring
 *   "small_kernel"    1 (default) = one small field (N <= 2^21) in one cooperative launch
 *   "multi_tile"      1 (default) = sel_estimate_multi runs its fused pass on the TMA tile
 *                     pipeline where the shape allows; 0 = one thread per block
 *   "batch_debug"     1 = the persistent k_batch kernel also dumps, per field, the
 *                     histogram its finalize tasks read and its per-(task, part) partials
 *                     (sel_debug_copy "batch_hist" / "batch_part"; tests)
 * None changes any result (tests).  Errors: SEL_EINVAL (unknown key, value out of range). */
int sel_set_option(sel_plan_t plan, const char *key, double value);

/* Estimate one field already in device memory (d_field: device, N floats).
 * Enqueues value range -> fused SZ/ZFP pass -> finalize on `stream`, copies the
 * result to pinned host memory, synchronises `stream`, fills *out.
 * Errors: SEL_EINVAL, SEL_ENONFINITE, SEL_EDEGENERATE, SEL_ECUDA. */
int sel_estimate(sel_plan_t plan, const float *d_field, void *stream, sel_result *out);

/* N3: the ZFP branch of Alg. 1 lines 11-15 -- "perform ZFP
 * compression on X_i with absolute error bound eb": the fixed-accuracy ZFP stream of the
 * plan's processed blocks (stride 1: the whole field), whose per-block lengths are the
 * bits the estimate counts (zfp_total_bits == *nbits).  Per block, row-major: 1 bit 0 if
 * the block is empty or keeps no bit plane; else 1 bit 1, 8 bits emax + 127, then the
 * group-testing embedded code of planes 31..kmin (R13); bits packed
 * LSB first into little-endian 32-bit words.
 *   d_out : device buffer owned by the caller, or NULL to query the length only;
 *           cap_bytes must be >= ceil(*nbits / 32) * 4 (else SEL_EINVAL, *nbits set).
 *   nbits : out, the stream length in bits.
 * Synchronises `stream`.  The SZ branch (line 12) is not built.
 * Errors: SEL_EINVAL, SEL_ENONFINITE, SEL_EDEGENERATE, SEL_ENOMEM, SEL_ECUDA. */
int sel_compress_zfp(sel_plan_t plan, const float *d_field, void *d_out, uint64_t cap_bytes, uint64_t *nbits,
                     void *stream);

/* N2: the paper-literal estimate of one device field with the plan's eb,
 * mode and stride (sel_paper_result above).  Two dependent passes, as Alg. 1 prints them:
 * the ZFP samples give PSNR_sp, whose delta fixes the SZ re-quantisation of the same
 * processed blocks.  d_field: device, float32, C order; synchronises `stream`.
 * Errors: SEL_EINVAL (NULL, options debug / kernel_timing set), SEL_ENONFINITE,
 * SEL_EDEGENERATE (status also in out->status), SEL_ENOMEM, SEL_ECUDA. */
int sel_estimate_paper(sel_plan_t plan, const float *d_field, void *stream, sel_paper_result *out);

/* N4: the log-scale and equal-probability quantisation estimates of one device
 * field (sel_variant_result above) with the plan's eb, mode and stride: value range, the
 * fused pass (its code histogram is the PDF), then one pass over the 65,535 bins.
 *   log_base : integer b >= 2;  eqp_n : n in 1..32768 (2n - 1 bins).
 * d_field: device, float32, C order; synchronises `stream`.  Errors: SEL_EINVAL (NULL,
 * b or n out of range, options debug / kernel_timing set), SEL_ENONFINITE, SEL_EDEGENERATE
 * (also when no code is in range; status also in out->status), SEL_ENOMEM, SEL_ECUDA. */
int sel_estimate_variants(sel_plan_t plan, const float *d_field, int log_base, int eqp_n, void *stream,
                          sel_variant_result *out);

/* N1: the rate-distortion curve of one field at k error bounds from ONE read
 * (P:384-392 -- rate-distortion compared over error bounds; Alg. 1 lines 2-10 per eb,
 * P:478-490).  ebs[0..k) (1 <= k <= 8) replace the plan's eb, interpreted in the plan's
 * mode (absolute, or x value range); dims, stride and block are the plan's.  The value
 * range is computed once, every processed block is read once, its Lorenzo residuals and
 * ZFP transform are formed once, and the eb-dependent stages (quantisation + histogram,
 * fixed-accuracy cut, bit count, error) run per eb (full-field 2D / 3D shapes with the
 * fastest extent % 4 == 0 and a 16-byte aligned field: on the TMA tile pipeline, one
 * shared-memory histogram window per eb).  out[e] (host, k entries) equals what
 * sel_estimate would return at ebs[e] (per-eb status in out[e].status: SEL_ENONFINITE,
 * SEL_EDEGENERATE, ...).  d_field: device, float32, C order, not modified; the call
 * synchronises `stream`.  Errors: SEL_EINVAL (NULL, k out of range, eb not finite or <= 0,
 * option kernel_timing or debug set), SEL_ENOMEM, SEL_ECUDA. */
int sel_estimate_multi(sel_plan_t plan, const float *d_field, int k, const double *ebs, void *stream,
                       sel_result *out);

/* Estimate n fields of the plan's shape (d_fields: HOST array of n DEVICE
 * pointers).  out[i].status holds each field's status; returns SEL_OK if the
 * launches succeeded (individual fields may still carry an error status). */
int sel_estimate_batch(sel_plan_t plan, const float *const *d_fields, int n, void *stream,
                       sel_result *out);

/* Stream-ordered variant of sel_estimate_batch: enqueues the estimate of the n fields
 * and a copy of the n results to `out` on `stream` and returns without waiting.
 *   out : DEVICE memory or page-locked HOST memory (cudaHostAlloc / pinned), room for n
 *         sel_result; valid once `stream` has been synchronised (caller's job).
 * The plan's workspace is reused by its next call, so successive calls on one plan must
 * be issued to the same stream (or ordered by the caller).  Not available while the
 * options debug or kernel_timing are set (they read back on the host).
 * Errors: SEL_EINVAL (NULL pointer, n < 0, debug/kernel_timing set), SEL_ENOMEM,
 * SEL_ECUDA; per-field errors land in out[i].status. */
int sel_estimate_batch_async(sel_plan_t plan, const float *const *d_fields, int n, void *stream,
                             sel_result *out);

/* End-to-end entry: fields in HOST memory (pinned for full speed).  The plan
 * stages each field into device buffers with cudaMemcpyAsync on an internal
 * copy stream, double-buffered so the copy of field i+1 overlaps the estimate
 * of field i.  h_fields: host array of n host pointers. */
int sel_estimate_batch_host(sel_plan_t plan, const float *const *h_fields, int n,
                            void *stream, sel_result *out);

/* Pure host: Alg.1 lines 7-10 recomputed from r's fields
 * (sz_bits_per_value, zfp_bits_per_value, zfp_psnr, zfp_mse, value_range, eb_abs).
 * Ties go to ZFP.  Errors: SEL_EINVAL (NULL). */
int sel_choose(const sel_result *r, int32_t *choice);

/* Pure host: the fixed-maximum-error selector the paper compares against (Lu et al.,
 * P:639-642, "selects the compressor with the highest compression ratio based on a fixed
 * error bound"): 0 (SZ) iff r->sz_bits_per_value < r->zfp_bits_per_value, both at the
 * user's eb; ties go to ZFP as in Alg.1.  Equals r->choice_eb.  Errors: SEL_EINVAL (NULL). */
int sel_choose_eb(const sel_result *r, int32_t *choice);

/* Test-only: copy a debug dump of the LAST sel_estimate (requires option debug=1):
 *   "codes"  int32[N]           slot per point, -1 where no code was formed
 *   "hist"   uint64[65536]
 *   "emax"   int32[n_blocks]    -127 for an all-zero block
 *   "coef"   int32[n_blocks*4^d] lifted coefficients, natural order
 *   "uword"  uint32[n_blocks*4^d] negabinary words, sequency order
 *   "bits"   uint32[n_blocks]
 *   "err"    double[n_blocks]   E_b
 * and of the LAST k_batch launch (requires option batch_debug=1; nf = its field count):
 *   "batch_hist" uint32[nf][65536] each field's histogram as the finalize tasks read it
 *   "batch_part" {uint64 bits, double err}[nf][nT * parts_per_task] per-(tile task, part)
 *                sums of the ZFP block bits / errors, layout from sel_batch_layout
 * bytes must equal the array size.  Errors: SEL_EINVAL, SEL_ECUDA. */
int sel_debug_copy(sel_plan_t plan, const char *what, void *host_dst, uint64_t bytes);

/* Test-only: geometry of the k_batch partials of this plan, out[0..7] =
 *   {nT tile tasks per field, parts per task, block rows per part, block rows per tile,
 *    tile columns ntk (32 blocks each), tile rows ntj, sampled (1: part p of task t covers
 *    processed blocks 32*(t*parts+p) .. +31 in row-major order), CTA groups of the last
 *    launch}.  Tile task t covers tile column t % ntk, tile row (t / ntk) % ntj, block
 *    layer t / (ntk*ntj) (3D); part p of it the block rows [p*rows_per_part, +rows_per_part)
 *    of the tile.  Errors: SEL_EINVAL (NULL). */
int sel_batch_layout(sel_plan_t plan, int64_t out[8]);

/* Per-kernel device time accumulated since the last reset (option kernel_timing=1):
 * ms[0] value range, ms[1] fused estimate, ms[2] finalize; launches[k] the count.
 * reset != 0 clears the accumulators after reading. */
int sel_kernel_times(sel_plan_t plan, double ms[3], uint64_t launches[3], int reset);

/* Number of processed blocks / values and the device workspace size of a plan. */
uint64_t sel_processed_blocks(sel_plan_t plan);
uint64_t sel_processed_values(sel_plan_t plan);
size_t sel_workspace_bytes(sel_plan_t plan);
/* Total kernel launches issued by this plan so far. */
uint64_t sel_launch_count(sel_plan_t plan);

void sel_plan_destroy(sel_plan_t plan);

/* Static description of a status; for SEL_ECUDA the last CUDA error message. */
const char *sel_strerror(int status);

#ifdef __cplusplus
}
#endif
#endif /* SEL_H */
