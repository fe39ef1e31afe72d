/*
 * orc.h -- CPU ORACLE for the SZ-vs-ZFP rate-distortion estimator of
 * Tao, Di, Liang, Chen, Cappello, "Optimizing Lossy Compression
 * Rate-Distortion from Automatic Online Selection between SZ and ZFP"
 * (arXiv 1806.08901, IEEE TPDS 2018), PAPER.md.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_1806_08901_b200/, include/sel.h) never links,
 * includes or calls anything here, and this file includes nothing from it.
 *
 * Every routine is a plain, sequential restatement of one step of the paper
 * (or of a DESIGN.md "reading" where the paper is silent); citations are
 * "P:<line>" into PAPER.md.  Floating point: fp64 except where the decision
 * that yields an integer is taken in fp32 on both sides (Lorenzo residual and
 * quantisation, R4/R5).
 */
#ifndef ORC_H
#define ORC_H
#include <stdint.h>

#define ORC_OK 0
#define ORC_EINVAL -1
#define ORC_ENONFINITE -4
#define ORC_EDEGENERATE -5

#define ORC_NSLOTS 65536       /* 65,535 code bins + 1 overflow slot */
#define ORC_OVF_SLOT 65535

typedef struct {
  double sz_bits_per_value, sz_psnr, zfp_bits_per_value, zfp_psnr;
  int32_t choice, matched;
  double value_range, eb_abs, sz_entropy, sz_overflow_frac;
  double sz_bits_matched, sz_eb_matched, zfp_mse;
  uint64_t n_sz_points, n_values, n_blocks, zfp_total_bits;
  double zfp_err_sum;   /* sum_b E_b (value units squared) */
  int32_t minexp;
  float r_f;
  int32_t choice_eb;    /* selection based on the error bound (Lu et al.) */
  int32_t pad_;
  uint64_t hist_total;  /* sum of the 65,536 histogram counts (== n_sz_points) */
  uint64_t hist_ovf;    /* count in the overflow slot 65,535 */
} orc_result;

/* Optional per-element dumps (any pointer may be NULL).
 * codes      : int32[N]   slot of every SZ point, -1 where no code was formed
 * hist       : uint64[65536]
 * emax       : int32[NP]  per processed block (row-major over processed blocks); -127 = empty
 * coef       : int32[NP*4^d] lifted coefficients, natural (row-major) order
 * uword      : uint32[NP*4^d] negabinary words in sequency order
 * bits       : uint32[NP]
 * err        : double[NP] E_b in value units squared                      */
typedef struct {
  int32_t *codes;
  uint64_t *hist;
  int32_t *emax;
  int32_t *coef;
  uint32_t *uword;
  uint32_t *bits;
  double *err;
} orc_debug;

/* ---- whole-field estimate (Alg. 1 lines 1-10) ---- */
int orc_estimate(const float *x, int ndims, const int64_t *dims, int eb_mode,
                 double eb, const int32_t *stride, double sz_offset,
                 orc_result *out, orc_debug *dbg);
/* Same, on nthreads threads (contiguous slabs of the slowest block axis); every
 * merge is exact and the per-block E_b are summed in block order, so the result is
 * bit-identical to orc_estimate (checked by tests/test_oracle_pins.py). */
#define ORC_MAX_THREADS 256
int orc_estimate_mt(const float *x, int ndims, const int64_t *dims, int eb_mode,
                    double eb, const int32_t *stride, double sz_offset,
                    orc_result *out, orc_debug *dbg, int nthreads);
uint64_t orc_processed_blocks(int ndims, const int64_t *dims, const int32_t *stride);

/* ---- the paper-literal estimator (Alg. 1 lines 3-10 as printed) ----
 * ZFP: n_sb of 3 / 9 / 16 sampled coefficients per 1D / 2D / 3D block, linear
 * interpolation of n_sb over the block's sequency order, average = BR_zfp;
 * MSE_sp = mean over the sampled coefficients of (truncated error x block exponent
 * offset)^2, unit weights.  SZ: delta from PSNR_sp (Alg. 1 line 7, Eq.
 * psnr-pdf-linear P:403), the Lorenzo residuals of the processed blocks re-quantised at
 * bin width delta, BR_sz = entropy (Eq. bitrate-sz) + offset + 32 p_ovf. */
typedef struct {
  double zfp_nsb_bits;    /* n_sb average: nsb2_total / 2 / n_values                       */
  double zfp_mse_sp;      /* sum of sampled squared errors / n_samples                      */
  double zfp_psnr_sp;     /* 20 log10 VR - 10 log10 MSE_sp; +INF if MSE_sp == 0             */
  double sz_delta;        /* sqrt(12 MSE_sp) (= VR sqrt(12) 10^(-PSNR_sp/20)); 2 eb_abs if   */
                          /* MSE_sp == 0 (matched = 0)                                      */
  double sz_bits;         /* H(delta) + offset + 32 p_ovf                                    */
  double sz_entropy;
  double sz_overflow_frac;
  double value_range, eb_abs;
  uint64_t nsb2_total;    /* 2 x sum of the interpolated n_sb (an exact integer)            */
  uint64_t n_samples;     /* sampled coefficients = m x processed blocks                    */
  uint64_t n_values;      /* real values in processed blocks                                */
  uint64_t hist_total, hist_ovf;
  float r_star;           /* float(1 / delta), the quantiser scale of the SZ re-quantisation */
  int32_t choice;         /* 0 = SZ iff sz_bits < zfp_nsb_bits (Alg. 1 line 10)              */
  int32_t matched;
  int32_t status;
} orc_paper_result;
int orc_estimate_paper(const float *x, int ndims, const int64_t *dims, int eb_mode, double eb,
                       const int32_t *stride, double sz_offset, orc_paper_result *out);
/* the sampled sequency positions j_i = round(i (4^d - 1) / (m - 1)), i < m */
int orc_paper_positions(int ndims, int32_t *pos);
/* one block: 2 x sum of the linearly interpolated n_sb and the sum of the sampled squared
 * errors (value units), from the sequency-ordered negabinary words */
void orc_block_paper(const uint32_t *u_seq, int ndims, int kmin, int32_t emax, uint64_t *nsb2,
                     double *mse_num);

/* ---- Alg. 1 line 13, "perform ZFP compression on X_i with absolute
 * error bound eb" -- the fixed-accuracy stream whose per-block lengths the estimator counts
 * (P:436).  Per processed block, row-major: 1 bit 0 if the block is
 * empty or p = 0; else 1 bit 1, 8 bits emax + 127 (LSB first), then the group-testing
 * embedded code of planes 31..kmin (orc_gt_encode).  Bits are packed LSB first within
 * bytes.  Returns ORC_OK and the stream length in *nbits; ORC_EINVAL if cap_bytes is too
 * small (with *nbits = the length needed). */
int orc_zfp_stream(const float *x, int ndims, const int64_t *dims, int eb_mode, double eb,
                   const int32_t *stride, uint8_t *buf, uint64_t cap_bytes, uint64_t *nbits);
/* decode such a stream into the field (processed blocks only; other values untouched):
 * words -> negabinary inverse -> sequency inverse -> inverse lift -> x 2^(emax-30) */
int orc_zfp_stream_decode(const uint8_t *buf, uint64_t nbits, int ndims, const int64_t *dims, int eb_mode,
                          double eb, double value_range, const int32_t *stride, float *out);

/* ---- the variant quantisers of Section 5.1.4 evaluated with
 * the general Stage-II estimators -- BR = -sum_i P_i log2 P_i (Eq. bit-rate-pdf),
 * MSE = (1/12) sum_i delta_i^2 P_i (delta_i^3 P(m_i) = delta_i^2 P_i), PSNR =
 * 20 log10 VR - 10 log10 MSE (Eq. psnr-pdf) -- on the approximate PDF the
 * selector stores: the n_pdf = 65,535-bin code histogram, cell q = [(q - 1/2)
 * delta, (q + 1/2) delta), delta = 2 eb_abs, mass c_q / N_in, uniform inside a cell
 * (reading R21; codes in the overflow slot lie outside the PDF's support).
 *  linear: the bins are the cells; BR = the entropy of the in-range codes,
 *    PSNR = Eq. psnr-pdf-linear.
 *  log-scale, integer base b >= 2: bin(q) = n + sign(q) floor(log_b |q|), the
 *    central bin n holds |q| < b (width 2b - 1 cells; printed delta_n = 2b on the
 *    continuum), bin n +- i holds b^i <= |q| < b^(i+1) (width b^(i+1) - b^i cells).
 *  equal-probability, 2n - 1 bins: edges at the quantiles k / (2n - 1) of the
 *    piecewise-linear CDF, s_0 / s_(2n-1) = the outer edges of the lowest / highest
 *    occupied cell; BR = 1 + log2 n as printed, MSE from the general equation with
 *    P_i = 1 / (2n - 1) (no K-means: P:428 calls it expensive, SURVEY A21 rules it out). */
typedef struct {
  double lin_bits, lin_psnr;
  double log_bits, log_psnr, log_mse;
  double eqp_bits, eqp_psnr, eqp_mse;
  double eqp_width_sum;        /* sum_k delta_k in cells = (highest - lowest occupied cell) + 1 */
  double value_range, eb_abs;
  uint64_t n_in;               /* in-range codes (the PDF's mass)                             */
  uint64_t hist_ovf;
  int32_t log_base, log_bins;  /* occupied log-scale bins                                     */
  int32_t eqp_n;
  int32_t status;
} orc_variant_result;
int orc_variants_from_hist(const uint64_t *hist, double value_range, double eb_abs, int log_base,
                           int eqp_n, orc_variant_result *out);
int orc_estimate_variants(const float *x, int ndims, const int64_t *dims, int eb_mode, double eb,
                          const int32_t *stride, int log_base, int eqp_n, orc_variant_result *out);

/* ---- single steps, exported for the pin tests ---- */
float orc_lorenzo(const float *x, int ndims, const int64_t *dims, const int64_t *idx);
int32_t orc_quantize(float d, float r_f);
double orc_entropy_counts(const uint64_t *c, int64_t n);
void orc_fwd_lift4(int32_t *v, int64_t stride);
void orc_inv_lift4(int32_t *v, int64_t stride);
void orc_fwd_xform(int32_t *blk, int ndims);
void orc_inv_xform(int32_t *blk, int ndims);
void orc_sequency_perm(int ndims, int32_t *perm);
uint32_t orc_negabinary(int32_t c);
int32_t orc_negabinary_inv(uint32_t u);
int32_t orc_block_emax(const float *blk, int n);
void orc_block_bfp(const float *blk, int n, int32_t emax, int32_t *out);
int32_t orc_precision(int32_t emax, int32_t minexp, int ndims);
uint64_t orc_gt_count(const uint32_t *u, int n, int kmin);
uint64_t orc_gt_encode(const uint32_t *u, int n, int kmin, uint8_t *buf, uint64_t cap_bits);
uint64_t orc_gt_decode(const uint8_t *buf, uint64_t nbits, int n, int kmin, uint32_t *u);
double orc_block_err(const int32_t *coef_nat, const uint32_t *u_seq, const int32_t *perm,
                     int ndims, int kmin, int32_t emax);
double orc_gain(int ndims, int nat_index);
/* selection based on the error bound: 0 = SZ iff its ratio is higher */
int orc_select_eb(double br_sz, double br_zfp);
int orc_select(double br_sz, double psnr_sz, double br_zfp, double psnr_zfp,
               double vr, double eb_abs, double zfp_mse, double *br_sz_matched,
               double *eb_sz_matched, int32_t *matched);
#endif
