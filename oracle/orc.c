/*
 * orc.c -- plain sequential CPU ORACLE (test infrastructure only; see orc.h).
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -fPIC -shared
 *        (x86-64 SSE: float arithmetic is evaluated in float, FLT_EVAL_METHOD 0).
 * No blocking, fusion or reordering beyond what each cited definition states.
 * Readings R1..R17 are listed in DESIGN.md section 3.
 */
#include "orc.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ */
/* small helpers                                                        */
/* ------------------------------------------------------------------ */
static int64_t ipow4(int d) { int64_t r = 1; while (d-- > 0) r *= 4; return r; }

/* floor(v / 2) for a signed integer, written out (the lifting network's ">>1"). */
static int64_t floor_half(int64_t v) { return (v >= 0) ? v / 2 : -((1 - v) / 2); }

/* value of x at multi-index idx; 0 outside the field (R4: zero boundary). */
static float at_or_zero(const float *x, int nd, const int64_t *dims, const int64_t *idx) {
  int64_t lin = 0;
  for (int a = 0; a < nd; ++a) {
    if (idx[a] < 0 || idx[a] >= dims[a]) return 0.0f;
    lin = lin * dims[a] + idx[a];
  }
  return x[lin];
}

/* ------------------------------------------------------------------ */
/* A4  Lorenzo residual on ORIGINAL values (P:151 footnote)     */
/*     nested first differences in fp32 (reading R4)                   */
/* ------------------------------------------------------------------ */
float orc_lorenzo(const float *x, int nd, const int64_t *dims, const int64_t *idx) {
  int64_t t[3];
  if (nd == 1) {
    t[0] = idx[0];     float x0 = at_or_zero(x, nd, dims, t);
    t[0] = idx[0] - 1; float x1 = at_or_zero(x, nd, dims, t);
    return x0 - x1;
  }
  if (nd == 2) {
    float v[2][2]; /* v[di][dj] = x[i-di][j-dj] */
    for (int di = 0; di < 2; ++di)
      for (int dj = 0; dj < 2; ++dj) {
        t[0] = idx[0] - di; t[1] = idx[1] - dj;
        v[di][dj] = at_or_zero(x, nd, dims, t);
      }
    float r0 = v[0][0] - v[0][1];
    float r1 = v[1][0] - v[1][1];
    return r0 - r1;
  }
  float v[2][2][2];
  for (int di = 0; di < 2; ++di)
    for (int dj = 0; dj < 2; ++dj)
      for (int dk = 0; dk < 2; ++dk) {
        t[0] = idx[0] - di; t[1] = idx[1] - dj; t[2] = idx[2] - dk;
        v[di][dj][dk] = at_or_zero(x, nd, dims, t);
      }
  float a = v[0][0][0] - v[0][0][1];
  float b = v[0][1][0] - v[0][1][1];
  float c = v[1][0][0] - v[1][0][1];
  float e = v[1][1][0] - v[1][1][1];
  return (a - b) - (c - e);
}

/* ------------------------------------------------------------------ */
/* A5  linear quantisation, bin width 2*eb, 65,535 bins     */
/*     (P:637); overflow -> slot 65535 (reading R5)                     */
/* ------------------------------------------------------------------ */
int32_t orc_quantize(float d, float r_f) {
  float q = fabsf(d) * r_f;
  if (!(q < 32767.5f)) return ORC_OVF_SLOT;
  int32_t m = (int32_t)lrintf(q); /* round half to even (default FE_TONEAREST) */
  int32_t code = (d < 0.0f) ? -m : m;
  return code + 32767;
}

/* ------------------------------------------------------------------ */
/* A6  Shannon entropy of bin probabilities, Eq. (entropy)   */
/*     BR = - sum_i P_i log2 P_i,  P_i = c_i / N                        */
/* ------------------------------------------------------------------ */
double orc_entropy_counts(const uint64_t *c, int64_t n) {
  uint64_t tot = 0;
  for (int64_t i = 0; i < n; ++i) tot += c[i];
  if (tot == 0) return 0.0;
  double H = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    if (c[i] == 0) continue;
    double p = (double)c[i] / (double)tot;
    H -= p * log2(p);
  }
  return H;
}

/* ------------------------------------------------------------------ */
/* A8  ZFP forward decorrelating lift on one 4-vector (reading R8).    */
/*     Exact-arithmetic map = A = (1/16)[[4,4,4,4],[5,1,-1,-5],         */
/*     [-4,4,4,-4],[-2,6,-6,2]]; ">>1" is floor(v/2).                   */
/* ------------------------------------------------------------------ */
void orc_fwd_lift4(int32_t *p, int64_t s) {
  int64_t x = p[0], y = p[s], z = p[2 * s], w = p[3 * s];
  /* stage 1: x <- (x+w)/2, w <- w - x */
  x = floor_half(x + w); w = w - x;
  /* stage 2: z <- (z+y)/2, y <- y - z */
  z = floor_half(z + y); y = y - z;
  /* stage 3: x <- (x+z)/2, z <- z - x */
  x = floor_half(x + z); z = z - x;
  /* stage 4: w <- (w+y)/2, y <- y - w */
  w = floor_half(w + y); y = y - w;
  /* stage 5: w <- w + y/2, y <- y - w/2 */
  w = w + floor_half(y); y = y - floor_half(w);
  p[0] = (int32_t)x; p[s] = (int32_t)y; p[2 * s] = (int32_t)z; p[3 * s] = (int32_t)w;
}

/* inverse network: the five stages undone in reverse order (linear part A^-1) */
void orc_inv_lift4(int32_t *p, int64_t s) {
  int64_t x = p[0], y = p[s], z = p[2 * s], w = p[3 * s];
  y = y + floor_half(w); w = w - floor_half(y);   /* undo stage 5 */
  y = y + w; w = 2 * w; w = w - y;                /* undo stage 4 */
  z = z + x; x = 2 * x; x = x - z;                /* undo stage 3 */
  y = y + z; z = 2 * z; z = z - y;                /* undo stage 2 */
  w = w + x; x = 2 * x; x = x - w;                /* undo stage 1 */
  p[0] = (int32_t)x; p[s] = (int32_t)y; p[2 * s] = (int32_t)z; p[3 * s] = (int32_t)w;
}

/* separable application, fastest axis first (P:218-233 unfold/fold along each
 * axis; ZFP order x -> y -> z, reading R8).  blk is 4^d int32 row-major. */
void orc_fwd_xform(int32_t *blk, int nd) {
  int64_t size = ipow4(nd);
  for (int a = nd - 1; a >= 0; --a) {
    int64_t s = ipow4(nd - 1 - a); /* stride of axis a */
    for (int64_t n = 0; n < size; ++n) {
      if ((n / s) % 4 != 0) continue; /* line start: coordinate along a == 0 */
      orc_fwd_lift4(blk + n, s);
    }
  }
}

void orc_inv_xform(int32_t *blk, int nd) {
  int64_t size = ipow4(nd);
  for (int a = 0; a < nd; ++a) {
    int64_t s = ipow4(nd - 1 - a);
    for (int64_t n = 0; n < size; ++n) {
      if ((n / s) % 4 != 0) continue;
      orc_inv_lift4(blk + n, s);
    }
  }
}

/* ------------------------------------------------------------------ */
/* A10 total-sequency order: sort multi-indices by (sum i, sum i^2, n)  */
/*     (reading R10; low frequencies first, the "staircase" P:436)      */
/* ------------------------------------------------------------------ */
void orc_sequency_perm(int nd, int32_t *perm) {
  int size = (int)ipow4(nd);
  int key1[64], key2[64];
  for (int n = 0; n < size; ++n) {
    int s1 = 0, s2 = 0, r = n;
    for (int a = 0; a < nd; ++a) { int i = r % 4; r /= 4; s1 += i; s2 += i * i; }
    key1[n] = s1; key2[n] = s2; perm[n] = n;
  }
  for (int i = 1; i < size; ++i) { /* insertion sort, stable on n */
    int32_t v = perm[i]; int j = i - 1;
    while (j >= 0) {
      int32_t u = perm[j];
      int gt = key1[u] > key1[v] || (key1[u] == key1[v] && (key2[u] > key2[v] ||
               (key2[u] == key2[v] && u > v)));
      if (!gt) break;
      perm[j + 1] = u; --j;
    }
    perm[j + 1] = v;
  }
}

/* ------------------------------------------------------------------ */
/* A11 negabinary (reading R11):  u = (c + 0xAAAAAAAA) xor 0xAAAAAAAA   */
/* ------------------------------------------------------------------ */
uint32_t orc_negabinary(int32_t c) {
  return ((uint32_t)c + 0xAAAAAAAAu) ^ 0xAAAAAAAAu;
}
int32_t orc_negabinary_inv(uint32_t u) {
  return (int32_t)((u ^ 0xAAAAAAAAu) - 0xAAAAAAAAu);
}

/* ------------------------------------------------------------------ */
/* A9  block exponent ("alignment of exponent"): max frexp        */
/*     exponent over nonzero values, clamped >= -126; -127 if empty     */
/* ------------------------------------------------------------------ */
int32_t orc_block_emax(const float *blk, int n) {
  int any = 0, emax = -1000;
  for (int i = 0; i < n; ++i) {
    if (blk[i] == 0.0f) continue;
    int e; frexpf(blk[i], &e);
    if (!any || e > emax) emax = e;
    any = 1;
  }
  if (!any) return -127;
  return emax < -126 ? -126 : emax;
}

/* "fixed-point integer conversion": i = trunc(x * 2^(30-emax)), exact */
void orc_block_bfp(const float *blk, int n, int32_t emax, int32_t *out) {
  for (int i = 0; i < n; ++i)
    out[i] = (int32_t)trunc(ldexp((double)blk[i], 30 - emax));
}

/* A12 fixed-accuracy precision (reading R12; ZFP-0.5 fixed accuracy P:507) */
int32_t orc_precision(int32_t emax, int32_t minexp, int nd) {
  int64_t p = (int64_t)emax - minexp + 2 * (nd + 1);
  if (p < 0) p = 0;
  if (p > 32) p = 32;
  return (int32_t)p;
}

/* ------------------------------------------------------------------ */
/* A13 group-testing embedded coder (EC; reading R13),    */
/*     simulated literally: planes 31..kmin, n carried across planes.   */
/* ------------------------------------------------------------------ */
static int plane_bit(const uint32_t *u, int j, int k) { return (int)((u[j] >> k) & 1u); }

uint64_t orc_gt_count(const uint32_t *u, int size, int kmin) {
  uint64_t bits = 0;
  int n = 0;
  for (int k = 31; k >= kmin; --k) {
    bits += (uint64_t)n;                       /* (i) verbatim bits of 0..n-1 */
    while (n < size) {                         /* (ii) group tests            */
      int any = 0;
      for (int j = n; j < size; ++j) any |= plane_bit(u, j, k);
      bits += 1;
      if (!any) break;
      for (;;) {
        if (n == size - 1) { n = size; break; }  /* last 1 implied */
        bits += 1;
        int b = plane_bit(u, n, k);
        ++n;
        if (b) break;
      }
    }
  }
  return bits;
}

static void put_bit(uint8_t *buf, uint64_t pos, int b) {
  if (b) buf[pos >> 3] |= (uint8_t)(1u << (pos & 7));
  else buf[pos >> 3] &= (uint8_t)~(1u << (pos & 7));
}
static int get_bit(const uint8_t *buf, uint64_t pos) { return (buf[pos >> 3] >> (pos & 7)) & 1; }

/* actually write the EC bitstream; returns its length in bits (0 on overflow) */
uint64_t orc_gt_encode(const uint32_t *u, int size, int kmin, uint8_t *buf, uint64_t cap) {
  uint64_t pos = 0;
  int n = 0;
#define PUT(b) do { if (pos >= cap) return 0; put_bit(buf, pos++, (b)); } while (0)
  for (int k = 31; k >= kmin; --k) {
    for (int j = 0; j < n; ++j) PUT(plane_bit(u, j, k));
    while (n < size) {
      int any = 0;
      for (int j = n; j < size; ++j) any |= plane_bit(u, j, k);
      PUT(any);
      if (!any) break;
      for (;;) {
        if (n == size - 1) { n = size; break; }
        int b = plane_bit(u, n, k);
        PUT(b);
        ++n;
        if (b) break;
      }
    }
  }
#undef PUT
  return pos;
}

/* decode the stream back into words (bits below kmin are zero); returns bits read */
uint64_t orc_gt_decode(const uint8_t *buf, uint64_t nbits, int size, int kmin, uint32_t *u) {
  uint64_t pos = 0;
  int n = 0;
  for (int j = 0; j < size; ++j) u[j] = 0;
#define GET() ((pos < nbits) ? get_bit(buf, pos++) : (pos++, 0))
  for (int k = 31; k >= kmin; --k) {
    for (int j = 0; j < n; ++j) if (GET()) u[j] |= 1u << k;
    while (n < size) {
      if (!GET()) break;
      for (;;) {
        if (n == size - 1) { u[n] |= 1u << k; n = size; break; }
        int b = GET();
        if (b) u[n] |= 1u << k;
        ++n;
        if (b) break;
      }
    }
  }
#undef GET
  return pos;
}

/* ------------------------------------------------------------------ */
/* A14 truncation error weighted by the squared column norms of the     */
/*     inverse transform (reading R14, Theorem thm:1 P:275)  */
/* ------------------------------------------------------------------ */
double orc_gain(int nd, int n) {
  static const double g[4] = {4.0, 5.0, 4.0, 3.25};
  double w = 1.0;
  for (int a = 0; a < nd; ++a) { w *= g[n % 4]; n /= 4; }
  return w;
}

double orc_block_err(const int32_t *coef_nat, const uint32_t *u_seq, const int32_t *perm,
                     int nd, int kmin, int32_t emax) {
  int size = (int)ipow4(nd);
  double E = 0.0;
  for (int j = 0; j < size; ++j) {
    uint32_t ut = (kmin >= 32) ? 0u : (u_seq[j] & ~((1u << kmin) - 1u));
    int32_t ct = orc_negabinary_inv(ut);
    int64_t e = (int64_t)coef_nat[perm[j]] - (int64_t)ct;
    double ed = (double)e;
    E += orc_gain(nd, perm[j]) * (ed * ed);
  }
  return E * ldexp(1.0, 2 * (emax - 30));
}

/* ------------------------------------------------------------------ */
/* The comparison selector of P:639-642 (Lu et al., "selection based on  */
/* error bound"): "simply selects the compressor with the highest        */
/* compression ratio based on a fixed error bound" -- the lower bit-rate */
/* at the user's eb (ratio = 32 / bit-rate for float32); ties -> ZFP as  */
/* in Alg. 1's ELSE (reading; the paper does not discuss ties).          */
/* ------------------------------------------------------------------ */
int orc_select_eb(double br_sz, double br_zfp) {
  double ratio_sz = 32.0 / br_sz, ratio_zfp = 32.0 / br_zfp;
  return (ratio_sz > ratio_zfp) ? 0 : 1;
}

/* ------------------------------------------------------------------ */
/* A16 selection, Alg. 1 lines 7-10, ties -> ZFP            */
/* ------------------------------------------------------------------ */
int orc_select(double br_sz, double psnr_sz, double br_zfp, double psnr_zfp,
               double vr, double eb_abs, double zfp_mse, double *bm, double *ebm,
               int32_t *matched) {
  (void)psnr_sz;
  if (!(zfp_mse > 0.0) || !(vr > 0.0) || !isfinite(psnr_zfp)) {
    /* reading R16(ii): matching impossible -> compare at the user's eb */
    *matched = 0; *bm = br_sz; *ebm = eb_abs;
    return (br_sz < br_zfp) ? 0 : 1;
  }
  /* line 7: delta from PSNR_sz = PSNR_zfp with Eq. (psnr-pdf-linear) */
  double delta = vr * sqrt(12.0) * pow(10.0, -psnr_zfp / 20.0);
  /* lines 8-9: Eq. (bitrate-sz) evaluated with the 2eb-histogram density
   * (reading R16(i)):  BR(delta) = BR(2eb) + log2(2eb / delta) */
  double b = br_sz + log2(2.0 * eb_abs / delta);
  if (b < 0.0) b = 0.0;
  *matched = 1; *bm = b; *ebm = delta / 2.0;
  return (b < br_zfp) ? 0 : 1;   /* line 10: IF BR_sz < BR_zfp -> SZ */
}

/* ------------------------------------------------------------------ */
/* A3 block sampling: block b processed iff b_a % s_a == 0  */
/* ------------------------------------------------------------------ */
uint64_t orc_processed_blocks(int nd, const int64_t *dims, const int32_t *stride) {
  uint64_t r = 1;
  for (int a = 0; a < nd; ++a) {
    int64_t nb = (dims[a] + 3) / 4;
    int64_t s = stride ? stride[a] : 1;
    r *= (uint64_t)((nb + s - 1) / s);
  }
  return r;
}

/* ------------------------------------------------------------------ */
/* whole field: Alg. 1 lines 1-10                                       */
/*                                                                      */
/* The loop bodies below are the plain per-point / per-block steps.     */
/* orc_estimate_mt splits the block grid into contiguous slabs of the   */
/* slowest block axis, one per thread (the paper's one-process-per-     */
/* field model, applied within a field); every merge is exact:   */
/* integer histogram / count sums, and the per-block E_b are stored by  */
/* processed-block ordinal and summed in that order after the join, so  */
/* the result is bit-identical to nthreads = 1.                         */
/* ------------------------------------------------------------------ */
typedef struct {
  /* inputs */
  const float *x;
  int nd;
  const int64_t *dims;
  int64_t nb[3];
  int32_t s[3];
  int size;
  const int32_t *perm;
  float r_f;
  int32_t minexp;
  orc_debug *dbg;
  double *E;          /* [processed blocks] E_b by processed-block ordinal */
  uint32_t *bitsv;    /* [processed blocks] bits_b */
  /* slab of the slowest block axis */
  int64_t b0_lo, b0_hi;
  /* value-range part: element range */
  int64_t i_lo, i_hi;
  float vmin, vmax;
  int bad;
  /* outputs */
  uint64_t *hist;
  uint64_t n_sz, n_values, n_blocks;
} orc_work;

/* A1 over x[i_lo, i_hi): min, max, non-finite flag */
static void work_range(orc_work *w) {
  w->bad = 0;
  w->vmin = w->x[w->i_lo];
  w->vmax = w->x[w->i_lo];
  for (int64_t i = w->i_lo; i < w->i_hi; ++i) {
    float v = w->x[i];
    if (!isfinite(v)) { w->bad = 1; continue; }
    if (v < w->vmin) w->vmin = v;
    if (v > w->vmax) w->vmax = v;
  }
}

/* A3-A14 for the processed blocks with b0 in [b0_lo, b0_hi), row-major */
static void work_blocks(orc_work *w) {
  const int nd = w->nd, size = w->size;
  const int64_t *dims = w->dims;
  const int64_t *nb = w->nb;
  const int32_t *s = w->s;
  /* processed-block ordinal of the first block of the slab */
  int64_t npb12 = ((nb[1] + s[1] - 1) / s[1]) * ((nb[2] + s[2] - 1) / s[2]);
  int64_t pb = ((w->b0_lo + s[0] - 1) / s[0]) * npb12;
  int64_t b[3];
  for (int64_t lb = w->b0_lo * nb[1] * nb[2]; lb < w->b0_hi * nb[1] * nb[2]; ++lb) {
    /* block coordinates, row-major (axis 0 slowest) */
    int64_t r = lb;
    for (int a = nd - 1; a >= 0; --a) { b[a] = r % nb[a]; r /= nb[a]; }
    int processed = 1;
    for (int a = 0; a < nd; ++a) if (b[a] % s[a] != 0) processed = 0;
    if (!processed) continue;

    /* ---- SZ part: A4-A5 for every real point of the block ---- */
    float blk[64];
    int nreal = 0;
    for (int n = 0; n < size; ++n) {
      int64_t idx[3], cl[3];
      int inside = 1, rr = n;
      for (int a = nd - 1; a >= 0; --a) {
        int o = rr % 4; rr /= 4;
        idx[a] = 4 * b[a] + o;
        if (idx[a] >= dims[a]) inside = 0;
        cl[a] = idx[a] < dims[a] ? idx[a] : dims[a] - 1; /* edge replication (R17) */
      }
      int64_t lin = 0;
      for (int a = 0; a < nd; ++a) lin = lin * dims[a] + cl[a];
      blk[n] = w->x[lin];
      if (!inside) continue;
      ++nreal;
      int origin = 1;
      for (int a = 0; a < nd; ++a) if (idx[a] != 0) origin = 0;
      if (origin) continue; /* R4: the first value is stored verbatim */
      float d = orc_lorenzo(w->x, nd, dims, idx);
      int32_t slot = orc_quantize(d, w->r_f);
      w->hist[slot] += 1;
      ++w->n_sz;
      if (w->dbg && w->dbg->codes) w->dbg->codes[lin] = slot;
    }
    w->n_values += (uint64_t)nreal;
    ++w->n_blocks;

    /* ---- ZFP part: A9-A14 on the (padded) block ---- */
    int32_t emax = orc_block_emax(blk, size);
    int32_t coef[64];
    uint32_t u[64];
    uint64_t bits;
    double E;
    if (emax == -127) { /* empty block: 1 header bit, no error */
      for (int n = 0; n < size; ++n) { coef[n] = 0; u[n] = 0; }
      bits = 1; E = 0.0;
    } else {
      orc_block_bfp(blk, size, emax, coef);
      orc_fwd_xform(coef, nd);
      for (int j = 0; j < size; ++j) u[j] = orc_negabinary(coef[w->perm[j]]);
      int32_t p = orc_precision(emax, w->minexp, nd);
      int kmin = 32 - p;
      bits = (p == 0) ? 1 : 9 + orc_gt_count(u, size, kmin);
      E = orc_block_err(coef, u, w->perm, nd, kmin, emax);
    }
    w->E[pb] = E;
    w->bitsv[pb] = (uint32_t)bits;
    if (w->dbg) {
      if (w->dbg->emax) w->dbg->emax[pb] = emax;
      if (w->dbg->coef) memcpy(w->dbg->coef + pb * size, coef, sizeof(int32_t) * size);
      if (w->dbg->uword) memcpy(w->dbg->uword + pb * size, u, sizeof(uint32_t) * size);
      if (w->dbg->bits) w->dbg->bits[pb] = (uint32_t)bits;
      if (w->dbg->err) w->dbg->err[pb] = E;
    }
    ++pb;
  }
}

static void *work_range_thread(void *p) { work_range((orc_work *)p); return NULL; }
static void *work_blocks_thread(void *p) { work_blocks((orc_work *)p); return NULL; }

/* run fn over w[0..n) on n threads (w[0] on the caller's thread) */
static void run_threads(orc_work *w, int n, void *(*fn)(void *)) {
  pthread_t th[ORC_MAX_THREADS];
  int started[ORC_MAX_THREADS];
  for (int t = 1; t < n; ++t) started[t] = pthread_create(&th[t], NULL, fn, &w[t]) == 0;
  fn(&w[0]);
  for (int t = 1; t < n; ++t) {
    if (started[t]) pthread_join(th[t], NULL);
    else fn(&w[t]);   /* could not start a thread: run it here (same result) */
  }
}

int orc_estimate_mt(const float *x, int nd, const int64_t *dims, int eb_mode, double eb,
                    const int32_t *stride, double sz_offset, orc_result *out, orc_debug *dbg,
                    int nthreads) {
  if (nd < 1 || nd > 3 || !x || !dims || !out) return ORC_EINVAL;
  int64_t N = 1;
  for (int a = 0; a < nd; ++a) { if (dims[a] < 1) return ORC_EINVAL; N *= dims[a]; }
  int32_t s[3] = {1, 1, 1};
  for (int a = 0; a < nd; ++a) { s[a] = stride ? stride[a] : 1; if (s[a] < 1) return ORC_EINVAL; }
  if (!isfinite(eb) || !(eb > 0.0)) return ORC_EINVAL;
  if (eb_mode != 0 && eb_mode != 1) return ORC_EINVAL;
  if (nthreads < 1) nthreads = 1;
  if (nthreads > ORC_MAX_THREADS) nthreads = ORC_MAX_THREADS;

  int64_t nb[3] = {1, 1, 1};
  for (int a = 0; a < nd; ++a) nb[a] = (dims[a] + 3) / 4;
  int nt = nthreads;
  if (nt > nb[0]) nt = (int)nb[0];
  if ((int64_t)nt > N) nt = (int)N;
  orc_work w[ORC_MAX_THREADS];
  memset(w, 0, sizeof(w));

  /* A1: value range over the whole field */
  for (int t = 0; t < nt; ++t) {
    w[t].x = x;
    w[t].i_lo = N * t / nt;
    w[t].i_hi = N * (t + 1) / nt;
  }
  run_threads(w, nt, work_range_thread);
  float vmin = w[0].vmin, vmax = w[0].vmax;
  for (int t = 0; t < nt; ++t) {
    if (w[t].bad) return ORC_ENONFINITE;
    if (w[t].vmin < vmin) vmin = w[t].vmin;
    if (w[t].vmax > vmax) vmax = w[t].vmax;
  }
  double VR = (double)vmax - (double)vmin;

  /* A2: error bound (Alg. 1 line 2) and derived scalars */
  double eb_abs = (eb_mode == 1) ? eb * VR : eb;
  if (eb_mode == 1 && VR == 0.0) return ORC_EDEGENERATE;
  float r_f = (float)(1.0 / (2.0 * eb_abs));
  if (!isfinite(r_f) || !(eb_abs > 0.0)) return ORC_EINVAL;
  int fe; frexp(eb_abs, &fe);
  int32_t minexp = fe - 1; /* floor(log2 eb_abs) */

  int size = (int)ipow4(nd);
  int32_t perm[64];
  orc_sequency_perm(nd, perm);
  uint64_t npb = orc_processed_blocks(nd, dims, stride);

  int rc = ORC_OK;
  uint64_t *hist = (uint64_t *)calloc((size_t)ORC_NSLOTS * nt, sizeof(uint64_t));
  double *E = (double *)malloc(sizeof(double) * (npb ? npb : 1));
  uint32_t *bitsv = (uint32_t *)malloc(sizeof(uint32_t) * (npb ? npb : 1));
  if (!hist || !E || !bitsv) { rc = ORC_EINVAL; goto done; }
  if (dbg && dbg->codes) for (int64_t i = 0; i < N; ++i) dbg->codes[i] = -1;

  for (int t = 0; t < nt; ++t) {
    w[t].nd = nd; w[t].dims = dims; w[t].size = size; w[t].perm = perm;
    for (int a = 0; a < 3; ++a) { w[t].nb[a] = nb[a]; w[t].s[a] = s[a]; }
    w[t].r_f = r_f; w[t].minexp = minexp; w[t].dbg = dbg; w[t].E = E; w[t].bitsv = bitsv;
    w[t].b0_lo = nb[0] * t / nt;
    w[t].b0_hi = nb[0] * (t + 1) / nt;
    w[t].hist = hist + (size_t)ORC_NSLOTS * t;
  }
  run_threads(w, nt, work_blocks_thread);

  /* exact merges: integer sums; E_b and bits_b in processed-block order */
  uint64_t n_sz = 0, n_values = 0, n_blocks = 0, total_bits = 0;
  for (int t = 0; t < nt; ++t) {
    n_sz += w[t].n_sz; n_values += w[t].n_values; n_blocks += w[t].n_blocks;
    if (t > 0)
      for (int k = 0; k < ORC_NSLOTS; ++k) hist[k] += w[t].hist[k];
  }
  double err_sum = 0.0;
  for (uint64_t pb = 0; pb < npb; ++pb) { total_bits += bitsv[pb]; err_sum += E[pb]; }

  if (n_sz == 0) { rc = ORC_EDEGENERATE; goto done; }
  {
    /* A6: entropy bit-rate (Eq. entropy, bitrate-sz P:402), +0.5 offset */
    double H = orc_entropy_counts(hist, ORC_NSLOTS);
    double p_ovf = (double)hist[ORC_OVF_SLOT] / (double)n_sz;
    double br_sz = H + sz_offset + 32.0 * p_ovf;
    /* A7: Eq. (psnr-sz) */
    double psnr_sz = 20.0 * log10(VR / eb_abs) + 10.0 * log10(3.0);
    /* A13/A15: EC bit-rate; A14 PSNR_sp */
    double br_zfp = (double)total_bits / (double)n_values;
    double mse = err_sum / (double)n_values;
    double psnr_zfp = (mse > 0.0) ? 20.0 * log10(VR) - 10.0 * log10(mse) : INFINITY;

    memset(out, 0, sizeof(*out));
    out->sz_bits_per_value = br_sz;
    out->sz_psnr = psnr_sz;
    out->zfp_bits_per_value = br_zfp;
    out->zfp_psnr = psnr_zfp;
    out->value_range = VR;
    out->eb_abs = eb_abs;
    out->sz_entropy = H;
    out->sz_overflow_frac = p_ovf;
    out->zfp_mse = mse;
    out->n_sz_points = n_sz;
    out->n_values = n_values;
    out->n_blocks = n_blocks;
    out->zfp_total_bits = total_bits;
    out->zfp_err_sum = err_sum;
    out->minexp = minexp;
    out->r_f = r_f;
    out->choice = orc_select(br_sz, psnr_sz, br_zfp, psnr_zfp, VR, eb_abs, mse,
                             &out->sz_bits_matched, &out->sz_eb_matched, &out->matched);
    out->choice_eb = orc_select_eb(br_sz, br_zfp);
    uint64_t tot = 0;
    for (int k = 0; k < ORC_NSLOTS; ++k) tot += hist[k];
    out->hist_total = tot;
    out->hist_ovf = hist[ORC_OVF_SLOT];
    if (dbg && dbg->hist) memcpy(dbg->hist, hist, sizeof(uint64_t) * ORC_NSLOTS);
  }
done:
  free(hist);
  free(E);
  free(bitsv);
  return rc;
}

int orc_estimate(const float *x, int nd, const int64_t *dims, int eb_mode, double eb,
                 const int32_t *stride, double sz_offset, orc_result *out, orc_debug *dbg) {
  return orc_estimate_mt(x, nd, dims, eb_mode, eb, stride, sz_offset, out, dbg, 1);
}

/* ------------------------------------------------------------------ */
/* the paper-literal estimator                         */
/* ------------------------------------------------------------------ */
/* "we sample 3 data points for one 1D data block, 9 data points for one 4x4 2D data
 * block, and 16 data points for one 3D 4x4x4 data block".  Which points the paper's
 * figure marks is not recoverable (figure missing); reading R19: evenly spaced
 * over the sequency order, first and last included, j_i = round(i (4^d-1) / (m-1)),
 * rounding halves up. */
int orc_paper_positions(int nd, int32_t *pos) {
  const int m = nd == 1 ? 3 : (nd == 2 ? 9 : 16);
  const int L = (int)ipow4(nd) - 1;
  for (int i = 0; i < m; ++i) pos[i] = (2 * i * L + (m - 1)) / (2 * (m - 1));
  return m;
}

/* number of significant bits of a coefficient at the cut kmin: the bit planes from its
 * leading one down to kmin (n_sb = max(0, f - kmin + 1)) */
static int nsb_of(uint32_t u, int kmin) {
  int f = -1;
  for (int k = 31; k >= 0; --k) if ((u >> k) & 1u) { f = k; break; }
  return f >= kmin ? f - kmin + 1 : 0;
}

void orc_block_paper(const uint32_t *u, int nd, int kmin, int32_t emax, uint64_t *nsb2, double *mse_num) {
  int32_t pos[16];
  const int m = orc_paper_positions(nd, pos);
  int64_t n[16] = {0};
  for (int i = 0; i < m; ++i) n[i] = nsb_of(u[pos[i]], kmin);
  /* "use these sampled data points and their n_sb to interpolate n_sb for the remaining
   * data points": linear interpolation along the sequency order between the
   * neighbouring samples; the block's sum of interpolated values, doubled, is an integer:
   * sum over segment a of (len n_a + (n_{a+1} - n_a) t) / len, t = 0..len-1 */
  int64_t two_sum = 0;
  for (int a = 0; a + 1 < m; ++a) {
    const int64_t len = pos[a + 1] - pos[a];
    int64_t num = 0;                          /* sum_t (len n_a + (n_{a+1} - n_a) t) */
    for (int64_t t = 0; t < len; ++t) num += len * n[a] + (n[a + 1] - n[a]) * t;
    two_sum += 2 * num / len;                 /* exact: = 2 len n_a + (n_{a+1}-n_a)(len-1) */
  }
  two_sum += 2 * n[m - 1];                     /* the last position */
  *nsb2 = (uint64_t)two_sum;
  /* MSE_sp: "each sampled data point's error is calculated by multiplication of its
   * truncated error in binary representation and its block's exponent offset value"
   * (P:456): e = value of the dropped bit planes (< kmin) of the negabinary word,
   * times 2^(emax - 30), squared; unit weights (the paper's reading; R14 is ours) */
  double acc = 0.0;
  const double scale = ldexp(1.0, 2 * (emax - 30));
  for (int i = 0; i < m; ++i) {
    const uint32_t uj = u[pos[i]];
    const uint32_t low = kmin >= 32 ? 0xffffffffu : ((1u << kmin) - 1u);
    const int64_t c = (int64_t)orc_negabinary_inv(uj);
    const int64_t ct = (int64_t)orc_negabinary_inv(uj & ~low);    /* planes >= kmin kept */
    const double e = (double)(c - ct);
    acc += e * e * scale;
  }
  *mse_num = acc;
}

int orc_estimate_paper(const float *x, int nd, const int64_t *dims, int eb_mode, double eb,
                       const int32_t *stride, double sz_offset, orc_paper_result *out) {
  if (nd < 1 || nd > 3 || !x || !dims || !out) return ORC_EINVAL;
  int64_t N = 1;
  for (int a = 0; a < nd; ++a) { if (dims[a] < 1) return ORC_EINVAL; N *= dims[a]; }
  int32_t s[3] = {1, 1, 1};
  for (int a = 0; a < nd; ++a) { s[a] = stride ? stride[a] : 1; if (s[a] < 1) return ORC_EINVAL; }
  if (!isfinite(eb) || !(eb > 0.0) || (eb_mode != 0 && eb_mode != 1)) return ORC_EINVAL;
  /* Alg. 1 line 2: VR and eb */
  float vmin = x[0], vmax = x[0];
  for (int64_t i = 0; i < N; ++i) {
    if (!isfinite(x[i])) return ORC_ENONFINITE;
    if (x[i] < vmin) vmin = x[i];
    if (x[i] > vmax) vmax = x[i];
  }
  const double VR = (double)vmax - (double)vmin;
  const double eb_abs = (eb_mode == 1) ? eb * VR : eb;
  if (eb_mode == 1 && VR == 0.0) return ORC_EDEGENERATE;
  if (!isfinite((float)(1.0 / (2.0 * eb_abs))) || !(eb_abs > 0.0)) return ORC_EINVAL;
  int fe; frexp(eb_abs, &fe);
  const int32_t minexp = fe - 1;
  const int size = (int)ipow4(nd);
  int32_t perm[64], pos[16];
  orc_sequency_perm(nd, perm);
  const int m = orc_paper_positions(nd, pos);
  int64_t nb[3] = {1, 1, 1};
  for (int a = 0; a < nd; ++a) nb[a] = (dims[a] + 3) / 4;
  const int64_t nblocks_all = nb[0] * nb[1] * nb[2];
  /* Alg. 1 lines 3-6: blockwise sample, then the ZFP estimate of each block
   * from its sampled coefficients */
  uint64_t nsb2_total = 0, n_samples = 0, n_values = 0;
  double mse_sum = 0.0;
  for (int64_t lb = 0; lb < nblocks_all; ++lb) {
    int64_t b[3], r = lb;
    for (int a = nd - 1; a >= 0; --a) { b[a] = r % nb[a]; r /= nb[a]; }
    int processed = 1;
    for (int a = 0; a < nd; ++a) if (b[a] % s[a] != 0) processed = 0;
    if (!processed) continue;
    float blk[64];
    for (int n = 0; n < size; ++n) {
      int64_t idx[3], cl[3];
      int inside = 1, rr = n;
      for (int a = nd - 1; a >= 0; --a) {
        int o = rr % 4; rr /= 4;
        idx[a] = 4 * b[a] + o;
        if (idx[a] >= dims[a]) inside = 0;
        cl[a] = idx[a] < dims[a] ? idx[a] : dims[a] - 1;     /* edge replication (R17) */
      }
      int64_t lin = 0;
      for (int a = 0; a < nd; ++a) lin = lin * dims[a] + cl[a];
      blk[n] = x[lin];
      n_values += inside ? 1 : 0;
    }
    uint32_t u[64];
    int32_t emax = orc_block_emax(blk, size);
    int kmin = 32;
    if (emax == -127) {
      for (int j = 0; j < size; ++j) u[j] = 0;
      emax = -126;                                /* (no error, no significant bit) */
    } else {
      int32_t coef[64];
      orc_block_bfp(blk, size, emax, coef);
      orc_fwd_xform(coef, nd);
      for (int j = 0; j < size; ++j) u[j] = orc_negabinary(coef[perm[j]]);
      kmin = 32 - orc_precision(emax, minexp, nd);
    }
    uint64_t nsb2;
    double mn;
    orc_block_paper(u, nd, kmin, emax, &nsb2, &mn);
    nsb2_total += nsb2;
    mse_sum += mn;
    n_samples += (uint64_t)m;
  }
  memset(out, 0, sizeof(*out));
  out->value_range = VR;
  out->eb_abs = eb_abs;
  out->nsb2_total = nsb2_total;
  out->n_samples = n_samples;
  out->n_values = n_values;
  out->zfp_nsb_bits = (double)nsb2_total / 2.0 / (double)n_values;
  out->zfp_mse_sp = mse_sum / (double)n_samples;
  /* PSNR_sp = -10 log10 MSE_sp + 20 log10 VR */
  out->zfp_psnr_sp = out->zfp_mse_sp > 0.0 ? 20.0 * log10(VR) - 10.0 * log10(out->zfp_mse_sp) : INFINITY;
  /* Alg. 1 line 7: delta with PSNR_sz = PSNR_sp in Eq. psnr-pdf-linear:
   * delta = VR sqrt(12) 10^(-PSNR_sp/20) = sqrt(12 MSE_sp).  MSE_sp == 0 (or VR == 0):
   * no PSNR to match -- SZ at the user's bound (delta = 2 eb_abs), matched = 0 (R16 ii) */
  double delta = out->zfp_mse_sp > 0.0 && VR > 0.0 ? sqrt(12.0 * out->zfp_mse_sp) : 2.0 * eb_abs;
  float rs = (float)(1.0 / delta);
  out->matched = out->zfp_mse_sp > 0.0 && VR > 0.0 && isfinite(rs) ? 1 : 0;
  if (!out->matched) { delta = 2.0 * eb_abs; rs = (float)(1.0 / delta); }
  out->sz_delta = delta;
  out->r_star = rs;
  /* Alg. 1 lines 8-9: the residual density of the sampled blocks at bin width delta
   * (linear quantisation R5 with r = 1/delta), Eq. bitrate-sz = its entropy,
   * + offset + 32 p_ovf (R6) */
  uint64_t *hist = (uint64_t *)calloc(ORC_NSLOTS, sizeof(uint64_t));
  if (!hist) return ORC_EINVAL;
  uint64_t n_sz = 0;
  for (int64_t lb = 0; lb < nblocks_all; ++lb) {
    int64_t b[3], r = lb;
    for (int a = nd - 1; a >= 0; --a) { b[a] = r % nb[a]; r /= nb[a]; }
    int processed = 1;
    for (int a = 0; a < nd; ++a) if (b[a] % s[a] != 0) processed = 0;
    if (!processed) continue;
    for (int n = 0; n < size; ++n) {
      int64_t idx[3];
      int inside = 1, origin = 1, rr = n;
      for (int a = nd - 1; a >= 0; --a) {
        int o = rr % 4; rr /= 4;
        idx[a] = 4 * b[a] + o;
        if (idx[a] >= dims[a]) inside = 0;
        if (idx[a] != 0) origin = 0;
      }
      if (!inside || origin) continue;
      hist[orc_quantize(orc_lorenzo(x, nd, dims, idx), rs)] += 1;
      ++n_sz;
    }
  }
  int rc = ORC_OK;
  if (n_sz == 0) rc = ORC_EDEGENERATE;
  else {
    out->sz_entropy = orc_entropy_counts(hist, ORC_NSLOTS);
    out->sz_overflow_frac = (double)hist[ORC_OVF_SLOT] / (double)n_sz;
    out->sz_bits = out->sz_entropy + sz_offset + 32.0 * out->sz_overflow_frac;
    uint64_t tot = 0;
    for (int k = 0; k < ORC_NSLOTS; ++k) tot += hist[k];
    out->hist_total = tot;
    out->hist_ovf = hist[ORC_OVF_SLOT];
    /* Alg. 1 line 10: SZ iff BR_sz < BR_zfp, else ZFP */
    out->choice = out->sz_bits < out->zfp_nsb_bits ? 0 : 1;
  }
  out->status = rc;
  free(hist);
  return rc;
}

/* ------------------------------------------------------------------ */
/* the fixed-accuracy ZFP stream (Alg. 1 line 13)       */
/* ------------------------------------------------------------------ */
static void put_bits(uint8_t *buf, uint64_t *pos, uint64_t cap_bits, uint32_t v, int n) {
  for (int i = 0; i < n; ++i) {
    if (*pos < cap_bits) put_bit(buf, *pos, (int)((v >> i) & 1u));
    ++*pos;
  }
}

/* derived scalars of Alg. 1 line 2 (A1/A2) for the stream routines */
static int stream_setup(const float *x, int nd, const int64_t *dims, int eb_mode, double eb, double *VR,
                        int32_t *minexp) {
  int64_t N = 1;
  for (int a = 0; a < nd; ++a) { if (dims[a] < 1) return ORC_EINVAL; N *= dims[a]; }
  if (!isfinite(eb) || !(eb > 0.0) || (eb_mode != 0 && eb_mode != 1)) return ORC_EINVAL;
  if (x) {
    float vmin = x[0], vmax = x[0];
    for (int64_t i = 0; i < N; ++i) {
      if (!isfinite(x[i])) return ORC_ENONFINITE;
      if (x[i] < vmin) vmin = x[i];
      if (x[i] > vmax) vmax = x[i];
    }
    *VR = (double)vmax - (double)vmin;
  }
  const double eb_abs = eb_mode == 1 ? eb * *VR : eb;
  if (eb_mode == 1 && *VR == 0.0) return ORC_EDEGENERATE;
  if (!(eb_abs > 0.0)) return ORC_EINVAL;
  int fe; frexp(eb_abs, &fe);
  *minexp = fe - 1;
  return ORC_OK;
}

int orc_zfp_stream(const float *x, int nd, const int64_t *dims, int eb_mode, double eb,
                   const int32_t *stride, uint8_t *buf, uint64_t cap_bytes, uint64_t *nbits) {
  if (nd < 1 || nd > 3 || !x || !dims || !nbits) return ORC_EINVAL;
  double VR = 0.0;
  int32_t minexp = 0;
  int rc = stream_setup(x, nd, dims, eb_mode, eb, &VR, &minexp);
  if (rc) return rc;
  int32_t s[3] = {1, 1, 1};
  for (int a = 0; a < nd; ++a) s[a] = stride ? stride[a] : 1;
  const int size = (int)ipow4(nd);
  int32_t perm[64];
  orc_sequency_perm(nd, perm);
  int64_t nb[3] = {1, 1, 1};
  for (int a = 0; a < nd; ++a) nb[a] = (dims[a] + 3) / 4;
  const uint64_t cap_bits = buf ? cap_bytes * 8 : 0;
  if (buf) memset(buf, 0, cap_bytes);
  uint8_t ec[64 * 33 / 8 + 64];                 /* one block's EC bits (<= 32 x (64 + 1) bits) */
  uint64_t pos = 0;
  for (int64_t lb = 0; lb < nb[0] * nb[1] * nb[2]; ++lb) {
    int64_t b[3], r = lb;
    for (int a = nd - 1; a >= 0; --a) { b[a] = r % nb[a]; r /= nb[a]; }
    int processed = 1;
    for (int a = 0; a < nd; ++a) if (b[a] % s[a] != 0) processed = 0;
    if (!processed) continue;
    float blk[64];
    for (int n = 0; n < size; ++n) {
      int64_t cl[3];
      int rr = n;
      for (int a = nd - 1; a >= 0; --a) {
        const int64_t i = 4 * b[a] + rr % 4;
        rr /= 4;
        cl[a] = i < dims[a] ? i : dims[a] - 1;        /* edge replication (R17) */
      }
      int64_t lin = 0;
      for (int a = 0; a < nd; ++a) lin = lin * dims[a] + cl[a];
      blk[n] = x[lin];
    }
    const int32_t emax = orc_block_emax(blk, size);
    if (emax == -127) { put_bits(buf, &pos, cap_bits, 0u, 1); continue; }   /* empty block */
    int32_t coef[64];
    uint32_t u[64];
    orc_block_bfp(blk, size, emax, coef);
    orc_fwd_xform(coef, nd);
    for (int j = 0; j < size; ++j) u[j] = orc_negabinary(coef[perm[j]]);
    const int32_t p = orc_precision(emax, minexp, nd);
    if (p == 0) { put_bits(buf, &pos, cap_bits, 0u, 1); continue; }      /* nothing kept */
    put_bits(buf, &pos, cap_bits, 1u, 1);
    put_bits(buf, &pos, cap_bits, (uint32_t)(emax + 127), 8);
    memset(ec, 0, sizeof ec);
    const uint64_t n = orc_gt_encode(u, size, 32 - p, ec, sizeof(ec) * 8);
    for (uint64_t i = 0; i < n; ++i) {
      if (pos < cap_bits) put_bit(buf, pos, get_bit(ec, i));
      ++pos;
    }
  }
  *nbits = pos;
  return (buf && pos > cap_bits) ? ORC_EINVAL : ORC_OK;
}

int orc_zfp_stream_decode(const uint8_t *buf, uint64_t nbits, int nd, const int64_t *dims, int eb_mode,
                          double eb, double VR, const int32_t *stride, float *out) {
  if (nd < 1 || nd > 3 || !buf || !dims || !out) return ORC_EINVAL;
  int32_t minexp = 0;
  int rc = stream_setup(NULL, nd, dims, eb_mode, eb, &VR, &minexp);
  if (rc) return rc;
  int32_t s[3] = {1, 1, 1};
  for (int a = 0; a < nd; ++a) s[a] = stride ? stride[a] : 1;
  const int size = (int)ipow4(nd);
  int32_t perm[64];
  orc_sequency_perm(nd, perm);
  int64_t nb[3] = {1, 1, 1};
  for (int a = 0; a < nd; ++a) nb[a] = (dims[a] + 3) / 4;
  uint64_t pos = 0;
  for (int64_t lb = 0; lb < nb[0] * nb[1] * nb[2]; ++lb) {
    int64_t b[3], r = lb;
    for (int a = nd - 1; a >= 0; --a) { b[a] = r % nb[a]; r /= nb[a]; }
    int processed = 1;
    for (int a = 0; a < nd; ++a) if (b[a] % s[a] != 0) processed = 0;
    if (!processed) continue;
    float blk[64];
    if (pos >= nbits) return ORC_EINVAL;
    if (!get_bit(buf, pos++)) {
      for (int n = 0; n < size; ++n) blk[n] = 0.0f;   /* empty or p = 0: decodes to zeros */
    } else {
      uint32_t e8 = 0;
      for (int i = 0; i < 8; ++i) e8 |= (uint32_t)get_bit(buf, pos++) << i;
      const int32_t emax = (int32_t)e8 - 127;
      const int kmin = 32 - orc_precision(emax, minexp, nd);
      /* the EC bits: decode from a copy starting at bit 0 */
      uint8_t ec[64 * 33 / 8 + 64];
      memset(ec, 0, sizeof ec);
      const uint64_t avail = nbits - pos < sizeof(ec) * 8 ? nbits - pos : sizeof(ec) * 8;
      for (uint64_t i = 0; i < avail; ++i) put_bit(ec, i, get_bit(buf, pos + i));
      uint32_t u[64];
      pos += orc_gt_decode(ec, avail, size, kmin, u);
      int32_t coef[64];
      for (int j = 0; j < size; ++j) coef[perm[j]] = orc_negabinary_inv(u[j]);
      orc_inv_xform(coef, nd);
      for (int n = 0; n < size; ++n) blk[n] = (float)ldexp((double)coef[n], emax - 30);
    }
    for (int n = 0; n < size; ++n) {
      int64_t idx[3];
      int inside = 1, rr = n;
      for (int a = nd - 1; a >= 0; --a) {
        idx[a] = 4 * b[a] + rr % 4;
        rr /= 4;
        if (idx[a] >= dims[a]) inside = 0;
      }
      if (!inside) continue;
      int64_t lin = 0;
      for (int a = 0; a < nd; ++a) lin = lin * dims[a] + idx[a];
      out[lin] = blk[n];
    }
  }
  return pos == nbits ? ORC_OK : ORC_EINVAL;
}

/* ------------------------------------------------------------------ */
/* log-scale and equal-probability quantisation         */
/* estimates on the stored PDF; see orc.h.          */
/* ------------------------------------------------------------------ */
int orc_variants_from_hist(const uint64_t *hist, double VR, double eb_abs, int b, int n,
                           orc_variant_result *out) {
  if (!hist || !out || b < 2 || n < 1 || n > 32768) return ORC_EINVAL;
  memset(out, 0, sizeof(*out));
  out->value_range = VR;
  out->eb_abs = eb_abs;
  out->log_base = b;
  out->eqp_n = n;
  out->hist_ovf = hist[ORC_OVF_SLOT];
  const int C0 = 32767;                         /* slot of code 0 */
  uint64_t N = 0;
  for (int s = 0; s < ORC_OVF_SLOT; ++s) N += hist[s];
  out->n_in = N;
  if (N == 0) { out->status = ORC_EDEGENERATE; return ORC_EDEGENERATE; }
  const double delta = 2.0 * eb_abs;
  /* linear: bins = cells */
  {
    double H = 0.0;
    for (int s = 0; s < ORC_OVF_SLOT; ++s) {
      if (!hist[s]) continue;
      const double p = (double)hist[s] / (double)N;
      H -= p * log2(p);
    }
    out->lin_bits = H;
    out->lin_psnr = 20.0 * log10(VR / delta) + 10.0 * log10(12.0);   /* Eq. psnr-pdf-linear */
  }
  /* log-scale: bin index i = floor(log_b |q|) by repeated multiplication */
  {
    uint64_t cnt[2][17];
    double width[17];
    memset(cnt, 0, sizeof cnt);
    uint64_t central = 0;
    for (int s = 0; s < ORC_OVF_SLOT; ++s) {
      if (!hist[s]) continue;
      const int q = s - C0;
      const int64_t a = q < 0 ? -(int64_t)q : q;
      if (a < b) { central += hist[s]; continue; }
      int i = 0;
      int64_t pw = b;                            /* b^(i+1) */
      while (pw * b <= a) { pw *= b; ++i; }
      /* now b^(i+1) <= a < b^(i+2): bin i + 1 */
      cnt[q < 0][i + 1] += hist[s];
    }
    {
      double pw = 1.0;                           /* width of bin i >= 1: b^(i+1) - b^i cells */
      for (int i = 1; i < 17; ++i) { pw *= (double)b; width[i] = pw * (double)b - pw; }
    }
    double H = 0.0, M = 0.0;
    int used = 0;
    if (central) {
      const double p = (double)central / (double)N, w = (double)(2 * b - 1) * delta;
      H -= p * log2(p);
      M += w * w * p;
      ++used;
    }
    for (int sg = 0; sg < 2; ++sg)
      for (int i = 1; i < 17; ++i) {
        if (!cnt[sg][i]) continue;
        const double p = (double)cnt[sg][i] / (double)N, w = width[i] * delta;
        H -= p * log2(p);
        M += w * w * p;
        ++used;
      }
    out->log_bits = H;
    out->log_mse = M / 12.0;
    out->log_psnr = 20.0 * log10(VR) - 10.0 * log10(out->log_mse);
    out->log_bins = used;
  }
  /* equal-probability: edges s_k = F^-1(k / (2n-1)) in cell units */
  {
    const uint64_t K = (uint64_t)(2 * n - 1);
    int lo = 0, hi = ORC_OVF_SLOT - 1;
    while (!hist[lo]) ++lo;
    while (!hist[hi]) --hi;
    double prev = (double)(lo - C0) - 0.5;        /* s_0 */
    double sum2 = 0.0, sumw = 0.0;
    uint64_t cum = 0;                             /* mass below cell s */
    int s = lo;
    for (uint64_t k = 1; k <= K; ++k) {
      double edge;
      if (k == K) {
        edge = (double)(hi - C0) + 0.5;           /* s_(2n-1) */
      } else {
        const uint64_t T = k * N;                 /* target mass x K */
        while ((cum + hist[s]) * K <= T) { cum += hist[s]; ++s; }   /* cum K <= T < (cum + c_s) K */
        const double frac = (double)(T - cum * K) / ((double)hist[s] * (double)K);
        edge = ((double)(s - C0) - 0.5) + frac;
      }
      const double w = edge - prev;
      sum2 += w * w;
      sumw += w;
      prev = edge;
    }
    out->eqp_width_sum = sumw;
    out->eqp_bits = 1.0 + log2((double)n);
    out->eqp_mse = delta * delta * sum2 / (12.0 * (double)K);
    out->eqp_psnr = 20.0 * log10(VR) - 10.0 * log10(out->eqp_mse);
  }
  out->status = ORC_OK;
  return ORC_OK;
}

int orc_estimate_variants(const float *x, int ndims, const int64_t *dims, int eb_mode, double eb,
                          const int32_t *stride, int log_base, int eqp_n, orc_variant_result *out) {
  if (!out) return ORC_EINVAL;
  uint64_t *hist = (uint64_t *)calloc(ORC_NSLOTS, sizeof(uint64_t));
  if (!hist) return ORC_EINVAL;
  orc_result r;
  orc_debug dbg;
  memset(&dbg, 0, sizeof dbg);
  dbg.hist = hist;
  int rc = orc_estimate(x, ndims, dims, eb_mode, eb, stride, 0.5, &r, &dbg);
  if (rc == ORC_OK) rc = orc_variants_from_hist(hist, r.value_range, r.eb_abs, log_base, eqp_n, out);
  free(hist);
  return rc;
}
