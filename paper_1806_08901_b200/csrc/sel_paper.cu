// sel_paper.cu -- SURVEY 8(f) N2: the paper-literal estimator (Alg. 1 lines 3-10 as printed,
// PAPER.md:478-490), next to the exact one of the hot path.
//
//   ZFP: per processed block, n_sb of the 3 / 9 / 16 sampled coefficients (1D / 2D / 3D,
//        P:459; positions evenly spaced over the sequency order, reading R19), linearly
//        interpolated over the block, averaged = BR_zfp; MSE_sp =
//        mean over the samples of (dropped-plane value x 2^(emax-30))^2, unit weights
//        (P:454-456); PSNR_sp = -10 log10 MSE_sp + 20 log10 VR.
//   SZ:  delta with PSNR_sz = PSNR_sp in Eq. psnr-pdf-linear (Alg. 1 line 7): delta =
//        VR sqrt(12) 10^(-PSNR_sp/20) = sqrt(12 MSE_sp); the processed blocks' Lorenzo
//        residuals re-quantised at bin width delta (lines 8-9), entropy + 0.5 + 32 p_ovf.
//   line 10: SZ iff BR_sz < BR_zfp.
// Launches: k_minmax -> k_paper_zfp -> k_paper_mid -> fused pass at r* = 1/delta (k_tile /
// k_estimate; only its histogram is used) -> k_finalize (entropy) -> k_paper_assemble.
#include "sel_device.cuh"

namespace sel {

// sampled sequency positions j_i = round(i (4^d - 1) / (m - 1)), halves up (reading R19)
template <int D>
struct PaperTab {
  static constexpr int M = D == 1 ? 3 : (D == 2 ? 9 : 16);
  static constexpr int L = Tab<D>::SIZE - 1;
  static constexpr int pos(int i) { return (2 * i * L + (M - 1)) / (2 * (M - 1)); }
};

struct PaperMid {
  unsigned long long nsb2;     // 2 x sum of interpolated n_sb
  unsigned long long nsamp;    // sampled coefficients
  double mse_sp, psnr_sp, delta;
  double vr, eb_abs;           // the value range and the user's bound (Alg. 1 line 2)
  float r_star;
  int matched;
  int status;
};

template <int D, bool VEC>
__global__ void __launch_bounds__(256) k_paper_zfp(const float *__restrict__ x, Geo g, const Params *prm_,
                                                   unsigned long long *part_nsb, double *part_mse) {
  constexpr int SZ = Tab<D>::SIZE;
  constexpr int M = PaperTab<D>::M;
  constexpr int PL = D == 3 ? 4 : 1;
  constexpr int RW = D >= 2 ? 4 : 1;
  const Params prm = *prm_;
  unsigned long long nsb2 = 0;
  double mse = 0.0;
  if (prm.status == SEL_OK) {
    const int64_t gstride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < g.n_pb; t += gstride) {
      const int64_t p2 = t % g.npb[2];
      const int64_t q = t / g.npb[2];
      const int64_t p1 = q % g.npb[1];
      const int64_t p0 = q / g.npb[1];
      const int64_t I0 = 4 * p0 * g.s[0], J0 = 4 * p1 * g.s[1], K0 = 4 * p2 * g.s[2];
      float blk[SZ];
#pragma unroll
      for (int p = 0; p < PL; ++p)
#pragma unroll
        for (int r = 0; r < RW; ++r) {
          float v[4], h;
          load_row<VEC>(x, g, I0 + p, J0 + r, K0, v, h);   // edge-replicated (R17)
#pragma unroll
          for (int c = 0; c < 4; ++c) blk[(p * RW + r) * 4 + c] = v[c];
        }
      int emax;
      int cf[SZ];
      if (!zfp_transform<D>(blk, emax, cf)) continue;     // all-zero block: n_sb = 0, e = 0
      int prec = emax - prm.minexp + 2 * (D + 1);
      prec = prec < 0 ? 0 : (prec > 32 ? 32 : prec);
      const int kmin = 32 - prec;
      const uint32_t low = kmin >= 32 ? 0xffffffffu : ((1u << kmin) - 1u);
      const uint32_t Mk = 0xAAAAAAAAu & low;
      const double scale = pow2d(2 * (emax - 30));
      int ns[M];
      static_for<0, M>([&](auto I) {
        constexpr int i = decltype(I)::value;
        constexpr int j = PaperTab<D>::pos(i);
        constexpr int n = Tab<D>::make_perm().v[j];
        const uint32_t uj = to_negabinary(cf[n]);
        const int f = flo(uj);
        ns[i] = f >= kmin ? f - kmin + 1 : 0;              // significant bits at the cut
        const long long e = (long long)((uj & low) ^ Mk) - (long long)Mk;   // dropped planes
        const double ed = (double)e;
        mse = __dadd_rn(mse, __dmul_rn(__dmul_rn(ed, ed), scale));
      });
      // 2 x sum of the linear interpolation between neighbouring samples (integer)
      long long s2 = 2LL * ns[M - 1];
      static_for<0, M - 1>([&](auto A) {
        constexpr int a = decltype(A)::value;
        constexpr int len = PaperTab<D>::pos(a + 1) - PaperTab<D>::pos(a);
        s2 += 2LL * len * ns[a] + (long long)(ns[a + 1] - ns[a]) * (len - 1);
      });
      nsb2 += (unsigned long long)s2;
    }
  }
  // per-CTA partial, fixed order: warp tree, then warps in order
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    nsb2 += __shfl_down_sync(0xffffffffu, nsb2, o);
    mse += __shfl_down_sync(0xffffffffu, mse, o);
  }
  __shared__ unsigned long long sn[8];
  __shared__ double sm[8];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) { sn[wid] = nsb2; sm[wid] = mse; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) { nsb2 += sn[w]; mse += sm[w]; }
    part_nsb[blockIdx.x] = nsb2;
    part_mse[blockIdx.x] = mse;
  }
}

// one thread: the CTA partials in order, PSNR_sp, delta (Alg. 1 line 7) and the params of
// the SZ re-quantisation at bin width delta (r* = float(1/delta))
__global__ void k_paper_mid(const Params *base, int nparts, const unsigned long long *part_nsb,
                            const double *part_mse, unsigned long long nsamp, PaperMid *mid, Params *pprm) {
  if (threadIdx.x != 0) return;
  const Params b = *base;
  PaperMid m{};
  m.status = b.status;
  m.nsamp = nsamp;
  m.vr = b.vr;
  m.eb_abs = b.eb_abs;
  double s = 0.0;
  unsigned long long n2 = 0;
  for (int i = 0; i < nparts; ++i) { n2 += part_nsb[i]; s += part_mse[i]; }
  m.nsb2 = n2;
  m.mse_sp = s / (double)nsamp;
  m.psnr_sp = m.mse_sp > 0.0 ? 20.0 * log10(b.vr) - 10.0 * log10(m.mse_sp) : __longlong_as_double(0x7ff0000000000000LL);
  // delta = VR sqrt(12) 10^(-PSNR_sp/20) = sqrt(12 MSE_sp); no PSNR to match (MSE_sp = 0 or
  // VR = 0): SZ at the user's bound, delta = 2 eb_abs, matched = 0 (R16 ii)
  double delta = (m.mse_sp > 0.0 && b.vr > 0.0) ? sqrt(12.0 * m.mse_sp) : 2.0 * b.eb_abs;
  float rs = __double2float_rn(1.0 / delta);
  m.matched = (m.mse_sp > 0.0 && b.vr > 0.0 && !is_nonfinite(rs)) ? 1 : 0;
  if (!m.matched) {
    delta = 2.0 * b.eb_abs;
    rs = __double2float_rn(1.0 / delta);
  }
  m.delta = delta;
  m.r_star = rs;
  *mid = m;
  Params p = b;
  p.r_f = rs;
  p.eb_abs = delta / 2.0;
  *pprm = p;
}

__global__ void k_paper_assemble(const PaperMid *mid, const sel_result *sz, uint64_t n_values,
                                 sel_paper_result *out) {
  if (threadIdx.x != 0) return;
  const PaperMid m = *mid;
  const sel_result r = *sz;
  sel_paper_result o = {};
  o.status = m.status != SEL_OK ? m.status : r.status;
  o.value_range = m.vr;
  o.eb_abs = m.eb_abs;
  o.nsb2_total = m.nsb2;
  o.n_samples = m.nsamp;
  o.n_values = n_values;
  o.zfp_nsb_bits = (double)m.nsb2 / 2.0 / (double)n_values;
  o.zfp_mse_sp = m.mse_sp;
  o.zfp_psnr_sp = m.psnr_sp;
  o.sz_delta = m.delta;
  o.r_star = m.r_star;
  o.matched = m.matched;
  o.sz_entropy = r.sz_entropy;
  o.sz_overflow_frac = r.sz_overflow_frac;
  o.sz_bits = r.sz_bits_per_value;
  o.hist_total = r.hist_total;
  o.hist_ovf = r.hist_ovf;
  o.choice = o.sz_bits < o.zfp_nsb_bits ? 0 : 1;      // Alg. 1 line 10
  *out = o;
}

namespace {
template <int D, bool VEC>
const void *pzfp_fn() { return (const void *)k_paper_zfp<D, VEC>; }
const void *pick_pzfp(int D, bool vec) {
  if (D == 1) return vec ? pzfp_fn<1, true>() : pzfp_fn<1, false>();
  if (D == 2) return vec ? pzfp_fn<2, true>() : pzfp_fn<2, false>();
  return vec ? pzfp_fn<3, true>() : pzfp_fn<3, false>();
}
}  // namespace

size_t paper_ws_bytes(int max_ctas) {
  return (size_t)max_ctas * 16 + sizeof(PaperMid) + sizeof(Params) + 1024;
}

// K2p + mid: the ZFP half of the paper-literal estimate; writes the params of the SZ pass
int launch_paper_zfp(const float *x, const Geo &g, int sm_count, int max_ctas, const Params *base, void *pws,
                     Params *pprm, cudaStream_t st) {
  const void *fn = pick_pzfp(g.ndims, g.vec != 0);
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, 256, 0) != cudaSuccess || occ < 1) return SEL_ECUDA;
  int64_t ctas = (g.n_pb + 255) / 256;
  if (ctas > (int64_t)occ * sm_count) ctas = (int64_t)occ * sm_count;
  if (ctas > max_ctas) ctas = max_ctas;
  if (ctas < 1) ctas = 1;
  char *b = (char *)pws;
  unsigned long long *pn = (unsigned long long *)b;
  double *pm = (double *)(b + (size_t)max_ctas * 8);
  PaperMid *mid = (PaperMid *)(b + (size_t)max_ctas * 16);
  Geo gg = g;
  void *args[] = {(void *)&x, (void *)&gg, (void *)&base, (void *)&pn, (void *)&pm};
  if (cudaLaunchKernel(fn, dim3((unsigned)ctas), dim3(256), args, 0, st) != cudaSuccess) return SEL_ECUDA;
  const int M = g.ndims == 1 ? 3 : (g.ndims == 2 ? 9 : 16);
  k_paper_mid<<<1, 32, 0, st>>>(base, (int)ctas, pn, pm, (unsigned long long)M * (unsigned long long)g.n_pb, mid,
                                pprm);
  return cudaGetLastError() == cudaSuccess ? SEL_OK : SEL_ECUDA;
}

int launch_paper_assemble(void *pws, int max_ctas, const sel_result *sz, uint64_t n_values, sel_paper_result *out,
                          cudaStream_t st) {
  const PaperMid *mid = (const PaperMid *)((char *)pws + (size_t)max_ctas * 16);
  k_paper_assemble<<<1, 32, 0, st>>>(mid, sz, n_values, out);
  return cudaGetLastError() == cudaSuccess ? SEL_OK : SEL_ECUDA;
}

}  // namespace sel
