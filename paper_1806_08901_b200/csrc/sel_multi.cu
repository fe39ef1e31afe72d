// sel_multi.cu -- SURVEY 8(f) N1: the rate-distortion curve of one field at k error
// bounds from ONE read of the field (rate-distortion is compared over error
// bounds; Alg. 1 loops per field).
//
// Only the error bound separates the k estimates: the value range (Alg. 1 line 2) is
// shared; SZ quantises the same Lorenzo residual d (R4) at k bin widths (k histograms);
// ZFP's block exponent, block floating point and lift (R8, R9) do not depend on eb at all
// and the fixed-accuracy cut, bit count and error (R12-R14) depend on it only through the
// integer minexp.  So one pass reads every processed block once, forms d and the lifted
// block once, and runs the eb-dependent stages k times (zfp_cost per eb, one smem
// histogram window per eb).  Each eb's result then goes through the regular finalize
// (entropy, PSNRs, Alg. 1 selection) -- bit-identical to k single-eb estimates.
//
// Launches: k_minmax (value range) -> k_multi (fused pass, k ebs) -> k x k_finalize.
#include "sel_device.cuh"

namespace sel {

constexpr int kMaxEb = 8;          // error bounds per call
constexpr int kMWin = 2048;        // per-eb shared-memory window: codes [-1024, 1024)

struct MultiArgs {
  int k, mode;
  double eb[kMaxEb];
  const Params *base;              // k_minmax output: vmin, vmax, non-finite status
  Params *prm;                     // [k] per-eb params (written by CTA 0)
  unsigned long long *hist;        // [k][kNSlots]
  Partial *part;                   // [k][gridDim.x] per-CTA (bits, err) partials
};

template <int D, bool VEC>
__global__ void __launch_bounds__(256) k_multi(const float *__restrict__ x, Geo g, MultiArgs ma) {
  constexpr int SZ = Tab<D>::SIZE;
  constexpr int PL = D == 3 ? 4 : 1;   // planes per block (axis 0 of the 3-axis view)
  constexpr int RW = D >= 2 ? 4 : 1;   // rows per block   (axis 1)
  constexpr uint32_t kMOff = kSlotOff + (uint32_t)(kCenter - kMWin / 2);   // bits(q+M) -> window bin
  extern __shared__ unsigned int win[];                                    // [k][kMWin]
  __shared__ float s_rf[kMaxEb];
  __shared__ int s_minexp[kMaxEb];
  __shared__ unsigned int s_ovf[kMaxEb];
  __shared__ uint64_t sb[kMaxEb][8];
  __shared__ double se[kMaxEb][8];
  const int k = ma.k;
  for (int i = threadIdx.x; i < k * kMWin; i += blockDim.x) win[i] = 0u;
  if (threadIdx.x == 0) {
    const Params b = *ma.base;
    for (int i = 0; i < k; ++i) {
      // per-eb derived scalars from the shared value range (R1, R2)
      const Params p = make_params(b.vmin, b.vmax, b.status == SEL_ENONFINITE, ma.mode, ma.eb[i]);
      s_rf[i] = p.r_f;
      s_minexp[i] = p.minexp;
      s_ovf[i] = 0u;
      if (blockIdx.x == 0) ma.prm[i] = p;
    }
  }
  __syncthreads();
  if (ma.base->status == SEL_ENONFINITE) return;   // every eb reports it (finalize)
  uint64_t bacc[kMaxEb];
  double eacc[kMaxEb];
#pragma unroll
  for (int i = 0; i < kMaxEb; ++i) { bacc[i] = 0; eacc[i] = 0.0; }

  const int64_t gstride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < g.n_pb; t += gstride) {
    const int64_t p2 = t % g.npb[2];
    const int64_t q = t / g.npb[2];
    const int64_t p1 = q % g.npb[1];
    const int64_t p0 = q / g.npb[1];
    const int64_t I0 = 4 * p0 * g.s[0], J0 = 4 * p1 * g.s[1], K0 = 4 * p2 * g.s[2];
    float blk[SZ];
    float dprev[RW][4];
    // ---------------- SZ: Lorenzo on original values, nested differences (R4), ONCE
#pragma unroll
    for (int r = 0; r < RW; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) dprev[r][c] = 0.0f;
    if (D == 3 && I0 > 0) {
      float up[4], uh = 0.0f;
#pragma unroll
      for (int c = 0; c < 4; ++c) up[c] = 0.0f;
      if (J0 > 0) load_row<VEC>(x, g, I0 - 1, J0 - 1, K0, up, uh);
      float d1up[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) d1up[c] = up[c] - (c ? up[c - 1] : uh);
#pragma unroll
      for (int r = 0; r < RW; ++r) {
        float v[4], h;
        load_row<VEC>(x, g, I0 - 1, J0 + r, K0, v, h);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const float d1 = v[c] - (c ? v[c - 1] : h);
          dprev[r][c] = d1 - d1up[c];
          d1up[c] = d1;
        }
      }
    }
#pragma unroll
    for (int p = 0; p < PL; ++p) {
      const int64_t i = I0 + p;
      float d1up[4];
      {
        float up[4], uh = 0.0f;
#pragma unroll
        for (int c = 0; c < 4; ++c) up[c] = 0.0f;
        if (D >= 2 && J0 > 0) load_row<VEC>(x, g, i, J0 - 1, K0, up, uh);
#pragma unroll
        for (int c = 0; c < 4; ++c) d1up[c] = up[c] - (c ? up[c - 1] : uh);
      }
#pragma unroll
      for (int r = 0; r < RW; ++r) {
        const int64_t j = J0 + r;
        float v[4], h;
        load_row<VEC>(x, g, i, j, K0, v, h);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          blk[(p * RW + r) * 4 + c] = v[c];
          const float d1 = v[c] - (c ? v[c - 1] : h);
          const float d2 = d1 - d1up[c];
          d1up[c] = d1;
          const float d = d2 - dprev[r][c];
          dprev[r][c] = d2;
          const int64_t kk = K0 + c;
          const bool real = (i < g.n[0]) && (j < g.n[1]) && (kk < g.n[2]);
          const bool origin = (i == 0) && (j == 0) && (kk == 0);
          if (real && !origin) {
            // quantisation (R5) of the same residual at every eb
#pragma unroll 1
            for (int e = 0; e < k; ++e) {
              const uint32_t bq = __float_as_uint(__fadd_rn(__fmul_rn(d, s_rf[e]), kMagic));
              const uint32_t w = bq - kMOff;
              if (w < (uint32_t)kMWin) {
                atomicAdd(win + e * kMWin + w, 1u);
              } else {
                const uint32_t s = bq - kSlotOff;
                if (s > 65534u) atomicAdd(&s_ovf[e], 1u);
                else atomicAdd(ma.hist + (size_t)e * kNSlots + s, 1ull);
              }
            }
          }
        }
      }
    }
    // ---------------- ZFP: transform once (R8, R9), cut / bits / error per eb (R12-R14)
    int emax;
    int cf[SZ];
    uint32_t u[SZ];
    if (!zfp_transform<D>(blk, emax, cf)) {
#pragma unroll
      for (int e = 0; e < kMaxEb; ++e) bacc[e] += e < k ? 1u : 0u;   // empty block: 1 bit
      continue;
    }
#pragma unroll
    for (int e = 0; e < kMaxEb; ++e) {
      if (e < k) {
        uint32_t bits;
        double E;
        zfp_cost<D, false>(cf, emax, s_minexp[e], bits, E, u);
        bacc[e] += bits;
        eacc[e] += E;
      }
    }
  }
  // per-CTA partials per eb in a fixed order (deterministic): warp tree, then warps in order
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int e = 0; e < kMaxEb; ++e) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      bacc[e] += __shfl_down_sync(0xffffffffu, bacc[e], o);
      eacc[e] += __shfl_down_sync(0xffffffffu, eacc[e], o);
    }
    if (lane == 0) { sb[e][wid] = bacc[e]; se[e][wid] = eacc[e]; }
  }
  __syncthreads();
  if (threadIdx.x < k) {
    const int e = threadIdx.x;
    uint64_t b = sb[e][0];
    double er = se[e][0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) { b += sb[e][w]; er += se[e][w]; }
    Partial pr;
    pr.bits = b;
    pr.err = er;
    ma.part[(size_t)e * gridDim.x + blockIdx.x] = pr;
    if (s_ovf[e]) atomicAdd(ma.hist + (size_t)e * kNSlots + kOvfSlot, (unsigned long long)s_ovf[e]);
  }
  // windows -> global histograms
  for (int i = threadIdx.x; i < k * kMWin; i += blockDim.x) {
    const unsigned int c = win[i];
    if (c) {
      const int e = i / kMWin, w = i - e * kMWin;
      atomicAdd(ma.hist + (size_t)e * kNSlots + (kCenter - kMWin / 2) + w, (unsigned long long)c);
    }
  }
}

namespace {
template <int D, bool VEC>
const void *multi_fn() { return (const void *)k_multi<D, VEC>; }
const void *pick_multi(int D, bool vec) {
  if (D == 1) return vec ? multi_fn<1, true>() : multi_fn<1, false>();
  if (D == 2) return vec ? multi_fn<2, true>() : multi_fn<2, false>();
  return vec ? multi_fn<3, true>() : multi_fn<3, false>();
}
}  // namespace

int multi_ctas(const Geo &g, int k, int sm_count, int *ctas) {
  const void *fn = pick_multi(g.ndims, g.vec != 0);
  const size_t smem = (size_t)k * kMWin * 4;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(kMaxEb * kMWin * 4)) !=
      cudaSuccess)
    return SEL_ECUDA;
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, 256, smem) != cudaSuccess || occ < 1)
    return SEL_ECUDA;
  const int64_t want = (g.n_pb + 255) / 256;
  const int64_t cap = (int64_t)occ * sm_count;
  *ctas = (int)(want < cap ? (want < 1 ? 1 : want) : cap);
  return SEL_OK;
}

int launch_multi(const float *x, const Geo &g, int ctas, int k, const double *ebs, int mode,
                 const Params *base, Params *prm, unsigned long long *hist, Partial *part, cudaStream_t st) {
  if (k < 1 || k > kMaxEb) return SEL_EINVAL;
  MultiArgs ma;
  ma.k = k;
  ma.mode = mode;
  for (int i = 0; i < kMaxEb; ++i) ma.eb[i] = i < k ? ebs[i] : 1.0;
  ma.base = base;
  ma.prm = prm;
  ma.hist = hist;
  ma.part = part;
  Geo gg = g;
  void *args[] = {(void *)&x, (void *)&gg, (void *)&ma};
  const void *fn = pick_multi(g.ndims, g.vec != 0);
  return cudaLaunchKernel(fn, dim3(ctas), dim3(256), args, (size_t)k * kMWin * 4, st) == cudaSuccess ? SEL_OK
                                                                                                      : SEL_ECUDA;
}

}  // namespace sel
