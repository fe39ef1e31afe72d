// sel_variants.cu -- SURVEY 8(f) N4: the variant quantisers of the paper's Section 5.1.4
// (log-scale P:414-422, equal-probability, and the linear one P:396-403 by the
// same general equations) evaluated on the PDF the selector stores: the field's 65,535-bin
// code histogram.  General Stage-II estimators: BR = -sum_i P_i log2 P_i (Eq.
// bit-rate-pdf), MSE = (1/12) sum_i delta_i^2 P_i, PSNR = 20 log10 VR
// - 10 log10 MSE (Eq. psnr-pdf).  DESIGN.md reading R21: cell q of the PDF is
// [(q - 1/2) delta, (q + 1/2) delta), delta = 2 eb_abs, mass c_q / N_in, uniform inside.
//
// One CTA of 1,024 threads, 64 consecutive histogram slots per thread (the histogram is
// 512 KB and sits in L2 right after the finalize wrote it):
//   pass 1  per-thread mass -> CTA exclusive scan (mass below each thread's slots), lowest /
//           highest occupied cell, linear entropy, log-scale bin masses (shared-memory
//           u64 atomics on <= 35 bins);
//   pass 2  equal-probability edges: the slot holding mass cum <= k N / K < cum + c owns
//           edge k (exact 64-bit integer test), s_k = (q - 1/2) + (k N - cum K) / (c K),
//           written to a K + 1 entry scratch; then sum_k (s_(k+1) - s_k)^2 by a fixed-order
//           CTA reduction;
//   thread 0 assembles the result.
#include <cmath>

#include "sel_internal.h"

namespace sel {
namespace {

constexpr int kVarThreads = 1024;
constexpr int kVarPer = kNSlots / kVarThreads;   // 64 slots per thread
constexpr int kLogMax = 17;                      // log-scale bins per side (b >= 2: 2^15 > 32,767)

__device__ __forceinline__ double block_sum(double v, double *sh) {   // fixed order: lanes, then warps
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < kVarThreads / 32; ++w) s += sh[w];
  return s;
}

__global__ void __launch_bounds__(kVarThreads) k_variants(const unsigned long long *__restrict__ hist,
                                                          const Params *prm_p, int b, int n,
                                                          double *edges, sel_variant_result *out) {
  __shared__ unsigned long long s_warp[kVarThreads / 32];
  __shared__ unsigned long long s_log[2][kLogMax], s_central, s_N;
  __shared__ int s_lo, s_hi;
  __shared__ double s_red[kVarThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const Params prm = *prm_p;
  const int s0 = tid * kVarPer;
  if (tid < 2 * kLogMax) s_log[tid / kLogMax][tid % kLogMax] = 0ull;
  if (tid == 0) { s_central = 0ull; s_lo = kNSlots; s_hi = -1; }
  // ---- pass 1: this thread's mass (the overflow slot 65,535 is outside the PDF)
  unsigned long long mine = 0;
  int lo = kNSlots, hi = -1;
#pragma unroll 8
  for (int k = 0; k < kVarPer; ++k) {
    const int s = s0 + k;
    const unsigned long long c = s < kOvfSlot ? __ldcg(hist + s) : 0ull;
    mine += c;
    if (c) { lo = min(lo, s); hi = max(hi, s); }
  }
  // exclusive scan over threads: warp scan, then warp totals
  unsigned long long inc = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  __syncthreads();
  if (lane == 31) s_warp[wid] = inc;
  if (lo < kNSlots) { atomicMin(&s_lo, lo); atomicMax(&s_hi, hi); }
  __syncthreads();
  unsigned long long below = inc - mine;
  for (int w = 0; w < wid; ++w) below += s_warp[w];
  if (tid == kVarThreads - 1) s_N = below + mine;
  __syncthreads();
  const unsigned long long N = s_N;
  if (N == 0ull || prm.status != SEL_OK) {
    if (tid == 0) {
      sel_variant_result r{};
      r.status = prm.status != SEL_OK ? prm.status : SEL_EDEGENERATE;
      r.value_range = prm.vr;
      r.eb_abs = prm.eb_abs;
      r.log_base = b;
      r.eqp_n = n;
      r.hist_ovf = __ldcg(hist + kOvfSlot);
      *out = r;
    }
    return;
  }
  // ---- linear entropy and the log-scale bin masses
  const double Nd = (double)N, lN = log2(Nd);
  double hlin = 0.0;
  const unsigned long long K = (unsigned long long)(2 * n - 1);
  unsigned long long cum = below;
  for (int k = 0; k < kVarPer; ++k) {
    const int s = s0 + k;
    const unsigned long long c = s < kOvfSlot ? __ldcg(hist + s) : 0ull;
    if (!c) continue;
    const double cd = (double)c;
    hlin += cd * (lN - log2(cd));
    // log-scale bin of code q: central if |q| < b, else i with b^i <= |q| < b^(i+1)
    const int q = s - kCenter;
    const long long a = q < 0 ? -(long long)q : (long long)q;
    if (a < b) {
      atomicAdd(&s_central, c);
    } else {
      int i = 1;
      long long pw = b;                 // b^i
      while (pw * b <= a) { pw *= b; ++i; }
      atomicAdd(&s_log[q < 0][i], c);
    }
    // ---- equal-probability edges owned by this slot: cum K <= k N < (cum + c) K, 1 <= k < K
    unsigned long long k0 = (cum * K + N - 1) / N;          // ceil(cum K / N)
    if (k0 < 1) k0 = 1;
    for (unsigned long long kk = k0; kk < K && kk * N < (cum + c) * K; ++kk) {
      const double frac = (double)(kk * N - cum * K) / ((double)c * (double)K);
      edges[kk] = ((double)q - 0.5) + frac;
    }
    cum += c;
  }
  if (tid == 0) {
    edges[0] = (double)(s_lo - kCenter) - 0.5;
    edges[K] = (double)(s_hi - kCenter) + 0.5;
  }
  __threadfence_block();
  __syncthreads();
  double sum2 = 0.0;
  for (unsigned long long kk = tid; kk < K; kk += kVarThreads) {
    const double w = __ldcg(edges + kk + 1) - __ldcg(edges + kk);
    sum2 += w * w;
  }
  sum2 = block_sum(sum2, s_red);
  hlin = block_sum(hlin, s_red);
  if (tid != 0) return;
  // ---- result (thread 0), bins in the oracle's order: central, positive side, negative side
  sel_variant_result r{};
  const double delta = 2.0 * prm.eb_abs;
  r.value_range = prm.vr;
  r.eb_abs = prm.eb_abs;
  r.n_in = N;
  r.hist_ovf = __ldcg(hist + kOvfSlot);
  r.log_base = b;
  r.eqp_n = n;
  r.lin_bits = hlin / Nd;
  r.lin_psnr = 20.0 * log10(prm.vr / delta) + 10.0 * log10(12.0);
  double H = 0.0, M = 0.0;
  int used = 0;
  if (s_central) {
    const double p = (double)s_central / Nd, w = (double)(2 * b - 1) * delta;
    H -= p * log2(p);
    M += w * w * p;
    ++used;
  }
  for (int sg = 0; sg < 2; ++sg) {
    double pw = 1.0;
    for (int i = 1; i < kLogMax; ++i) {
      pw *= (double)b;
      const unsigned long long c = s_log[sg][i];
      if (!c) continue;
      const double p = (double)c / Nd, w = (pw * (double)b - pw) * delta;
      H -= p * log2(p);
      M += w * w * p;
      ++used;
    }
  }
  r.log_bits = H;
  r.log_mse = M / 12.0;
  r.log_psnr = 20.0 * log10(prm.vr) - 10.0 * log10(r.log_mse);
  r.log_bins = used;
  r.eqp_width_sum = edges[K] - edges[0];
  r.eqp_bits = 1.0 + log2((double)n);
  r.eqp_mse = delta * delta * sum2 / (12.0 * (double)K);
  r.eqp_psnr = 20.0 * log10(prm.vr) - 10.0 * log10(r.eqp_mse);
  r.status = SEL_OK;
  *out = r;
}

}  // namespace

size_t variants_ws_bytes() {   // [hist copy u64 x 65,536 | edges double x 65,536 | result]
  return (size_t)kNSlots * 8 + (size_t)kNSlots * 8 + 256;
}

int launch_variants(void *vws, const Params *prm, int log_base, int eqp_n, cudaStream_t st) {
  char *b = (char *)vws;
  const unsigned long long *hist = (const unsigned long long *)b;
  double *edges = (double *)(b + (size_t)kNSlots * 8);
  sel_variant_result *out = (sel_variant_result *)(b + (size_t)kNSlots * 16);
  k_variants<<<1, kVarThreads, 0, st>>>(hist, prm, log_base, eqp_n, edges, out);
  return cudaGetLastError() == cudaSuccess ? SEL_OK : SEL_ECUDA;
}

}  // namespace sel
