// sel_device.cuh -- device building blocks shared by the fused-pass kernels
// (sel_kernels.cu: march / generic; sel_tile.cu: TMA tile pipeline).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "sel_internal.h"

namespace sel {

// ============================================================ compile-time tables
template <int D>
struct Tab {
  static constexpr int SIZE = D == 1 ? 4 : (D == 2 ? 16 : 64);
  static constexpr int NCLS = D == 1 ? 3 : (D == 2 ? 6 : 10);
  struct IArr { int v[64]; };
  // total-sequency order: sort multi-indices by (sum i, sum i^2, n) (reading R10)
  static constexpr IArr make_perm() {
    IArr a{};
    int k1[64] = {}, k2[64] = {};
    for (int n = 0; n < SIZE; ++n) {
      int r = n, s1 = 0, s2 = 0;
      for (int d = 0; d < D; ++d) { int i = r % 4; r /= 4; s1 += i; s2 += i * i; }
      k1[n] = s1; k2[n] = s2; a.v[n] = n;
    }
    for (int i = 1; i < SIZE; ++i) {
      int v = a.v[i], j = i - 1;
      while (j >= 0) {
        int u = a.v[j];
        bool gt = k1[u] > k1[v] || (k1[u] == k1[v] && (k2[u] > k2[v] || (k2[u] == k2[v] && u > v)));
        if (!gt) break;
        a.v[j + 1] = u; --j;
      }
      a.v[j + 1] = v;
    }
    return a;
  }
  // weight class of natural coefficient n: the squared column norm of the inverse
  // lift per axis is g = (4, 5, 4, 13/4) (reading R14); class = (#axes with g=5,
  // #axes with g=13/4) -> index nB*(D+1) - ... packed densely below.
  static constexpr int cls_of(int n) {
    int nb = 0, nc = 0, r = n;
    for (int d = 0; d < D; ++d) { int i = r % 4; r /= 4; nb += (i == 1); nc += (i == 3); }
    // dense index over pairs (nb, nc) with nb + nc <= D
    int idx = 0;
    for (int b = 0; b < nb; ++b) idx += D + 1 - b;
    return idx + nc;
  }
  static constexpr double cls_weight(int c) {
    for (int b = 0; b <= D; ++b)
      for (int cc = 0; cc <= D - b; ++cc) {
        int idx = 0;
        for (int t = 0; t < b; ++t) idx += D + 1 - t;
        if (idx + cc == c) {
          double w = 1.0;
          for (int t = 0; t < D - b - cc; ++t) w *= 4.0;
          for (int t = 0; t < b; ++t) w *= 5.0;
          for (int t = 0; t < cc; ++t) w *= 3.25;
          return w;
        }
      }
    return 0.0;
  }
  static constexpr double gain(int n) {
    const double g[4] = {4.0, 5.0, 4.0, 3.25};
    double w = 1.0;
    int r = n;
    for (int d = 0; d < D; ++d) { w *= g[r % 4]; r /= 4; }
    return w;
  }
};

template <int B, int E, typename F>
__device__ __forceinline__ void static_for(F &&f) {
  if constexpr (B < E) {
    f(std::integral_constant<int, B>{});
    static_for<B + 1, E>(f);
  }
}

// ============================================================ device helpers
__device__ __forceinline__ bool is_nonfinite(float v) {
  return (__float_as_uint(v) & 0x7f800000u) == 0x7f800000u;
}

// position of the most significant set bit, -1 for 0 (SASS FLO)
__device__ __forceinline__ int flo(uint32_t u) {
  int r;
  asm("bfind.u32 %0, %1;" : "=r"(r) : "r"(u));
  return r;
}

__device__ __forceinline__ void grid_dep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void grid_dep_launch() { asm volatile("griddepcontrol.launch_dependents;"); }

// ---- SZ quantisation code -> histogram (reading R5) --------------------------------
// q = d * r_f (fp32, sign-symmetric so equal to sign(d) * (|d| r_f)); adding the even
// constant M = 1.5*2^23 rounds q to the nearest integer, ties to even, and leaves
// rint(q) in the low mantissa bits for |q| < 2^22.  slot = bits(q + M) - bits(M) + 32767.
// Every q with !(|q| < 32767.5) (including NaN/Inf) maps to an unsigned slot > 65534.
constexpr float kMagic = 12582912.0f;                       // 1.5 * 2^23
constexpr uint32_t kSlotOff = 0x4B400000u - (uint32_t)kCenter;
constexpr uint32_t kWinOff = kSlotOff + (uint32_t)(kCenter - kWinHalf);

// rare path (out of the smem window): overflow -> counted by the caller, else a global
// atomic on the full-width histogram.  Kept out of line: it is inlined at every site.
static __device__ __noinline__ unsigned int sz_tail(uint32_t s, unsigned long long *gh) {
  if (s > 65534u) return 1u;
  atomicAdd(gh + s, 1ull);
  return 0u;
}

template <bool DBG>
__device__ __forceinline__ void sz_put(float d, float r_f, bool valid, unsigned int *sh,
                                       unsigned long long *gh, unsigned int &ovf,
                                       int32_t *dbg_code) {
  const uint32_t b = __float_as_uint(__fadd_rn(__fmul_rn(d, r_f), kMagic));
  const uint32_t w = b - kWinOff;
  if (valid) {
    if (w < (uint32_t)kWinBins) atomicAdd(sh + w, 1u);
    else ovf += sz_tail(b - kSlotOff, gh);
    if constexpr (DBG) {
      const uint32_t s = b - kSlotOff;
      *dbg_code = s > 65534u ? kOvfSlot : (int32_t)s;
    }
  }
}

// ---- ZFP --------------------------------------------------------------------------
// Forward decorrelating lift on one 4-vector (reading R8): five add / arithmetic-shift /
// subtract stages; exact-arithmetic map A = (1/16)[[4,4,4,4],[5,1,-1,-5],[-4,4,4,-4],[-2,6,-6,2]].
__device__ __forceinline__ void fwd_lift(int &x, int &y, int &z, int &w) {
  x += w; x >>= 1; w -= x;
  z += y; z >>= 1; y -= z;
  x += z; x >>= 1; z -= x;
  w += y; w >>= 1; y -= w;
  w += y >> 1; y -= w >> 1;
}

__device__ __forceinline__ uint32_t to_negabinary(int c) {
  return ((uint32_t)c + 0xAAAAAAAAu) ^ 0xAAAAAAAAu;
}

__device__ __forceinline__ double pow2d(int k) {   // 2^k, k in [-1022, 1023]
  return __hiloint2double((1023 + k) << 20, 0);
}

// Error sum in double, coefficient by coefficient in sequency order (used when kmin >= 30,
// incl. p == 0, where the squared errors no longer fit exact 64-bit class sums).
template <int D>
__device__ __forceinline__ double zfp_err_double(const int (&cf)[Tab<D>::SIZE], int kmin, int emax) {
  constexpr int SZ = Tab<D>::SIZE;
  const uint32_t low = kmin >= 32 ? 0xffffffffu : ((1u << kmin) - 1u);
  const uint32_t Mk = 0xAAAAAAAAu & low;
  double E = 0.0;
  static_for<0, SZ>([&](auto J) {
    constexpr int j = decltype(J)::value;
    constexpr int n = Tab<D>::make_perm().v[j];
    constexpr double w = Tab<D>::gain(n);
    const uint32_t uj = to_negabinary(cf[n]);
    const long long e = (long long)((uj & low) ^ Mk) - (long long)Mk;
    const double ed = (double)e;
    E = __dadd_rn(E, __dmul_rn(w, __dmul_rn(ed, ed)));
  });
  return __dmul_rn(E, pow2d(2 * (emax - 30)));
}

// ZFP stage 1 (R9, R8): block exponent, block floating point, decorrelating lift.
// Returns false for an all-zero block (emax = -127; no transform, cf untouched).
template <int D>
__device__ __forceinline__ bool zfp_transform(const float (&v)[Tab<D>::SIZE], int &emax,
                                              int (&cf)[Tab<D>::SIZE]) {
  constexpr int SZ = Tab<D>::SIZE;
  // exponent (R9): max |x| as float; exponent field - 126 (subnormal max -> -126)
  float m = 0.0f;
#pragma unroll
  for (int n = 0; n < SZ; ++n) m = fmaxf(m, fabsf(v[n]));
  if (m == 0.0f) {
    emax = -127;
    return false;
  }
  emax = (int)(__float_as_uint(m) >> 23) - 126;
  // block floating point: i = trunc(x 2^(30-emax)), exact (R9)
  if (emax >= -97) {
    const float sc = __uint_as_float((uint32_t)(157 - emax) << 23);
#pragma unroll
    for (int n = 0; n < SZ; ++n) cf[n] = __float2int_rz(__fmul_rn(v[n], sc));
  } else {
    // (rare: blocks below 2^-97.  The empty volatile asm keeps this a real branch -- without
    // it the compiler evaluates both scalings for every block and selects: 3 FMUL + 1 FSEL
    // per value instead of 1 FMUL.)
    const float sc = __uint_as_float((uint32_t)(93 - emax) << 23);
#pragma unroll
    for (int n = 0; n < SZ; ++n) {
      float t = __fmul_rn(v[n], 0x1p64f);
      asm volatile("" : "+f"(t));
      cf[n] = __float2int_rz(__fmul_rn(t, sc));
    }
  }
  // decorrelating lift along the fastest axis first, then slower (R8)
#pragma unroll
  for (int l = 0; l < SZ / 4; ++l) fwd_lift(cf[4 * l], cf[4 * l + 1], cf[4 * l + 2], cf[4 * l + 3]);
  if constexpr (D >= 2) {
#pragma unroll
    for (int p = 0; p < SZ / 16; ++p)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int b = p * 16 + c;
        fwd_lift(cf[b], cf[b + 4], cf[b + 8], cf[b + 12]);
      }
  }
  if constexpr (D == 3) {
#pragma unroll
    for (int l = 0; l < 16; ++l) fwd_lift(cf[l], cf[l + 16], cf[l + 32], cf[l + 48]);
  }
  return true;
}

// ZFP stage 2 (R10-R14) for one tolerance exponent minexp: fixed-accuracy cut, exact EC
// bit count and gain-weighted truncation error of a transformed (non-empty) block.  The
// sequency-ordered negabinary words are formed on the fly in ONE descending pass that
// does both the bit count and the error classes, so a lifted coefficient dies as soon as
// it is consumed (register pressure: the 3D block is 64 words).  Only this stage depends
// on the error bound (through the integer minexp): the multi-eb path runs it per eb on
// one transform.
template <int D, bool DBG>
__device__ __forceinline__ void zfp_cost(const int (&cf)[Tab<D>::SIZE], int emax, int minexp,
                                         uint32_t &bits, double &E, uint32_t (&u)[Tab<D>::SIZE]) {
  constexpr int SZ = Tab<D>::SIZE;
  constexpr int NC = Tab<D>::NCLS;
  // fixed-accuracy cut (R12)
  int prec = emax - minexp + 2 * (D + 1);
  prec = prec < 0 ? 0 : (prec > 32 ? 32 : prec);
  const int kmin = 32 - prec;
  // kmin >= 30 (incl. p == 0, where every plane is dropped): the error in double, first
  double Ed = 0.0;
  if (kmin >= 30) Ed = zfp_err_double<D>(cf, kmin, emax);
  // ONE pass over the sequency order j = SZ-1 .. 0 (R10 reorder + R11 negabinary on the
  // fly): the closed-form group-testing count (R13) and the exact error class sums (R14).
  //   bit count: f_j = floor(log2 u_j) (-1 for 0), S_j = max_{j'>=j} f_j',
  //   Q_j = max(kmin-1, S_j):
  //   GT = sum_j max(0, S_j-kmin+1)                = sum_j Q_j - SZ (kmin-1)
  //      + #{j : f_j >= kmin and f_j >= S_{j+1}}   (f_j >= kmin and f_j >= Q_{j+1})
  //      + 32 - max(f_L+1, kmin) - [f_L >= kmin]
  //   evaluated with R_j = max(kmin, S_j): the middle set is C = {j : f_j >= R_{j+1}}
  //   (a bit mask, counted by popc), and sum_j Q_j = sum_j R_j - z with z = #{j : S_j <
  //   kmin} = SZ-1-max(C) (the highest j of C is the last significant coefficient).
  //   error: e_j = value of the dropped negabinary digits = ((u & low) ^ M) - M; e_j^2
  //   summed EXACTLY in 64-bit integers per weight class (|e| < 2^29 for kmin <= 29, so
  //   the class sums fit), then weighted in double.
  const uint32_t low = (1u << (kmin & 31)) - 1u;   // (only used when kmin < 30)
  const uint32_t Mk = 0xAAAAAAAAu & low;
  unsigned long long acc[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) acc[c] = 0ull;
  int R = kmin, sR = 0;
  uint32_t cm0 = 0u, cm1 = 0u;   // C for j < 32 / j >= 32
  int fL = -1;
  static_for<0, SZ>([&](auto JJ) {
    constexpr int j = SZ - 1 - decltype(JJ)::value;
    constexpr int n = Tab<D>::make_perm().v[j];
    constexpr int c = Tab<D>::cls_of(n);
    // negabinary u = (c + M) ^ M; its dropped digits (u & low) ^ (M & low) = (c + M) & low
    const uint32_t tj = (uint32_t)cf[n] + 0xAAAAAAAAu;
    const uint32_t uj = tj ^ 0xAAAAAAAAu;
    if constexpr (DBG) u[j] = uj;
    const int f = flo(uj);
    if constexpr (j == SZ - 1) fL = f;
    if (f >= R) {
      if (j < 32) cm0 |= 1u << (j & 31);
      else cm1 |= 1u << (j & 31);
    }
    R = max(R, f);
    sR += R;
    const int e = (int)(tj & low) - (int)Mk;
    acc[c] += (unsigned long long)((long long)e * (long long)e);
  });
  if (prec == 0) {
    bits = 1u;
  } else {
    const int last = cm1 ? 32 + flo(cm1) : flo(cm0);       // -1 if C is empty
    const int t1 = sR - (SZ - 1 - last);
    const int t2 = __popc(cm0) + __popc(cm1);
    const int t3 = 32 - max(fL + 1, kmin) - (fL >= kmin ? 1 : 0);
    bits = (uint32_t)(9 + t1 - SZ * (kmin - 1) + t2 + t3);
  }
  if (kmin >= 30) {
    E = Ed;
    return;
  }
  double s = 0.0;
  static_for<0, NC>([&](auto Cc) {
    constexpr int c = decltype(Cc)::value;
    constexpr double w = Tab<D>::cls_weight(c);
    s = __dadd_rn(s, __dmul_rn(w, (double)acc[c]));
  });
  E = __dmul_rn(s, pow2d(2 * (emax - 30)));
}

// One 4^d block: v (natural order, edge-replicated) -> EC bits and gain-weighted error.
template <int D, bool DBG>
__device__ __forceinline__ void zfp_block(const float (&v)[Tab<D>::SIZE], int minexp,
                                          uint32_t &bits, double &E, int &emax,
                                          int (&cf)[Tab<D>::SIZE], uint32_t (&u)[Tab<D>::SIZE]) {
  constexpr int SZ = Tab<D>::SIZE;
  if (!zfp_transform<D>(v, emax, cf)) {
    bits = 1u;
    E = 0.0;
    if constexpr (DBG) {
#pragma unroll
      for (int n = 0; n < SZ; ++n) { cf[n] = 0; u[n] = 0u; }
    }
    return;
  }
  zfp_cost<D, DBG>(cf, emax, minexp, bits, E, u);
}


// one 4-value row of a block (+ its left neighbour h) from global memory; rows / planes
// past the field edge are replicated (R17), the left neighbour is 0 at k = 0 (R4)
template <bool VEC>
__device__ __forceinline__ void load_row(const float *__restrict__ x, const Geo &g, int64_t i,
                                         int64_t j, int64_t k0, float v[4], float &h) {
  const int64_t ic = i < g.n[0] ? i : g.n[0] - 1;   // edge replication for padded rows (R17)
  const int64_t jc = j < g.n[1] ? j : g.n[1] - 1;
  const float *row = x + (ic * g.n[1] + jc) * g.n[2];
  if constexpr (VEC) {
    const float4 q = __ldg(reinterpret_cast<const float4 *>(row + k0));
    v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
  } else {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      int64_t k = k0 + c;
      v[c] = __ldg(row + (k < g.n[2] ? k : g.n[2] - 1));
    }
  }
  h = k0 > 0 ? __ldg(row + k0 - 1) : 0.0f;
}

// Per-field result from the reduced sums (Eq. entropy, Eq. psnr-sz
// P:410) and the Alg. 1 lines 7-10 selection (reading R16).
// S = sum_s c_s log2(N/c_s); lg_* are log10(VR/eb), log10(VR), log10(MSE).
__device__ __forceinline__ sel_result assemble_result(const Params &prm, double S, double errs,
                                                      uint64_t tb, uint64_t novf, uint64_t hcnt,
                                                      const FinalizeArgs &fa, double lg_vr_eb,
                                                      double lg_vr, double lg_mse) {
  sel_result r = {};
  r.status = prm.status;
  r.value_range = prm.vr;
  r.eb_abs = prm.eb_abs;
  r.minexp = prm.minexp;
  r.r_f = prm.r_f;
  r.n_sz_points = fa.n_sz;
  r.n_values = fa.n_values;
  r.n_blocks = fa.n_blocks;
  r.hist_total = hcnt;
  r.hist_ovf = novf;
  if (r.status == SEL_OK && fa.n_sz == 0) r.status = SEL_EDEGENERATE;   // single-value field
  if (r.status != SEL_OK) return r;
  const double Nsz = (double)fa.n_sz;
  const double vr = prm.vr, eb = prm.eb_abs;
  const double mse = errs / (double)fa.n_values;
  const double H = S / Nsz;
  const double povf = (double)novf / Nsz;
  r.sz_entropy = H;
  r.sz_overflow_frac = povf;
  r.sz_bits_per_value = H + fa.sz_offset + 32.0 * povf;
  r.sz_psnr = 20.0 * lg_vr_eb + 10.0 * log10(3.0);
  r.zfp_total_bits = tb;
  r.zfp_err_sum = errs;
  r.zfp_bits_per_value = (double)tb / (double)fa.n_values;
  r.zfp_mse = mse;
  r.zfp_psnr = mse > 0.0 ? 20.0 * lg_vr - 10.0 * lg_mse : __longlong_as_double(0x7ff0000000000000LL);
  // selection based on the error bound (Lu et al.): lower bit-rate at eb
  r.choice_eb = r.sz_bits_per_value < r.zfp_bits_per_value ? 0 : 1;
  if (!(r.zfp_mse > 0.0) || !(vr > 0.0) || !isfinite(r.zfp_psnr)) {
    r.matched = 0;
    r.sz_bits_matched = r.sz_bits_per_value;
    r.sz_eb_matched = eb;
    r.choice = r.sz_bits_per_value < r.zfp_bits_per_value ? 0 : 1;
  } else {
    const double delta = vr * sqrt(12.0) * pow(10.0, -r.zfp_psnr / 20.0);
    double bm = r.sz_bits_per_value + log2(2.0 * eb / delta);
    if (bm < 0.0) bm = 0.0;
    r.matched = 1;
    r.sz_bits_matched = bm;
    r.sz_eb_matched = delta / 2.0;
    r.choice = bm < r.zfp_bits_per_value ? 0 : 1;
  }
  return r;
}

// value-range derived scalars (Alg. 1 line 2; readings R1, R2)
__device__ __forceinline__ Params make_params(float mn, float mx, int bad, int mode, double eb) {
  Params p;
  p.vmin = mn; p.vmax = mx; p.pad = 0;
  p.vr = (double)mx - (double)mn;
  p.status = bad ? SEL_ENONFINITE : SEL_OK;
  p.eb_abs = (mode == SEL_EB_REL) ? eb * p.vr : eb;
  if (p.status == SEL_OK && mode == SEL_EB_REL && p.vr == 0.0) p.status = SEL_EDEGENERATE;
  p.r_f = __double2float_rn(1.0 / (2.0 * p.eb_abs));
  if (p.status == SEL_OK && (is_nonfinite(p.r_f) || !(p.eb_abs > 0.0))) p.status = SEL_EINVAL;
  int e = 0;
  frexp(p.eb_abs, &e);
  p.minexp = e - 1;
  return p;
}

__device__ __forceinline__ unsigned int ld_acquire(const unsigned int *p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned int *p, unsigned int v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// ============================================================ shared K2 prologue/epilogue
__device__ __forceinline__ void hist_zero(unsigned int *sh) {
  uint4 *s4 = reinterpret_cast<uint4 *>(sh);
  for (int i = threadIdx.x; i < kWinBins / 4; i += blockDim.x) s4[i] = make_uint4(0, 0, 0, 0);
}

__device__ __forceinline__ void hist_flush(const unsigned int *sh, unsigned long long *gh) {
  const uint4 *s4 = reinterpret_cast<const uint4 *>(sh);
  for (int i = threadIdx.x; i < kWinBins / 4; i += blockDim.x) {
    const uint4 c = s4[i];
    unsigned long long *g = gh + (kCenter - kWinHalf) + 4 * i;
    if (c.x) atomicAdd(g + 0, (unsigned long long)c.x);
    if (c.y) atomicAdd(g + 1, (unsigned long long)c.y);
    if (c.z) atomicAdd(g + 2, (unsigned long long)c.z);
    if (c.w) atomicAdd(g + 3, (unsigned long long)c.w);
  }
}

__device__ __forceinline__ void ovf_flush(unsigned int ovf, unsigned long long *gh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ovf += __shfl_xor_sync(0xffffffffu, ovf, o);
  if ((threadIdx.x & 31) == 0 && ovf) atomicAdd(gh + kOvfSlot, (unsigned long long)ovf);
}

// warp-reduce a task's (bits, err) in a fixed shuffle order; lane 0 stores the partial
__device__ __forceinline__ void task_store(Partial *part, int task, uint64_t bits, double err) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    bits += __shfl_down_sync(0xffffffffu, bits, o);
    err += __shfl_down_sync(0xffffffffu, err, o);
  }
  if ((threadIdx.x & 31) == 0) {
    Partial p;
    p.bits = bits;
    p.err = err;
    part[task] = p;
  }
}

__device__ __forceinline__ int next_task(unsigned int *ctr) {
  int t = 0;
  if ((threadIdx.x & 31) == 0) t = (int)atomicAdd(ctr, 1u);
  return __shfl_sync(0xffffffffu, t, 0);
}

}  // namespace sel
