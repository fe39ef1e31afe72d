// sel_kernels.cu -- sm_100a kernels of the SZ/ZFP rate-distortion estimator.
//
//   K1 k_minmax    : value range over the whole field (Alg.1 line 2) and the
//                    derived scalars eb_abs, r_f, minexp (last-block-done finalise)
//   K2 k_estimate  : one fused pass over the processed 4^d blocks.  One thread owns
//                    one block: it loads the block rows (float4, coalesced across the
//                    warp: lanes own consecutive blocks along the fastest axis) plus the
//                    -1 halo, computes the SZ Lorenzo residuals and
//                    quantisation codes into a shared-memory privatised
//                    histogram, then runs ZFP's block pipeline on the same
//                    registers: exponent, block floating point, decorrelating lift,
//                    sequency reorder, negabinary, closed-form group-testing EC bit count
//                    at the fixed-accuracy cut and the gain-weighted
//                    truncation error.
//   K3 k_finalize  : entropy of the 65,536-slot histogram (Eq. entropy), PSNRs
//                     and the Alg.1 selection; re-zeroes the
//                    histogram for the next field.
//
// Arithmetic readings are implemented from the math spec, not
// from the oracle: the two share no code.  Built with -fmad=false, IEEE div/sqrt.
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "sel_internal.h"

namespace sel {

// ============================================================ compile-time tables
template <int D>
struct Tab {
  static constexpr int SIZE = D == 1 ? 4 : (D == 2 ? 16 : 64);
  struct IArr { int v[64]; };
  struct DArr { double v[64]; };
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
  // squared column norms of the inverse lift, per axis (4, 5, 4, 13/4) (reading R14)
  static constexpr DArr make_gain() {
    DArr a{};
    const double g[4] = {4.0, 5.0, 4.0, 3.25};
    for (int n = 0; n < SIZE; ++n) {
      double w = 1.0;
      int r = n;
      for (int d = 0; d < D; ++d) { w *= g[r % 4]; r /= 4; }
      a.v[n] = w;
    }
    return a;
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

// Quantisation code slot (reading R5): q = |d| * r_f in fp32; overflow slot if
// !(q < 32767.5); else round half-even; slot = code + 32767.
__device__ __forceinline__ int quant_slot(float d, float r_f) {
  float q = __fmul_rn(fabsf(d), r_f);
  if (!(q < 32767.5f)) return kOvfSlot;
  int m = __float2int_rn(q);
  return kCenter + (d < 0.0f ? -m : m);
}

// ZFP's forward decorrelating lift on one 4-vector (reading R8): five
// add / arithmetic-shift / subtract stages; exact-arithmetic map is
// A = (1/16)[[4,4,4,4],[5,1,-1,-5],[-4,4,4,-4],[-2,6,-6,2]].
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

// 2^k as a double, k in [-1022, 1023]
__device__ __forceinline__ double pow2d(int k) {
  return __hiloint2double((1023 + k) << 20, 0);
}

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

// ============================================================ K1: value range
template <int THREADS>
__global__ void __launch_bounds__(THREADS) k_minmax(const float *__restrict__ x, int64_t N,
                                                    Workspace ws, int mode, double eb) {
  float mn = INFINITY, mx = -INFINITY;
  int bad = 0;
  const int64_t tid = (int64_t)blockIdx.x * THREADS + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * THREADS;
  int64_t head = (int64_t)(((16u - ((uintptr_t)x & 15u)) & 15u) >> 2);
  if (head > N) head = N;
  for (int64_t i = tid; i < head; i += nth) {
    float v = x[i];
    bad |= is_nonfinite(v); mn = fminf(mn, v); mx = fmaxf(mx, v);
  }
  const float4 *x4 = reinterpret_cast<const float4 *>(x + head);
  const int64_t n4 = (N - head) >> 2;
  int64_t i = tid;
  for (; i + 3 * nth < n4; i += 4 * nth) {
    float4 a = __ldcs(x4 + i), b = __ldcs(x4 + i + nth), c = __ldcs(x4 + i + 2 * nth),
           d = __ldcs(x4 + i + 3 * nth);
    float4 q[4] = {a, b, c, d};
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      bad |= is_nonfinite(q[t].x) | is_nonfinite(q[t].y) | is_nonfinite(q[t].z) | is_nonfinite(q[t].w);
      mn = fminf(mn, fminf(fminf(q[t].x, q[t].y), fminf(q[t].z, q[t].w)));
      mx = fmaxf(mx, fmaxf(fmaxf(q[t].x, q[t].y), fmaxf(q[t].z, q[t].w)));
    }
  }
  for (; i < n4; i += nth) {
    float4 q = __ldcs(x4 + i);
    bad |= is_nonfinite(q.x) | is_nonfinite(q.y) | is_nonfinite(q.z) | is_nonfinite(q.w);
    mn = fminf(mn, fminf(fminf(q.x, q.y), fminf(q.z, q.w)));
    mx = fmaxf(mx, fmaxf(fmaxf(q.x, q.y), fmaxf(q.z, q.w)));
  }
  for (int64_t k = head + 4 * n4 + tid; k < N; k += nth) {
    float v = x[k];
    bad |= is_nonfinite(v); mn = fminf(mn, v); mx = fmaxf(mx, v);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    bad |= __shfl_xor_sync(0xffffffffu, bad, o);
  }
  __shared__ float smn[THREADS / 32], smx[THREADS / 32];
  __shared__ int sbad[THREADS / 32];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) { smn[wid] = mn; smx[wid] = mx; sbad[wid] = bad; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < THREADS / 32; ++w) {
      mn = fminf(mn, smn[w]); mx = fmaxf(mx, smx[w]); bad |= sbad[w];
    }
    ws.mm_part[blockIdx.x] = make_float2(mn, mx);
    ws.mm_flag[blockIdx.x] = bad;
    __threadfence();
    unsigned t = atomicAdd(&ws.tickets[0], 1u);
    last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return;
  // last block: reduce the per-CTA partials, derive the per-field scalars
  __threadfence();
  mn = INFINITY; mx = -INFINITY; bad = 0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += THREADS) {
    float2 p = __ldcg(ws.mm_part + b);
    mn = fminf(mn, p.x); mx = fmaxf(mx, p.y); bad |= __ldcg(ws.mm_flag + b);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    bad |= __shfl_xor_sync(0xffffffffu, bad, o);
  }
  __syncthreads();
  if (lane == 0) { smn[wid] = mn; smx[wid] = mx; sbad[wid] = bad; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < THREADS / 32; ++w) {
      mn = fminf(mn, smn[w]); mx = fmaxf(mx, smx[w]); bad |= sbad[w];
    }
    Params p;
    p.vmin = mn; p.vmax = mx; p.pad = 0;
    p.vr = (double)mx - (double)mn;                       // A1
    p.status = bad ? SEL_ENONFINITE : SEL_OK;
    p.eb_abs = (mode == SEL_EB_REL) ? eb * p.vr : eb;     // A2 (Alg.1 line 2)
    if (p.status == SEL_OK && mode == SEL_EB_REL && p.vr == 0.0) p.status = SEL_EDEGENERATE;
    p.r_f = __double2float_rn(1.0 / (2.0 * p.eb_abs));
    if (p.status == SEL_OK && (is_nonfinite(p.r_f) || !(p.eb_abs > 0.0))) p.status = SEL_EINVAL;
    int e = 0;
    frexp(p.eb_abs, &e);
    p.minexp = e - 1;                                     // floor(log2 eb_abs)
    *ws.params = p;
    ws.tickets[0] = 0;
  }
}

// ============================================================ K2: fused SZ + ZFP pass
template <int D, bool VEC, bool DBG>
__global__ void __launch_bounds__(256) k_estimate(const float *__restrict__ x, Geo g,
                                                  Workspace ws, DebugPtrs dbg) {
  constexpr int SIZE = Tab<D>::SIZE;
  constexpr int PL = D == 3 ? 4 : 1;   // planes per block (axis 0 of the 3-axis view)
  constexpr int RW = D >= 2 ? 4 : 1;   // rows per block   (axis 1)
  extern __shared__ unsigned int sh_hist[];

  const Params prm = *ws.params;
  if (prm.status != SEL_OK) return;
  for (int i = threadIdx.x; i < kWinBins; i += blockDim.x) sh_hist[i] = 0u;
  __syncthreads();

  const float r_f = prm.r_f;
  const int minexp = prm.minexp;
  uint64_t bits_acc = 0;
  double err_acc = 0.0;
  unsigned int ovf = 0;

  const int64_t gstride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < g.n_pb; t += gstride) {
    const int64_t p2 = t % g.npb[2];
    const int64_t q = t / g.npb[2];
    const int64_t p1 = q % g.npb[1];
    const int64_t p0 = q / g.npb[1];
    const int64_t I0 = 4 * p0 * g.s[0], J0 = 4 * p1 * g.s[1], K0 = 4 * p2 * g.s[2];

    float blk[PL][RW][4];
    float dprev[RW][4];
    // ---------------- SZ: Lorenzo on original values, nested differences (R4)
    // halo plane i = I0-1 -> its 2D difference D2 becomes dprev
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
          float d1 = v[c] - (c ? v[c - 1] : h);
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
          blk[p][r][c] = v[c];
          const float d1 = v[c] - (c ? v[c - 1] : h);
          const float d2 = d1 - d1up[c];
          d1up[c] = d1;
          const float d = d2 - dprev[r][c];
          dprev[r][c] = d2;
          const int64_t k = K0 + c;
          const bool real = (i < g.n[0]) && (j < g.n[1]) && (k < g.n[2]);
          const bool origin = (i == 0) && (j == 0) && (k == 0);
          if (real && !origin) {
            const int slot = quant_slot(d, r_f);
            if (slot == kOvfSlot) {
              ++ovf;
            } else {
              const unsigned w = (unsigned)(slot - (kCenter - kWinHalf));
              if (w < (unsigned)kWinBins) atomicAdd(&sh_hist[w], 1u);
              else atomicAdd(&ws.hist[slot], 1ull);
            }
            if constexpr (DBG) dbg.codes[(i * g.n[1] + j) * g.n[2] + k] = slot;
          }
        }
      }
    }

    // ---------------- ZFP: exponent (R9)
    uint32_t mbits = 0;
#pragma unroll
    for (int p = 0; p < PL; ++p)
#pragma unroll
      for (int r = 0; r < RW; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) mbits = max(mbits, __float_as_uint(blk[p][r][c]) & 0x7fffffffu);

    uint32_t bits;
    double E = 0.0;
    int emax;
    int cf[SIZE];
    uint32_t u[SIZE];
    if (mbits == 0u) {              // empty block: 1 header bit, no error
      emax = -127;
      bits = 1u;
      if constexpr (DBG) {
#pragma unroll
        for (int n = 0; n < SIZE; ++n) { cf[n] = 0; u[n] = 0u; }
      }
    } else {
      emax = (int)(mbits >> 23) - 126;
      // block floating point: i = trunc(x 2^(30-emax)), exact (R9)
      if (emax >= -97) {
        const float sc = __uint_as_float((uint32_t)(157 - emax) << 23);
#pragma unroll
        for (int p = 0; p < PL; ++p)
#pragma unroll
          for (int r = 0; r < RW; ++r)
#pragma unroll
            for (int c = 0; c < 4; ++c) cf[(p * RW + r) * 4 + c] = __float2int_rz(__fmul_rn(blk[p][r][c], sc));
      } else {
        const float sc = __uint_as_float((uint32_t)(93 - emax) << 23);
#pragma unroll
        for (int p = 0; p < PL; ++p)
#pragma unroll
          for (int r = 0; r < RW; ++r)
#pragma unroll
            for (int c = 0; c < 4; ++c)
              cf[(p * RW + r) * 4 + c] =
                  __float2int_rz(__fmul_rn(__fmul_rn(blk[p][r][c], 0x1p64f), sc));
      }
      // decorrelating lift along the fastest axis first, then slower (R8)
#pragma unroll
      for (int l = 0; l < SIZE / 4; ++l) fwd_lift(cf[4 * l], cf[4 * l + 1], cf[4 * l + 2], cf[4 * l + 3]);
      if constexpr (D >= 2) {
#pragma unroll
        for (int p = 0; p < PL; ++p)
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
      // sequency reorder + negabinary (R10, R11)
      static_for<0, SIZE>([&](auto J) {
        constexpr int j = decltype(J)::value;
        constexpr int n = Tab<D>::make_perm().v[j];
        u[j] = to_negabinary(cf[n]);
      });
      // fixed-accuracy cut (R12)
      int prec = emax - minexp + 2 * (D + 1);
      prec = prec < 0 ? 0 : (prec > 32 ? 32 : prec);
      const int kmin = 32 - prec;
      if (prec == 0) {
        bits = 1u;
      } else {
        // closed-form group-testing count (R13): with O_j = u_j | ... | u_L,
        //   GT = sum_j max(bitlen O_j, kmin) - SIZE*kmin
        //      + #{j : u_j > max(O_j >> 1, 2^kmin - 1)}
        //      + 32 - max(bitlen u_L, kmin) - [bitlen u_L > kmin]
        const uint32_t thr = (1u << kmin) - 1u;
        uint32_t O = 0u;
        int t1 = 0, t2 = 0;
#pragma unroll
        for (int j = SIZE - 1; j >= 0; --j) {
          O |= u[j];
          const int bl = 32 - __clz(O);
          t1 += max(bl, kmin);
          t2 += (u[j] > max(O >> 1, thr)) ? 1 : 0;
        }
        const int blL = 32 - __clz(u[SIZE - 1]);
        const int t3 = 32 - max(blL, kmin) - (blL > kmin ? 1 : 0);
        bits = (uint32_t)(9 + t1 - SIZE * kmin + t2 + t3);
      }
      // gain-weighted truncation error (R14): e_j = value of the dropped
      // negabinary digits = (lo ^ M) - M with M the digit-sign mask below kmin
      const uint32_t low = kmin >= 32 ? 0xffffffffu : ((1u << kmin) - 1u);
      const uint32_t Mk = 0xAAAAAAAAu & low;
      static_for<0, SIZE>([&](auto J) {
        constexpr int j = decltype(J)::value;
        const uint32_t lo = u[j] & low;
        const long long e = (long long)(lo ^ Mk) - (long long)Mk;
        const double ed = (double)e;
        constexpr int n = Tab<D>::make_perm().v[j];
        constexpr double w = Tab<D>::make_gain().v[n];
        E = __dadd_rn(E, __dmul_rn(w, __dmul_rn(ed, ed)));
      });
      E = __dmul_rn(E, pow2d(2 * (emax - 30)));
    }
    bits_acc += bits;
    err_acc += E;
    if constexpr (DBG) {
      dbg.emax[t] = emax;
      dbg.bits[t] = bits;
      dbg.err[t] = E;
#pragma unroll
      for (int n = 0; n < SIZE; ++n) {
        dbg.coef[t * SIZE + n] = cf[n];
        dbg.uword[t * SIZE + n] = u[n];
      }
    }
  }

  // ---------------- per-CTA reduction in a fixed order (deterministic)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    bits_acc += __shfl_down_sync(0xffffffffu, bits_acc, o);
    err_acc += __shfl_down_sync(0xffffffffu, err_acc, o);
    ovf += __shfl_down_sync(0xffffffffu, ovf, o);
  }
  __shared__ uint64_t sb[8];
  __shared__ double se[8];
  __shared__ unsigned int so[8];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) { sb[wid] = bits_acc; se[wid] = err_acc; so[wid] = ovf; }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int nw = blockDim.x >> 5;
    for (int w = 1; w < nw; ++w) { bits_acc += sb[w]; err_acc += se[w]; ovf += so[w]; }
    Partial pr;
    pr.bits = bits_acc;
    pr.err = err_acc;
    ws.est_part[blockIdx.x] = pr;
    if (ovf) atomicAdd(&ws.hist[kOvfSlot], (unsigned long long)ovf);
  }
  // flush the privatised window
  for (int i = threadIdx.x; i < kWinBins; i += blockDim.x) {
    const unsigned int c = sh_hist[i];
    if (c) atomicAdd(&ws.hist[kCenter - kWinHalf + i], (unsigned long long)c);
  }
}

// ============================================================ K3: finalize
__global__ void __launch_bounds__(kFinThreads) k_finalize(Workspace ws, FinalizeArgs fa,
                                                         sel_result *out,
                                                         unsigned long long *dbg_hist) {
  const Params prm = *ws.params;
  const double Nsz = (double)fa.n_sz;
  const double lN = log2(Nsz);
  double acc = 0.0;
  constexpr int PER = kNSlots / kFinCTAs;
  for (int s = blockIdx.x * PER + threadIdx.x; s < (blockIdx.x + 1) * PER; s += kFinThreads) {
    const unsigned long long c = ws.hist[s];
    if (c) {
      const double cd = (double)c;
      acc += cd * (lN - log2(cd));          // c log2(N/c): exactly 0 for a single slot
      ws.hist[s] = 0ull;
      if (dbg_hist) dbg_hist[s] = c;
    } else if (dbg_hist) {
      dbg_hist[s] = 0ull;
    }
    if (s == kOvfSlot) *ws.fin_ovf = c;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  __shared__ double sacc[kFinThreads / 32];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) sacc[wid] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < kFinThreads / 32; ++w) acc += sacc[w];
    ws.fin_part[blockIdx.x] = acc;
    __threadfence();
    unsigned t = atomicAdd(&ws.tickets[1], 1u);
    last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!last || threadIdx.x != 0) return;
  __threadfence();
  ws.tickets[1] = 0;

  sel_result r = {};
  r.status = prm.status;
  r.value_range = prm.vr;
  r.eb_abs = prm.eb_abs;
  r.minexp = prm.minexp;
  r.r_f = prm.r_f;
  r.n_sz_points = fa.n_sz;
  r.n_values = fa.n_values;
  r.n_blocks = fa.n_blocks;
  if (r.status == SEL_OK && fa.n_sz == 0) r.status = SEL_EDEGENERATE;   // single-value field
  if (r.status == SEL_OK) {
    double S = 0.0;
    for (int b = 0; b < kFinCTAs; ++b) S += __ldcg(ws.fin_part + b);
    uint64_t bits = 0;
    double err = 0.0;
    for (int b = 0; b < fa.est_ctas; ++b) {
      bits += __ldcg(&ws.est_part[b].bits);
      err += __ldcg(&ws.est_part[b].err);
    }
    const double vr = prm.vr, eb = prm.eb_abs;
    const double H = S / Nsz;                                        // Eq. entropy
    const double povf = (double)__ldcg(ws.fin_ovf) / Nsz;
    r.sz_entropy = H;
    r.sz_overflow_frac = povf;
    r.sz_bits_per_value = H + fa.sz_offset + 32.0 * povf;            // P:402, R6
    r.sz_psnr = 20.0 * log10(vr / eb) + 10.0 * log10(3.0);           // Eq. psnr-sz
    r.zfp_total_bits = bits;
    r.zfp_err_sum = err;
    r.zfp_bits_per_value = (double)bits / (double)fa.n_values;
    r.zfp_mse = err / (double)fa.n_values;
    r.zfp_psnr = r.zfp_mse > 0.0 ? 20.0 * log10(vr) - 10.0 * log10(r.zfp_mse)
                                 : __longlong_as_double(0x7ff0000000000000LL);
    // Alg.1 lines 7-10 (R16)
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
  }
  *out = r;
}

// ============================================================ launchers
int minmax_ctas(int64_t N, int sm_count) {
  int64_t want = (N + 512 * 16 - 1) / (512 * 16);
  int64_t cap = 2LL * sm_count;
  return (int)(want < 1 ? 1 : (want > cap ? cap : want));
}

int launch_minmax(const float *x, int64_t N, int ctas, const Workspace &ws, int mode, double eb,
                  cudaStream_t st) {
  k_minmax<512><<<ctas, 512, 0, st>>>(x, N, ws, mode, eb);
  return cudaGetLastError() == cudaSuccess ? SEL_OK : SEL_ECUDA;
}

template <int D, bool VEC, bool DBG>
static const void *est_fn() { return (const void *)k_estimate<D, VEC, DBG>; }

static const void *pick_est(int D, bool vec, bool dbg) {
  if (D == 1) return vec ? (dbg ? est_fn<1, true, true>() : est_fn<1, true, false>())
                         : (dbg ? est_fn<1, false, true>() : est_fn<1, false, false>());
  if (D == 2) return vec ? (dbg ? est_fn<2, true, true>() : est_fn<2, true, false>())
                         : (dbg ? est_fn<2, false, true>() : est_fn<2, false, false>());
  return vec ? (dbg ? est_fn<3, true, true>() : est_fn<3, true, false>())
             : (dbg ? est_fn<3, false, true>() : est_fn<3, false, false>());
}

static constexpr int kEstThreads = 256;
static constexpr size_t kEstSmem = kWinBins * sizeof(unsigned int);

int estimate_max_ctas(const Geo &g, int debug, int sm_count) {
  const void *fn = pick_est(g.ndims, g.vec != 0, debug != 0);
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kEstSmem) !=
      cudaSuccess)
    return -1;
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kEstThreads, kEstSmem) != cudaSuccess)
    return -1;
  if (occ < 1) occ = 1;
  int64_t want = (g.n_pb + kEstThreads - 1) / kEstThreads;
  int64_t cap = (int64_t)occ * sm_count;
  return (int)(want < 1 ? 1 : (want > cap ? cap : want));
}

int launch_estimate(const float *x, const Geo &g, int ctas, const Workspace &ws,
                    const DebugPtrs *dbg, cudaStream_t st) {
  DebugPtrs d{};
  if (dbg) d = *dbg;
  const void *fn = pick_est(g.ndims, g.vec != 0, dbg != nullptr);
  Geo gg = g;
  Workspace w = ws;
  void *args[] = {(void *)&x, (void *)&gg, (void *)&w, (void *)&d};
  cudaError_t e = cudaLaunchKernel(fn, dim3(ctas), dim3(kEstThreads), args, kEstSmem, st);
  return e == cudaSuccess ? SEL_OK : SEL_ECUDA;
}

int launch_finalize(const Workspace &ws, const FinalizeArgs &fa, sel_result *d_out,
                    unsigned long long *dbg_hist, cudaStream_t st) {
  k_finalize<<<kFinCTAs, kFinThreads, 0, st>>>(ws, fa, d_out, dbg_hist);
  return cudaGetLastError() == cudaSuccess ? SEL_OK : SEL_ECUDA;
}

}  // namespace sel
