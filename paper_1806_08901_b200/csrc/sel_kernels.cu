// sel_kernels.cu -- sm_100a kernels of the SZ/ZFP rate-distortion estimator.
//
//   K1 k_minmax   : value range over the whole field (Alg.1 line 2) and the derived
//                   scalars eb_abs, r_f, minexp (last-block-done).
//   K2 k_march    : full-field fused SZ+ZFP pass for 2D/3D fields.  One warp owns 32
//                   consecutive 4^d blocks along the fastest axis (lane = block, float4
//                   rows -> 512 B coalesced per warp row) and MARCHES along the slowest
//                   block axis, carrying the Lorenzo partial differences of the previous
//                   plane/row in registers, so every value is loaded once (+ one halo row
//                   per plane); the left halo comes from lane-1 by shuffle.
//      k_estimate : generic fused pass (sampled blocks, 1D): one thread per processed
//                   block with explicit halo loads.
//      Both feed one shared-memory privatised histogram window per CTA
//      and run the same per-block ZFP routine (zfp_block): exponent, block floating
//      point, decorrelating lift, sequency reorder, negabinary, closed-form group-testing
//      EC bit count at the fixed-accuracy cut and the gain-weighted
//      truncation error, accumulated exactly in integers per weight class.
//   K3 k_finalize : entropy of the 65,536-slot histogram (Eq. entropy), PSNRs
//                    and the Alg.1 selection; re-zeroes state.
//
// Work decomposition is dynamic (a task counter) but every floating-point partial is
// produced per TASK and summed in task order, so results are bit-reproducible.
// Readings are implemented from the math spec, not from the
// oracle: the two share no code.  Built with -fmad=false, IEEE div/sqrt, no fast math.
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "sel_device.cuh"

#ifndef SEL_MARCH3_MINB
#define SEL_MARCH3_MINB 1   // CTAs/SM the 3D march kernel is register-capped for
#endif

namespace sel {

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
  constexpr int U = 8;
  int64_t i = tid;
  for (; i + (U - 1) * nth < n4; i += U * nth) {
    float4 q[U];
#pragma unroll
    for (int t = 0; t < U; ++t) q[t] = __ldg(x4 + i + t * nth);
#pragma unroll
    for (int t = 0; t < U; ++t) {
      bad |= is_nonfinite(q[t].x) | is_nonfinite(q[t].y) | is_nonfinite(q[t].z) | is_nonfinite(q[t].w);
      mn = fminf(mn, fminf(fminf(q[t].x, q[t].y), fminf(q[t].z, q[t].w)));
      mx = fmaxf(mx, fmaxf(fmaxf(q[t].x, q[t].y), fmaxf(q[t].z, q[t].w)));
    }
  }
  for (; i < n4; i += nth) {
    float4 q = __ldg(x4 + i);
    bad |= is_nonfinite(q.x) | is_nonfinite(q.y) | is_nonfinite(q.z) | is_nonfinite(q.w);
    mn = fminf(mn, fminf(fminf(q.x, q.y), fminf(q.z, q.w)));
    mx = fmaxf(mx, fmaxf(fmaxf(q.x, q.y), fmaxf(q.z, q.w)));
  }
  for (int64_t k = head + 4 * n4 + tid; k < N; k += nth) {
    float v = x[k];
    bad |= is_nonfinite(v); mn = fminf(mn, v); mx = fmaxf(mx, v);
  }
  grid_dep_launch();   // let the fused pass stage its prologue (PDL)
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
    const Params p = make_params(mn, mx, bad, mode, eb);
    *ws.params = p;    // this field's own params slot
    ws.tickets[0] = 0;
  }
}

// ============================================================ K2a: marching full-field pass
template <bool VEC>
__device__ __forceinline__ void mrow(const float *__restrict__ x, int64_t rowoff, int64_t K0,
                                     int64_t n2, bool active, int lane, float (&v)[4], float &h) {
  const float *row = x + rowoff;
  float hl = 0.0f;
  if (lane == 0 && K0 > 0) hl = __ldg(row + K0 - 1);
  if (active) {
    if constexpr (VEC) {
      const float4 q = __ldg(reinterpret_cast<const float4 *>(row + K0));
      v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
    } else {
#pragma unroll
      for (int c = 0; c < 4; ++c) v[c] = __ldg(row + (K0 + c < n2 ? K0 + c : n2 - 1));
    }
  } else {
#pragma unroll
    for (int c = 0; c < 4; ++c) v[c] = 0.0f;
  }
  const float hs = __shfl_up_sync(0xffffffffu, v[3], 1);
  h = lane == 0 ? hl : hs;
}

template <int D, bool VEC, bool DBG>
__global__ void __launch_bounds__(256, (D == 3 ? SEL_MARCH3_MINB : 3)) k_march(const float *__restrict__ x, MarchGeo mg,
                                               Workspace ws, DebugPtrs dbg) {
  static_assert(D == 2 || D == 3, "march kernel is for 2D/3D fields");
  constexpr int SZ = Tab<D>::SIZE;
  constexpr int PL = D == 3 ? 4 : 1;
  extern __shared__ unsigned int sh_hist[];
  hist_zero(sh_hist);
  grid_dep_wait();                 // params come from k_minmax
  __syncthreads();
  const Params prm = *ws.params;
  if (prm.status != SEL_OK) return;
  const float r_f = prm.r_f;
  const int minexp = prm.minexp;
  const int lane = threadIdx.x & 31;
  const int64_t n0 = mg.n[0], n1 = mg.n[1], n2 = mg.n[2];
  const int nbm = (int)(D == 3 ? mg.nb[0] : mg.nb[1]);     // marching axis blocks
  unsigned int ovf = 0;

  for (int task = next_task(ws.task_ctr); task < mg.ntasks; task = next_task(ws.task_ctr)) {
    const int chunk = task % mg.nchunk;
    const int rest = task / mg.nchunk;
    const int other = rest % mg.nother;
    const int seg = rest / mg.nother;
    const int64_t bk = (int64_t)chunk * 32 + lane;
    const bool active = bk < mg.nb[2];
    const int64_t K0 = 4 * bk;
    const int cm = !active ? 0 : (n2 - K0 >= 4 ? 0xF : (int)((1u << (n2 - K0)) - 1u));
    const int bm0 = seg * mg.L;
    const int bm1 = min(bm0 + mg.L, nbm);
    uint64_t tbits = 0;
    double terr = 0.0;

    if constexpr (D == 3) {
      const int64_t J0 = 4 * (int64_t)other;
      float carry[4][4];   // D2 of the previous plane
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) carry[r][c] = 0.0f;
      auto plane_d1up = [&](int64_t ic, float (&d1up)[4]) {
        float v[4], h;
        if (J0 > 0) {
          mrow<VEC>(x, (ic * n1 + (J0 - 1)) * n2, K0, n2, active, lane, v, h);
#pragma unroll
          for (int c = 0; c < 4; ++c) d1up[c] = v[c] - (c ? v[c - 1] : h);
        } else {
#pragma unroll
          for (int c = 0; c < 4; ++c) d1up[c] = 0.0f;
        }
      };
      if (bm0 > 0) {     // carry from plane 4*bm0 - 1
        const int64_t ic = 4 * (int64_t)bm0 - 1;
        float d1up[4];
        plane_d1up(ic, d1up);
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int64_t jc = min(J0 + r, n1 - 1);
          float v[4], h;
          mrow<VEC>(x, (ic * n1 + jc) * n2, K0, n2, active, lane, v, h);
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const float d1 = v[c] - (c ? v[c - 1] : h);
            carry[r][c] = d1 - d1up[c];
            d1up[c] = d1;
          }
        }
      }
      for (int bm = bm0; bm < bm1; ++bm) {
        float blk[SZ];
#pragma unroll
        for (int p = 0; p < PL; ++p) {
          const int64_t i = 4 * (int64_t)bm + p;
          const int64_t ic = min(i, n0 - 1);
          float d1up[4];
          plane_d1up(ic, d1up);
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            const int64_t j = J0 + r;
            const int64_t jc = min(j, n1 - 1);
            float v[4], h;
            mrow<VEC>(x, (ic * n1 + jc) * n2, K0, n2, active, lane, v, h);
            const bool rowok = (i < n0) && (j < n1);
            const bool orow = (i == 0) && (j == 0) && (K0 == 0);
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              blk[(p * 4 + r) * 4 + c] = v[c];
              const float d1 = v[c] - (c ? v[c - 1] : h);
              const float d2 = d1 - d1up[c];
              d1up[c] = d1;
              const float d = d2 - carry[r][c];
              carry[r][c] = d2;
              const bool valid = rowok && ((cm >> c) & 1) && !(c == 0 && orow);
              sz_put<DBG>(d, r_f, valid, sh_hist, ws.hist, ovf,
                          DBG ? dbg.codes + (i * n1 + j) * n2 + K0 + c : nullptr);
            }
          }
        }
        if (active) {
          uint32_t bits;
          double E;
          int emax;
          int cf[SZ];
          uint32_t u[SZ];
          zfp_block<D, DBG>(blk, minexp, bits, E, emax, cf, u);
          tbits += bits;
          terr += E;
          if constexpr (DBG) {
            const int64_t t = ((int64_t)bm * mg.nb[1] + other) * mg.nb[2] + bk;
            dbg.emax[t] = emax; dbg.bits[t] = bits; dbg.err[t] = E;
#pragma unroll
            for (int n = 0; n < SZ; ++n) { dbg.coef[t * SZ + n] = cf[n]; dbg.uword[t * SZ + n] = u[n]; }
          }
        }
      }
    } else {   // D == 2: rows of the 2D field are axis 1 of the view
      float carry[4];   // D1 of the previous row
#pragma unroll
      for (int c = 0; c < 4; ++c) carry[c] = 0.0f;
      if (bm0 > 0) {
        const int64_t j = 4 * (int64_t)bm0 - 1;
        float v[4], h;
        mrow<VEC>(x, j * n2, K0, n2, active, lane, v, h);
#pragma unroll
        for (int c = 0; c < 4; ++c) carry[c] = v[c] - (c ? v[c - 1] : h);
      }
      for (int bm = bm0; bm < bm1; ++bm) {
        float blk[SZ];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int64_t j = 4 * (int64_t)bm + r;
          const int64_t jc = min(j, n1 - 1);
          float v[4], h;
          mrow<VEC>(x, jc * n2, K0, n2, active, lane, v, h);
          const bool rowok = j < n1;
          const bool orow = (j == 0) && (K0 == 0);
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            blk[r * 4 + c] = v[c];
            const float d1 = v[c] - (c ? v[c - 1] : h);
            const float d = d1 - carry[c];
            carry[c] = d1;
            const bool valid = rowok && ((cm >> c) & 1) && !(c == 0 && orow);
            sz_put<DBG>(d, r_f, valid, sh_hist, ws.hist, ovf,
                        DBG ? dbg.codes + j * n2 + K0 + c : nullptr);
          }
        }
        if (active) {
          uint32_t bits;
          double E;
          int emax;
          int cf[SZ];
          uint32_t u[SZ];
          zfp_block<D, DBG>(blk, minexp, bits, E, emax, cf, u);
          tbits += bits;
          terr += E;
          if constexpr (DBG) {
            const int64_t t = (int64_t)bm * mg.nb[2] + bk;
            dbg.emax[t] = emax; dbg.bits[t] = bits; dbg.err[t] = E;
#pragma unroll
            for (int n = 0; n < SZ; ++n) { dbg.coef[t * SZ + n] = cf[n]; dbg.uword[t * SZ + n] = u[n]; }
          }
        }
      }
    }
    task_store(ws.task_part, task, tbits, terr);
  }
  ovf_flush(ovf, ws.hist);
  __syncthreads();
  hist_flush(sh_hist, ws.hist);
}

// ============================================================ K2b: generic pass (sampled, 1D)
// One processed block t (row-major over processed blocks): SZ residuals of its real points
// with neighbours from the full field (R4, R5: codes into the smem window sh_hist or the
// global histogram), then the ZFP block (R8-R14).  Shared by k_estimate and k_small.
template <int D, bool VEC, bool DBG>
__device__ __forceinline__ void block_estimate(const float *__restrict__ x, const Geo &g, int64_t t, float r_f,
                                               int minexp, unsigned int *sh_hist, unsigned long long *gh,
                                               unsigned int &ovf, const DebugPtrs &dbg, uint32_t &bits,
                                               double &E) {
  constexpr int SZ = Tab<D>::SIZE;
  constexpr int PL = D == 3 ? 4 : 1;   // planes per block (axis 0 of the 3-axis view)
  constexpr int RW = D >= 2 ? 4 : 1;   // rows per block   (axis 1)
  const int64_t p2 = t % g.npb[2];
  const int64_t q = t / g.npb[2];
  const int64_t p1 = q % g.npb[1];
  const int64_t p0 = q / g.npb[1];
  const int64_t I0 = 4 * p0 * g.s[0], J0 = 4 * p1 * g.s[1], K0 = 4 * p2 * g.s[2];

  float blk[SZ];
  float dprev[RW][4];
  // ---------------- SZ: Lorenzo on original values, nested differences (R4)
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
        blk[(p * RW + r) * 4 + c] = v[c];
        const float d1 = v[c] - (c ? v[c - 1] : h);
        const float d2 = d1 - d1up[c];
        d1up[c] = d1;
        const float d = d2 - dprev[r][c];
        dprev[r][c] = d2;
        const int64_t k = K0 + c;
        const bool real = (i < g.n[0]) && (j < g.n[1]) && (k < g.n[2]);
        const bool origin = (i == 0) && (j == 0) && (k == 0);
        sz_put<DBG>(d, r_f, real && !origin, sh_hist, gh, ovf,
                    DBG ? dbg.codes + (i * g.n[1] + j) * g.n[2] + k : nullptr);
      }
    }
  }
  int emax;
  int cf[SZ];
  uint32_t u[SZ];
  zfp_block<D, DBG>(blk, minexp, bits, E, emax, cf, u);
  if constexpr (DBG) {
    dbg.emax[t] = emax;
    dbg.bits[t] = bits;
    dbg.err[t] = E;
#pragma unroll
    for (int n = 0; n < SZ; ++n) {
      dbg.coef[t * SZ + n] = cf[n];
      dbg.uword[t * SZ + n] = u[n];
    }
  }
}

template <int D, bool VEC, bool DBG>
__global__ void __launch_bounds__(256) k_estimate(const float *__restrict__ x, Geo g,
                                                  Workspace ws, DebugPtrs dbg) {
  extern __shared__ unsigned int sh_hist[];
  hist_zero(sh_hist);
  grid_dep_wait();
  __syncthreads();
  const Params prm = *ws.params;
  if (prm.status != SEL_OK) return;
  const float r_f = prm.r_f;
  const int minexp = prm.minexp;
  unsigned int ovf = 0;
  uint64_t bits_acc = 0;
  double err_acc = 0.0;

  const int64_t gstride = (int64_t)gridDim.x * blockDim.x;
  // static thread -> block mapping; the per-CTA partial is this CTA's "task"
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < g.n_pb; t += gstride) {
    uint32_t bits;
    double E;
    block_estimate<D, VEC, DBG>(x, g, t, r_f, minexp, sh_hist, ws.hist, ovf, dbg, bits, E);
    bits_acc += bits;
    err_acc += E;
  }
  // per-CTA partial in a fixed order (deterministic): warp tree, then warps in order
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    bits_acc += __shfl_down_sync(0xffffffffu, bits_acc, o);
    err_acc += __shfl_down_sync(0xffffffffu, err_acc, o);
  }
  __shared__ uint64_t sb[8];
  __shared__ double se[8];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) { sb[wid] = bits_acc; se[wid] = err_acc; }
  ovf_flush(ovf, ws.hist);
  __syncthreads();
  if (threadIdx.x == 0) {
    const int nw = blockDim.x >> 5;
    for (int w = 1; w < nw; ++w) { bits_acc += sb[w]; err_acc += se[w]; }
    Partial pr;
    pr.bits = bits_acc;
    pr.err = err_acc;
    ws.task_part[blockIdx.x] = pr;
  }
  hist_flush(sh_hist, ws.hist);
}

// ============================================================ K3: finalize
__global__ void __launch_bounds__(kFinThreads) k_finalize(Workspace ws, FinalizeArgs fa,
                                                         sel_result *out,
                                                         unsigned long long *dbg_hist) {
  grid_dep_wait();
  const Params prm = *ws.params;
  const double Nsz = (double)fa.n_sz;
  const double lN = log2(Nsz);
  double acc = 0.0;
  unsigned long long hcnt = 0;                       // device count of the slice's codes
  constexpr int PER = kNSlots / kFinCTAs;            // 1024 slots per CTA
  constexpr int SPT = PER / kFinThreads;             // slots per thread, all loads in flight
  unsigned long long cs[SPT];
#pragma unroll
  for (int k = 0; k < SPT; ++k) cs[k] = __ldcg(ws.hist + blockIdx.x * PER + k * kFinThreads + threadIdx.x);
#pragma unroll
  for (int k = 0; k < SPT; ++k) {
    const int s = blockIdx.x * PER + k * kFinThreads + threadIdx.x;
    const unsigned long long c = cs[k];
    hcnt += c;
    if (c) {
      const double cd = (double)c;
      acc += cd * (lN - log2(cd));          // c log2(N/c): exactly 0 for a single slot
      ws.hist[s] = 0ull;
    }
    if (dbg_hist) dbg_hist[s] = c;
    if (s == kOvfSlot) *ws.fin_ovf = c;
  }
  // this CTA's contiguous slice of the task partials, fixed order
  uint64_t bits = 0;
  double err = 0.0;
  {
    const int per = (fa.ntasks + kFinCTAs - 1) / kFinCTAs;
    const int t0 = blockIdx.x * per, t1 = min(t0 + per, fa.ntasks);
#pragma unroll 4
    for (int t = t0 + threadIdx.x; t < t1; t += kFinThreads) {
      bits += __ldcg(&ws.task_part[t].bits);
      err += __ldcg(&ws.task_part[t].err);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    acc += __shfl_down_sync(0xffffffffu, acc, o);
    err += __shfl_down_sync(0xffffffffu, err, o);
    bits += __shfl_down_sync(0xffffffffu, bits, o);
    hcnt += __shfl_down_sync(0xffffffffu, hcnt, o);
  }
  if ((threadIdx.x & 31) == 0 && hcnt) atomicAdd(ws.fin_ovf + 1, hcnt);   // exact integer total
  __shared__ double sacc[kFinThreads / 32], serr[kFinThreads / 32];
  __shared__ uint64_t sbits[kFinThreads / 32];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) { sacc[wid] = acc; serr[wid] = err; sbits[wid] = bits; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < kFinThreads / 32; ++w) { acc += sacc[w]; err += serr[w]; bits += sbits[w]; }
    ws.fin_part[blockIdx.x] = acc;
    ws.fin_err[blockIdx.x] = err;
    ws.fin_bits[blockIdx.x] = bits;
    __threadfence();
    unsigned t = atomicAdd(&ws.tickets[1], 1u);
    last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return;
  // ---- last CTA: fixed-order reduction of the 64 CTA partials (warps 0-1), and the
  // independent transcendentals spread over threads, then thread 0 assembles the result
  __threadfence();
  __shared__ double sfin[4];
  __shared__ uint64_t sfb[2];
  __shared__ double slog[3];
  if (threadIdx.x < kFinCTAs) {
    double a = __ldcg(ws.fin_part + threadIdx.x), e = __ldcg(ws.fin_err + threadIdx.x);
    uint64_t tb = __ldcg(ws.fin_bits + threadIdx.x);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a += __shfl_down_sync(0xffffffffu, a, o);
      e += __shfl_down_sync(0xffffffffu, e, o);
      tb += __shfl_down_sync(0xffffffffu, tb, o);
    }
    if (lane == 0) { sfin[wid * 2] = a; sfin[wid * 2 + 1] = e; sfb[wid] = tb; }
  }
  __syncthreads();
  const double vr = prm.vr, eb = prm.eb_abs;
  const double errs = sfin[1] + sfin[3];
  const double mse = errs / (double)fa.n_values;
  if (threadIdx.x == 32) slog[0] = log10(vr / eb);
  if (threadIdx.x == 64) slog[1] = log10(vr);
  if (threadIdx.x == 96) slog[2] = mse > 0.0 ? log10(mse) : 0.0;
  __syncthreads();
  if (threadIdx.x != 0) return;
  ws.tickets[1] = 0;
  *ws.task_ctr = 0;

  const double S = sfin[0] + sfin[2];
  const uint64_t tb = sfb[0] + sfb[1];
  const uint64_t hc = __ldcg(ws.fin_ovf + 1);
  ws.fin_ovf[1] = 0ull;
  sel_result r = assemble_result(prm, S, errs, tb, __ldcg(ws.fin_ovf), hc, fa, slog[0], slog[1], slog[2]);
  *out = r;
}

// ============================================================ launchers
static cudaError_t launch_pdl(const void *fn, dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              void **args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelExC(&cfg, fn, args);
}

// One 256-thread CTA per SM at most: small enough (regs, no smem) to co-reside with the
// persistent fused-pass CTA, so the batch pipeline can overlap the two.
int minmax_ctas(int64_t N, int sm_count) {
  int64_t want = (N + 256 * 32 - 1) / (256 * 32);
  int64_t cap = 4 * (int64_t)sm_count;   // 4 CTAs per SM: 128 KB of loads in flight per SM
  return (int)(want < 1 ? 1 : (want > cap ? cap : want));
}

int launch_minmax(const float *x, int64_t N, int ctas, const Workspace &ws, int mode, double eb,
                  cudaStream_t st) {
  k_minmax<256><<<ctas, 256, 0, st>>>(x, N, ws, mode, eb);
  return cudaGetLastError() == cudaSuccess ? SEL_OK : SEL_ECUDA;
}

template <int D, bool VEC, bool DBG>
static const void *est_fn() { return (const void *)k_estimate<D, VEC, DBG>; }
template <int D, bool VEC, bool DBG>
static const void *march_fn() { return (const void *)k_march<D, VEC, DBG>; }

static const void *pick_kernel(int D, bool vec, bool dbg, bool march) {
  if (march) {
    if (D == 2) return vec ? (dbg ? march_fn<2, true, true>() : march_fn<2, true, false>())
                           : (dbg ? march_fn<2, false, true>() : march_fn<2, false, false>());
    return vec ? (dbg ? march_fn<3, true, true>() : march_fn<3, true, false>())
               : (dbg ? march_fn<3, false, true>() : march_fn<3, false, false>());
  }
  if (D == 1) return vec ? (dbg ? est_fn<1, true, true>() : est_fn<1, true, false>())
                         : (dbg ? est_fn<1, false, true>() : est_fn<1, false, false>());
  if (D == 2) return vec ? (dbg ? est_fn<2, true, true>() : est_fn<2, true, false>())
                         : (dbg ? est_fn<2, false, true>() : est_fn<2, false, false>());
  return vec ? (dbg ? est_fn<3, true, true>() : est_fn<3, true, false>())
             : (dbg ? est_fn<3, false, true>() : est_fn<3, false, false>());
}

static constexpr int kEstThreads = 256;
static constexpr size_t kEstSmem = kWinBins * sizeof(unsigned int);

bool use_march(const Geo &g) {
  return g.ndims >= 2 && g.s[0] == 1 && g.s[1] == 1 && g.s[2] == 1;
}

int occupancy(const Geo &g, int debug, int *occ_out) {
  const void *fn = pick_kernel(g.ndims, g.vec != 0, debug != 0, use_march(g));
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kEstSmem) !=
      cudaSuccess)
    return SEL_ECUDA;
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kEstThreads, kEstSmem) != cudaSuccess)
    return SEL_ECUDA;
  *occ_out = occ < 1 ? 1 : occ;
  return SEL_OK;
}

// Work decomposition for the fused pass (host): grid size and, for the marching
// kernel, the segment length L (block layers per warp task).
int plan_estimate(const Geo &g, int debug, int sm_count, EstLaunch *el) {
  int occ = 0;
  int rc = occupancy(g, debug, &occ);
  if (rc) return rc;
  el->march = use_march(g);
  if (el->march) {
    MarchGeo &m = el->mg;
    for (int a = 0; a < 3; ++a) { m.n[a] = g.n[a]; m.nb[a] = g.nb[a]; }
    const int64_t nbm = g.ndims == 3 ? g.nb[0] : g.nb[1];
    m.nchunk = (int)((g.nb[2] + 31) / 32);
    m.nother = g.ndims == 3 ? (int)g.nb[1] : 1;
    const int64_t resident_warps = (int64_t)occ * sm_count * (kEstThreads / 32);
    const int64_t cols = (int64_t)m.nchunk * m.nother;
    int64_t segs = (4 * resident_warps + cols - 1) / cols;
    if (segs < 1) segs = 1;
    int64_t L = (nbm + segs - 1) / segs;
    if (L < 1) L = 1;
    if (L > 32) L = 32;
    m.L = (int)L;
    m.nseg = (int)((nbm + L - 1) / L);
    const int64_t nt = (int64_t)m.nseg * cols;
    if (nt > (int64_t)1 << 30) return SEL_EINVAL;
    m.ntasks = (int)nt;
    const int64_t want = (nt + (kEstThreads / 32) - 1) / (kEstThreads / 32);
    const int64_t cap = (int64_t)occ * sm_count;
    el->ctas = (int)(want < cap ? want : cap);
    el->ntasks = m.ntasks;
  } else {
    const int64_t want = (g.n_pb + kEstThreads - 1) / kEstThreads;
    const int64_t cap = (int64_t)occ * sm_count;
    el->ctas = (int)(want < 1 ? 1 : (want > cap ? cap : want));
    el->ntasks = el->ctas;
  }
  if (el->ctas < 1) el->ctas = 1;
  return SEL_OK;
}

int launch_estimate(const float *x, const Geo &g, const EstLaunch &el, const Workspace &ws,
                    const DebugPtrs *dbg, cudaStream_t st) {
  DebugPtrs d{};
  if (dbg) d = *dbg;
  const void *fn = pick_kernel(g.ndims, g.vec != 0, dbg != nullptr, el.march);
  Geo gg = g;
  MarchGeo mg = el.mg;
  Workspace w = ws;
  void *args_e[] = {(void *)&x, (void *)&gg, (void *)&w, (void *)&d};
  void *args_m[] = {(void *)&x, (void *)&mg, (void *)&w, (void *)&d};
  cudaError_t e = launch_pdl(fn, dim3(el.ctas), dim3(kEstThreads), kEstSmem, st,
                             el.march ? args_m : args_e);
  return e == cudaSuccess ? SEL_OK : SEL_ECUDA;
}

int launch_finalize(const Workspace &ws, const FinalizeArgs &fa, sel_result *d_out,
                    unsigned long long *dbg_hist, cudaStream_t st) {
  Workspace w = ws;
  FinalizeArgs f = fa;
  void *args[] = {(void *)&w, (void *)&f, (void *)&d_out, (void *)&dbg_hist};
  return launch_pdl((const void *)k_finalize, dim3(kFinCTAs), dim3(kFinThreads), 0, st, args) ==
                 cudaSuccess
             ? SEL_OK : SEL_ECUDA;
}

// ============================================================ small single field
// k_small: one launch estimates one small field (N <= 2^21): value range -> per-block SZ
// + ZFP -> entropy / result, separated by two grid-wide barriers on a co-resident grid
// (cooperative launch) instead of three launches or k_batch's cross-CTA task hand-offs
// (k_batch: ~44 us for one 256x256 field).  The last CTA resets the
// barrier counters, the range keys and (as every CTA does for its slice) the histogram,
// so the next call starts from the same state; results are bit-identical to the per-field
// kernels (same per-block code, fixed-order partial sums).
struct SmallState {
  unsigned int rmin, rmax, rbad, ctr, ticket, pad[3];
};
struct SmallFin { double acc; unsigned long long hcnt, ovf; };
#ifndef SEL_SMALL_PROF
#define SEL_SMALL_PROF 0               // developer probe: %globaltimer at k_small's phase ends (CTA 0)
#endif
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ unsigned int sk_key(float v) {   // order-preserving float key
  const unsigned int b = __float_as_uint(v);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float sk_float(unsigned int k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}
__device__ __forceinline__ void grid_barrier(unsigned int *ctr, unsigned int target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(ctr, 1u);
    long long guard = 0;
    while (ld_acquire(ctr) < target) {
      __nanosleep(32);
      if (++guard > (1LL << 26)) __trap();
    }
  }
  __syncthreads();
}

template <int D, bool VEC>
__global__ void __launch_bounds__(256) k_small(const float *__restrict__ x, Geo g, SmallState *st,
                                               unsigned long long *gh, Partial *part, SmallFin *fin,
                                               Params *prm_out, FinalizeArgs fa, sel_result *out) {
  extern __shared__ unsigned int sh_hist[];
  const unsigned long long T0 = SEL_SMALL_PROF ? gtimer() : 0ull;
  __shared__ float s_mn[8], s_mx[8];
  __shared__ int s_bad[8];
  __shared__ bool s_last;
  hist_zero(sh_hist);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  // ---- phase 1: value range (Alg. 1 line 2, R1); NaN-propagating min, +-inf in min / max
  {
    float mn = INFINITY, mx = -INFINITY;
    const int64_t gs = (int64_t)gridDim.x * blockDim.x;
    auto take = [&](float v) {
      mn = (v != v || v < mn) ? v : mn;
      mx = fmaxf(mx, v);
    };
    if (VEC) {   // float4 loads, 4 in flight per thread (one L2 round trip for C1)
      const float4 *x4 = reinterpret_cast<const float4 *>(x);
      const int64_t n4 = g.N / 4;
      for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < n4; i0 += 4 * gs) {
        float4 q[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int64_t i = i0 + u * gs;
          q[u] = i < n4 ? __ldg(x4 + i) : make_float4(x[0], x[0], x[0], x[0]);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) { take(q[u].x); take(q[u].y); take(q[u].z); take(q[u].w); }
      }
    } else {
      for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < g.N; i0 += 4 * gs) {
        float q[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int64_t i = i0 + u * gs;
          q[u] = i < g.N ? __ldg(x + i) : x[0];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) take(q[u]);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float a = __shfl_xor_sync(0xffffffffu, mn, o);
      mn = (a != a || a < mn) ? a : mn;
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if (lane == 0) { s_mn[wid] = mn; s_mx[wid] = mx; }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int w = 1; w < nw; ++w) {
        mn = (s_mn[w] != s_mn[w] || s_mn[w] < mn) ? s_mn[w] : mn;
        mx = fmaxf(mx, s_mx[w]);
      }
      const int bad = (mn != mn) | ((mn <= mx) & (is_nonfinite(mn) | is_nonfinite(mx)));
      if (mn <= mx) {
        atomicMin(&st->rmin, sk_key(mn));
        atomicMax(&st->rmax, sk_key(mx));
      }
      if (bad) atomicOr(&st->rbad, 1u);
    }
  }
  const unsigned long long T1 = SEL_SMALL_PROF ? gtimer() : 0ull;
  grid_barrier(&st->ctr, gridDim.x);
  const unsigned long long T2 = SEL_SMALL_PROF ? gtimer() : 0ull;
  const Params prm = make_params(sk_float(__ldcg(&st->rmin)), sk_float(__ldcg(&st->rmax)), (int)__ldcg(&st->rbad),
                                 fa.mode, fa.eb);
  // ---- phase 2: every processed block (R3-R14), per-CTA partial in a fixed order
  uint64_t bits_acc = 0;
  double err_acc = 0.0;
  unsigned int ovf = 0;
  if (prm.status == SEL_OK) {
    const DebugPtrs nd{};
    const int64_t gs = (int64_t)gridDim.x * blockDim.x;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < g.n_pb; t += gs) {
      uint32_t bits;
      double E;
      block_estimate<D, VEC, false>(x, g, t, prm.r_f, prm.minexp, sh_hist, gh, ovf, nd, bits, E);
      bits_acc += bits;
      err_acc += E;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    bits_acc += __shfl_down_sync(0xffffffffu, bits_acc, o);
    err_acc += __shfl_down_sync(0xffffffffu, err_acc, o);
  }
  __shared__ uint64_t sb[8];
  __shared__ double se[8];
  if (lane == 0) { sb[wid] = bits_acc; se[wid] = err_acc; }
  ovf_flush(ovf, gh);
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < nw; ++w) { bits_acc += sb[w]; err_acc += se[w]; }
    Partial pr;
    pr.bits = bits_acc;
    pr.err = err_acc;
    part[blockIdx.x] = pr;
  }
  const unsigned long long T3 = SEL_SMALL_PROF ? gtimer() : 0ull;
  hist_flush(sh_hist, gh);
  const unsigned long long T4 = SEL_SMALL_PROF ? gtimer() : 0ull;
  grid_barrier(&st->ctr, 2 * gridDim.x);
  const unsigned long long T5 = SEL_SMALL_PROF ? gtimer() : 0ull;
  if (SEL_SMALL_PROF && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long *pr = (unsigned long long *)(fin + gridDim.x);
    pr[0] = T1 - T0; pr[1] = T2 - T1; pr[2] = T3 - T2; pr[3] = T4 - T3; pr[4] = T5 - T4;
  }
  // ---- phase 3: this CTA's slice of the histogram: sum c log2(N/c), re-zero (R6)
  {
    const int per = (kNSlots + gridDim.x - 1) / gridDim.x;
    const int s0 = blockIdx.x * per, s1 = min(s0 + per, kNSlots);
    const double lN = log2((double)fa.n_sz);
    double acc = 0.0;
    unsigned long long hcnt = 0, novf = 0;
    for (int sl = s0 + threadIdx.x; sl < s1; sl += blockDim.x) {
      const unsigned long long c = __ldcg(gh + sl);
      hcnt += c;
      if (c) {
        const double cd = (double)c;
        acc += cd * (lN - log2(cd));
        gh[sl] = 0ull;
      }
      if (sl == kOvfSlot) novf = c;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      acc += __shfl_down_sync(0xffffffffu, acc, o);
      hcnt += __shfl_down_sync(0xffffffffu, hcnt, o);
      novf += __shfl_down_sync(0xffffffffu, novf, o);
    }
    __shared__ double sa[8];
    __shared__ unsigned long long sh[8], so[8];
    if (lane == 0) { sa[wid] = acc; sh[wid] = hcnt; so[wid] = novf; }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int w = 1; w < nw; ++w) { acc += sa[w]; hcnt += sh[w]; novf += so[w]; }
      SmallFin f;
      f.acc = acc;
      f.hcnt = hcnt;
      f.ovf = novf;
      fin[blockIdx.x] = f;
      __threadfence();
      s_last = atomicAdd(&st->ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
  }
  if (!s_last || wid != 0) return;
  // ---- the last CTA, warp 0: fixed-order sums (lane-strided loads, one shuffle tree),
  // the result (Eq. entropy, psnr-sz, ZFP, Alg. 1 lines 7-10), and the reset
  __threadfence();
  double S = 0.0, errs = 0.0;
  unsigned long long tb = 0, hc = 0, ov = 0;
  for (unsigned int c = lane; c < gridDim.x; c += 32) {
    S += __ldcg(&fin[c].acc);
    hc += __ldcg(&fin[c].hcnt);
    ov += __ldcg(&fin[c].ovf);
    tb += __ldcg(&part[c].bits);
    errs += __ldcg(&part[c].err);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    S += __shfl_down_sync(0xffffffffu, S, o);
    errs += __shfl_down_sync(0xffffffffu, errs, o);
    tb += __shfl_down_sync(0xffffffffu, tb, o);
    hc += __shfl_down_sync(0xffffffffu, hc, o);
    ov += __shfl_down_sync(0xffffffffu, ov, o);
  }
  // the three logarithms of the result on three lanes at once (as k_finalize does)
  const double mse = __shfl_sync(0xffffffffu, errs, 0) / (double)fa.n_values;
  const bool okp = prm.status == SEL_OK;
  double lg = 0.0;
  if (lane == 1 && okp) lg = log10(prm.vr / prm.eb_abs);
  if (lane == 2 && okp) lg = log10(prm.vr);
  if (lane == 3 && mse > 0.0) lg = log10(mse);
  const double lg_vr_eb = __shfl_sync(0xffffffffu, lg, 1), lg_vr = __shfl_sync(0xffffffffu, lg, 2),
               lg_mse = __shfl_sync(0xffffffffu, lg, 3);
  if (lane != 0) return;
  if (SEL_SMALL_PROF) {
    unsigned long long *pr = (unsigned long long *)(fin + gridDim.x);
    pr[5] = gtimer() - T5;   // phase 3 + the last CTA (the last CTA's own T5)
    pr[6] = blockIdx.x;
  }
  *prm_out = prm;
  *out = assemble_result(prm, S, errs, tb, ov, hc, fa, lg_vr_eb, lg_vr, lg_mse);
  st->rmin = 0xffffffffu;
  st->rmax = 0u;
  st->rbad = 0u;
  st->ctr = 0u;
  st->ticket = 0u;
}

namespace {
template <int D, bool VEC>
const void *small_fn() { return (const void *)k_small<D, VEC>; }
const void *pick_small(int D, bool vec) {
  if (D == 1) return vec ? small_fn<1, true>() : small_fn<1, false>();
  if (D == 2) return vec ? small_fn<2, true>() : small_fn<2, false>();
  return vec ? small_fn<3, true>() : small_fn<3, false>();
}
}  // namespace

size_t small_state_bytes(int sm_count) {
  return 256 + (size_t)sm_count * (sizeof(Partial) + sizeof(SmallFin)) + 512;
}

// one-time init of the small-field state (range keys at their neutral values)
int init_small_state(void *state, cudaStream_t st) {
  SmallState s{};
  s.rmin = 0xffffffffu;
  return cudaMemcpyAsync(state, &s, sizeof(s), cudaMemcpyHostToDevice, st) == cudaSuccess ? SEL_OK : SEL_ECUDA;
}

int launch_small(const float *x, const Geo &g, int sm_count, void *state, const Workspace &ws,
                 const FinalizeArgs &fa, sel_result *d_out, cudaStream_t st) {
  const void *fn = pick_small(g.ndims, g.vec != 0);
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, 256, kEstSmem) != cudaSuccess || occ < 1)
    return SEL_ECUDA;
  const int64_t ctas = sm_count;                         // one CTA per SM: co-resident
  SmallState *ss = (SmallState *)state;
  Partial *part = (Partial *)((char *)state + 256);
  SmallFin *fin = (SmallFin *)(part + sm_count);
  Geo gg = g;
  FinalizeArgs f = fa;
  unsigned long long *gh = ws.hist;
  Params *prm = ws.params;
  void *args[] = {(void *)&x, (void *)&gg, (void *)&ss, (void *)&gh, (void *)&part, (void *)&fin,
                  (void *)&prm, (void *)&f, (void *)&d_out};
#ifndef SEL_SMALL_PLAIN
#define SEL_SMALL_PLAIN 0              // developer probe: plain (non-cooperative) launch
#endif
  if (SEL_SMALL_PLAIN)
    return cudaLaunchKernel(fn, dim3((unsigned)ctas), dim3(256), args, kEstSmem, st) == cudaSuccess ? SEL_OK : SEL_ECUDA;
  return cudaLaunchCooperativeKernel(fn, dim3((unsigned)ctas), dim3(256), args, kEstSmem, st) == cudaSuccess
             ? SEL_OK
             : SEL_ECUDA;
}

}  // namespace sel
