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
// Launches: k_minmax (value range) -> the fused pass for k ebs -> k x k_finalize.  The fused
// pass is k_tile_multi (the TMA tile pipeline of sel_tile.cu with the eb-dependent stages in a
// loop over the ebs) for full-field 2D / 3D estimates, else k_multi (one thread per block).
#include <cmath>
#include <cstdlib>

#include "sel_tile_common.cuh"

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

// ============================================================ tile pipeline, k ebs
// Same producer / stage ring / tile geometry as k_tile (sel_tile.cu).  The consumer forms a
// plane's 16 Lorenzo residuals per lane once and quantises them in a loop over the ebs, each
// eb into its own shared-memory window; the windows share the single-eb kernel's budget of
// TileCfg<D>::W bins, split in proportion to 1 / eb (a 10x finer bound spreads the codes 10x
// wider), so the finest bound keeps nearly the whole window.  The ZFP block is transformed
// once (zfp_transform) and cut / counted / measured per eb (zfp_cost).  Partials are per
// (task, warp, block row) and eb, summed in index order by k_finalize: bit-reproducible.
struct MultiTileArgs {
  int k, mode;
  double eb[kMaxEb];
  int wsize[kMaxEb];               // per-eb window: bins (codes [-wsize/2, wsize/2)), multiple of 4
  int wbase[kMaxEb];               // first word of the window; word wbase + wsize is its pad bin
  const Params *base;              // k_minmax output
  Params *prm;                     // [k] per-eb params (written by CTA 0)
  unsigned long long *hist;        // [k][kNSlots]
  Partial *part;                   // [k][part_stride]
  size_t part_stride;
  unsigned int *task_ctr;          // [2]: task counter, departed producers (zero between launches)
};

template <int D>
__device__ __forceinline__ void tile_consume_multi(const float *S, int t, int btk, int btj, int bi,
                                                   const TileGeo &tg, int warp, int lane, bool ok,
                                                   const MultiTileArgs &ma, const float *s_rf,
                                                   const int *s_minexp, const int *s_wsize,
                                                   const int *s_wbase, unsigned int *win,
                                                   unsigned int *s_ovf) {
  using Cfg = TileCfg<D>;
  constexpr int SZ = Tab<D>::SIZE;
  constexpr int NPL = D == 3 ? 4 : 1;
  const int k = ma.k;
  const int n0 = (int)tg.n[0], n1 = (int)tg.n[1];
  const int bk = btk * 32 + lane;
#pragma unroll 1
  for (int rb = 0; rb < Cfg::BR; ++rb) {
    const int wr = warp * Cfg::BR + rb;           // block row within the tile
    const int bj = btj * Cfg::ROWS + wr;
    const size_t pidx = ((size_t)t * Cfg::CW + warp) * Cfg::BR + rb;
    if (!(ok && bj < tg.nb[1])) {
      if (lane == 0) {
        Partial z;
        z.bits = 0; z.err = 0.0;
        for (int e = 0; e < k; ++e) ma.part[(size_t)e * ma.part_stride + pidx] = z;
      }
      continue;
    }
    const bool activeK = bk < tg.nb[2];
    const int I0 = 4 * bi, J0 = 4 * bj;
    const float *wrow = S + (4 * wr) * kBoxK;     // smem row of j = J0 - 1 (plane 0)
    const bool edge = J0 + 4 > n1 || (D == 3 && I0 + 4 > n0);
    // ---------------- SZ: nested differences once (R4), codes per eb (R5)
    float blk2[D == 2 ? 16 : 1];
    float dprev[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) dprev[r][c] = 0.0f;
    if constexpr (D == 3) {     // plane i = I0 - 1 (smem plane 0; zeros at i < 0)
      float v[5][4], h[5], d1up[4];
      load_plane(wrow, lane, v, h);
#pragma unroll
      for (int c = 0; c < 4; ++c) d1up[c] = v[0][c] - (c ? v[0][c - 1] : h[0]);
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const float d1 = v[r + 1][c] - (c ? v[r + 1][c - 1] : h[r + 1]);
          dprev[r][c] = d1 - d1up[c];
          d1up[c] = d1;
        }
    }
#pragma unroll 1
    for (int p = 0; p < NPL; ++p) {
      const int i = I0 + p;
      float d[4][4];
      {
        float v[5][4], h[5], d1up[4];
        load_plane(wrow + (D == 3 ? (p + 1) * Cfg::PLANE : 0), lane, v, h);
        if constexpr (D == 2) {       // rows past the field's edge replicate the last (R17)
#pragma unroll
          for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int c = 0; c < 4; ++c)
              blk2[4 * r + c] = (r == 0 || !edge || J0 + r < n1) ? v[r + 1][c] : blk2[4 * (r - 1) + c];
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) d1up[c] = v[0][c] - (c ? v[0][c - 1] : h[0]);
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const float d1 = v[r + 1][c] - (c ? v[r + 1][c - 1] : h[r + 1]);
            const float d2 = d1 - d1up[c];
            d1up[c] = d1;
            if constexpr (D == 3) {
              d[r][c] = d2 - dprev[r][c];
              dprev[r][c] = d2;
            } else {
              d[r][c] = d2;
            }
          }
      }
      if (D == 3 && i >= n0) continue;             // padded plane: no SZ point (warp-uniform)
      const int nrow = edge ? min(4, n1 - J0) : 4; // real rows of the block (warp-uniform)
      const bool orow = (i == 0) && (J0 == 0) && (btk == 0) && (lane == 0);   // the field origin (R4)
#pragma unroll 1
      for (int e = 0; e < k; ++e) {
        const float rf = lane_rf(activeK, s_rf[e]);
        const uint32_t wsz = (uint32_t)s_wsize[e];
        const uint32_t woff = kSlotOff + (uint32_t)kCenter - (wsz >> 1);
        unsigned int *wb = win + s_wbase[e];
        unsigned long long *gh = ma.hist + (size_t)e * kNSlots;
        unsigned int o = 0;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          if (r < nrow) {
            uint32_t w[4];
            uint32_t any = 0;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const uint32_t b = __float_as_uint(__fadd_rn(__fmul_rn(d[r][c], rf), kMagic));
              w[c] = b - woff;
              atomicAdd(wb + min(w[c], wsz), 1u);
              any |= w[c];
            }
            if (r == 0 && orow) {                   // stored verbatim, not coded: undo its count
              if (w[0] < wsz) atomicSub(wb + w[0], 1u);
              w[0] = 0u;
              any = w[1] | w[2] | w[3];
            }
            if (__any_sync(0xffffffffu, activeK && any >= wsz)) {
#pragma unroll
              for (int c = 0; c < 4; ++c)
                if (activeK && w[c] >= wsz) {
                  const uint32_t sl = w[c] + (woff - kSlotOff);
                  if (sl > 65534u) ++o;
                  else atomicAdd(gh + sl, 1ull);
                }
            }
          }
        }
        if (__any_sync(0xffffffffu, o != 0u)) {
          o = __reduce_add_sync(0xffffffffu, o);
          if (lane == 0) atomicAdd(s_ovf + e, o);
        }
      }
    }
    // ---------------- ZFP: transform once (R8, R9), cut / bits / error per eb (R12-R14)
    int emax = 0;
    int cf[SZ];
    bool nz = false;
    if (activeK) {
      float blk[SZ];
      if constexpr (D == 2) {
#pragma unroll
        for (int n = 0; n < 16; ++n) blk[n] = blk2[n];
      } else {
        const float *bbase = S + Cfg::PLANE + (4 * wr + 1) * kBoxK + 4 + 4 * lane;
#pragma unroll
        for (int p = 0; p < NPL; ++p) {
          const int ic = edge ? min(I0 + p, n0 - 1) - I0 : p;          // edge-replicated (R17)
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            const int jc = edge ? min(J0 + r, n1 - 1) - J0 : r;
            const float4 q = *reinterpret_cast<const float4 *>(bbase + ic * Cfg::PLANE + jc * kBoxK);
            const int o = (p * 4 + r) * 4;
            blk[o] = q.x; blk[o + 1] = q.y; blk[o + 2] = q.z; blk[o + 3] = q.w;
          }
        }
      }
      nz = zfp_transform<D>(blk, emax, cf);
    }
#pragma unroll 1
    for (int e = 0; e < k; ++e) {
      uint32_t bits = 0;
      double E = 0.0;
      if (activeK) {
        if (nz) {
          uint32_t u[SZ];
          zfp_cost<D, false>(cf, emax, s_minexp[e], bits, E, u);
        } else {
          bits = 1u;                                // empty block: 1 bit, no error
        }
      }
      task_store(ma.part + (size_t)e * ma.part_stride, (int)pidx, (uint64_t)bits, E);
    }
  }
}

template <int D>
__global__ void __launch_bounds__(TileCfg<D>::THREADS, 1)
    k_tile_multi(const __grid_constant__ CUtensorMap tmap, TileGeo tg, MultiTileArgs ma) {
  using Cfg = TileCfg<D>;
  constexpr int CW = Cfg::CW;
  extern __shared__ float smem_dyn[];
  float *const base = smem_dyn + (((128u - (smem_u32(smem_dyn) & 127u)) & 127u) >> 2);
  unsigned int *const hist = reinterpret_cast<unsigned int *>(base + Cfg::STAGES * Cfg::STAGE_FLOATS);
  uint64_t *const full_bar = reinterpret_cast<uint64_t *>(hist + Cfg::HIST_WORDS);
  uint64_t *const empty_bar = full_bar + Cfg::STAGES;
  int4 *const stage_task = reinterpret_cast<int4 *>(empty_bar + Cfg::STAGES);   // {t, btk, btj, bi}
  __shared__ float s_rf[kMaxEb];
  __shared__ int s_minexp[kMaxEb];
  __shared__ unsigned int s_ovf[kMaxEb];
  __shared__ int s_wsize[kMaxEb], s_wbase[kMaxEb];
  __shared__ int s_status;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], CW);
    }
    fence_barrier_init();
    const Params b = *ma.base;
    s_status = b.status;
    for (int i = 0; i < ma.k; ++i) {
      // per-eb derived scalars from the shared value range (R1, R2)
      const Params p = make_params(b.vmin, b.vmax, b.status == SEL_ENONFINITE, ma.mode, ma.eb[i]);
      s_rf[i] = p.r_f;
      s_minexp[i] = p.minexp;
      s_ovf[i] = 0u;
      s_wsize[i] = ma.wsize[i];
      s_wbase[i] = ma.wbase[i];
      if (p.status != SEL_OK) s_status = p.status;     // every eb's finalize reports its own status
      if (blockIdx.x == 0) ma.prm[i] = p;
    }
  }
  for (int i = threadIdx.x; i < Cfg::HIST_WORDS; i += Cfg::THREADS) hist[i] = 0u;
  __syncthreads();

  // ------------------------------------------------------------------ producer (as k_tile)
  if (warp == CW) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
      int stage = 0;
      uint32_t ph = 0;
      int next = (int)atomicAdd(ma.task_ctr, 1u);     // fetched one task ahead
      for (;;) {
        const int t = next;
        if (t < tg.ntasks) next = (int)atomicAdd(ma.task_ctr, 1u);
        mbar_wait_sleep(&empty_bar[stage], ph ^ 1u);
        if (t >= tg.ntasks) {           // sentinel stage: consumers stop here
          stage_task[stage] = make_int4(t, 0, 0, 0);
          mbar_arrive(&full_bar[stage]);
          break;
        }
        const int btk = t % tg.ntk;
        const int rest = t / tg.ntk;
        const int btj = rest % tg.ntj;
        const int bi = rest / tg.ntj;
        stage_task[stage] = make_int4(t, btk, btj, bi);
        float *dst = base + stage * Cfg::STAGE_FLOATS;
        mbar_arrive_expect_tx(&full_bar[stage], Cfg::STAGE_BYTES);
        if constexpr (D == 3)
          tma_load_3d(dst, &tmap, 128 * btk - 4, 4 * Cfg::ROWS * btj - 1, 4 * bi - 1, &full_bar[stage]);
        else
          tma_load_2d(dst, &tmap, 128 * btk - 4, 4 * Cfg::ROWS * btj - 1, &full_bar[stage]);
        if (++stage == Cfg::STAGES) { stage = 0; ph ^= 1u; }
      }
      // the last producer to leave (every CTA has made its final claim) re-zeroes the
      // counters for the next call
      if (atomicAdd(ma.task_ctr + 1, 1u) == gridDim.x - 1) {
        ma.task_ctr[0] = 0u;
        ma.task_ctr[1] = 0u;
      }
    }
    return;
  }

  // ------------------------------------------------------------------ consumers
  const bool ok = s_status == SEL_OK;
  int stage = 0;
  uint32_t ph = 0;
  for (;;) {
    mbar_wait(&full_bar[stage], ph);
    const int4 td = stage_task[stage];
    const int t = td.x;
    if (t >= tg.ntasks) break;
    const float *S = base + stage * Cfg::STAGE_FLOATS;
    tile_consume_multi<D>(S, t, td.y, td.z, td.w, tg, warp, lane, ok, ma, s_rf, s_minexp, s_wsize, s_wbase,
                          hist, s_ovf);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty_bar[stage]);    // stage free for the producer
    if (++stage == Cfg::STAGES) { stage = 0; ph ^= 1u; }
  }
  consumer_sync<CW * 32>();
  // windows (without their pad bins) and overflow counts -> global histograms
  for (int e = 0; e < ma.k; ++e) {
    unsigned long long *gh = ma.hist + (size_t)e * kNSlots;
    const int wsz = s_wsize[e];
    const unsigned int *wb = hist + s_wbase[e];
    for (int i = threadIdx.x; i < wsz; i += CW * 32) {
      const unsigned int c = wb[i];
      if (c) atomicAdd(gh + (kCenter - wsz / 2) + i, (unsigned long long)c);
    }
    if (threadIdx.x == 0 && s_ovf[e]) atomicAdd(gh + kOvfSlot, (unsigned long long)s_ovf[e]);
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

// ---- tile pipeline, k ebs (host side)
long long multi_tile_parts(const Geo &g, const TileLaunch &tl) {       // partials per eb
  return (long long)tl.tg.ntasks *
         (g.ndims == 3 ? TileCfg<3>::CW * TileCfg<3>::BR : TileCfg<2>::CW * TileCfg<2>::BR);
}

int launch_multi_tile(const float *x, const Geo &g, const TileLaunch &tl, int sm_count, int k, const double *ebs,
                      int mode, const Params *base, Params *prm, unsigned long long *hist, Partial *part,
                      size_t part_stride, unsigned int *task_ctr, cudaStream_t st) {
  if (k < 1 || k > kMaxEb) return SEL_EINVAL;
  const int W = g.ndims == 3 ? TileCfg<3>::W : TileCfg<2>::W;
  MultiTileArgs ma;
  ma.k = k;
  ma.mode = mode;
  // window split: every eb gets 64 bins + its pad word, the rest in proportion to eb^-0.3.
  // In proportion to 1 / eb every eb would cut the residual distribution at the same
  // absolute value: the coarse bounds, whose codes sit on a few bins, would then send their
  // tails to a few global addresses (same-address atomics serialise).  Measured on C3 / C4 /
  // C5 (scripts/probe_multi.py): exponent 1: C4 field 1 2.7 ms, noisy C5 11.8 ms; 0.5: 1.28 /
  // 11.6; 0.25-0.35: 1.23 / 3.4-3.7; 0 (equal windows): 1.55 / 2.6.  SEL_MULTI_WEXP: developer
  // override.
  double wexp = 0.3;
  if (const char *ev = getenv("SEL_MULTI_WEXP")) wexp = atof(ev);
  double wt[kMaxEb], wsum = 0.0;
  for (int i = 0; i < k; ++i) {
    wt[i] = pow(ebs[i], -wexp);
    wsum += wt[i];
  }
  const int spare = (W - k * 68) / 64;            // 64-bin granules to distribute
  int used = 0;
  for (int i = 0; i < kMaxEb; ++i) {
    ma.eb[i] = i < k ? ebs[i] : 1.0;
    ma.wsize[i] = 0;
    ma.wbase[i] = 0;
    if (i < k) {
      int gran = (int)((double)spare * (wt[i] / wsum));
      if (gran < 0) gran = 0;
      if (gran > spare) gran = spare;
      ma.wsize[i] = 64 + 64 * gran;
      ma.wbase[i] = used;
      used += ma.wsize[i] + 4;                     // + pad bin, 16-byte aligned windows
    }
  }
  if (used > W + 4) return SEL_EINVAL;
  ma.base = base;
  ma.prm = prm;
  ma.hist = hist;
  ma.part = part;
  ma.part_stride = part_stride;
  ma.task_ctr = task_ctr;
  CUtensorMap map;
  if (make_tile_map(&map, x, g)) return SEL_ECUDA;
  const void *fn = g.ndims == 3 ? (const void *)k_tile_multi<3> : (const void *)k_tile_multi<2>;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tl.smem) != cudaSuccess)
    return SEL_ECUDA;
  TileGeo tg = tl.tg;
  const int ctas = tg.ntasks < sm_count ? (tg.ntasks < 1 ? 1 : tg.ntasks) : sm_count;
  void *args[] = {(void *)&map, (void *)&tg, (void *)&ma};
  return cudaLaunchKernel(fn, dim3(ctas), dim3(tl.threads), args, tl.smem, st) == cudaSuccess ? SEL_OK : SEL_ECUDA;
}

}  // namespace sel
