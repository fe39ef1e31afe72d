// sel_tile.cu -- TMA-fed fused SZ+ZFP pass (the hot path for 2D/3D full-field estimates).
//
// One persistent CTA per SM: the last warp is the producer, the CW warps before it are
// consumers.  A task is a tile of CW block rows (one per consumer warp) x 32 blocks along
// the fastest axis (one per lane) x one 4-plane block layer (3D).  The producer fetches
// task ids from a global counter and streams each tile, extended by its -1 halo (one
// column, one row and, in 3D, one plane), into a ring of shared-memory stages with one
// cp.async.bulk.tensor (TMA) per task, completing on an mbarrier (expect_tx).  TMA's
// out-of-bounds zero fill IS the Lorenzo zero boundary (P:151 footnote; reading R4), so
// the consumer code has no boundary branches.  Consumers compute the SZ residuals (nested
// first differences, R4) and quantisation codes (R5) from shared memory into a
// lane-replicated shared-memory histogram window (C copies: a smooth field sends all 32
// lanes to the same code, and copies turn a 32-way same-address conflict into a
// 32/C-way one), then each lane runs the ZFP block pipeline (zfp_block, R8-R14) on its
// block, re-read from shared memory with the far-edge replication (R17) folded into the
// row/plane index.  Every (task, warp) writes one partial, summed in task order by the
// finalize kernel: bit-reproducible regardless of the dynamic schedule.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include "sel_device.cuh"

namespace sel {

constexpr int kBoxK = 4 * 32 + 4;             // 132 floats: 4 halo columns (last one used) + 128
constexpr int kHBins = 1024;                  // histogram window: codes [-512, 512)
constexpr int kHStride = kHBins + 1;          // copy stride (words): copy c of a bin -> bank + c
constexpr uint32_t kHOff = kSlotOff + (uint32_t)(kCenter - kHBins / 2);

template <int D>
struct TileCfg {
  static constexpr int CW = D == 3 ? 8 : 16;                      // consumer warps
  static constexpr int THREADS = (CW + 1) * 32;
  static constexpr int BOXJ = 4 * CW + 1;                         // halo row + 4 per warp
  static constexpr int BOXI = D == 3 ? 5 : 1;                     // halo plane + 4 (3D)
  static constexpr int PLANE = kBoxK * BOXJ;                      // floats per smem plane
  static constexpr uint32_t STAGE_BYTES = PLANE * BOXI * 4;
  static constexpr int STAGE_FLOATS = ((STAGE_BYTES + 127) & ~127) / 4;
  static constexpr int STAGES = D == 3 ? 2 : 4;
  static constexpr int COPIES = D == 3 ? 4 : 8;                   // histogram lane copies
  static constexpr int HIST_WORDS = (COPIES + 1) * kHStride;   // + trash copy
  // second level: one packed 16-bit-counter table of TB slots centred on code 0 for the
  // codes outside the lane-copy window (wide distributions: noise, coarse data)
  static constexpr int TB = D == 3 ? 17408 : 27392;   // leaves ~2.5 KB of the SM for k_minmax + k_finalize
  static constexpr int TBL_WORDS = TB / 2;
  static constexpr size_t SMEM = 128 + (size_t)STAGES * STAGE_FLOATS * 4 + HIST_WORDS * 4 +
                                 TBL_WORDS * 4 + STAGES * 16 + 16;
};

// ------------------------------------------------------------ mbarrier / TMA PTX
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 10000000;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, int c0, int c1,
                                            int c2, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, int c0, int c1,
                                            uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
template <int N>
__device__ __forceinline__ void consumer_sync() {   // the consumer threads only
  asm volatile("bar.sync 1, %0;" ::"n"(N) : "memory");
}

// One plane of a warp's tile rows: the 5 smem rows (halo row + 4) of the lane's block
// columns, each with its left neighbour (lane-1's last value; lane 0 reads the halo
// column, which TMA zero-filled at the field's left edge).  All loads are issued first.
__device__ __forceinline__ void load_plane(const float *prow, int lane, float (&v)[5][4],
                                           float (&h)[5]) {
  float h0[5];
#pragma unroll
  for (int r = 0; r < 5; ++r) {
    const float4 q = *reinterpret_cast<const float4 *>(prow + r * kBoxK + 4 + 4 * lane);
    v[r][0] = q.x; v[r][1] = q.y; v[r][2] = q.z; v[r][3] = q.w;
    h0[r] = prow[r * kBoxK + 3];
  }
#pragma unroll
  for (int r = 0; r < 5; ++r) {
    const float hs = __shfl_up_sync(0xffffffffu, v[r][3], 1);
    h[r] = lane == 0 ? h0[r] : hs;
  }
}

// SZ code of one residual: b = bits(q + M) (reading R5, see sel_device.cuh), w = its
// offset in the window; one unconditional increment of the lane's copy (no divergence):
// out-of-window values land in the copy's pad word (index kHBins), ignored at the flush.
__device__ __forceinline__ uint32_t sz_win(float d, float r_f, unsigned int *hcopy) {
  const uint32_t b = __float_as_uint(__fadd_rn(__fmul_rn(d, r_f), kMagic));
  const uint32_t w = b - kHOff;
  atomicAdd(hcopy + min(w, (uint32_t)kHBins), 1u);
  return w;
}

template <int D, bool DBG>
__global__ void __launch_bounds__(TileCfg<D>::THREADS, 1)
    k_tile(const __grid_constant__ CUtensorMap tmap, TileGeo tg, Workspace ws, DebugPtrs dbg) {
  using Cfg = TileCfg<D>;
  constexpr int CW = Cfg::CW;
  constexpr int SZ = Tab<D>::SIZE;
  constexpr int NPL = D == 3 ? 4 : 1;          // data planes per tile
  extern __shared__ float smem_dyn[];
  // 128-byte align the stage ring (TMA destination) without leaving the shared window
  float *const base = smem_dyn + (((128u - (smem_u32(smem_dyn) & 127u)) & 127u) >> 2);
  unsigned int *const hist = reinterpret_cast<unsigned int *>(base + Cfg::STAGES * Cfg::STAGE_FLOATS);
  unsigned int *const tbl = hist + Cfg::HIST_WORDS;
  uint64_t *const full_bar =
      reinterpret_cast<uint64_t *>(tbl + Cfg::TBL_WORDS + ((Cfg::HIST_WORDS + Cfg::TBL_WORDS) & 1));
  uint64_t *const empty_bar = full_bar + Cfg::STAGES;
  int *const stage_task = reinterpret_cast<int *>(empty_bar + Cfg::STAGES);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], CW);
    }
    fence_barrier_init();
  }
  for (int i = threadIdx.x; i < Cfg::HIST_WORDS + Cfg::TBL_WORDS; i += Cfg::THREADS) hist[i] = 0u;
  __syncthreads();
  grid_dep_wait();   // k_minmax done: params valid, the task counter was reset by the
                     // previous field's finalize (which k_minmax waited for)

  // ------------------------------------------------------------------ producer
  if (warp == CW) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
      int stage = 0;
      uint32_t ph = 0;
      for (;;) {
        const int t = (int)atomicAdd(ws.task_ctr, 1u);
        mbar_wait(&empty_bar[stage], ph ^ 1u);
        stage_task[stage] = t;
        if (t >= tg.ntasks) {           // sentinel stage: consumers stop here
          mbar_arrive(&full_bar[stage]);
          break;
        }
        const int btk = t % tg.ntk;
        const int rest = t / tg.ntk;
        const int btj = rest % tg.ntj;
        const int bi = rest / tg.ntj;
        float *dst = base + stage * Cfg::STAGE_FLOATS;
        mbar_arrive_expect_tx(&full_bar[stage], Cfg::STAGE_BYTES);
        if constexpr (D == 3)
          tma_load_3d(dst, &tmap, 128 * btk - 4, 4 * CW * btj - 1, 4 * bi - 1, &full_bar[stage]);
        else
          tma_load_2d(dst, &tmap, 128 * btk - 4, 4 * CW * btj - 1, &full_bar[stage]);
        if (++stage == Cfg::STAGES) { stage = 0; ph ^= 1u; }
      }
    }
    return;
  }

  // ------------------------------------------------------------------ consumers
  const Params prm = *ws.params;
  const bool ok = prm.status == SEL_OK;
  const float r_f = prm.r_f;
  const int minexp = prm.minexp;
  const int64_t n0 = tg.n[0], n1 = tg.n[1], n2 = tg.n[2];
  unsigned int *const hlane = hist + (lane % Cfg::COPIES) * kHStride;
  unsigned int *const htrash = hist + Cfg::COPIES * kHStride;   // inactive lanes count here
  unsigned int ovf = 0;
  int stage = 0;
  uint32_t ph = 0;
  for (;;) {
    mbar_wait(&full_bar[stage], ph);
    const int t = stage_task[stage];
    if (t >= tg.ntasks) break;
    const float *S = base + stage * Cfg::STAGE_FLOATS;
    const int btk = t % tg.ntk;
    const int rest = t / tg.ntk;
    const int btj = rest % tg.ntj;
    const int bi = rest / tg.ntj;
    const int bj = btj * CW + warp;
    const int64_t bk = (int64_t)btk * 32 + lane;
    uint64_t tbits = 0;
    double terr = 0.0;
    if (ok && bj < tg.nb[1]) {
      const bool activeK = bk < tg.nb[2];
      const int64_t I0 = 4 * (int64_t)bi, J0 = 4 * (int64_t)bj, K0 = 4 * bk;
      const float *wrow = S + (4 * warp) * kBoxK;   // smem row of j = J0 - 1 (plane 0)
      unsigned int *const hcopy = activeK ? hlane : htrash;
      // ---------------- SZ: nested differences on the tile (R4), codes -> histogram (R5)
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
        const int64_t i = I0 + p;
        float v[5][4], h[5], d1up[4];
        load_plane(wrow + (D == 3 ? (p + 1) * Cfg::PLANE : 0), lane, v, h);
#pragma unroll
        for (int c = 0; c < 4; ++c) d1up[c] = v[0][c] - (c ? v[0][c - 1] : h[0]);
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int64_t j = J0 + r;
          if (i >= n0 || j >= n1) break;              // padded rows/planes: no SZ point
          uint32_t w[4];
          uint32_t any = 0;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const float d1 = v[r + 1][c] - (c ? v[r + 1][c - 1] : h[r + 1]);
            const float d2 = d1 - d1up[c];
            d1up[c] = d1;
            float d;
            if constexpr (D == 3) {
              d = d2 - dprev[r][c];
              dprev[r][c] = d2;
            } else {
              d = d2;
            }
            w[c] = sz_win(d, r_f, hcopy);
            any |= w[c];
          }
          // the field origin is stored verbatim, not coded (R4): undo its count
          const bool orow = (i == 0) && (j == 0) && (btk == 0);
          if (orow && lane == 0) {
            if (w[0] < (uint32_t)kHBins) atomicSub(hcopy + w[0], 1u);
            w[0] = 0u;
          }
          if constexpr (DBG) {
            if (activeK) {
#pragma unroll
              for (int c = 0; c < 4; ++c) {
                if (orow && lane == 0 && c == 0) continue;
                const uint32_t sl = w[c] + (kHOff - kSlotOff);
                dbg.codes[(i * n1 + j) * n2 + K0 + c] = sl > 65534u ? kOvfSlot : (int32_t)sl;
              }
            }
          }
          // out-of-window codes: one warp-uniform branch per row
          if (__any_sync(0xffffffffu, activeK && any >= (uint32_t)kHBins)) {
            if (activeK) {
#pragma unroll
              for (int c = 0; c < 4; ++c)
                if (w[c] >= (uint32_t)kHBins) {
                  const uint32_t sl = w[c] + (kHOff - kSlotOff);
                  const uint32_t tb = sl - (uint32_t)(kCenter - Cfg::TB / 2);
                  if (sl > 65534u) {
                    ++ovf;
                  } else if (tb < (uint32_t)Cfg::TB) {
                    // packed 16-bit counter; the increment that takes it to 0x8000 moves
                    // 0x8000 counts to the global histogram, so it never carries
                    const uint32_t sh = (tb & 1u) << 4;
                    const uint32_t old = atomicAdd(tbl + (tb >> 1), 1u << sh);
                    if (((old >> sh) & 0xffffu) == 0x7fffu) {
                      atomicSub(tbl + (tb >> 1), 0x8000u << sh);
                      atomicAdd(ws.hist + sl, 0x8000ull);
                    }
                  } else {
                    atomicAdd(ws.hist + sl, 1ull);
                  }
                }
            }
          }
        }
      }
      // ---------------- ZFP on the lane's block, edge-replicated at the far edges (R17)
      if (activeK) {
        float blk[SZ];
#pragma unroll
        for (int p = 0; p < NPL; ++p) {
          const int64_t ic = min(I0 + p, n0 - 1) - I0;          // 0..3 (3D)
          const float *pbase = S + (D == 3 ? (ic + 1) * Cfg::PLANE : 0);
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            const int64_t jc = min(J0 + r, n1 - 1) - J0;         // 0..3
            const float4 q = *reinterpret_cast<const float4 *>(
                pbase + (4 * warp + 1 + jc) * kBoxK + 4 + 4 * lane);
            const int o = (p * 4 + r) * 4;
            blk[o] = q.x; blk[o + 1] = q.y; blk[o + 2] = q.z; blk[o + 3] = q.w;
          }
        }
        uint32_t bits;
        double E;
        int emax;
        int cf[SZ];
        uint32_t u[SZ];
        zfp_block<D, DBG>(blk, minexp, bits, E, emax, cf, u);
        tbits = bits;
        terr = E;
        if constexpr (DBG) {
          const int64_t tb = (D == 3 ? ((int64_t)bi * tg.nb[1] + bj) : (int64_t)bj) * tg.nb[2] + bk;
          dbg.emax[tb] = emax; dbg.bits[tb] = bits; dbg.err[tb] = E;
#pragma unroll
          for (int n = 0; n < SZ; ++n) { dbg.coef[tb * SZ + n] = cf[n]; dbg.uword[tb * SZ + n] = u[n]; }
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty_bar[stage]);      // stage free for the producer
    task_store(ws.task_part, t * CW + warp, tbits, terr);
    if (++stage == Cfg::STAGES) { stage = 0; ph ^= 1u; }
  }
  ovf_flush(ovf, ws.hist);
  consumer_sync<CW * 32>();
  for (int i = threadIdx.x; i < kHBins; i += CW * 32) {
    unsigned long long c = 0;
#pragma unroll
    for (int k = 0; k < Cfg::COPIES; ++k) c += hist[k * kHStride + i];
    if (c) atomicAdd(ws.hist + (kCenter - kHBins / 2) + i, c);
  }
  for (int i = threadIdx.x; i < Cfg::TBL_WORDS; i += CW * 32) {
    const uint32_t v = tbl[i];
    unsigned long long *g = ws.hist + (kCenter - Cfg::TB / 2) + 2 * i;
    if (v & 0xffffu) atomicAdd(g, (unsigned long long)(v & 0xffffu));
    if (v >> 16) atomicAdd(g + 1, (unsigned long long)(v >> 16));
  }
}

// ============================================================ host side
namespace {
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

int get_encode() {
  if (g_encode) return SEL_OK;
  void *fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !fn)
    return SEL_ECUDA;
  g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  return SEL_OK;
}

template <int D>
const void *tile_fn(bool dbg) {
  return dbg ? (const void *)k_tile<D, true> : (const void *)k_tile<D, false>;
}
}  // namespace

bool tile_supported(const Geo &g) {
  return (g.ndims == 2 || g.ndims == 3) && g.s[0] == 1 && g.s[1] == 1 && g.s[2] == 1 &&
         g.n[2] % 4 == 0 && g.n[2] < (1LL << 31) && g.n[1] < (1LL << 31) && g.n[0] < (1LL << 31);
}

int plan_tile(const Geo &g, int sm_count, int debug, TileLaunch *tl) {
  TileGeo &t = tl->tg;
  const int cw = g.ndims == 3 ? TileCfg<3>::CW : TileCfg<2>::CW;
  for (int a = 0; a < 3; ++a) { t.n[a] = g.n[a]; t.nb[a] = (int)g.nb[a]; }
  t.ntj = (int)((g.nb[1] + cw - 1) / cw);
  t.ntk = (int)((g.nb[2] + 31) / 32);
  const int64_t nt = (int64_t)t.ntj * t.ntk * (g.ndims == 3 ? g.nb[0] : 1);
  if (nt > (1LL << 26)) return SEL_EINVAL;
  t.ntasks = (int)nt;
  const size_t smem = g.ndims == 3 ? TileCfg<3>::SMEM : TileCfg<2>::SMEM;
  const int threads = g.ndims == 3 ? TileCfg<3>::THREADS : TileCfg<2>::THREADS;
  const void *fn = g.ndims == 3 ? tile_fn<3>(debug) : tile_fn<2>(debug);
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return SEL_ECUDA;
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, smem) != cudaSuccess)
    return SEL_ECUDA;
  if (occ < 1) return SEL_ECUDA;
  const int64_t cap = (int64_t)occ * sm_count;
  tl->ctas = (int)(nt < cap ? nt : cap);
  if (tl->ctas < 1) tl->ctas = 1;
  tl->smem = smem;
  tl->threads = threads;
  tl->npart = t.ntasks * cw;
  return SEL_OK;
}

int launch_tile(const float *x, const Geo &g, const TileLaunch &tl, const Workspace &ws,
                const DebugPtrs *dbg, cudaStream_t st) {
  if (get_encode()) return SEL_ECUDA;
  CUtensorMap map;
  const int rank = g.ndims;
  cuuint64_t gdim[3], gstride[2];
  cuuint32_t box[3], estr[3] = {1, 1, 1};
  gdim[0] = (cuuint64_t)g.n[2];
  gdim[1] = (cuuint64_t)g.n[1];
  gdim[2] = (cuuint64_t)g.n[0];
  gstride[0] = (cuuint64_t)g.n[2] * 4;
  gstride[1] = (cuuint64_t)g.n[2] * g.n[1] * 4;
  box[0] = kBoxK;
  box[1] = rank == 3 ? TileCfg<3>::BOXJ : TileCfg<2>::BOXJ;
  box[2] = rank == 3 ? TileCfg<3>::BOXI : 1;
  CUresult r = g_encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, const_cast<float *>(x), gdim,
                        gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return SEL_ECUDA;
  DebugPtrs d{};
  if (dbg) d = *dbg;
  TileGeo tg = tl.tg;
  Workspace w = ws;
  void *args[] = {(void *)&map, (void *)&tg, (void *)&w, (void *)&d};
  const void *fn = rank == 3 ? tile_fn<3>(dbg != nullptr) : tile_fn<2>(dbg != nullptr);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(tl.ctas);
  cfg.blockDim = dim3(tl.threads);
  cfg.dynamicSmemBytes = tl.smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelExC(&cfg, fn, args) == cudaSuccess ? SEL_OK : SEL_ECUDA;
}

}  // namespace sel
