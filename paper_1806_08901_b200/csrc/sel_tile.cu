// sel_tile.cu -- TMA-fed fused SZ+ZFP pass (the hot path for 2D/3D full-field estimates).
//
// One persistent CTA per SM: warp 8 is the producer, warps 0-7 are consumers.  A task
// is a tile of 8 block rows (one per consumer warp) x 32 blocks along the fastest axis
// (one per lane) x one 4-plane block layer (3D).  The producer fetches task ids from a
// global counter and streams each tile, extended by its -1 halo (one column, one row
// and, in 3D, one plane), into a ring of shared-memory stages with one
// cp.async.bulk.tensor (TMA) per task, completing on an mbarrier (expect_tx).  TMA's
// out-of-bounds zero fill IS the Lorenzo zero boundary (P:151 footnote; reading R4),
// so the consumer code has no boundary branches.  Consumers compute the SZ residuals
// (nested first differences, R4) and quantisation codes (R5) from shared memory into
// the CTA's privatised histogram window, then each lane runs the ZFP block pipeline
// (zfp_block, R8-R14) on its block, re-read from shared memory with the far-edge
// replication (R17) folded into the row/plane index.  Every (task, warp) writes one
// partial, summed in task order by the finalize kernel: bit-reproducible.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include "sel_device.cuh"

namespace sel {

constexpr int kTileWarps = 8;                 // consumer warps = block rows per tile
constexpr int kTileThreads = (kTileWarps + 1) * 32;
constexpr int kBoxK = 4 * 32 + 4;             // 132 floats: 4 halo columns (last one used) + 128
constexpr int kBoxJ = 4 * kTileWarps + 1;     // 33 rows: halo row + 32

template <int D>
struct TileCfg {
  static constexpr int BOXI = D == 3 ? 5 : 1;                     // halo plane + 4 (3D)
  static constexpr int PLANE = kBoxK * kBoxJ;                     // floats per smem plane
  static constexpr int STAGE_FLOATS = PLANE * BOXI;
  static constexpr uint32_t STAGE_BYTES = STAGE_FLOATS * 4;
  static constexpr int STAGE_STRIDE = (STAGE_BYTES + 127) & ~127;
  static constexpr int STAGES = D == 3 ? 2 : 8;
  static constexpr size_t SMEM = (size_t)STAGES * STAGE_STRIDE + kWinBins * 4 + 128;
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
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
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
__device__ __forceinline__ void consumer_sync() {   // the 256 consumer threads only
  asm volatile("bar.sync 1, %0;" ::"n"(kTileWarps * 32) : "memory");
}

// one smem row of the lane's block columns: 4 values + left halo (lane-1's last value;
// lane 0 reads the halo column, which TMA zero-filled at the field's left edge)
__device__ __forceinline__ void srow(const float *row, int lane, float (&v)[4], float &h) {
  const float4 q = *reinterpret_cast<const float4 *>(row + 4 + 4 * lane);
  v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
  const float hs = __shfl_up_sync(0xffffffffu, q.w, 1);
  h = lane == 0 ? row[3] : hs;
}

template <int D, bool DBG>
__global__ void __launch_bounds__(kTileThreads, 1)
    k_tile(const __grid_constant__ CUtensorMap tmap, TileGeo tg, Workspace ws, DebugPtrs dbg) {
  using Cfg = TileCfg<D>;
  constexpr int SZ = Tab<D>::SIZE;
  constexpr int NPL = D == 3 ? 4 : 1;          // data planes per tile
  extern __shared__ unsigned char smem_raw[];
  unsigned char *base =
      reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~(uintptr_t)127);
  unsigned int *sh_hist = reinterpret_cast<unsigned int *>(base + Cfg::STAGES * Cfg::STAGE_STRIDE);
  __shared__ __align__(8) uint64_t full_bar[Cfg::STAGES];
  __shared__ __align__(8) uint64_t empty_bar[Cfg::STAGES];
  __shared__ int stage_task[Cfg::STAGES];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], kTileWarps);
    }
    fence_barrier_init();
  }
  if (warp < kTileWarps) {
    uint4 *s4 = reinterpret_cast<uint4 *>(sh_hist);
    for (int i = threadIdx.x; i < kWinBins / 4; i += kTileWarps * 32) s4[i] = make_uint4(0, 0, 0, 0);
  }
  __syncthreads();
  grid_dep_wait();   // k_minmax done: params valid, the task counter was reset by the
                     // previous field's finalize (which k_minmax waited for)

  // ------------------------------------------------------------------ producer
  if (warp == kTileWarps) {
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
        float *dst = reinterpret_cast<float *>(base + stage * Cfg::STAGE_STRIDE);
        mbar_arrive_expect_tx(&full_bar[stage], Cfg::STAGE_BYTES);
        if constexpr (D == 3)
          tma_load_3d(dst, &tmap, 128 * btk - 4, 32 * btj - 1, 4 * bi - 1, &full_bar[stage]);
        else
          tma_load_2d(dst, &tmap, 128 * btk - 4, 32 * btj - 1, &full_bar[stage]);
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
  unsigned int ovf = 0;
  int stage = 0;
  uint32_t ph = 0;
  for (;;) {
    mbar_wait(&full_bar[stage], ph);
    const int t = stage_task[stage];
    if (t >= tg.ntasks) break;
    const float *S = reinterpret_cast<const float *>(base + stage * Cfg::STAGE_STRIDE);
    const int btk = t % tg.ntk;
    const int rest = t / tg.ntk;
    const int btj = rest % tg.ntj;
    const int bi = rest / tg.ntj;
    const int bj = btj * kTileWarps + warp;
    const int64_t bk = (int64_t)btk * 32 + lane;
    uint64_t tbits = 0;
    double terr = 0.0;
    if (ok && bj < tg.nb[1]) {
      const bool activeK = bk < tg.nb[2];
      const int64_t I0 = 4 * (int64_t)bi, J0 = 4 * (int64_t)bj, K0 = 4 * bk;
      const float *wrow = S + (4 * warp) * kBoxK;   // smem row of j = J0 - 1 (plane 0)
      // ---------------- SZ: nested differences on the tile (R4), codes -> histogram (R5)
      float dprev[4][4];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) dprev[r][c] = 0.0f;
      if constexpr (D == 3) {     // plane i = I0 - 1 (smem plane 0; zeros at i < 0)
        float v[4], h, d1up[4];
        srow(wrow, lane, v, h);
#pragma unroll
        for (int c = 0; c < 4; ++c) d1up[c] = v[c] - (c ? v[c - 1] : h);
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          srow(wrow + (r + 1) * kBoxK, lane, v, h);
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const float d1 = v[c] - (c ? v[c - 1] : h);
            dprev[r][c] = d1 - d1up[c];
            d1up[c] = d1;
          }
        }
      }
#pragma unroll 1
      for (int p = 0; p < NPL; ++p) {
        const int64_t i = I0 + p;
        const float *prow = wrow + (D == 3 ? (p + 1) * Cfg::PLANE : 0);
        float v[4], h, d1up[4];
        srow(prow, lane, v, h);
#pragma unroll
        for (int c = 0; c < 4; ++c) d1up[c] = v[c] - (c ? v[c - 1] : h);
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int64_t j = J0 + r;
          srow(prow + (r + 1) * kBoxK, lane, v, h);
          const bool rowok = activeK && (i < n0) && (j < n1);
          const bool orow = (i == 0) && (j == 0) && (K0 == 0);
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const float d1 = v[c] - (c ? v[c - 1] : h);
            const float d2 = d1 - d1up[c];
            d1up[c] = d1;
            float d;
            if constexpr (D == 3) {
              d = d2 - dprev[r][c];
              dprev[r][c] = d2;
            } else {
              d = d2;
            }
            const bool valid = rowok && !(c == 0 && orow);
            sz_put<DBG>(d, r_f, valid, sh_hist, ws.hist, ovf,
                        DBG ? dbg.codes + (i * n1 + j) * n2 + K0 + c : nullptr);
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
    task_store(ws.task_part, t * kTileWarps + warp, tbits, terr);
    if (++stage == Cfg::STAGES) { stage = 0; ph ^= 1u; }
  }
  ovf_flush(ovf, ws.hist);
  consumer_sync();
  {
    const uint4 *s4 = reinterpret_cast<const uint4 *>(sh_hist);
    for (int i = threadIdx.x; i < kWinBins / 4; i += kTileWarps * 32) {
      const uint4 c = s4[i];
      unsigned long long *g = ws.hist + (kCenter - kWinHalf) + 4 * i;
      if (c.x) atomicAdd(g + 0, (unsigned long long)c.x);
      if (c.y) atomicAdd(g + 1, (unsigned long long)c.y);
      if (c.z) atomicAdd(g + 2, (unsigned long long)c.z);
      if (c.w) atomicAdd(g + 3, (unsigned long long)c.w);
    }
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
  for (int a = 0; a < 3; ++a) { t.n[a] = g.n[a]; t.nb[a] = (int)g.nb[a]; }
  t.ntj = (int)((g.nb[1] + kTileWarps - 1) / kTileWarps);
  t.ntk = (int)((g.nb[2] + 31) / 32);
  const int64_t nt = (int64_t)t.ntj * t.ntk * (g.ndims == 3 ? g.nb[0] : 1);
  if (nt > (1LL << 27)) return SEL_EINVAL;
  t.ntasks = (int)nt;
  const size_t smem = g.ndims == 3 ? TileCfg<3>::SMEM : TileCfg<2>::SMEM;
  const void *fn = g.ndims == 3 ? tile_fn<3>(debug) : tile_fn<2>(debug);
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return SEL_ECUDA;
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kTileThreads, smem) != cudaSuccess)
    return SEL_ECUDA;
  if (occ < 1) return SEL_ECUDA;
  const int64_t cap = (int64_t)occ * sm_count;
  tl->ctas = (int)(nt < cap ? nt : cap);
  if (tl->ctas < 1) tl->ctas = 1;
  tl->smem = smem;
  tl->npart = t.ntasks * kTileWarps;
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
  box[1] = kBoxJ;
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
  cfg.blockDim = dim3(kTileThreads);
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
