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
// first differences, R4) and quantisation codes (R5) from shared memory into one CTA-wide
// shared-memory histogram window (atomicAdd with an unused result compiles to
// ATOMS.POPC.INC, which merges the lanes of a warp hitting the same bin), then each lane
// runs the ZFP block pipeline (zfp_block, R8-R14) on its
// block, re-read from shared memory with the far-edge replication (R17) folded into the
// row/plane index.  Every (task, warp) writes one partial, summed in task order by the
// finalize kernel: bit-reproducible regardless of the dynamic schedule.
#include "sel_tile_common.cuh"

namespace sel {

template <int D, bool DBG>
__global__ void __launch_bounds__(TileCfg<D>::THREADS, 1)
    k_tile(const __grid_constant__ CUtensorMap tmap, TileGeo tg, Workspace ws, DebugPtrs dbg) {
  using Cfg = TileCfg<D>;
  constexpr int CW = Cfg::CW;
  extern __shared__ float smem_dyn[];
  // 128-byte align the stage ring (TMA destination) without leaving the shared window
  float *const base = smem_dyn + (((128u - (smem_u32(smem_dyn) & 127u)) & 127u) >> 2);
  unsigned int *const hist = reinterpret_cast<unsigned int *>(base + Cfg::STAGES * Cfg::STAGE_FLOATS);
  // barriers + per-stage descriptors, 16-byte aligned (hist starts 128-byte aligned)
  uint64_t *const full_bar =
      reinterpret_cast<uint64_t *>(hist + Cfg::HIST_WORDS);
  uint64_t *const empty_bar = full_bar + Cfg::STAGES;
  int4 *const stage_task = reinterpret_cast<int4 *>(empty_bar + Cfg::STAGES);   // {t, btk, btj, bi}

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], CW);
    }
    fence_barrier_init();
  }
  for (int i = threadIdx.x; i < Cfg::HIST_WORDS; i += Cfg::THREADS) hist[i] = 0u;
  __syncthreads();
  grid_dep_wait();   // k_minmax done: params valid, the task counter was reset by the
                     // previous field's finalize (which k_minmax waited for)

  // ------------------------------------------------------------------ producer
  if (warp == CW) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
      int stage = 0;
      uint32_t ph = 0;
      int next = (int)atomicAdd(ws.task_ctr, 1u);     // fetched one task ahead
      for (;;) {
        const int t = next;
        if (t < tg.ntasks) next = (int)atomicAdd(ws.task_ctr, 1u);
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
    }
    return;
  }

  // ------------------------------------------------------------------ consumers
  const Params prm = *ws.params;
  const bool ok = prm.status == SEL_OK;
  const float r_f = prm.r_f;
  const int minexp = prm.minexp;
  unsigned int ovf = 0;
  int stage = 0;
  uint32_t ph = 0;
  for (;;) {
    mbar_wait(&full_bar[stage], ph);
    const int4 td = stage_task[stage];
    const int t = td.x;
    if (t >= tg.ntasks) break;
    const float *S = base + stage * Cfg::STAGE_FLOATS;
    uint64_t tbits = 0;
    double terr = 0.0;
    tile_consume<D, DBG>(S, td.y, td.z, td.w, tg, warp, lane, ok, r_f, minexp, hist, ws.hist, ovf,
                         dbg, tbits, terr);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty_bar[stage]);    // stage free for the producer
    task_store(ws.task_part, t * CW + warp, tbits, terr);
    if (++stage == Cfg::STAGES) { stage = 0; ph ^= 1u; }
  }
  ovf_flush(ovf, ws.hist);
  consumer_sync<CW * 32>();
  tile_hist_flush<D>(hist, ws.hist, threadIdx.x, CW * 32);
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
         g.n[2] % 4 == 0 && g.n[2] < (1LL << 30) && g.n[1] < (1LL << 30) && g.n[0] < (1LL << 30);
}

int plan_tile(const Geo &g, int sm_count, int debug, TileLaunch *tl) {
  TileGeo &t = tl->tg;
  const int cw = g.ndims == 3 ? TileCfg<3>::CW : TileCfg<2>::CW;
  const int rows = g.ndims == 3 ? TileCfg<3>::ROWS : TileCfg<2>::ROWS;   // block rows per tile
  for (int a = 0; a < 3; ++a) { t.n[a] = g.n[a]; t.nb[a] = (int)g.nb[a]; }
  t.ntj = (int)((g.nb[1] + rows - 1) / rows);
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

// TMA descriptor of a field for the tile box (x: 16-B aligned, fastest extent % 4 == 0)
int make_tile_map(CUtensorMap *map, const float *x, const Geo &g) {
  if (get_encode()) return SEL_ECUDA;
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
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, const_cast<float *>(x), gdim,
                        gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? SEL_OK : SEL_ECUDA;
}

int launch_tile(const float *x, const Geo &g, const TileLaunch &tl, const Workspace &ws,
                const DebugPtrs *dbg, cudaStream_t st) {
  CUtensorMap map;
  if (make_tile_map(&map, x, g)) return SEL_ECUDA;
  const int rank = g.ndims;
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
