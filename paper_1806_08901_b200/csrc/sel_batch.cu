// sel_batch.cu -- one persistent launch for a whole batch of fields (2D/3D tile shapes).
//
// The estimate of a field is three dependent phases: value range (needs every value,
// Alg.1 line 2), the fused SZ+ZFP tile pass (needs eb, r_f, minexp), and the histogram
// entropy / selection (needs every tile).  Instead of three launches per field, one
// persistent CTA per SM pulls tasks of three kinds from a single global sequence laid out
// in phases:   phase p = [ F(p-4) | R(p) and T(p-2) interleaved ]
//   R(f, i): TMA bulk copy of chunk i of field f into a stage, min/max/non-finite;
//            the last R task of f writes params(f) and raises params_ready[f]
//   T(f, i): the TMA tile task of k_tile (same consumer code, sel_tile_common.cuh)
//   F(f, k): 1/8 of the histogram entropy + tile partials of f (needs tdone[f] == nT);
//            the last F task of f writes result f and raises fin_ready[f]
// A task only ever waits (spin on a flag) for tasks earlier in the sequence, every CTA
// processes its tasks in fetch order, and a CTA flushes its shared-memory histogram
// before it starts any task that may block (T of another field, F) -- so the earliest
// unfinished task can always run: no deadlock.  The value range of field f+1 (DRAM) and
// the finalize of f-1 overlap the tiles of f (ALU), there is no launch or ramp between
// fields, and field f arrives in L2 two phases before its tiles.  Histogram/partial
// buffers rotate over f % 3 (T(f) waits fin_ready[f-3]).  All floating-point sums
// are per task and reduced in task order: results are bit-identical to the per-field path.
// The sequence is decoded once on the host (build_group_sequence, cached per key) into a
// 16-byte-per-task table the producer reads: decoding on the producer thread itself was
// the kernel's critical path.
#include <vector>

#include "sel_tile_common.cuh"

namespace sel {

constexpr int kFinTasks = 8;                   // F tasks per field (8192 slots each)
constexpr int kRing = 3;                       // histogram / partial buffers (field % 3)
// phase p: R(p), T(p - lagT), F(p - lagF) with lagF = lagT + 2 (BatchArgs; default 2 / 4)
// Global histograms are u32 (a field has < 2^32 values: batch_ok) with slot s at word
// 1 + s of its ring slot, so the smem window / table land on 16-byte aligned global
// addresses for cp.reduce.async.bulk; stride 65,540 words keeps every ring slot aligned.
constexpr int kH32Stride = kNSlots + 4;
#ifndef SEL_RWARPS
#define SEL_RWARPS 6                           // range chunk split over min(this, CW) warps (rotating)
#endif
#ifndef SEL_NO_PF
#define SEL_NO_PF 0                            // developer probe: no L2 prefetch at claim time
#endif
#ifndef SEL_CLAIM
#define SEL_CLAIM 1                            // producer: task ids claimed per atomic
#endif
#ifndef SEL_PWAIT
#define SEL_PWAIT 1000                          // producer stage wait: 0 probe loop, > 0 try_wait hint (ns)
#endif
#ifndef SEL_RSLEEP
#define SEL_RSLEEP 32                          // release warp: first / reset sleep between queue polls (ns)
#endif
#ifndef SEL_PBACKOFF
#define SEL_PBACKOFF 64                        // producer: longest sleep between stage probes (ns)
#endif
#ifndef SEL_BATCH_PROF
#define SEL_BATCH_PROF 0                       // 1: per-CTA cycle counters (sel_dev_batch_profile)
#endif
#if SEL_BATCH_PROF
#define PROF(stmt) stmt
#define PCLOCK() clock64()
#else
#define PROF(stmt)
#define PCLOCK() 0LL
#pragma nv_diag_suppress 177                    // timestamps unused without profiling
#endif

// float -> unsigned key with the same order (for atomicMin/atomicMax), and back
__device__ __forceinline__ unsigned int float_key(float v) {
  const unsigned int b = __float_as_uint(v);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float key_float(unsigned int k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}
struct FPart { double acc, err; unsigned long long bits, ovf, cnt; };

struct BatchArgs {
  const CUtensorMap *tmaps;       // [nf], 64-B aligned, global
  const float *const *xs;         // [nf] device pointers
  int nf;
  TileGeo tg;
  Geo g;                          // sampling geometry (sampled != 0: strides > 1)
  int sampled;                    // T tasks are sampled-block tasks (no TMA tile)
  int64_t N;
  int nR, nT, phase;              // tasks per field (F: kFinTasks); phase = kFinTasks + nR + nT
  const uint4 *ttab;              // decoded task sequences of all groups (host-built)
  int rchunk;                     // floats per R task
  int rw;                         // 1: the value range is streamed by the range warps (no R tasks)
  int nRc, rcf;                   // range-warp chunks per field, floats per chunk
  unsigned int *rtask_ctr;        // [G] range-warp chunk counter of each group
  FinalizeArgs fa;
  int mode;
  double eb;
  // state
  Params *params;                 // [nf]
  unsigned int *rmin, *rmax, *rbad; // [nf] order-preserving keys of min / max, non-finite flag
  unsigned int *rdone;            // [nf] range slices done (nR * CW per field)
  unsigned int *params_ready;     // [nf]
  unsigned int *tdone;            // [nf] tile tasks whose histogram counts are flushed
  unsigned int *fdone;            // [nf]
  unsigned int *fin_ready;        // [nf]
  int lagT, lagF;                 // phases from a field's range pass to its tiles / finalize
  int G;                          // CTA groups: group g = blockIdx % G runs fields f = g (mod G)
  unsigned int *hist;             // [G * kRing][kH32Stride] (slot s at 1 + s), slot ring(f)
  Partial *tpart;                 // [G * kRing][nT * CW]
  FPart *fpart;                   // [G * kRing][kFinTasks]
  unsigned int *task_ctr;         // [G]
  sel_result *results;            // [nf]
  unsigned int *hdump;            // optional [nf][kNSlots]: each field's histogram as the F tasks read it
  Partial *pdump;                 // optional [nf][nT * CW]: each field's per-(task, warp) partials
  unsigned long long *prof;       // optional [gridDim * 8] cycle counters (warp 0 of each CTA)
};

enum { KIND_NONE = 0, KIND_R = 1, KIND_T = 2, KIND_F = 3 };

// Task sequence without padding.  Phase p holds F(p-kLagF) [kFinTasks] first, then
// R(p) [nR] and T(p-kLagT) [nT] interleaved (Bresenham); absent fields contribute nothing.
// R runs kLagT phases ahead of its tiles (its results are published at the next phase
// boundary), F runs two phases after them (every CTA has flushed by then).
// With G CTA groups every group runs this sequence over its own fields (local index
// l <-> field l * G + g) with its own task counter, so a CTA meets G x fewer fields.
__device__ __forceinline__ bool in_range(int nfl, int f) { return f >= 0 && f < nfl; }

__device__ __forceinline__ long long phase_size(const BatchArgs &a, int nfl, int p) {
  return (long long)(in_range(nfl, p - a.lagF) ? kFinTasks : 0) + (in_range(nfl, p) ? a.nR : 0) +
         (in_range(nfl, p - a.lagT) ? a.nT : 0);
}

// buffer slot of field f: kRing per group, reused by field f + kRing * G
__device__ __forceinline__ int ring(const BatchArgs &a, int f) {
  return (f % a.G) * kRing + (f / a.G) % kRing;
}

__device__ __forceinline__ void bulk_load(void *dst, const void *src, uint32_t bytes, uint64_t *bar,
                                          uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d_hint(void *dst, const CUtensorMap *map, int c0, int c1,
                                                 int c2, uint64_t *bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)),
      "l"(policy)
      : "memory");
}
__device__ __forceinline__ void bulk_prefetch(const void *src, uint32_t bytes, uint64_t policy) {
  asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(src),
               "r"(bytes), "l"(policy)
               : "memory");
}
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap *map, int c0, int c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap *map, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
__device__ __forceinline__ void tma_load_2d_hint(void *dst, const CUtensorMap *map, int c0, int c1,
                                                 uint64_t *bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// Bulk reduction shared -> global by the TMA engine (the histogram flush): one instruction
// adds a whole smem array into global memory at L2, instead of one atomic per bin.
__device__ __forceinline__ void bulk_reduce_add_u32(unsigned int *gdst, const void *ssrc, uint32_t bytes) {
  asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.u32 [%0], [%1], %2;" ::"l"(gdst),
               "r"(smem_u32(ssrc)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ float fmin_nan(float a, float b) {   // NaN if either is NaN
  float r;
  asm("min.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float fmin3_nan(float a, float b, float c) {   // sm_100 FMNMX3
  float r;
  asm("min.NaN.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
__device__ __forceinline__ unsigned int ld_acquire_cta(const unsigned int *p) {
  unsigned int v;
  asm volatile("ld.acquire.cta.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_cta(unsigned int *p, unsigned int v) {
  asm volatile("st.release.cta.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Release requests, consumer tid 0 -> release warp (shared-memory ring).  The release warp
// makes a flush / range publication visible (fence.acq_rel.gpu + counter increment) so the
// fence's wait for the CTA's outstanding atomics never stalls the consumer warps.  The
// chain consumer atomics -> bar.sync -> st.release.cta(head) -> ld.acquire.cta(head) ->
// fence.acq_rel.gpu -> atomicAdd is cumulative (PTX memory model), so the increment
// publishes every consumer thread's atomics.  A request never waits on another CTA.
enum { REQ_T = 1, REQ_R = 2, REQ_END = 3 };
struct RelReq { int kind, f; unsigned int cnt, rmin, rmax, rbad; };
constexpr int kRelQ = 16;

// Range warps: extra warps that stream the value range of the fields ahead of the
// tiles straight from global memory into registers (LDG.128, 32 in flight per lane), so the
// stage ring carries tiles only and a tile loads while the previous one is computed (with R
// tasks interleaved on a 2-stage ring every tile load waited for the tile before it).
#ifndef SEL_RW3
#define SEL_RW3 1              // 3D: one range warp (C4 1.59 -> 1.62 TB/s, C3 +2-3 % against two; waiting consumers help)
#endif
#ifndef SEL_RW2
#define SEL_RW2 2              // 2D: 2 range warps (C2 1.73 -> 1.95 TB/s with 20 consumer warps, 1.92 with 16 -- kept: stride (1,10) 2.41 -> 3.04; 1 or 3-4 range warps: no gain)
#endif
template <int D>
constexpr int range_warps() { return D == 3 ? SEL_RW3 : SEL_RW2; }
template <int D>
constexpr int batch_threads() { return (TileCfg<D>::CW + 2 + range_warps<D>()) * 32; }   // + producer + release warp
constexpr int kRwChunk = 16384;                // floats per range-warp chunk (64 KB)

// producer: wait until a stage is free.  SEL_PWAIT = 0: probe + nanosleep back-off;
// otherwise a hardware-suspended mbarrier.try_wait with that time hint (ns): the thread
// sleeps until the phase completes (or the hint expires) instead of re-issuing probes --
// the probe loop took ~8 % of the 3D kernel's issued instructions (ncu r02b)
__device__ __forceinline__ void mbar_wait_backoff(uint64_t *bar, uint32_t parity) {
  if (SEL_PWAIT > 0) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAITP_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
        "@!p bra WAITP_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "n"(SEL_PWAIT)
        : "memory");
    return;
  }
  unsigned int ns = 64;
  while (!mbar_test(bar, parity)) {
    __nanosleep(ns);
    if (ns < SEL_PBACKOFF) ns <<= 1;
  }
}

// Named barriers for the waits inside the CTA.  A warp blocked in bar.sync issues nothing;
// an mbarrier try_wait / nanosleep poll does not stay asleep while bulk copies land in the
// CTA (every complete_tx wakes NANOSLEEP.SYNCS: ncu showed the producer's stage wait looping
// every ~8 ns, ~10 % of the kernel's issued instructions, and the release warp's queue poll
// another ~5 %).  Ids: 0 __syncthreads, 1 consumers, 2 + s "stage s is free" (consumer
// warps arrive, the producer warp syncs), kBarReq the consumer warp 0 <-> release warp
// hand-over (both sync: a rendezvous per request).
constexpr int kBarStage = 2, kBarReq = 8;
__device__ __forceinline__ void bar_sync_n(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_arrive_n(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// warp 0 lane 0 spins until *flag >= target (acquire); the caller syncs the consumers
__device__ __forceinline__ void spin_until(const unsigned int *flag, unsigned int target) {
  unsigned int ns = 32;
  long long guard = 0;
  while (ld_acquire(flag) < target) {
    __nanosleep(ns);
    if (ns < 1024) ns <<= 1;
    if (++guard > (1LL << 24)) __trap();     // never hang the GPU on a logic error
  }
}


// ---- value range by streaming warps (rw mode): chunk c of a group = (local field c / nRc,
// chunk c % nRc), claimed in order from the group's counter by the range warps and by
// consumer warps that are waiting for a field's parameters.
__device__ __forceinline__ float4 ldg_keep(const float4 *p, uint64_t pol) {
  float4 v;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
      : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
      : "l"(p), "l"(pol));
  return v;
}
struct RangeAcc { float mn, mx, mn2, mx2; unsigned int cnt; };
__device__ __forceinline__ void range_reset(RangeAcc &r) {
  r.mn = r.mn2 = INFINITY;
  r.mx = r.mx2 = -INFINITY;
  r.cnt = 0u;
}
// min / max of one chunk (n4 float4, 16-byte aligned) into the warp's accumulators; NaN
// propagates through min.NaN (R1), 32 loads in flight per lane
__device__ __forceinline__ void range_chunk(const float4 *__restrict__ src, int n4, int lane,
                                            uint64_t pol, RangeAcc &r) {
  constexpr int U = 32;
  int i = lane;
#pragma unroll 1
  for (; i + (U - 1) * 32 < n4; i += U * 32) {
    float4 q[U];
#pragma unroll
    for (int k = 0; k < U; ++k) q[k] = ldg_keep(src + i + k * 32, pol);
#pragma unroll
    for (int k = 0; k < U; ++k) {
      r.mn = fmin3_nan(r.mn, q[k].x, q[k].y);
      r.mx = fmax3(r.mx, q[k].x, q[k].y);
      r.mn2 = fmin3_nan(r.mn2, q[k].z, q[k].w);
      r.mx2 = fmax3(r.mx2, q[k].z, q[k].w);
    }
  }
#pragma unroll 1
  for (; i < n4; i += 32) {
    const float4 q = ldg_keep(src + i, pol);
    r.mn = fmin3_nan(r.mn, q.x, q.y);
    r.mx = fmax3(r.mx, q.x, q.y);
    r.mn2 = fmin3_nan(r.mn2, q.z, q.w);
    r.mx2 = fmax3(r.mx2, q.z, q.w);
  }
  ++r.cnt;
}

template <int D>
__global__ void __launch_bounds__(batch_threads<D>(), 1) k_batch(const BatchArgs a) {
  using Cfg = TileCfg<D>;
  constexpr int CW = Cfg::CW;
  constexpr int NC = CW * 32;                  // consumer threads
  constexpr int kRWarps = SEL_RWARPS > CW ? CW : SEL_RWARPS;   // consumer warps reducing one range chunk
  extern __shared__ float smem_dyn[];
  float *const base = smem_dyn + (((128u - (smem_u32(smem_dyn) & 127u)) & 127u) >> 2);
  unsigned int *const hist = reinterpret_cast<unsigned int *>(base + Cfg::STAGES * Cfg::STAGE_FLOATS);
  // barriers + per-stage descriptors, 16-byte aligned (hist starts 128-byte aligned)
  uint64_t *const full_bar =
      reinterpret_cast<uint64_t *>(hist + Cfg::HIST_WORDS);
  uint64_t *const empty_bar = full_bar + Cfg::STAGES;
  // per stage, decoded once by the producer: {kind | end flag, f, id, phase} and the tile
  // coordinates {btk, btj, bi}
  int4 *const stage_desc = reinterpret_cast<int4 *>(empty_bar + Cfg::STAGES);
  int4 *const stage_tile = stage_desc + Cfg::STAGES;
  __shared__ double s_red[3][CW];
  __shared__ unsigned long long s_redu[3][CW];
  constexpr int NCHUNK = Cfg::W / kChunk;
  __shared__ int s_chunk[NCHUNK];                // window chunks with a nonzero bin (flush)
  __shared__ unsigned int s_rmin[2], s_rmax[2], s_rbad[2], s_rcnt[2];
  __shared__ RelReq s_q[kRelQ];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  const int grp = (int)(blockIdx.x % (unsigned)a.G);
  const int nfl = (a.nf - grp + a.G - 1) / a.G;                  // this group's fields
  const long long ntot = (long long)nfl * (a.nR + a.nT + kFinTasks);
  // this group's task table: groups before it hold (fields with f % G < grp) sequences
  const uint4 *const ttab = a.ttab + (long long)a.phase * ((long long)grp * (a.nf / a.G) + min(grp, a.nf % a.G));
  if (tid == 0) {
    for (int k = 0; k < 2; ++k) {
      s_rmin[k] = 0xffffffffu; s_rmax[k] = 0u; s_rbad[k] = 0u; s_rcnt[k] = 0u;
    }
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
    }
    fence_barrier_init();
  }
  for (int i = tid; i < Cfg::HIST_WORDS; i += (int)blockDim.x) hist[i] = 0u;
  __syncthreads();

  // ---- rw mode: chunk claim / publish (range warps, and consumer warps waiting for params)
  const bool rw_on = range_warps<D>() > 0 && a.rw != 0;     // (compiled out of the 2D kernel)
  const unsigned int rw_total = rw_on ? (unsigned)nfl * (unsigned)a.nRc : 0u;
  auto rw_claim = [&]() -> unsigned int {
    unsigned int c = 0u;
    if (lane == 0) c = atomicAdd(a.rtask_ctr + grp, 1u);
    return __shfl_sync(0xffffffffu, c, 0);
  };
  // the warp's accumulated chunks of local field l -> the field's global min / max keys;
  // the last contributor of the field writes params(f) (Alg. 1 line 2)
  auto rw_publish = [&](int l, RangeAcc &r) {
    if (r.cnt) {
      float mn = fmin_nan(r.mn, r.mn2), mx = fmaxf(r.mx, r.mx2);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        mn = fmin_nan(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      }
      if (lane == 0) {
        const int g = l * a.G + grp;
        const int bad = (mn != mn) | ((mn <= mx) & (is_nonfinite(mn) | is_nonfinite(mx)));
        if (mn <= mx) {
          atomicMin(a.rmin + g, float_key(mn));
          atomicMax(a.rmax + g, float_key(mx));
        }
        if (bad) atomicOr(a.rbad + g, 1u);
        fence_acq_rel_gpu();
        if (atomicAdd(a.rdone + g, r.cnt) + r.cnt == (unsigned)a.nRc) {   // last
          fence_acq_rel_gpu();
          const float fmn = key_float(ld_acquire(a.rmin + g)), fmx = key_float(ld_acquire(a.rmax + g));
          a.params[g] = make_params(fmn, fmx, (int)ld_acquire(a.rbad + g), a.mode, a.eb);
          fence_acq_rel_gpu();
          st_release(a.params_ready + g, 1u);
        }
      }
      __syncwarp();
    }
    range_reset(r);
  };
  auto rw_chunk = [&](unsigned int c, uint64_t pol, RangeAcc &r) {   // chunk c of this group
    const int l = (int)(c / (unsigned)a.nRc), i = (int)(c % (unsigned)a.nRc);
    const long long lo = (long long)i * a.rcf;
    const int n4 = (int)(min((long long)a.rcf, a.N - lo) >> 2);
    range_chunk(reinterpret_cast<const float4 *>(a.xs[l * a.G + grp] + lo), n4, lane, pol, r);
  };

  // ------------------------------------------------------------------ producer
  if (warp == CW) {
    {
      int stage = 0;
      uint32_t ph = 0;
      // L2 policies: a range task's chunk is read again by the field's tiles two phases
      // later (keep it: evict_last); a tile is the last use (evict_first)
      uint64_t pol_keep, pol_last;
      asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_keep));
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_last));
      // Task ids are claimed two tasks ahead: a claimed task is decoded and its data
      // prefetched into L2 (range chunks come from HBM; tiles of big fields too) while
      // earlier stages are consumed; the claim's atomic itself is issued one iteration
      // before its result is needed.
      struct Dec { int kind, f, id, phase, btk, btj, bi, slot; };
      // A task is decoded from one task-table entry (instead of decoding the sequence
      // on this issue-starved thread); the entry is fetched one task before it is decoded
      auto fetch = [&](long long tau) -> uint4 {
        return tau < ntot ? __ldg(ttab + tau) : make_uint4(0u, 0u, 0u, 0u);
      };
      auto decode_pf = [&](long long tau, const uint4 e, Dec &d) {
        d.kind = KIND_NONE; d.f = 0; d.id = 0; d.phase = 0; d.btk = d.btj = d.bi = 0; d.slot = 0;
        if (tau >= ntot) { d.kind = -1; return; }
        d.kind = (int)(e.x & 3u);
        d.phase = (int)(e.x >> 2);
        d.id = (int)e.y;
        d.f = d.phase - (d.kind == KIND_R ? 0 : d.kind == KIND_T ? a.lagT : a.lagF);
        d.slot = grp * kRing + d.f % kRing;  // = ring(a, global field)
        d.f = d.f * a.G + grp;             // global field index
        if (d.kind == KIND_T && !a.sampled) {
          d.btk = (int)(e.z & 0xffffu);
          d.btj = (int)(e.z >> 16);
          d.bi = (int)e.w;
          if (!SEL_NO_PF) {
            if constexpr (D == 3)
              tma_prefetch_3d(a.tmaps + d.f, 128 * d.btk - 4, 4 * Cfg::ROWS * d.btj - 1, 4 * d.bi - 1);
            else
              tma_prefetch_2d(a.tmaps + d.f, 128 * d.btk - 4, 4 * Cfg::ROWS * d.btj - 1);
          }
        } else if (d.kind == KIND_R) {
          const long long lo = (long long)d.id * a.rchunk;
          const long long cnt = min((long long)a.rchunk, a.N - lo);
          if (!SEL_NO_PF) bulk_prefetch(a.xs[d.f] + lo, (uint32_t)(cnt * 4), pol_keep);
        }
      };
      // Tasks are claimed SEL_CLAIM consecutive ids per atomic, the next batch's atomic
      // one batch ahead: the claim's round trip to L2 (a counter shared by the group's
      // CTAs) is off the producer's critical path (it was ~2,000 cycles per task).
      constexpr unsigned int K = SEL_CLAIM;
      long long cb = ntot, nb = ntot;
      if (lane == 0) {
        cb = (long long)atomicAdd(a.task_ctr + grp, K);
        nb = cb < ntot ? (long long)atomicAdd(a.task_ctr + grp, K) : ntot;
      }
      unsigned int ck = 0;
      auto next_tau = [&]() -> long long {
        if (ck == K) {
          cb = nb;
          ck = 0;
          nb = cb < ntot ? (long long)atomicAdd(a.task_ctr + grp, K) : ntot;
        }
        const long long t = cb + ck++;
        return t < ntot ? t : ntot;
      };
      Dec t0, t1;
      t0.kind = t1.kind = -1;
      long long tau_n = ntot;
      uint4 e_n = make_uint4(0u, 0u, 0u, 0u);
      if (lane == 0) {
        tau_n = next_tau();
        decode_pf(tau_n, fetch(tau_n), t0);
        tau_n = next_tau();
        decode_pf(tau_n, fetch(tau_n), t1);
        tau_n = t1.kind < 0 ? ntot : next_tau();
        e_n = fetch(tau_n);              // in flight: the task after t1
      }
      __syncwarp();
      long long pp_start = PCLOCK(), pp_wait = 0, pp_dec = 0, pp_n = 0;
      long long posted = 0;
      // every lane walks the loop (the stage wait is a warp-level bar.sync); lane 0 works
      for (;;) {
        const long long pw0 = PCLOCK();
        if (posted >= Cfg::STAGES) bar_sync_n(kBarStage + stage, (CW + 1) * 32);
        ++posted;
        PROF(pp_wait += clock64() - pw0; ++pp_n);
        int done = 0;
        if (lane == 0) {
        stage_desc[stage] = make_int4(t0.kind, t0.f, t0.id, t0.phase);
        stage_tile[stage] = make_int4(t0.btk, t0.btj, t0.bi, t0.slot);
        float *dst = base + stage * Cfg::STAGE_FLOATS;
        if (t0.kind == KIND_T && !a.sampled) {
          mbar_arrive_expect_tx(&full_bar[stage], Cfg::STAGE_BYTES);
          if constexpr (D == 3)
            tma_load_3d_hint(dst, a.tmaps + t0.f, 128 * t0.btk - 4, 4 * Cfg::ROWS * t0.btj - 1,
                             4 * t0.bi - 1, &full_bar[stage], pol_last);
          else
            tma_load_2d_hint(dst, a.tmaps + t0.f, 128 * t0.btk - 4, 4 * Cfg::ROWS * t0.btj - 1,
                             &full_bar[stage], pol_last);
        } else if (t0.kind == KIND_R) {
          const long long lo = (long long)t0.id * a.rchunk;
          const long long cnt = min((long long)a.rchunk, a.N - lo);   // multiple of 4 floats
          mbar_arrive_expect_tx(&full_bar[stage], (uint32_t)(cnt * 4));
          bulk_load(dst, a.xs[t0.f] + lo, (uint32_t)(cnt * 4), &full_bar[stage], pol_keep);
        } else {
          mbar_arrive(&full_bar[stage]);   // F / sampled T / sentinel: no staged data
        }
        done = t0.kind < 0;
        }
        done = __shfl_sync(0xffffffffu, done, 0);
        if (++stage == Cfg::STAGES) { stage = 0; ph ^= 1u; }
        if (done) break;                   // the sentinel went out: done
        if (lane == 0) {
        t0 = t1;
        const long long pd0 = PCLOCK();
        decode_pf(tau_n, e_n, t1);
        tau_n = t1.kind < 0 ? ntot : next_tau();
        e_n = fetch(tau_n);
        PROF(pp_dec += clock64() - pd0);
        }
        __syncwarp();
      }
#if SEL_BATCH_PROF
      if (a.prof && lane == 0) {
        atomicAdd(a.prof + 148 * 8 + 8, (unsigned long long)(clock64() - pp_start));
        atomicAdd(a.prof + 148 * 8 + 9, (unsigned long long)pp_wait);
        atomicAdd(a.prof + 148 * 8 + 10, (unsigned long long)pp_dec);
        atomicAdd(a.prof + 148 * 8 + 11, (unsigned long long)pp_n);
      }
#endif
    }
    return;
  }

  // ------------------------------------------------------------------ release warp
  if (warp == CW + 1) {
    // one rendezvous (bar.sync kBarReq) per request: consumer warp 0 wrote s_q[t % kRelQ]
    // before it; blocked in the barrier the warp issues nothing
    for (unsigned int t = 0;; ++t) {
      bar_sync_n(kBarReq, 64);
      const RelReq r = s_q[t % kRelQ];
      if (r.kind == REQ_END) break;
      if (lane == 0) {
        if (r.kind == REQ_T) {
          fence_acq_rel_gpu();
          atomicAdd(a.tdone + r.f, r.cnt);
        } else {                     // REQ_R: this CTA's range slices of field r.f
          const int g = r.f;
          if (r.rmin != 0xffffffffu) atomicMin(a.rmin + g, r.rmin);
          if (r.rmax != 0u) atomicMax(a.rmax + g, r.rmax);
          if (r.rbad) atomicOr(a.rbad + g, 1u);
          fence_acq_rel_gpu();
          if (atomicAdd(a.rdone + g, r.cnt) + r.cnt == (unsigned)a.nR * kRWarps) {   // last
            fence_acq_rel_gpu();
            const float fmn = key_float(ld_acquire(a.rmin + g)), fmx = key_float(ld_acquire(a.rmax + g));
            a.params[g] = make_params(fmn, fmx, (int)ld_acquire(a.rbad + g), a.mode, a.eb);
            fence_acq_rel_gpu();
            st_release(a.params_ready + g, 1u);
          }
        }
      }
      __syncwarp();
    }
    return;
  }

  // ------------------------------------------------------------------ range warps
  if (warp >= CW + 2) {
    if (rw_on) {
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
      RangeAcc r;
      range_reset(r);
      int curl = -1;
      unsigned int c = rw_claim();
      while (c < rw_total) {
        const unsigned int cn = rw_claim();     // the next claim's round trip overlaps this chunk
        const int l = (int)(c / (unsigned)a.nRc);
        if (l != curl) {
          if (curl >= 0) rw_publish(curl, r);   // nothing is held across the wait below
          curl = l;
          // (no pacing against the tiles: a wait here would be a poll loop, and polls steal
          // issue slots from the consumer warps; the range simply runs ahead of the tiles)
        }
        rw_chunk(c, pol, r);
        c = cn;
      }
      if (curl >= 0) rw_publish(curl, r);
    }
    return;
  }

  // ------------------------------------------------------------------ consumers
  int cur = -1;                    // field owning the smem histogram
  int cur_slot = 0;                // its ring slot
  unsigned int cur_tasks = 0;      // its T tasks since the last flush
  unsigned int ovf = 0;
  bool ok = false;
  float r_f = 0.f;
  int minexp = 0;
  DebugPtrs nodbg{};

#if SEL_BATCH_PROF
  long long pc[8] = {0, 0, 0, 0, 0, 0, 0, 0};   // wait, flush, T, R, F, release, #flush, #publish
#endif

  unsigned int qh = 0;             // consumer warp 0: next request slot
  auto enqueue = [&](int kind, int f, unsigned int cnt, unsigned int rmn, unsigned int rmx,
                     unsigned int rbd) {   // every lane of consumer warp 0
    const long long tp0 = PCLOCK();
    if (lane == 0) {
      RelReq r;
      r.kind = kind; r.f = f; r.cnt = cnt; r.rmin = rmn; r.rmax = rmx; r.rbad = rbd;
      s_q[qh % kRelQ] = r;
    }
    ++qh;
    __syncwarp();
    bar_sync_n(kBarReq, 64);        // hand-over: the release warp reads the slot after it
    PROF(pc[5] += clock64() - tp0);
  };

  // Histogram flush (all consumers, same task): the warps mark the window's nonzero
  // 1024-bin chunks, tid 0 adds those chunks into the field's global histogram with bulk
  // reductions (the TMA engine, cp.reduce.async.bulk .add.u32), the consumers clear them
  // once they have been read, and the publication (tdone) waits for the reductions to
  // complete.
  auto flush = [&]() {
    unsigned int *gh = a.hist + (size_t)cur_slot * kH32Stride + 1;
    const long long q0 = PCLOCK();
    {
      unsigned int o = ovf;
#pragma unroll
      for (int k = 16; k > 0; k >>= 1) o += __shfl_xor_sync(0xffffffffu, o, k);
      if (lane == 0 && o) atomicAdd(gh + kOvfSlot, o);
    }
    ovf = 0;
    const long long q1 = PCLOCK();
    consumer_sync<NC>();
    const long long q2 = PCLOCK();
    for (int c = warp; c < NCHUNK; c += CW) {
      const uint4 *h4 = reinterpret_cast<const uint4 *>(hist + c * kChunk);
      uint32_t any = 0u;
#pragma unroll
      for (int k = 0; k < kChunk / 128; ++k) {
        const uint4 v = h4[k * 32 + lane];
        any |= v.x | v.y | v.z | v.w;
      }
      any = __any_sync(0xffffffffu, any != 0u);
      if (lane == 0) s_chunk[c] = (int)any;
    }
    consumer_sync<NC>();
    if (tid == 0) {
      fence_proxy_async_global();
      int n = 0;
      for (int c = 0; c < NCHUNK; ++c)
        if (s_chunk[c]) {
          bulk_reduce_add_u32(gh + (kCenter - Cfg::W / 2) + c * kChunk, hist + c * kChunk, kChunk * 4);
          ++n;
        }
      bulk_commit();
      if (n) bulk_wait_read();
    }
    consumer_sync<NC>();
    for (int c = warp; c < NCHUNK; c += CW)
      if (s_chunk[c]) {
        uint4 *h4 = reinterpret_cast<uint4 *>(hist + c * kChunk);
#pragma unroll
        for (int k = 0; k < kChunk / 128; ++k) h4[k * 32 + lane] = make_uint4(0u, 0u, 0u, 0u);
      }
    const long long q3 = PCLOCK();
    consumer_sync<NC>();           // cleared before anyone counts again
    if (tid == 0) {                // the reductions are complete before tdone publishes them
      bulk_wait_all();
      fence_proxy_async_global();
    }
    const long long q4 = PCLOCK();
    if (SEL_BATCH_PROF && a.prof && tid == 0) {
      atomicAdd(a.prof + 148 * 8 + 0, (unsigned long long)(q1 - q0));
      atomicAdd(a.prof + 148 * 8 + 1, (unsigned long long)(q2 - q1));
      atomicAdd(a.prof + 148 * 8 + 2, (unsigned long long)(q3 - q2));
      atomicAdd(a.prof + 148 * 8 + 3, (unsigned long long)(q4 - q3));
    }
    if (warp == 0) enqueue(REQ_T, cur, cur_tasks, 0u, 0u, 0u);
    cur = -1;
    cur_tasks = 0;
  };

  // Range results are accumulated per CTA in shared memory (slot = phase parity).  At a
  // phase change every consumer warp meets at a barrier (they all walk the same task
  // sequence, so they all see the change at the same task); after it, every range slice
  // of the phase is in the slot and tid 0 publishes it.  Warps can then only move one
  // phase ahead (into the other slot) before the next such barrier.
  int cur_phase = 0;
  auto leave_phase = [&]() {
    consumer_sync<NC>();
    if (warp == 0) {
      const int pp = cur_phase & 1;
      const unsigned int cnt = s_rcnt[pp], rmn = s_rmin[pp], rmx = s_rmax[pp], rbd = s_rbad[pp];
      __syncwarp();
      if (lane == 0) {
        s_rmin[pp] = 0xffffffffu;
        s_rmax[pp] = 0u;
        s_rbad[pp] = 0u;
        s_rcnt[pp] = 0u;
      }
      if (cnt) {
        const int g = cur_phase * a.G + grp;                      // R(p) belongs to local field p
        enqueue(REQ_R, g, cnt, rmn, rmx, rbd);
        PROF(pc[7] += 1);
      }
    }
  };

  int stage = 0;
  uint32_t ph = 0;
  for (;;) {
    const long long t_w0 = PCLOCK();
    mbar_wait(&full_bar[stage], ph);
    const long long t_w1 = PCLOCK();
    PROF(pc[0] += t_w1 - t_w0);      // waiting for data
    const int4 sd = stage_desc[stage];
    const bool end = sd.x < 0;
    const int kind = end ? KIND_NONE : sd.x, f = sd.y, id = sd.z, phase = sd.w;
    if (SEL_BATCH_PROF && a.prof && tid == 0)
      atomicAdd(a.prof + 148 * 8 + 4 + (kind == KIND_T ? 0 : kind == KIND_R ? 1 : 2),
                (unsigned long long)(t_w1 - t_w0));
    // flush before anything that may block (another field's tiles wait on params /
    // fin_ready, finalize waits on tdone) and at the end; range tasks never block
    const bool may_block = end || kind == KIND_F || (kind == KIND_T && f != cur);
    while (cur_phase < (end ? nfl + a.lagF + 1 : phase)) {        // phase change(s)
      leave_phase();
      ++cur_phase;
    }
    // flush before anything that may block: what we hold is then handed to the release
    // warp, which completes it without waiting on anyone
    if (cur >= 0 && may_block) flush();
    const long long t_k0 = PCLOCK();
    PROF(pc[1] += t_k0 - t_w1);      // publish + flush
    if (end) {
      if (warp == 0) enqueue(REQ_END, 0, 0u, 0u, 0u, 0u);
      break;
    }
    const float *S = base + stage * Cfg::STAGE_FLOATS;

    if (kind == KIND_T) {
      const int4 tc = stage_tile[stage];
      if (cur < 0) {               // first tile of field f here: params, ring slot free
        // per warp (no CTA barrier): lane 0 acquires the flags, the warp barrier orders
        // the lanes' L2 reads (ld.cg: never a stale L1 line) after it
        if (rw_on) {               // help with the value range while waiting for params(f)
          uint64_t pol;
          asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
          RangeAcc r;
          range_reset(r);
          bool more = true;
          for (;;) {
            unsigned int rdy = 0u;
            if (lane == 0) rdy = ld_acquire(a.params_ready + f);
            if (__shfl_sync(0xffffffffu, rdy, 0)) break;
            const unsigned int c = more ? rw_claim() : rw_total;
            if (c < rw_total) {
              rw_chunk(c, pol, r);
              rw_publish((int)(c / (unsigned)a.nRc), r);      // at once: nothing held while waiting
            } else {
              more = false;
              __nanosleep(256);
            }
          }
          if (lane == 0 && f >= kRing * a.G) spin_until(a.fin_ready + f - kRing * a.G, 1u);
        } else if (lane == 0) {
          spin_until(a.params_ready + f, 1u);
          if (f >= kRing * a.G) spin_until(a.fin_ready + f - kRing * a.G, 1u);   // slot's last user
        }
        __syncwarp();
        ok = __ldcg(&a.params[f].status) == SEL_OK;
        r_f = __ldcg(&a.params[f].r_f);
        minexp = __ldcg(&a.params[f].minexp);
        cur = f;
        cur_slot = tc.w;
      }
      uint64_t tbits = 0;
      double terr = 0.0;
      if (a.sampled) {             // processed blocks id*NC .. +NC-1, one per consumer lane
        const int64_t t = ((int64_t)id * CW + warp) * 32 + lane;
        sampled_consume<D>(a.xs[f], a.g, t, ok && t < a.g.n_pb, r_f, minexp, hist,
                           a.hist + (size_t)tc.w * kH32Stride + 1, ovf, tbits,
                           terr);
      } else {
        PROF(const long long tq0 = clock64());
        tile_consume<D, false>(S, tc.x, tc.y, tc.z, a.tg, warp, lane, ok, r_f, minexp, hist,
                               a.hist + (size_t)tc.w * kH32Stride + 1, ovf,
                               nodbg, tbits, terr);
        PROF(pc[6] += clock64() - tq0);   // the tile compute alone
      }
      ++cur_tasks;
      __syncwarp();
      bar_arrive_n(kBarStage + stage, (CW + 1) * 32);
      task_store(a.tpart + (size_t)tc.w * a.nT * CW, id * CW + warp, tbits, terr);
    } else if (kind == KIND_R) {
      // ---- min / max / non-finite of the staged chunk (R1) by kRWarps consumer warps
      // (rotating with the task id); the others release the stage at once and move on.
      // Order-preserving integer keys make the combines plain atomicMin/Max.
      const int slot = (warp - (id * kRWarps) % CW + CW) % CW;
      if (slot >= kRWarps) {
        __syncwarp();
        bar_arrive_n(kBarStage + stage, (CW + 1) * 32);
      } else {
        const long long lo = (long long)id * a.rchunk;
        const int n4 = (int)min((long long)a.rchunk, a.N - lo) / 4;
        const float4 *src = reinterpret_cast<const float4 *>(S);
        // min propagates NaN (min.NaN), so non-finite values show up in the reduced
        // min / max themselves: NaN -> mn is NaN, +-inf -> mx / mn infinite
        // 3-input min / max (sm_100 FMNMX3), two accumulator pairs to break the chains
        float mn = INFINITY, mx = -INFINITY, mn2 = INFINITY, mx2 = -INFINITY;
#pragma unroll 8
        for (int i = slot * 32 + lane; i < n4; i += kRWarps * 32) {
          const float4 q = src[i];
          mn = fmin3_nan(mn, q.x, q.y);
          mx = fmax3(mx, q.x, q.y);
          mn2 = fmin3_nan(mn2, q.z, q.w);
          mx2 = fmax3(mx2, q.z, q.w);
        }
        mn = fmin_nan(mn, mn2);
        mx = fmaxf(mx, mx2);
        __syncwarp();
        bar_arrive_n(kBarStage + stage, (CW + 1) * 32);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          mn = fmin_nan(mn, __shfl_xor_sync(0xffffffffu, mn, o));
          mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        }
        // (a slice with no values keeps mn = +inf > mx = -inf: not bad)
        const int bad = (mn != mn) | ((mn <= mx) & (is_nonfinite(mn) | is_nonfinite(mx)));
        if (lane == 0) {
          const int pp = phase & 1;
          if (mn <= mx) {
            atomicMin(&s_rmin[pp], float_key(mn));
            atomicMax(&s_rmax[pp], float_key(mx));
          }
          if (bad) atomicOr(&s_rbad[pp], 1u);
          atomicAdd(&s_rcnt[pp], 1u);
        }
      }
    } else if (kind == KIND_F) {
      const int slot = stage_tile[stage].w;   // read before the stage is released
      __syncwarp();
      bar_arrive_n(kBarStage + stage, (CW + 1) * 32);
      if (tid == 0) spin_until(a.tdone + f, (unsigned)a.nT);
      consumer_sync<NC>();
      unsigned int *gh = a.hist + (size_t)slot * kH32Stride + 1;
      const Partial *tpf = a.tpart + (size_t)slot * a.nT * CW;
      FPart *fpf = a.fpart + (size_t)slot * kFinTasks;
      // ---- 1/8 of the histogram: sum c log2(N/c), re-zero; and 1/8 of the tile partials
      const double Nsz = (double)a.fa.n_sz;
      const double lN = log2(Nsz);
      constexpr int PER = kNSlots / kFinTasks;
      constexpr int NIT = (PER + NC - 1) / NC;
      double acc = 0.0;
      unsigned long long novf = 0, hcnt = 0;
      // every load first (one L2 round trip instead of one per bin), then the bins in the
      // same order as before (the per-thread sum order, hence the result, is unchanged)
      unsigned int cv[NIT];
#pragma unroll
      for (int k = 0; k < NIT; ++k)
        cv[k] = (tid + k * NC < PER) ? __ldcg(gh + id * PER + tid + k * NC) : 0u;
#pragma unroll
      for (int k = 0; k < NIT; ++k) {
        const int s = id * PER + tid + k * NC;
        const unsigned int c = cv[k];
        hcnt += c;
        if (c) {
          const double cd = (double)c;
          acc += cd * (lN - log2(cd));
          gh[s] = 0u;
        }
        if (s == kOvfSlot && tid + k * NC < PER) novf = c;
        if (a.hdump && tid + k * NC < PER) a.hdump[(size_t)f * kNSlots + s] = c;   // test dump
      }
      const int np = a.nT * CW;
      const int per = (np + kFinTasks - 1) / kFinTasks;
      const int p0 = id * per, p1 = min(p0 + per, np);
      double err = 0.0;
      unsigned long long bits = 0;
      for (int t = p0 + tid; t < p1; t += NC) {
        bits += __ldcg(&tpf[t].bits);
        err += __ldcg(&tpf[t].err);
        if (a.pdump) a.pdump[(size_t)f * np + t] = tpf[t];   // test dump
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        acc += __shfl_down_sync(0xffffffffu, acc, o);
        err += __shfl_down_sync(0xffffffffu, err, o);
        bits += __shfl_down_sync(0xffffffffu, bits, o);
        novf += __shfl_down_sync(0xffffffffu, novf, o);
        hcnt += __shfl_down_sync(0xffffffffu, hcnt, o);
      }
      consumer_sync<NC>();
      if (lane == 0) {
        s_red[0][warp] = acc; s_red[1][warp] = err;
        s_redu[0][warp] = bits; s_redu[1][warp] = novf; s_redu[2][warp] = hcnt;
      }
      consumer_sync<NC>();
      if (tid == 0) {
        for (int w = 1; w < CW; ++w) {
          acc += s_red[0][w]; err += s_red[1][w];
          bits += s_redu[0][w]; novf += s_redu[1][w]; hcnt += s_redu[2][w];
        }
        FPart fp;
        fp.acc = acc; fp.err = err; fp.bits = bits; fp.ovf = novf; fp.cnt = hcnt;
        fpf[id] = fp;
        fence_acq_rel_gpu();
        if (atomicAdd(a.fdone + f, 1u) == (unsigned)kFinTasks - 1) {   // last: result f
          fence_acq_rel_gpu();
          double S = 0.0, errs = 0.0;
          unsigned long long tb = 0, ov = 0, hc = 0;
          for (int k = 0; k < kFinTasks; ++k) {
            S += __ldcg(&fpf[k].acc);
            errs += __ldcg(&fpf[k].err);
            tb += __ldcg(&fpf[k].bits);
            ov += __ldcg(&fpf[k].ovf);
            hc += __ldcg(&fpf[k].cnt);
          }
          const Params prm = a.params[f];
          const double mse = errs / (double)a.fa.n_values;
          a.results[f] = assemble_result(prm, S, errs, tb, ov, hc, a.fa, log10(prm.vr / prm.eb_abs),
                                         log10(prm.vr), mse > 0.0 ? log10(mse) : 0.0);
          fence_acq_rel_gpu();
          st_release(a.fin_ready + f, 1u);
        }
      }
    } else {
      __syncwarp();
      bar_arrive_n(kBarStage + stage, (CW + 1) * 32);
    }
#if SEL_BATCH_PROF
    {
      const long long dt = clock64() - t_k0;
      if (kind == KIND_T) pc[2] += dt;
      else if (kind == KIND_R) pc[3] += dt;
      else pc[4] += dt;
    }
#endif
    if (++stage == Cfg::STAGES) { stage = 0; ph ^= 1u; }
  }
#if SEL_BATCH_PROF
  if (a.prof && tid == 0)
    for (int k = 0; k < 8; ++k) a.prof[blockIdx.x * 8 + k] = (unsigned long long)pc[k];
#endif
}

// ============================================================ host side
unsigned long long *g_batch_prof = nullptr;   // developer profiling hook (sel_batch_profile)
namespace {
template <int D>
const void *batch_fn() { return (const void *)k_batch<D>; }
}  // namespace

int batch_sizes(const Geo &g, BatchSizes *bs) {
  const int d3 = g.ndims == 3;
  // range chunk: one smem stage
  bs->rchunk = d3 ? (TileCfg<3>::STAGE_FLOATS & ~3) : (TileCfg<2>::STAGE_FLOATS & ~3);
  bs->nR = (int)((g.N + bs->rchunk - 1) / bs->rchunk);
  bs->smem = d3 ? TileCfg<3>::SMEM : TileCfg<2>::SMEM;
  bs->threads = d3 ? batch_threads<3>() : batch_threads<2>();
  bs->cw = d3 ? TileCfg<3>::CW : TileCfg<2>::CW;
  const void *fn = d3 ? batch_fn<3>() : batch_fn<2>();
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bs->smem) != cudaSuccess)
    return SEL_ECUDA;
  return SEL_OK;
}

int batch_parts_per_task(const Geo &g) { return g.ndims == 3 ? TileCfg<3>::CW : TileCfg<2>::CW; }
int batch_rows_per_part(const Geo &g) { return g.ndims == 3 ? TileCfg<3>::BR : TileCfg<2>::BR; }

bool batch_fits(const Geo &g, const TileLaunch &tl, const BatchSizes &bs, int nf) {
  if (tl.tg.ntk >= (1 << 16) || tl.tg.ntj >= (1 << 16)) return false;
  const long long phase = kFinTasks + bs.nR + batch_ntasks(g, tl, bs);
  return (long long)nf * phase < (1LL << 31);
}

// T tasks per field: TMA tiles, or (strides > 1) groups of one processed block per lane
int batch_ntasks(const Geo &g, const TileLaunch &tl, const BatchSizes &bs) {
  if (g.s[0] > 1 || g.s[1] > 1 || g.s[2] > 1) {
    const int64_t per = (int64_t)bs.cw * 32;
    return (int)((g.n_pb + per - 1) / per);
  }
  return tl.tg.ntasks;
}

size_t batch_state_bytes(int nf, const BatchSizes &bs, int nT, int G) {
  return (size_t)nf * (sizeof(Params) + 8 * 4 + sizeof(CUtensorMap) + 8) + 64 +
         (size_t)G * 8 + (size_t)G * kRing * ((size_t)kH32Stride * 4 + (size_t)nT * bs.cw * sizeof(Partial) +
                              kFinTasks * sizeof(FPart)) +
         8192;
}

// The task sequence of one CTA group with nfl fields, decoded: phase p = F(p - lagF) [kFinTasks] then R(p) [nR] and T(p - lagT) [nT]
// interleaved (Bresenham).  Entry: {kind | phase << 2, id, btk | btj << 16, bi}.
static void build_group_sequence(int nfl, int nR, int nT, int lagT, int lagF, const TileGeo &tg,
                                 bool sampled, std::vector<uint4> &out) {
  auto inr = [&](int f) { return f >= 0 && f < nfl; };
  for (int p = 0; p < nfl + lagF; ++p) {
    if (inr(p - lagF))
      for (int k = 0; k < kFinTasks; ++k) out.push_back(make_uint4(KIND_F | (uint32_t)p << 2, (uint32_t)k, 0u, 0u));
    const long long nRp = inr(p) ? nR : 0, nTp = inr(p - lagT) ? nT : 0, M = nRp + nTp;
    for (long long m = 0; m < M; ++m) {
      const long long r0 = m * nRp / M, r1 = (m + 1) * nRp / M;
      if (r1 > r0) {
        out.push_back(make_uint4(KIND_R | (uint32_t)p << 2, (uint32_t)r0, 0u, 0u));
      } else {
        const int id = (int)(m - r0);
        uint32_t z = 0, w = 0;
        if (!sampled && tg.ntk > 0 && tg.ntj > 0) {
          const int btk = id % tg.ntk, rest = id / tg.ntk;
          z = (uint32_t)btk | (uint32_t)(rest % tg.ntj) << 16;
          w = (uint32_t)(rest / tg.ntj);
        }
        out.push_back(make_uint4(KIND_T | (uint32_t)p << 2, (uint32_t)id, z, w));
      }
    }
  }
}

int launch_batch(const Geo &g, const TileLaunch &tl, const BatchSizes &bs, const float *const *d_fields,
                 int nf, void *state, size_t state_bytes, const FinalizeArgs &fa, int mode, double eb,
                 sel_result *d_results, int sm_count, int G, int lagT, int range_warps_on, BatchTable *tab,
                 const BatchDump &dump, cudaStream_t st, cudaEvent_t *ev) {
  if (!tab || !batch_fits(g, tl, bs, nf)) return SEL_EINVAL;
  if (G < 1 || G > nf || G > sm_count || lagT < 1 || lagT > 4) return SEL_EINVAL;
  // state layout (device): tmaps | xs | params | counters | hist x2 | tpart x2 | fpart x2
  char *b = (char *)state;
  size_t off = 0;
  auto take = [&](size_t bytes, size_t align = 256) {
    off = (off + align - 1) & ~(align - 1);
    size_t o = off;
    off += bytes;
    return b + o;
  };
  const int nT = batch_ntasks(g, tl, bs);
  const bool sampled = g.s[0] > 1 || g.s[1] > 1 || g.s[2] > 1;
  // range warps (3D full-field stacks): no R tasks in the sequence
  const bool rw = range_warps_on && !sampled &&
                  (g.ndims == 3 ? range_warps<3>() > 0 : g.ndims == 2 && range_warps<2>() > 0);
  const int nRs = rw ? 0 : bs.nR;
  // the histogram ring first, at a fixed offset: its slots stay zero between launches
  const size_t nslot = (size_t)G * kRing;
  unsigned int *hst = (unsigned int *)take((size_t)kH32Stride * 4 * nslot);
  CUtensorMap *tmaps = (CUtensorMap *)take(sizeof(CUtensorMap) * nf, 128);
  const float **xs = (const float **)take(sizeof(float *) * nf);
  Params *params = (Params *)take(sizeof(Params) * nf);
  const size_t nctr = 8 * (size_t)nf + 2 * (size_t)G;
  unsigned int *ctrs = (unsigned int *)take(sizeof(unsigned int) * nctr);
  Partial *tp = (Partial *)take(sizeof(Partial) * (size_t)nT * bs.cw * nslot);
  FPart *fp = (FPart *)take(sizeof(FPart) * kFinTasks * nslot);
  if (off > state_bytes) return SEL_EINVAL;
  // host-built tensor maps and pointer table, one H2D copy each (staged in pinned memory
  // by the caller? small: a few KB -> plain cudaMemcpyAsync from pageable is fine)
  static thread_local std::vector<CUtensorMap> h_maps;
  h_maps.resize(nf);
  if (sampled) memset(h_maps.data(), 0, sizeof(CUtensorMap) * nf);   // no tiles
  else
    for (int f = 0; f < nf; ++f)
      if (make_tile_map(&h_maps[f], d_fields[f], g)) return SEL_ECUDA;
  // The histogram ring stays zero between launches (the F tasks re-zero every nonzero bin
  // they read, and every field is finalized); only slots not known to be zero -- a fresh
  // state, or more groups than before (the ring grew into other state) -- are cleared.
  if (tab->hist_clean < nslot) {
    if (cudaMemsetAsync(hst, 0, (size_t)kH32Stride * 4 * nslot, st) != cudaSuccess) return SEL_ECUDA;
  }
  tab->hist_clean = nslot;
  if (cudaMemcpyAsync(tmaps, h_maps.data(), sizeof(CUtensorMap) * nf, cudaMemcpyHostToDevice, st) !=
          cudaSuccess ||
      cudaMemcpyAsync(xs, d_fields, sizeof(float *) * nf, cudaMemcpyHostToDevice, st) != cudaSuccess ||
      cudaMemsetAsync(ctrs, 0, sizeof(unsigned int) * nctr, st) != cudaSuccess ||
      cudaMemsetAsync(ctrs + 6 * (size_t)nf, 0xff, sizeof(unsigned int) * nf, st) != cudaSuccess)
    return SEL_ECUDA;
  BatchArgs a;
  a.tmaps = tmaps;
  a.xs = xs;
  a.nf = nf;
  a.tg = tl.tg;
  a.g = g;
  a.sampled = sampled ? 1 : 0;
  a.N = g.N;
  a.nR = nRs;
  a.nT = nT;
  a.phase = kFinTasks + nRs + nT;
  a.rw = rw ? 1 : 0;
  a.rcf = kRwChunk;
  a.nRc = (int)((g.N + kRwChunk - 1) / kRwChunk);
  if ((long long)nf * a.phase >= (1LL << 31)) return SEL_EINVAL;   // 32-bit task indices
  {   // task table, rebuilt only when its key changes
    const long long key[8] = {nf, G, nRs, nT, lagT, sampled ? 1 : 0, tl.tg.ntk, tl.tg.ntj};
    if (memcmp(key, tab->key, sizeof(key)) != 0) {
      static thread_local std::vector<uint4> h;
      h.clear();
      h.reserve((size_t)nf * a.phase);
      for (int gi = 0; gi < G; ++gi)
        build_group_sequence((nf - gi + G - 1) / G, nRs, nT, lagT, lagT + 2, tl.tg, sampled, h);
      const size_t bytes = h.size() * sizeof(uint4);
      if (bytes > tab->cap) {
        if (tab->d) { cudaStreamSynchronize(st); cudaFree(tab->d); }
        tab->d = nullptr;
        tab->cap = 0;
        if (cudaMalloc(&tab->d, bytes) != cudaSuccess) return SEL_ENOMEM;
        tab->cap = bytes;
      }
      if (cudaMemcpyAsync(tab->d, h.data(), bytes, cudaMemcpyHostToDevice, st) != cudaSuccess) return SEL_ECUDA;
      memcpy(tab->key, key, sizeof(key));
    }
  }
  a.ttab = (const uint4 *)tab->d;
  a.rchunk = bs.rchunk;
  a.fa = fa;
  a.mode = mode;
  a.eb = eb;
  a.params = params;
  a.rdone = ctrs;
  a.params_ready = ctrs + nf;
  a.tdone = ctrs + 2 * nf;
  a.fdone = ctrs + 3 * nf;
  a.fin_ready = ctrs + 4 * nf;
  a.rmax = ctrs + 5 * nf;
  a.rmin = ctrs + 6 * nf;
  a.rbad = ctrs + 7 * nf;
  a.task_ctr = ctrs + 8 * nf;
  a.rtask_ctr = ctrs + 8 * nf + G;
  a.G = G;
  a.lagT = lagT;
  a.lagF = lagT + 2;
  a.hist = hst;
  a.tpart = tp;
  a.fpart = fp;
  a.results = d_results;
  a.hdump = dump.hist;
  a.pdump = dump.part;
  a.prof = g_batch_prof;
  const void *fn = g.ndims == 3 ? batch_fn<3>() : batch_fn<2>();
  void *args[] = {(void *)&a};
  if (ev && cudaEventRecord(ev[0], st) != cudaSuccess) return SEL_ECUDA;
  if (cudaLaunchKernel(fn, dim3(sm_count), dim3(bs.threads), args, bs.smem, st) != cudaSuccess)
    return SEL_ECUDA;
  if (ev && cudaEventRecord(ev[1], st) != cudaSuccess) return SEL_ECUDA;
  return SEL_OK;
}

}  // namespace sel

// Developer hook (not part of include/sel.h): per-CTA cycle counters of k_batch's warp 0
// {data wait, publish+flush, T, R, F, other} into dev_buf[ctas * 8]; NULL disables.
extern "C" void sel_dev_batch_profile(unsigned long long *dev_buf) { sel::g_batch_prof = dev_buf; }
