// sel_api.cu -- host runtime behind include/sel.h: plans own the device workspace,
// launches are stream-ordered (K1 value range -> K2 fused estimate -> K3 finalize),
// one small D2H of the result per call.  No CPU fallback: every estimate runs in
// the kernels of sel_kernels.cu.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <algorithm>
#include <vector>

#include "sel_internal.h"

using namespace sel;

namespace {

thread_local std::string g_cuda_msg = "no CUDA error recorded";

int cuda_fail(cudaError_t e, const char *what) {
  char buf[256];
  snprintf(buf, sizeof buf, "%s: %s (%s)", what, cudaGetErrorString(e), cudaGetErrorName(e));
  g_cuda_msg = buf;
  return SEL_ECUDA;
}

#define CK(call)                                         \
  do {                                                   \
    cudaError_t e_ = (call);                             \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call);  \
  } while (0)

struct TimingSlot {
  cudaEvent_t ev[4];   // before K1, after K1, after K2, after K3
};

}  // namespace

struct sel_plan_st {
  int device = 0;
  int sm_count = 0;
  Geo geo{};
  int mode = 0;
  double eb = 0.0;
  double sz_offset = 0.5;
  int debug = 0;
  int timing = 0;
  int mm_ctas = 0;
  EstLaunch el[2][2] = {};                        // [vec][debug]
  bool tile_ok = false;                           // TMA tile path available for this shape
  bool sampled_ok = false;                        // k_batch sampled-block tasks available
  TileLaunch tl[2] = {};                          // [debug]
  BatchSizes bs{};                                // persistent batch kernel sizes
  int use_batch = 1;
  int groups = 0;                 // k_batch CTA groups (0: auto, batch_groups)
  int lag_t = 2;                  // k_batch phases from a field's range pass to its tiles
  int batch_debug = 0;            // k_batch test dumps (histograms, partials) per field
  BatchDump bdump;
  int bdump_cap = 0;              // fields the dump buffers hold
  int last_batch_nf = 0;          // fields of the last k_batch launch
  int last_batch_G = 0;
  void *bstate = nullptr;                         // batch kernel state (grows with n)
  BatchTable btab;                                // k_batch task table (device, cached)
  cudaEvent_t bev[2] = {nullptr, nullptr};        // kernel_timing around k_batch
  bool batch_timed = false;
  size_t bstate_cap = 0;
  int max_tasks = 0;
  uint64_t n_sz = 0, n_values = 0;
  int size = 0;                                   // 4^d

  void *ws_mem = nullptr;
  size_t ws_bytes = 0;
  Workspace ws{};          // parity-0 copy (sequential path)
  Workspace wsk[2]{};      // per field parity (batch pipeline)

  sel_result *d_res = nullptr;
  sel_result *h_res = nullptr;   // pinned
  int res_cap = 0;

  // debug dumps
  void *dbg_mem = nullptr;
  DebugPtrs dbg{};
  unsigned long long *dbg_hist = nullptr;

  // end-to-end staging
  float *d_stage[2] = {nullptr, nullptr};
  size_t stage_cap = 0;                           // bytes of each staging buffer
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_copied[2] = {nullptr, nullptr};
  cudaEvent_t ev_done[2] = {nullptr, nullptr};

  // per-field params (capacity res_cap) and the batch pipeline's aux stream/events
  Params *d_params = nullptr;
  cudaStream_t aux_stream = nullptr, fin_stream = nullptr;
  std::vector<cudaEvent_t> ev_mm, ev_k2, ev_k3;
  int pipeline = 1;

  // kernel timing
  std::vector<TimingSlot> tslots;
  double ms[3] = {0, 0, 0};
  uint64_t tcount[3] = {0, 0, 0};

  // N1 multi-eb workspace (allocated on first use): per eb a Workspace view
  void *multi_mem = nullptr;
  Workspace mws[kMultiMaxEb]{};
  Params *mprm = nullptr;                         // [kMultiMaxEb]
  Partial *mpart = nullptr;                       // [kMultiMaxEb][mcap]
  int mcap = 0;                                   // CTA partials per eb
  void *mtile_mem = nullptr;                      // tile-pipeline multi-eb pass: [task counter | partials]
  int use_multi_tile = 1;                         // option "multi_tile"

  // small-field single-launch state (first use)
  void *small_mem = nullptr;
  int use_small = 1;              // option "small_kernel"
  int range_warps = 1;            // option "range_warps": k_batch<3> streams the value range on its own warps
  // N3 ZFP stream workspace (first use): per-block lengths, CTA bases, total
  void *zs_mem = nullptr;
  // N2 paper-literal workspace (first use): CTA partials, mid scalars, params, result
  void *paper_mem = nullptr;
  void *var_mem = nullptr;        // N4 variant-quantiser workspace (first use)
  int paper_cap = 0;

  uint64_t launches = 0;
};

namespace {

int ensure_results(sel_plan_t p, int n) {
  if (n <= p->res_cap) return SEL_OK;
  if (p->d_res) cudaFree(p->d_res);
  if (p->h_res) cudaFreeHost(p->h_res);
  if (p->d_params) cudaFree(p->d_params);
  p->d_res = nullptr;
  p->h_res = nullptr;
  p->d_params = nullptr;
  p->res_cap = 0;
  CK(cudaMalloc(&p->d_res, sizeof(sel_result) * (size_t)n));
  CK(cudaMallocHost(&p->h_res, sizeof(sel_result) * (size_t)n));
  CK(cudaMalloc(&p->d_params, sizeof(Params) * (size_t)n));
  p->res_cap = n;
  return SEL_OK;
}

int ensure_timing(sel_plan_t p, int n) {
  while ((int)p->tslots.size() < n) {
    TimingSlot s;
    for (auto &e : s.ev) CK(cudaEventCreate(&e));
    p->tslots.push_back(s);
  }
  return SEL_OK;
}

int ensure_debug(sel_plan_t p) {
  if (p->dbg_mem) return SEL_OK;
  const size_t N = (size_t)p->geo.N, B = (size_t)p->geo.n_pb, S = (size_t)p->size;
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 255) & ~(size_t)255; return o; };
  size_t o_codes = take(N * 4), o_emax = take(B * 4), o_coef = take(B * S * 4),
         o_uw = take(B * S * 4), o_bits = take(B * 4), o_err = take(B * 8),
         o_hist = take((size_t)kNSlots * 8);
  void *m = nullptr;
  if (cudaMalloc(&m, off) != cudaSuccess) return SEL_ENOMEM;
  char *b = (char *)m;
  p->dbg_mem = m;
  p->dbg.codes = (int32_t *)(b + o_codes);
  p->dbg.emax = (int32_t *)(b + o_emax);
  p->dbg.coef = (int32_t *)(b + o_coef);
  p->dbg.uword = (uint32_t *)(b + o_uw);
  p->dbg.bits = (uint32_t *)(b + o_bits);
  p->dbg.err = (double *)(b + o_err);
  p->dbg_hist = (unsigned long long *)(b + o_hist);
  return SEL_OK;
}

// Per-field launches.  Each field f owns params slot f (written by its k_minmax, read
// by its fused pass and finalize), so value-range passes may run ahead of the fused
// passes of earlier fields on another stream (batch pipeline below).
Workspace field_ws(sel_plan_t p, int f, int parity = 0) {
  Workspace w = p->wsk[parity];
  w.params = p->d_params + f;
  return w;
}

int enqueue_minmax(sel_plan_t p, const float *x, int f, cudaStream_t st) {
  const Workspace w = field_ws(p, f);
  int rc = launch_minmax(x, p->geo.N, p->mm_ctas, w, p->mode, p->eb, st);
  if (rc) return cuda_fail(cudaGetLastError(), "k_minmax launch");
  p->launches += 1;
  return SEL_OK;
}

int enqueue_est(sel_plan_t p, const float *x, int f, cudaStream_t st, TimingSlot *ts,
                int parity = 0, cudaStream_t fin_st = nullptr, cudaEvent_t k2_done = nullptr) {
  const int vec = (p->geo.n[2] % 4 == 0) && (((uintptr_t)x & 15u) == 0);
  const int dbg = p->debug ? 1 : 0;
  const EstLaunch &el = p->el[vec][dbg];
  Geo g = p->geo;
  g.vec = vec;
  const bool tile = p->tile_ok && vec;
  const Workspace w = field_ws(p, f, parity);
  int rc = tile ? launch_tile(x, g, p->tl[dbg], w, dbg ? &p->dbg : nullptr, st)
                : launch_estimate(x, g, el, w, dbg ? &p->dbg : nullptr, st);
  if (rc) return cuda_fail(cudaGetLastError(), tile ? "k_tile launch" : "k_estimate launch");
  if (ts) CK(cudaEventRecord(ts->ev[2], st));
  FinalizeArgs fa;
  fa.mode = p->mode;
  fa.eb = p->eb;
  fa.sz_offset = p->sz_offset;
  fa.n_sz = p->n_sz;
  fa.n_values = p->n_values;
  fa.n_blocks = (uint64_t)p->geo.n_pb;
  fa.ntasks = tile ? p->tl[dbg].npart : el.ntasks;
  if (k2_done) {                      // finalize on its own stream, after this fused pass
    CK(cudaEventRecord(k2_done, st));
    CK(cudaStreamWaitEvent(fin_st, k2_done, 0));
    st = fin_st;
  }
  rc = launch_finalize(w, fa, p->d_res + f, dbg ? p->dbg_hist : nullptr, st);
  if (rc) return cuda_fail(cudaGetLastError(), "k_finalize launch");
  if (ts) CK(cudaEventRecord(ts->ev[3], st));
  p->launches += 2;
  return SEL_OK;
}

// One persistent launch for the whole batch (sel_batch.cu): value range, tiles and
// finalize of every field as one task stream; results land in d_res[0..n).
bool batch_ok(sel_plan_t p, const float *const *x, int n) {
  if (!(p->tile_ok || p->sampled_ok) || !p->use_batch || p->debug) return false;
  if (p->geo.N >= (int64_t)1 << 32) return false;   // k_batch histograms are u32
  // task-table limits (16-bit tile coordinates, 32-bit task indices): otherwise the
  // per-field kernels run the shape
  if (!batch_fits(p->geo, p->tl[0], p->bs, n)) return false;
  for (int f = 0; f < n; ++f)
    if (((uintptr_t)x[f] & 15u) != 0) return false;
  return true;
}

// CTA groups for k_batch: G groups each run every G-th field on sm_count / G CTAs, so a
// CTA flushes its histogram G x less often; the fields whose range pass is ahead of
// their tiles (kLagT per group) must stay in L2 (~126 MB), hence the byte budget.
int batch_groups(sel_plan_t p, int n) {
  int G = p->groups;
  if (G <= 0) {                   // measured: ~160 MB of fields per
    const double fb = (double)p->geo.N * 4.0;   // group sequence (C2: G = 6; 100 MB C3: 1)
    G = (int)(160e6 / fb);
    // sampled strides: little tile work per field, so the per-field pipeline latency
    // dominates -- more groups in flight (C2 at stride (1,10): G 3 -> 10, +42%)
    if (p->sampled_ok && G < 16) G = 16;
    if (G > 64) G = 64;             // (C1, 256 small fields: 32 -> 64 groups +4 %)
    if (G > n / 2) G = n / 2;     // keep >= 2 fields per group (tail balance)
    // CTAs join group blockIdx % G and fields are split evenly over the groups, so a G
    // that does not divide the SM count leaves the smaller groups setting the makespan
    // (G = 64 on 148 SMs: 2- and 3-CTA groups): snap larger G to a divisor
    if (G > 8) {
      int d = G;
      while (d > 1 && p->sm_count % d != 0) --d;
      if (2 * d >= G) G = d;
    }
  }
  if (G > n) G = n;
  if (G > p->sm_count) G = p->sm_count;
  return G < 1 ? 1 : G;
}

int enqueue_batch(sel_plan_t p, const float *const *x, int n, cudaStream_t st,
                  sel_result *d_res = nullptr) {
  const int G = batch_groups(p, n);
  const size_t need = batch_state_bytes(n, p->bs, batch_ntasks(p->geo, p->tl[0], p->bs), G);
  if (need > p->bstate_cap) {
    if (p->bstate) {
      CK(cudaStreamSynchronize(st));
      cudaFree(p->bstate);
    }
    p->bstate = nullptr;
    p->bstate_cap = 0;
    if (cudaMalloc(&p->bstate, need) != cudaSuccess) return SEL_ENOMEM;
    p->bstate_cap = need;
    p->btab.hist_clean = 0;          // launch_batch zeroes the histogram ring
  }
  BatchDump dump;
  if (p->batch_debug) {
    if (n > p->bdump_cap) {
      CK(cudaStreamSynchronize(st));
      if (p->bdump.hist) cudaFree(p->bdump.hist);
      if (p->bdump.part) cudaFree(p->bdump.part);
      p->bdump = BatchDump();
      p->bdump_cap = 0;
      const size_t np = (size_t)batch_ntasks(p->geo, p->tl[0], p->bs) * batch_parts_per_task(p->geo);
      if (cudaMalloc(&p->bdump.hist, (size_t)n * kNSlots * 4) != cudaSuccess ||
          cudaMalloc(&p->bdump.part, (size_t)n * np * sizeof(Partial)) != cudaSuccess)
        return SEL_ENOMEM;
      p->bdump_cap = n;
    }
    dump = p->bdump;
  }
  p->last_batch_nf = n;
  p->last_batch_G = G;
  FinalizeArgs fa;
  fa.mode = p->mode;
  fa.eb = p->eb;
  fa.sz_offset = p->sz_offset;
  fa.n_sz = p->n_sz;
  fa.n_values = p->n_values;
  fa.n_blocks = (uint64_t)p->geo.n_pb;
  fa.ntasks = 0;
  Geo g = p->geo;
  g.vec = 1;
  if (p->timing) {
    if (!p->bev[0]) {
      CK(cudaEventCreate(&p->bev[0]));
      CK(cudaEventCreate(&p->bev[1]));
    }
  }
  int rc = launch_batch(g, p->tl[0], p->bs, x, n, p->bstate, p->bstate_cap, fa, p->mode, p->eb,
                        d_res ? d_res : p->d_res, p->sm_count, G, p->lag_t, p->range_warps, &p->btab, dump, st,
                        p->timing ? p->bev : nullptr);
  if (rc == SEL_ECUDA) return cuda_fail(cudaGetLastError(), "k_batch launch");
  if (rc) return rc;
  p->launches += 1;
  p->batch_timed = p->timing;
  return SEL_OK;
}

// one small field (N <= 2^21): one cooperative launch, k_small (sel_kernels.cu)
bool small_ok(sel_plan_t p) {
  return p->use_small && p->use_batch && !p->timing && !p->debug && p->geo.N <= ((int64_t)1 << 21);
}

int enqueue_small(sel_plan_t p, const float *d_field, cudaStream_t st) {
  int rc;
  if (!p->small_mem) {
    if (cudaMalloc(&p->small_mem, small_state_bytes(p->sm_count)) != cudaSuccess) {
      cudaGetLastError();
      p->small_mem = nullptr;
      return SEL_ENOMEM;
    }
    if ((rc = init_small_state(p->small_mem, st))) return cuda_fail(cudaGetLastError(), "small state");
  }
  Geo g = p->geo;
  g.vec = (g.n[2] % 4 == 0) && (((uintptr_t)d_field & 15u) == 0);
  FinalizeArgs fa;
  fa.mode = p->mode;
  fa.eb = p->eb;
  fa.sz_offset = p->sz_offset;
  fa.n_sz = p->n_sz;
  fa.n_values = p->n_values;
  fa.n_blocks = (uint64_t)p->geo.n_pb;
  fa.ntasks = 0;
  if ((rc = launch_small(d_field, g, p->sm_count, p->small_mem, field_ws(p, 0), fa, p->d_res, st)))
    return cuda_fail(cudaGetLastError(), "k_small launch");
  p->launches += 1;
  return SEL_OK;
}

// Sequential K1 -> K2 -> K3 for one field on one stream; result lands in d_res[f].
int enqueue_field(sel_plan_t p, const float *x, cudaStream_t st, int f) {
  if (p->debug) CK(cudaMemsetAsync(p->dbg.codes, 0xff, (size_t)p->geo.N * 4, st));
  TimingSlot *ts = p->timing ? &p->tslots[f] : nullptr;
  if (ts) CK(cudaEventRecord(ts->ev[0], st));
  int rc = enqueue_minmax(p, x, f, st);
  if (rc) return rc;
  if (ts) CK(cudaEventRecord(ts->ev[1], st));
  return enqueue_est(p, x, f, st, ts);
}

int ensure_aux(sel_plan_t p, int n) {
  if (!p->aux_stream) CK(cudaStreamCreateWithFlags(&p->aux_stream, cudaStreamNonBlocking));
  if (!p->fin_stream) CK(cudaStreamCreateWithFlags(&p->fin_stream, cudaStreamNonBlocking));
  while ((int)p->ev_mm.size() < n + 1) {
    cudaEvent_t a, b, c;
    CK(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c, cudaEventDisableTiming));
    p->ev_mm.push_back(a);
    p->ev_k2.push_back(b);
    p->ev_k3.push_back(c);
  }
  return SEL_OK;
}

// Batch pipeline over three streams.  aux: k_minmax(f) (DRAM-bound, one small CTA per
// SM); main: the fused pass of f (ALU-bound, one persistent CTA per SM); fin: finalize
// of f (latency-bound).  The three kinds co-reside on the SMs, so the value range of
// f+1 and the finalize of f-1 run under the fused pass of f; field f+1 is left in L2
// for its own fused pass.  k_minmax(f+2) is released by the fused pass of f (at most one
// field runs ahead); the fused pass of f+2 waits for the finalize of f, the other user
// of its parity's workspace.
int enqueue_pipelined(sel_plan_t p, const float *const *x, int n, cudaStream_t st) {
  int rc = ensure_aux(p, n);
  if (rc) return rc;
  cudaEvent_t start = p->ev_mm[n];
  CK(cudaEventRecord(start, st));                 // prior work on the caller's stream
  CK(cudaStreamWaitEvent(p->aux_stream, start, 0));
  CK(cudaStreamWaitEvent(p->fin_stream, start, 0));
  auto minmax = [&](int f) -> int {
    if (f >= 2) CK(cudaStreamWaitEvent(p->aux_stream, p->ev_k2[f - 2], 0));
    int r = enqueue_minmax(p, x[f], f, p->aux_stream);
    if (r) return r;
    CK(cudaEventRecord(p->ev_mm[f], p->aux_stream));
    return SEL_OK;
  };
  if ((rc = minmax(0))) return rc;
  if (n > 1 && (rc = minmax(1))) return rc;
  for (int f = 0; f < n; ++f) {
    CK(cudaStreamWaitEvent(st, p->ev_mm[f], 0));
    if (f >= 2) CK(cudaStreamWaitEvent(st, p->ev_k3[f - 2], 0));
    if ((rc = enqueue_est(p, x[f], f, st, nullptr, f & 1, p->fin_stream, p->ev_k2[f]))) return rc;
    CK(cudaEventRecord(p->ev_k3[f], p->fin_stream));
    if (f + 2 < n && (rc = minmax(f + 2))) return rc;
  }
  CK(cudaStreamWaitEvent(st, p->ev_k3[n - 1], 0));   // results complete on the caller's stream
  CK(cudaStreamWaitEvent(st, p->ev_mm[n - 1], 0));
  return SEL_OK;
}

int collect_timing(sel_plan_t p, int n) {
  if (!p->timing) return SEL_OK;
  if (p->batch_timed) {           // one k_batch launch: all of it counts as the fused pass
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, p->bev[0], p->bev[1]));
    p->ms[1] += ms;
    p->tcount[1] += 1;
    p->batch_timed = false;
    return SEL_OK;
  }
  for (int f = 0; f < n; ++f) {
    for (int k = 0; k < 3; ++k) {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, p->tslots[f].ev[k], p->tslots[f].ev[k + 1]));
      p->ms[k] += ms;
      p->tcount[k] += 1;
    }
  }
  return SEL_OK;
}

int finish(sel_plan_t p, cudaStream_t st, int n, sel_result *out) {
  CK(cudaMemcpyAsync(p->h_res, p->d_res, sizeof(sel_result) * (size_t)n, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  int rc = collect_timing(p, n);
  if (rc) return rc;
  memcpy(out, p->h_res, sizeof(sel_result) * (size_t)n);
  return SEL_OK;
}

uint64_t real_in_processed(int64_t n, int64_t s) {
  // sum over processed blocks b (b % s == 0) of the real values min(4, n - 4b)
  uint64_t r = 0;
  const int64_t nb = (n + 3) / 4;
  for (int64_t b = 0; b < nb; b += s) r += (uint64_t)((n - 4 * b) < 4 ? (n - 4 * b) : 4);
  return r;
}

// N1 multi-eb workspace: per eb a 65,536-slot histogram, CTA partials and the
// finalize state of a Workspace (k_finalize runs once per eb on its own view)
int ensure_multi(sel_plan_t p) {
  if (p->multi_mem) return SEL_OK;
  const int cap = p->sm_count * 8;                // 256-thread CTAs: occupancy <= 8
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 255) & ~(size_t)255; return o; };
  const size_t o_prm = take(sizeof(Params) * kMultiMaxEb);
  const size_t o_part = take(sizeof(Partial) * (size_t)cap * kMultiMaxEb);
  const size_t o_h = take((size_t)kNSlots * 8 * kMultiMaxEb);   // contiguous: k_multi indexes e * kNSlots
  size_t o_tc[kMultiMaxEb], o_fp[kMultiMaxEb], o_fe[kMultiMaxEb], o_fb[kMultiMaxEb], o_fo[kMultiMaxEb],
      o_tk[kMultiMaxEb];
  for (int e = 0; e < kMultiMaxEb; ++e) {
    o_tc[e] = take(4);
    o_fp[e] = take((size_t)kFinCTAs * 8);
    o_fe[e] = take((size_t)kFinCTAs * 8);
    o_fb[e] = take((size_t)kFinCTAs * 8);
    o_fo[e] = take(16);
    o_tk[e] = take(8);
  }
  if (cudaMalloc(&p->multi_mem, off) != cudaSuccess) {
    cudaGetLastError();
    p->multi_mem = nullptr;
    return SEL_ENOMEM;
  }
  if (cudaMemset(p->multi_mem, 0, off) != cudaSuccess) return cuda_fail(cudaGetLastError(), "multi workspace");
  char *b = (char *)p->multi_mem;
  p->mprm = (Params *)(b + o_prm);
  p->mpart = (Partial *)(b + o_part);
  p->mcap = cap;
  for (int e = 0; e < kMultiMaxEb; ++e) {
    Workspace &w = p->mws[e];
    w = p->ws;
    w.hist = (unsigned long long *)(b + o_h) + (size_t)e * kNSlots;
    w.params = p->mprm + e;
    w.task_part = p->mpart + (size_t)e * cap;
    w.task_ctr = (unsigned int *)(b + o_tc[e]);
    w.fin_part = (double *)(b + o_fp[e]);
    w.fin_err = (double *)(b + o_fe[e]);
    w.fin_bits = (unsigned long long *)(b + o_fb[e]);
    w.fin_ovf = (unsigned long long *)(b + o_fo[e]);
    w.tickets = (unsigned int *)(b + o_tk[e]);
  }
  return SEL_OK;
}

}  // namespace

extern "C" {

const char *sel_strerror(int status) {
  switch (status) {
    case SEL_OK: return "ok";
    case SEL_EINVAL: return "invalid argument";
    case SEL_ENOMEM: return "out of memory";
    case SEL_ECUDA: return g_cuda_msg.c_str();
    case SEL_ENONFINITE: return "field contains NaN or Inf";
    case SEL_EDEGENERATE: return "degenerate field (relative bound with zero value range, or no SZ point)";
    case SEL_ENOTIMPL: return "not implemented";
    default: return "unknown status";
  }
}

int sel_plan(sel_plan_t *out, int ndims, const int64_t *dims, sel_eb_mode mode, double eb,
             const int32_t *stride, int32_t block) {
  if (!out || !dims || ndims < 1 || ndims > 3) return SEL_EINVAL;
  if (block != 4) return SEL_EINVAL;
  if (mode != SEL_EB_ABS && mode != SEL_EB_REL) return SEL_EINVAL;
  if (!std::isfinite(eb) || !(eb > 0.0)) return SEL_EINVAL;
  if (mode == SEL_EB_ABS && !std::isfinite((float)(1.0 / (2.0 * eb)))) return SEL_EINVAL;
  Geo g{};
  for (int a = 0; a < 3; ++a) { g.n[a] = 1; g.s[a] = 1; }
  int64_t N = 1;
  for (int a = 0; a < ndims; ++a) {
    const int ax = 3 - ndims + a;
    if (dims[a] < 1) return SEL_EINVAL;
    if (N > INT64_MAX / 4 / dims[a]) return SEL_EINVAL;
    N *= dims[a];
    g.n[ax] = dims[a];
    if (stride) {
      if (stride[a] < 1) return SEL_EINVAL;
      g.s[ax] = stride[a];
    }
  }
  g.N = N;
  g.ndims = ndims;
  g.n_pb = 1;
  uint64_t nv = 1;
  for (int a = 0; a < 3; ++a) {
    g.nb[a] = (g.n[a] + 3) / 4;
    g.npb[a] = (g.nb[a] + g.s[a] - 1) / g.s[a];
    g.n_pb *= g.npb[a];
    nv *= real_in_processed(g.n[a], g.s[a]);
  }
  // the 3-axis view pads missing leading axes with extent 1: they contribute
  // real_in_processed(1, 1) = 1 value, as they should.
  auto *p = new (std::nothrow) sel_plan_st();
  if (!p) return SEL_ENOMEM;
  p->geo = g;
  p->mode = mode;
  p->eb = eb;
  p->size = ndims == 1 ? 4 : (ndims == 2 ? 16 : 64);
  p->n_values = nv;
  p->n_sz = nv - 1;   // the field origin is always in a processed block
  if (cudaGetDevice(&p->device) != cudaSuccess ||
      cudaDeviceGetAttribute(&p->sm_count, cudaDevAttrMultiProcessorCount, p->device) != cudaSuccess) {
    cuda_fail(cudaGetLastError(), "cudaGetDevice");
    delete p;
    return SEL_ECUDA;
  }
  p->mm_ctas = minmax_ctas(N, p->sm_count);
  for (int v = 0; v < 2; ++v)
    for (int d = 0; d < 2; ++d) {
      Geo gv = g;
      gv.vec = v;
      if (plan_estimate(gv, d, p->sm_count, &p->el[v][d]) != SEL_OK) {
        cuda_fail(cudaGetLastError(), "plan_estimate (occupancy)");
        delete p;
        return SEL_ECUDA;
      }
      if (p->el[v][d].ntasks > p->max_tasks) p->max_tasks = p->el[v][d].ntasks;
    }
  p->tile_ok = tile_supported(g);
  for (int d = 0; d < 2 && p->tile_ok; ++d) {
    if (plan_tile(g, p->sm_count, d, &p->tl[d]) != SEL_OK) {
      cuda_fail(cudaGetLastError(), "plan_tile");
      delete p;
      return SEL_ECUDA;
    }
    if (p->tl[d].npart > p->max_tasks) p->max_tasks = p->tl[d].npart;
  }
  // sampled strides: k_batch runs one processed block per lane (2D/3D, float4 rows)
  p->sampled_ok = (g.ndims == 2 || g.ndims == 3) && (g.s[0] > 1 || g.s[1] > 1 || g.s[2] > 1) &&
                  g.n[2] % 4 == 0 && g.n_pb < (1LL << 31);
  if ((p->tile_ok || p->sampled_ok) && batch_sizes(g, &p->bs) != SEL_OK) {
    cuda_fail(cudaGetLastError(), "batch_sizes");
    delete p;
    return SEL_ECUDA;
  }
  // workspace layout: two copies (field parity) of the fused-pass/finalize state so
  // the finalize of field f can overlap the fused pass of field f+1 (batch pipeline)
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 255) & ~(size_t)255; return o; };
  size_t o_hist[2], o_ep[2], o_tc[2], o_fp[2], o_fe[2], o_fb[2], o_fo[2], o_tk[2];
  const size_t o_mmp = take((size_t)p->mm_ctas * sizeof(float2)), o_mmf = take((size_t)p->mm_ctas * 4),
               o_prm = take(sizeof(Params));
  for (int k = 0; k < 2; ++k) {
    o_hist[k] = take((size_t)kNSlots * 8);
    o_ep[k] = take((size_t)p->max_tasks * sizeof(Partial));
    o_tc[k] = take(4);
    o_fp[k] = take((size_t)kFinCTAs * 8);
    o_fe[k] = take((size_t)kFinCTAs * 8);
    o_fb[k] = take((size_t)kFinCTAs * 8);
    o_fo[k] = take(16);   // [0] overflow count, [1] histogram total
    o_tk[k] = take(2 * 4);
  }
  if (cudaMalloc(&p->ws_mem, off) != cudaSuccess) {
    cudaGetLastError();
    delete p;
    return SEL_ENOMEM;
  }
  p->ws_bytes = off;
  char *b = (char *)p->ws_mem;
  for (int k = 0; k < 2; ++k) {
    Workspace &w = p->wsk[k];
    w.hist = (unsigned long long *)(b + o_hist[k]);
    w.mm_part = (float2 *)(b + o_mmp);
    w.mm_flag = (int32_t *)(b + o_mmf);
    w.params = (Params *)(b + o_prm);
    w.task_part = (Partial *)(b + o_ep[k]);
    w.task_ctr = (unsigned int *)(b + o_tc[k]);
    w.fin_part = (double *)(b + o_fp[k]);
    w.fin_err = (double *)(b + o_fe[k]);
    w.fin_bits = (unsigned long long *)(b + o_fb[k]);
    w.fin_ovf = (unsigned long long *)(b + o_fo[k]);
    w.tickets = (unsigned int *)(b + o_tk[k]);
  }
  p->ws = p->wsk[0];
  if (cudaMemset(p->ws_mem, 0, off) != cudaSuccess || ensure_results(p, 1) != SEL_OK) {
    cuda_fail(cudaGetLastError(), "workspace init");
    sel_plan_destroy(p);
    return SEL_ECUDA;
  }
  *out = p;
  return SEL_OK;
}

int sel_set_option(sel_plan_t p, const char *key, double value) {
  if (!p || !key) return SEL_EINVAL;
  if (!strcmp(key, "sz_offset_bits")) {
    if (!std::isfinite(value)) return SEL_EINVAL;
    p->sz_offset = value;
    return SEL_OK;
  }
  if (!strcmp(key, "debug")) {
    p->debug = value != 0.0;
    if (p->debug) return ensure_debug(p);
    return SEL_OK;
  }
  if (!strcmp(key, "lag")) {
    if (!(value >= 1.0 && value <= 4.0)) return SEL_EINVAL;
    p->lag_t = (int)value;
    return SEL_OK;
  }
  if (!strcmp(key, "groups")) {
    if (!(value >= 0.0 && value <= 148.0)) return SEL_EINVAL;
    p->groups = (int)value;
    return SEL_OK;
  }
  if (!strcmp(key, "batch_debug")) {
    p->batch_debug = value != 0.0;
    return SEL_OK;
  }
  if (!strcmp(key, "range_warps")) {
    p->range_warps = value != 0.0;
    return SEL_OK;
  }
  if (!strcmp(key, "small_kernel")) {
    p->use_small = value != 0.0;
    return SEL_OK;
  }
  if (!strcmp(key, "multi_tile")) {
    p->use_multi_tile = value != 0.0;
    return SEL_OK;
  }
  if (!strcmp(key, "batch_kernel")) {
    p->use_batch = value != 0.0;
    return SEL_OK;
  }
  if (!strcmp(key, "pipeline")) {
    p->pipeline = value != 0.0;
    return SEL_OK;
  }
  if (!strcmp(key, "kernel_timing")) {
    p->timing = value != 0.0;
    return SEL_OK;
  }
  return SEL_EINVAL;
}

int sel_estimate(sel_plan_t p, const float *d_field, void *stream, sel_result *out) {
  if (!p || !d_field || !out) return SEL_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  int rc = ensure_results(p, 1);
  if (rc) return rc;
  if (p->timing && (rc = ensure_timing(p, 1))) return rc;
  if (small_ok(p)) {
    if ((rc = enqueue_small(p, d_field, st))) return rc;
  } else if (batch_ok(p, &d_field, 1)) {
    if ((rc = enqueue_batch(p, &d_field, 1, st))) return rc;
  } else if ((rc = enqueue_field(p, d_field, st, 0))) {
    return rc;
  }
  sel_result r;
  if ((rc = finish(p, st, 1, &r))) return rc;
  if (r.status != SEL_OK) return r.status;
  *out = r;
  return SEL_OK;
}

int sel_compress_zfp(sel_plan_t p, const float *d_field, void *d_out, uint64_t cap_bytes, uint64_t *nbits,
                     void *stream) {
  if (!p || !d_field || !nbits || p->timing || p->debug) return SEL_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  const size_t wsb = zstream_ws_bytes(p->geo.n_pb);
  if (!p->zs_mem) {
    if (cudaMalloc(&p->zs_mem, wsb + 256) != cudaSuccess) {
      cudaGetLastError();
      p->zs_mem = nullptr;
      return SEL_ENOMEM;
    }
  }
  unsigned long long *d_total = (unsigned long long *)((char *)p->zs_mem + ((wsb + 127) & ~(size_t)127));
  Geo g = p->geo;
  g.vec = (g.n[2] % 4 == 0) && (((uintptr_t)d_field & 15u) == 0);
  const Workspace w0 = field_ws(p, 0);
  int rc = launch_minmax(d_field, g.N, p->mm_ctas, w0, p->mode, p->eb, st);   // Alg. 1 line 2
  if (rc) return cuda_fail(cudaGetLastError(), "k_minmax launch");
  if ((rc = launch_zstream_bits(d_field, g, p->sm_count, w0.params, p->zs_mem, d_total, st)))
    return cuda_fail(cudaGetLastError(), "stream length launch");
  unsigned long long total = 0;
  Params prm;
  CK(cudaMemcpyAsync(&total, d_total, sizeof(total), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&prm, w0.params, sizeof(prm), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  p->launches += 4;
  if (prm.status != SEL_OK) return prm.status;
  *nbits = total;
  if (!d_out) return SEL_OK;                                  // size query
  const uint64_t bytes = (total + 31) / 32 * 4;
  if (cap_bytes < bytes) return SEL_EINVAL;
  CK(cudaMemsetAsync(d_out, 0, bytes, st));
  if ((rc = launch_zstream_write(d_field, g, w0.params, p->zs_mem, (uint32_t *)d_out, st)))
    return cuda_fail(cudaGetLastError(), "stream write launch");
  p->launches += 1;
  CK(cudaStreamSynchronize(st));
  return SEL_OK;
}

int sel_estimate_paper(sel_plan_t p, const float *d_field, void *stream, sel_paper_result *out) {
  if (!p || !d_field || !out || p->timing || p->debug) return SEL_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  int rc = ensure_results(p, 1);
  if (rc) return rc;
  // workspace: [CTA partials | mid | Params | sel_paper_result], allocated once per plan
  const int cap = p->sm_count * 8;
  const size_t pws = paper_ws_bytes(cap);
  if (!p->paper_mem) {
    if (cudaMalloc(&p->paper_mem, pws + 2 * sizeof(Params) + sizeof(sel_paper_result) + 512) != cudaSuccess) {
      cudaGetLastError();
      p->paper_mem = nullptr;
      return SEL_ENOMEM;
    }
    p->paper_cap = cap;
  }
  char *b = (char *)p->paper_mem;
  Params *pprm = (Params *)(b + ((pws + 255) & ~(size_t)255));
  sel_paper_result *dres = (sel_paper_result *)(pprm + 2);
  Geo g = p->geo;
  g.vec = (g.n[2] % 4 == 0) && (((uintptr_t)d_field & 15u) == 0);
  // Alg. 1 line 2: value range (params slot 0 of the plan)
  const Workspace w0 = field_ws(p, 0);
  if ((rc = launch_minmax(d_field, g.N, p->mm_ctas, w0, p->mode, p->eb, st)))
    return cuda_fail(cudaGetLastError(), "k_minmax launch");
  // lines 3-7: ZFP from the sampled coefficients -> PSNR_sp -> delta, r* = 1/delta
  if ((rc = launch_paper_zfp(d_field, g, p->sm_count, p->paper_cap, w0.params, p->paper_mem, pprm, st)))
    return cuda_fail(cudaGetLastError(), "k_paper_zfp launch");
  // lines 8-9: the processed blocks' residuals at bin width delta (the fused pass with
  // r_f = r*; only its histogram is used), entropy in the finalize
  Workspace ws = p->wsk[0];
  ws.params = pprm;
  const bool tile = p->tile_ok && g.vec;
  rc = tile ? launch_tile(d_field, g, p->tl[0], ws, nullptr, st)
            : launch_estimate(d_field, g, p->el[g.vec][0], ws, nullptr, st);
  if (rc) return cuda_fail(cudaGetLastError(), "paper SZ pass launch");
  FinalizeArgs fa;
  fa.mode = p->mode;
  fa.eb = p->eb;
  fa.sz_offset = p->sz_offset;
  fa.n_sz = p->n_sz;
  fa.n_values = p->n_values;
  fa.n_blocks = (uint64_t)p->geo.n_pb;
  fa.ntasks = tile ? p->tl[0].npart : p->el[g.vec][0].ntasks;
  if ((rc = launch_finalize(ws, fa, p->d_res, nullptr, st))) return cuda_fail(cudaGetLastError(), "k_finalize launch");
  // line 10 + the result
  if ((rc = launch_paper_assemble(p->paper_mem, p->paper_cap, p->d_res, p->n_values, dres, st)))
    return cuda_fail(cudaGetLastError(), "k_paper_assemble launch");
  p->launches += 6;
  sel_paper_result h;
  CK(cudaMemcpyAsync(&h, dres, sizeof(h), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (h.status != SEL_OK) return h.status;
  *out = h;
  return SEL_OK;
}

int sel_estimate_variants(sel_plan_t p, const float *d_field, int log_base, int eqp_n, void *stream,
                          sel_variant_result *out) {
  if (!p || !d_field || !out || p->timing || p->debug) return SEL_EINVAL;
  if (log_base < 2 || eqp_n < 1 || eqp_n > 32768) return SEL_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  int rc = ensure_results(p, 1);
  if (rc) return rc;
  if (!p->var_mem && cudaMalloc(&p->var_mem, variants_ws_bytes()) != cudaSuccess) {
    cudaGetLastError();
    p->var_mem = nullptr;
    return SEL_ENOMEM;
  }
  Geo g = p->geo;
  g.vec = (g.n[2] % 4 == 0) && (((uintptr_t)d_field & 15u) == 0);
  // Alg. 1 line 2, then the fused pass of the per-field pipeline: its histogram is the PDF
  const Workspace w = field_ws(p, 0);
  if ((rc = launch_minmax(d_field, g.N, p->mm_ctas, w, p->mode, p->eb, st)))
    return cuda_fail(cudaGetLastError(), "k_minmax launch");
  const bool tile = p->tile_ok && g.vec;
  rc = tile ? launch_tile(d_field, g, p->tl[0], w, nullptr, st)
            : launch_estimate(d_field, g, p->el[g.vec][0], w, nullptr, st);
  if (rc) return cuda_fail(cudaGetLastError(), "variants fused pass launch");
  FinalizeArgs fa;
  fa.mode = p->mode;
  fa.eb = p->eb;
  fa.sz_offset = p->sz_offset;
  fa.n_sz = p->n_sz;
  fa.n_values = p->n_values;
  fa.n_blocks = (uint64_t)p->geo.n_pb;
  fa.ntasks = tile ? p->tl[0].npart : p->el[g.vec][0].ntasks;
  // the finalize copies the histogram out before it re-zeroes the workspace
  if ((rc = launch_finalize(w, fa, p->d_res, (unsigned long long *)p->var_mem, st)))
    return cuda_fail(cudaGetLastError(), "k_finalize launch");
  if ((rc = launch_variants(p->var_mem, w.params, log_base, eqp_n, st)))
    return cuda_fail(cudaGetLastError(), "k_variants launch");
  p->launches += 4;
  sel_variant_result h;
  CK(cudaMemcpyAsync(&h, (char *)p->var_mem + (size_t)kNSlots * 16, sizeof(h), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (h.status != SEL_OK) return h.status;
  *out = h;
  return SEL_OK;
}

int sel_estimate_multi(sel_plan_t p, const float *d_field, int k, const double *ebs, void *stream,
                       sel_result *out) {
  if (!p || !d_field || !ebs || !out || k < 1 || k > kMultiMaxEb || p->timing || p->debug) return SEL_EINVAL;
  for (int e = 0; e < k; ++e) {
    if (!std::isfinite(ebs[e]) || !(ebs[e] > 0.0)) return SEL_EINVAL;
    if (p->mode == SEL_EB_ABS && !std::isfinite((float)(1.0 / (2.0 * ebs[e])))) return SEL_EINVAL;
  }
  cudaStream_t st = (cudaStream_t)stream;
  int rc = ensure_results(p, k);
  if (rc) return rc;
  if ((rc = ensure_multi(p))) return rc;
  Geo g = p->geo;
  g.vec = (g.n[2] % 4 == 0) && (((uintptr_t)d_field & 15u) == 0);
  // full-field 2D / 3D: the TMA tile pipeline with the eb loop inside (k_tile_multi)
  const long long tparts = p->tile_ok ? multi_tile_parts(g, p->tl[0]) : 0;
  const bool tile = p->tile_ok && g.vec && p->use_multi_tile && tparts < (1LL << 31);
  if (tile && !p->mtile_mem) {
    if (cudaMalloc(&p->mtile_mem, 256 + sizeof(Partial) * (size_t)tparts * kMultiMaxEb) != cudaSuccess) {
      cudaGetLastError();
      p->mtile_mem = nullptr;
      return SEL_ENOMEM;
    }
    if (cudaMemsetAsync(p->mtile_mem, 0, 256, st) != cudaSuccess) return cuda_fail(cudaGetLastError(), "multi tile state");
  }
  int ctas = 0;
  if (!tile) {
    if ((rc = multi_ctas(g, k, p->sm_count, &ctas))) return cuda_fail(cudaGetLastError(), "multi occupancy");
    if (ctas > p->mcap) ctas = p->mcap;
  }
  // value range once (K1 writes vmin / vmax / non-finite into the plan's params slot)
  const Workspace w0 = field_ws(p, 0);
  if ((rc = launch_minmax(d_field, g.N, p->mm_ctas, w0, p->mode, p->eb, st)))
    return cuda_fail(cudaGetLastError(), "k_minmax launch");
  Partial *const tpart = tile ? (Partial *)((char *)p->mtile_mem + 256) : nullptr;
  if (tile) {
    if ((rc = launch_multi_tile(d_field, g, p->tl[0], p->sm_count, k, ebs, p->mode, w0.params, p->mprm,
                                p->mws[0].hist, tpart, (size_t)tparts, (unsigned int *)p->mtile_mem, st)))
      return rc == SEL_ECUDA ? cuda_fail(cudaGetLastError(), "k_tile_multi launch") : rc;
  } else if ((rc = launch_multi(d_field, g, ctas, k, ebs, p->mode, w0.params, p->mprm, p->mws[0].hist, p->mpart,
                                st))) {
    return rc == SEL_ECUDA ? cuda_fail(cudaGetLastError(), "k_multi launch") : rc;
  }
  // the per-eb part arrays are [e][ctas] inside [e][mcap] slots: k_multi writes
  // part[e * ctas + cta] -- give every finalize its own view
  for (int e = 0; e < k; ++e) {
    Workspace w = p->mws[e];
    w.task_part = tile ? tpart + (size_t)e * (size_t)tparts : p->mpart + (size_t)e * ctas;
    FinalizeArgs fa;
    fa.mode = p->mode;
    fa.eb = ebs[e];
    fa.sz_offset = p->sz_offset;
    fa.n_sz = p->n_sz;
    fa.n_values = p->n_values;
    fa.n_blocks = (uint64_t)p->geo.n_pb;
    fa.ntasks = tile ? (int)tparts : ctas;
    if ((rc = launch_finalize(w, fa, p->d_res + e, nullptr, st))) return cuda_fail(cudaGetLastError(), "k_finalize launch");
  }
  p->launches += 2 + k;
  return finish(p, st, k, out);
}

int sel_estimate_batch(sel_plan_t p, const float *const *d_fields, int n, void *stream,
                       sel_result *out) {
  if (!p || !d_fields || !out || n < 0) return SEL_EINVAL;
  if (n == 0) return SEL_OK;
  for (int f = 0; f < n; ++f) if (!d_fields[f]) return SEL_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  int rc = ensure_results(p, n);
  if (rc) return rc;
  if (p->timing && (rc = ensure_timing(p, n))) return rc;
  if (batch_ok(p, d_fields, n)) {
    if ((rc = enqueue_batch(p, d_fields, n, st))) return rc;
  } else if (n >= 2 && p->pipeline && !p->timing && !p->debug) {
    if ((rc = enqueue_pipelined(p, d_fields, n, st))) return rc;
  } else {
    for (int f = 0; f < n; ++f)
      if ((rc = enqueue_field(p, d_fields[f], st, f))) return rc;
  }
  return finish(p, st, n, out);
}

int sel_estimate_batch_async(sel_plan_t p, const float *const *d_fields, int n, void *stream,
                             sel_result *out) {
  if (!p || !d_fields || !out || n < 0 || p->timing || p->debug) return SEL_EINVAL;
  if (n == 0) return SEL_OK;
  for (int f = 0; f < n; ++f) if (!d_fields[f]) return SEL_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  int rc = ensure_results(p, n);
  if (rc) return rc;
  if (n == 1 && small_ok(p)) {
    if ((rc = enqueue_small(p, d_fields[0], st))) return rc;
  } else if (batch_ok(p, d_fields, n)) {
    if ((rc = enqueue_batch(p, d_fields, n, st))) return rc;
  } else if (n >= 2 && p->pipeline) {
    if ((rc = enqueue_pipelined(p, d_fields, n, st))) return rc;
  } else {
    for (int f = 0; f < n; ++f)
      if ((rc = enqueue_field(p, d_fields[f], st, f))) return rc;
  }
  CK(cudaMemcpyAsync(out, p->d_res, sizeof(sel_result) * (size_t)n, cudaMemcpyDefault, st));
  return SEL_OK;
}

int sel_estimate_batch_host(sel_plan_t p, const float *const *h_fields, int n, void *stream,
                            sel_result *out) {
  if (!p || !h_fields || !out || n < 0) return SEL_EINVAL;
  if (n == 0) return SEL_OK;
  for (int f = 0; f < n; ++f) if (!h_fields[f]) return SEL_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  int rc = ensure_results(p, n);
  if (rc) return rc;
  if (p->timing && (rc = ensure_timing(p, n))) return rc;
  const size_t bytes = (size_t)p->geo.N * sizeof(float);
  if (!p->copy_stream) {
    CK(cudaStreamCreateWithFlags(&p->copy_stream, cudaStreamNonBlocking));
    for (int b = 0; b < 2; ++b) {
      CK(cudaEventCreateWithFlags(&p->ev_copied[b], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&p->ev_done[b], cudaEventDisableTiming));
    }
  }
  // Chunks of K fields (<= ~1 GB per staging buffer), double-buffered: the H2D copies of
  // chunk c+1 (copy stream) overlap the estimate of chunk c, which is ONE k_batch launch
  // over the chunk -- the same kernel as the device-resident entry points -- where the
  // shape allows it (else the per-field kernels, one field at a time).
  const bool kb = (p->tile_ok || p->sampled_ok) && p->use_batch && !p->debug && !p->timing &&
                  p->geo.N < ((int64_t)1 << 32) && (p->geo.N % 4 == 0);
  int K = 1;
  if (kb) {
    K = (int)std::max<size_t>(1, (size_t)1e9 / bytes);
    if (K > n) K = n;
  }
  if (p->stage_cap < (size_t)K * bytes) {
    if (p->d_stage[0] || p->d_stage[1]) {
      CK(cudaStreamSynchronize(st));
      CK(cudaStreamSynchronize(p->copy_stream));
    }
    for (int b = 0; b < 2; ++b) {
      if (p->d_stage[b]) cudaFree(p->d_stage[b]);
      p->d_stage[b] = nullptr;
    }
    p->stage_cap = 0;
    for (int b = 0; b < 2; ++b)
      if (cudaMalloc(&p->d_stage[b], (size_t)K * bytes) != cudaSuccess) return SEL_ENOMEM;
    p->stage_cap = (size_t)K * bytes;
  }
  std::vector<const float *> ptrs((size_t)K);
  const int nchunk = (n + K - 1) / K;
  for (int c = 0; c < nchunk; ++c) {
    const int b = c & 1, f0 = c * K, nfc = std::min(K, n - f0);
    if (c >= 2) CK(cudaStreamWaitEvent(p->copy_stream, p->ev_done[b], 0));
    for (int i = 0; i < nfc; ++i) {
      float *dst = p->d_stage[b] + (size_t)i * (size_t)p->geo.N;
      CK(cudaMemcpyAsync(dst, h_fields[f0 + i], bytes, cudaMemcpyHostToDevice, p->copy_stream));
      ptrs[(size_t)i] = dst;
    }
    CK(cudaEventRecord(p->ev_copied[b], p->copy_stream));
    CK(cudaStreamWaitEvent(st, p->ev_copied[b], 0));
    if (kb && batch_ok(p, ptrs.data(), nfc)) {
      if ((rc = enqueue_batch(p, ptrs.data(), nfc, st, p->d_res + f0))) return rc;
    } else {
      for (int i = 0; i < nfc; ++i)
        if ((rc = enqueue_field(p, ptrs[(size_t)i], st, f0 + i))) return rc;
    }
    CK(cudaEventRecord(p->ev_done[b], st));
  }
  return finish(p, st, n, out);
}

int sel_choose(const sel_result *r, int32_t *choice) {
  if (!r || !choice) return SEL_EINVAL;
  const double vr = r->value_range, eb = r->eb_abs, mse = r->zfp_mse;
  const double bsz = r->sz_bits_per_value, bzfp = r->zfp_bits_per_value, pz = r->zfp_psnr;
  if (!(mse > 0.0) || !(vr > 0.0) || !std::isfinite(pz)) {
    *choice = bsz < bzfp ? 0 : 1;
    return SEL_OK;
  }
  const double delta = vr * std::sqrt(12.0) * std::pow(10.0, -pz / 20.0);
  double bm = bsz + std::log2(2.0 * eb / delta);
  if (bm < 0.0) bm = 0.0;
  *choice = bm < bzfp ? 0 : 1;
  return SEL_OK;
}

int sel_choose_eb(const sel_result *r, int32_t *choice) {
  if (!r || !choice) return SEL_EINVAL;
  *choice = r->sz_bits_per_value < r->zfp_bits_per_value ? 0 : 1;   // P:639-642, ties -> ZFP
  return SEL_OK;
}

int sel_debug_copy(sel_plan_t p, const char *what, void *dst, uint64_t bytes) {
  if (p && what && !strcmp(what, "small_prof")) {   // developer probe (SEL_SMALL_PROF builds)
    if (!p->small_mem || !dst || bytes != 7 * 8) return SEL_EINVAL;
    const size_t off = 256 + (size_t)p->sm_count * (sizeof(Partial) + 24);
    CK(cudaMemcpy(dst, (char *)p->small_mem + off, bytes, cudaMemcpyDeviceToHost));
    return SEL_OK;
  }
  if (!p || !what || !dst) return SEL_EINVAL;
  if (!strncmp(what, "batch_", 6)) {     // k_batch dumps of the last batch launch
    if (!p->bdump.hist || p->last_batch_nf < 1 || p->last_batch_nf > p->bdump_cap) return SEL_EINVAL;
    const uint64_t nf = (uint64_t)p->last_batch_nf;
    const uint64_t np = (uint64_t)batch_ntasks(p->geo, p->tl[0], p->bs) * batch_parts_per_task(p->geo);
    const void *bsrc = nullptr;
    uint64_t bneed = 0;
    if (!strcmp(what, "batch_hist")) { bsrc = p->bdump.hist; bneed = nf * kNSlots * 4; }
    else if (!strcmp(what, "batch_part")) { bsrc = p->bdump.part; bneed = nf * np * sizeof(Partial); }
    else return SEL_EINVAL;
    if (bytes != bneed) return SEL_EINVAL;
    CK(cudaMemcpy(dst, bsrc, bneed, cudaMemcpyDeviceToHost));
    return SEL_OK;
  }
  if (!p->dbg_mem) return SEL_EINVAL;
  const uint64_t N = (uint64_t)p->geo.N, B = (uint64_t)p->geo.n_pb, S = (uint64_t)p->size;
  const void *src = nullptr;
  uint64_t need = 0;
  if (!strcmp(what, "codes")) { src = p->dbg.codes; need = N * 4; }
  else if (!strcmp(what, "hist")) { src = p->dbg_hist; need = (uint64_t)kNSlots * 8; }
  else if (!strcmp(what, "emax")) { src = p->dbg.emax; need = B * 4; }
  else if (!strcmp(what, "coef")) { src = p->dbg.coef; need = B * S * 4; }
  else if (!strcmp(what, "uword")) { src = p->dbg.uword; need = B * S * 4; }
  else if (!strcmp(what, "bits")) { src = p->dbg.bits; need = B * 4; }
  else if (!strcmp(what, "err")) { src = p->dbg.err; need = B * 8; }
  else return SEL_EINVAL;
  if (bytes != need) return SEL_EINVAL;
  CK(cudaMemcpy(dst, src, need, cudaMemcpyDeviceToHost));
  return SEL_OK;
}

int sel_kernel_times(sel_plan_t p, double ms[3], uint64_t launches[3], int reset) {
  if (!p || !ms || !launches) return SEL_EINVAL;
  for (int k = 0; k < 3; ++k) { ms[k] = p->ms[k]; launches[k] = p->tcount[k]; }
  if (reset) for (int k = 0; k < 3; ++k) { p->ms[k] = 0; p->tcount[k] = 0; }
  return SEL_OK;
}

int sel_batch_layout(sel_plan_t p, int64_t out[8]) {
  if (!p || !out) return SEL_EINVAL;
  const bool sampled = p->geo.s[0] > 1 || p->geo.s[1] > 1 || p->geo.s[2] > 1;
  out[0] = batch_ntasks(p->geo, p->tl[0], p->bs);
  out[1] = batch_parts_per_task(p->geo);
  out[2] = batch_rows_per_part(p->geo);           // block rows per part (tile tasks)
  out[3] = out[1] * out[2];                       // block rows per tile
  out[4] = p->tl[0].tg.ntk;
  out[5] = p->tl[0].tg.ntj;
  out[6] = sampled ? 1 : 0;
  out[7] = p->last_batch_G;
  return SEL_OK;
}

uint64_t sel_processed_blocks(sel_plan_t p) { return p ? (uint64_t)p->geo.n_pb : 0; }
uint64_t sel_processed_values(sel_plan_t p) { return p ? p->n_values : 0; }
size_t sel_workspace_bytes(sel_plan_t p) { return p ? p->ws_bytes : 0; }
uint64_t sel_launch_count(sel_plan_t p) { return p ? p->launches : 0; }

void sel_plan_destroy(sel_plan_t p) {
  if (!p) return;
  if (p->copy_stream) cudaStreamSynchronize(p->copy_stream);
  if (p->ws_mem) cudaFree(p->ws_mem);
  if (p->multi_mem) cudaFree(p->multi_mem);
  if (p->mtile_mem) cudaFree(p->mtile_mem);
  if (p->paper_mem) cudaFree(p->paper_mem);
  if (p->var_mem) cudaFree(p->var_mem);
  if (p->zs_mem) cudaFree(p->zs_mem);
  if (p->small_mem) cudaFree(p->small_mem);
  if (p->d_res) cudaFree(p->d_res);
  if (p->h_res) cudaFreeHost(p->h_res);
  if (p->dbg_mem) cudaFree(p->dbg_mem);
  for (int b = 0; b < 2; ++b) {
    if (p->d_stage[b]) cudaFree(p->d_stage[b]);
    if (p->ev_copied[b]) cudaEventDestroy(p->ev_copied[b]);
    if (p->ev_done[b]) cudaEventDestroy(p->ev_done[b]);
  }
  if (p->copy_stream) cudaStreamDestroy(p->copy_stream);
  if (p->aux_stream) {
    cudaStreamSynchronize(p->aux_stream);
    cudaStreamDestroy(p->aux_stream);
  }
  if (p->fin_stream) {
    cudaStreamSynchronize(p->fin_stream);
    cudaStreamDestroy(p->fin_stream);
  }
  for (auto e : p->ev_mm) cudaEventDestroy(e);
  for (auto e : p->ev_k2) cudaEventDestroy(e);
  for (auto e : p->ev_k3) cudaEventDestroy(e);
  if (p->d_params) cudaFree(p->d_params);
  if (p->bstate) cudaFree(p->bstate);
  if (p->bdump.hist) cudaFree(p->bdump.hist);
  if (p->bdump.part) cudaFree(p->bdump.part);
  if (p->btab.d) cudaFree(p->btab.d);
  for (auto e : p->bev)
    if (e) cudaEventDestroy(e);
  for (auto &s : p->tslots)
    for (auto &e : s.ev) cudaEventDestroy(e);
  delete p;
}

}  // extern "C"
