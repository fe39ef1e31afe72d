// sel_internal.h -- structures shared by the host runtime (sel_api.cu) and the
// sm_100a kernels (sel_kernels.cu).  Not part of the public ABI.
#pragma once
#include <cstdint>

#include "../../include/sel.h"

namespace sel {

constexpr int kNSlots = 65536;       // 65,535 code bins + overflow slot
constexpr int kOvfSlot = 65535;
constexpr int kCenter = 32767;       // slot of code 0
constexpr int kWinHalf = 4096;       // smem-privatised window: slots [kCenter-kWinHalf, kCenter+kWinHalf)
constexpr int kWinBins = 2 * kWinHalf;
constexpr int kFinCTAs = 64;         // finalize: 64 CTAs x 1024 slots
constexpr int kFinThreads = 128;

// Geometry, padded to 3 axes: axis 0 slowest.  For ndims < 3 the leading axes
// have n = nb = npb = s = 1.
struct Geo {
  int64_t n[3];     // field extents
  int64_t nb[3];    // blocks per axis = ceil(n/4)
  int64_t npb[3];   // processed blocks per axis = ceil(nb/s)
  int32_t s[3];     // sampling stride in blocks
  int64_t n_pb;     // total processed blocks
  int64_t N;        // total values
  int32_t ndims;
  int32_t vec;      // 1: fastest extent % 4 == 0 and field 16B-aligned -> float4 loads
};

// Derived per-field scalars written by the value-range kernel (Alg.1 line 2).
struct Params {
  float vmin, vmax;
  double vr;
  double eb_abs;
  float r_f;
  int32_t minexp;
  int32_t status;   // sel_status
  int32_t pad;
};

// Per-task partials of the fused pass (summed in task order by the finalize).
struct Partial {
  uint64_t bits;    // sum of per-block EC bits
  double err;       // sum of E_b
};

// Geometry of the marching kernel (2D/3D, every block processed).  The marching axis
// is the slowest block axis (view axis 0 for 3D, 1 for 2D); a warp task is 32
// consecutive blocks along the fastest axis x one "other" block row (3D) x L layers.
struct MarchGeo {
  int64_t n[3];
  int64_t nb[3];
  int32_t L;        // block layers per task
  int32_t nchunk;   // ceil(nb[2] / 32)
  int32_t nother;   // nb[1] for 3D, 1 for 2D
  int32_t nseg;     // ceil(nb_march / L)
  int32_t ntasks;   // nseg * nother * nchunk
  int32_t pad;
};

// Geometry of the TMA tile kernel (2D/3D, every block, fastest extent % 4 == 0).
struct TileGeo {
  int64_t n[3];
  int32_t nb[3];
  int32_t ntj;      // tiles along axis 1 (one block row per consumer warp)
  int32_t ntk;      // tiles along axis 2 (32 blocks each)
  int32_t ntasks;   // ntj * ntk * (nb[0] for 3D)
};

struct TileLaunch {
  int ctas;
  int threads;
  size_t smem;
  int npart;        // partials written = ntasks * consumer warps
  TileGeo tg;
};

struct EstLaunch {
  bool march;
  int ctas;
  int ntasks;       // partials written (march: tasks; generic: CTAs)
  MarchGeo mg;
};

// Debug dump pointers (device), all may be null.
struct DebugPtrs {
  int32_t *codes;
  int32_t *emax;
  int32_t *coef;
  uint32_t *uword;
  uint32_t *bits;
  double *err;
};

struct Workspace {
  unsigned long long *hist;   // [kNSlots] u64
  float2 *mm_part;            // [mm_ctas] (min,max)
  int32_t *mm_flag;           // [mm_ctas] nonfinite flags
  Params *params;             // [1]
  Partial *task_part;         // [max tasks]
  unsigned int *task_ctr;     // [1] dynamic task counter (reset by finalize)
  double *fin_part;           // [kFinCTAs]
  double *fin_err;            // [kFinCTAs]
  unsigned long long *fin_bits; // [kFinCTAs]
  unsigned long long *fin_ovf;// [2]: overflow count, histogram total (device-counted)
  unsigned int *tickets;      // [2] last-block-done counters (minmax, finalize)
};

struct FinalizeArgs {
  int32_t mode;             // SEL_EB_ABS / SEL_EB_REL
  double eb;
  double sz_offset;
  uint64_t n_sz;            // SZ points (host geometry)
  uint64_t n_values;        // N_P
  uint64_t n_blocks;
  int32_t ntasks;
};

// launchers (sel_kernels.cu)
int launch_minmax(const float *x, int64_t N, int ctas, const Workspace &ws, int mode, double eb,
                  cudaStream_t st);
int plan_estimate(const Geo &g, int debug, int sm_count, EstLaunch *el);
int launch_estimate(const float *x, const Geo &g, const EstLaunch &el, const Workspace &ws,
                    const DebugPtrs *dbg, cudaStream_t st);
struct BatchSizes {
  int rchunk;       // floats per value-range task
  int nR;           // value-range tasks per field
  size_t smem;
  int threads;
  int cw;           // consumer warps
};

// k_batch task table: the decoded task sequence of every CTA group (uint4 per task), built
// on the host and cached on the device per (fields, groups, task counts) key
struct BatchTable {
  void *d = nullptr;
  size_t cap = 0;
  long long key[8] = {-1, -1, -1, -1, -1, -1, -1, -1};
  size_t hist_clean = 0;   // leading histogram-ring slots of the batch state known to be zero
};

// optional k_batch test dumps (option "batch_debug"): per field, the histogram the F
// tasks read and the per-(task, part) partials
struct BatchDump {
  unsigned int *hist = nullptr;   // [nf][kNSlots]
  Partial *part = nullptr;        // [nf][nT * parts per task]
};

bool tile_supported(const Geo &g);
// k_batch limits: 16-bit tile coordinates in the task table, 32-bit task indices
bool batch_fits(const Geo &g, const TileLaunch &tl, const BatchSizes &bs, int nf);
int batch_parts_per_task(const Geo &g);
int batch_rows_per_part(const Geo &g);
int batch_sizes(const Geo &g, BatchSizes *bs);
size_t batch_state_bytes(int nf, const BatchSizes &bs, int nT, int G);
int batch_ntasks(const Geo &g, const TileLaunch &tl, const BatchSizes &bs);
int launch_batch(const Geo &g, const TileLaunch &tl, const BatchSizes &bs, const float *const *d_fields,
                 int nf, void *state, size_t state_bytes, const FinalizeArgs &fa, int mode, double eb,
                 sel_result *d_results, int sm_count, int G, int lagT, int range_warps_on, BatchTable *tab,
                 const BatchDump &dump, cudaStream_t st, cudaEvent_t *ev);
int plan_tile(const Geo &g, int sm_count, int debug, TileLaunch *tl);
int launch_tile(const float *x, const Geo &g, const TileLaunch &tl, const Workspace &ws,
                const DebugPtrs *dbg, cudaStream_t st);
int launch_finalize(const Workspace &ws, const FinalizeArgs &fa, sel_result *d_out,
                    unsigned long long *dbg_hist, cudaStream_t st);
int minmax_ctas(int64_t N, int sm_count);
// small single field in one cooperative launch (sel_kernels.cu)
size_t small_state_bytes(int sm_count);
int init_small_state(void *state, cudaStream_t st);
int launch_small(const float *x, const Geo &g, int sm_count, void *state, const Workspace &ws,
                 const FinalizeArgs &fa, sel_result *d_out, cudaStream_t st);
// N3 ZFP stream (sel_stream.cu)
size_t zstream_ws_bytes(int64_t n_pb);
int launch_zstream_bits(const float *x, const Geo &g, int sm_count, const Params *prm, void *ws,
                        unsigned long long *d_total, cudaStream_t st);
int launch_zstream_write(const float *x, const Geo &g, const Params *prm, void *ws, uint32_t *out, cudaStream_t st);
// N4 variant quantisers (sel_variants.cu): workspace = [hist copy | edges | result]
size_t variants_ws_bytes();
int launch_variants(void *vws, const Params *prm, int log_base, int eqp_n, cudaStream_t st);

// N2 paper-literal estimator (sel_paper.cu)
size_t paper_ws_bytes(int max_ctas);
int launch_paper_zfp(const float *x, const Geo &g, int sm_count, int max_ctas, const Params *base, void *pws,
                     Params *pprm, cudaStream_t st);
int launch_paper_assemble(void *pws, int max_ctas, const sel_result *sz, uint64_t n_values, sel_paper_result *out,
                          cudaStream_t st);
// N1 multi-eb pass (sel_multi.cu)
constexpr int kMultiMaxEb = 8;
int multi_ctas(const Geo &g, int k, int sm_count, int *ctas);
int launch_multi(const float *x, const Geo &g, int ctas, int k, const double *ebs, int mode,
                 const Params *base, Params *prm, unsigned long long *hist, Partial *part, cudaStream_t st);
// ... on the TMA tile pipeline (full-field 2D / 3D, tile_supported shapes)
long long multi_tile_parts(const Geo &g, const TileLaunch &tl);
int launch_multi_tile(const float *x, const Geo &g, const TileLaunch &tl, int sm_count, int k, const double *ebs,
                      int mode, const Params *base, Params *prm, unsigned long long *hist, Partial *part,
                      size_t part_stride, unsigned int *task_ctr, cudaStream_t st);

}  // namespace sel
