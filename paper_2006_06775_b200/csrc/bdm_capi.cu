// bdm_capi.cu -- host runtime behind include/bdm.h (libbdm.so).
//
// Owns the device state of one population, sequences the kernels of bdm_kernels.cuh on one
// CUDA stream and maps every failure to a BDM_E* code (never aborts).  Device layout:
//   agents  double4 (x, y, z, D), 32 B = one sector per agent, two buffers (sorted / stepped)
//   ids     uint32, two buffers (agent id = input index)
//   table   uint32[n_boxes + 1]: per-box count, scanned in place into the start table
//   sort    key / slot / tsrc / tid / tkey uint32 scratch
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/bdm.h"
#include "bdm_kernels.cuh"

using namespace bdm;

namespace {

thread_local std::string g_tls_error;
const bool g_debug = std::getenv("BDM_DEBUG") != nullptr;  // sync + check after every launch
// BDM_DEFER=k: at most k consecutive deferred builds (no host round trip); 0 = off
// (default 8 since round 2: cfg3 2.303 -> 2.282 ms/step; bdm_set_defer sets it per handle)
const int g_defer = std::getenv("BDM_DEFER") ? std::atoi(std::getenv("BDM_DEFER")) : 8;
// BDM_HTILE=1: pass A with the TMA-staged neighbourhood (k_half_search_tile, warp-specialised producer);
// measured slower than k_half_search on cfg3, so off by default
const bool g_htile = std::getenv("BDM_HTILE") && std::getenv("BDM_HTILE")[0] == '1';
// BDM_BANDS=b: the force phase in b bands of the sorted order, the sum pass of band k on a second
// stream as soon as the searches of bands 0..k are done; 1 = one launch per pass
const int g_bands = std::getenv("BDM_BANDS") ? std::max(1, std::min(32, std::atoi(std::getenv("BDM_BANDS")))) : 1;
// BDM_PBOX=0: the key pass re-reads the state instead of the sum pass's packed boxes
const bool g_pbox = !(std::getenv("BDM_PBOX") && std::getenv("BDM_PBOX")[0] == '0');
// BDM_FUSE=0: no fused column pass in the sum pass (the build runs its own column pass)
const bool g_fuse = !(std::getenv("BDM_FUSE") && std::getenv("BDM_FUSE")[0] == '0');
// BDM_TZERO=0: the build zeroes its histogram itself (default: the last sum pass zeroed it, table2)
const bool g_tzero = !(std::getenv("BDM_TZERO") && std::getenv("BDM_TZERO")[0] == '0');
// BDM_RING=k: the banded force phase with a ring of 2^k pair rows even when the rows would fit (tests)
const int g_ring_log = std::getenv("BDM_RING") ? std::atoi(std::getenv("BDM_RING")) : 0;
// BDM_PDL=0: the step's launch chain without programmatic dependent launch (lx below)
const bool g_pdl = !(std::getenv("BDM_PDL") && std::getenv("BDM_PDL")[0] == '0');

enum class State { NoGrid, Fresh, Stepped };

struct TimedStep {
  cudaEvent_t e0, e1, e2;
  cudaEvent_t e3 = nullptr;  // half-shell path: between the search and the sum pass
};

struct DistGroup;  // distributed x-slab runtime (bdm_dist.cuh)

}  // namespace

struct bdm_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bdm_params prm{};
  int64_t n = 0;
  // state buffers: 'srt' holds the box-sorted agents after a grid build; 'cur' holds the newest
  // positions (after a step: in srt's order, ids shared with srt).
  double4* ag[2] = {nullptr, nullptr};
  float4* agf = nullptr;  // fp32 copy of the sorted positions (candidate prefilter)
  uint32_t* id[2] = {nullptr, nullptr};
  int cur = 0;  // index of the buffer holding the newest state
  uint32_t *key = nullptr, *slot = nullptr, *tsrc = nullptr, *tid = nullptr, *tkey = nullptr;
  uint32_t* table = nullptr;
  size_t table_cap = 0;  // entries
  // the next build's histogram buffer (same capacity), zeroed by the last sum pass up to ext->zeroed
  // entries while the current table was still in use (table_pre: that happened; the build swaps them)
  uint32_t* table2 = nullptr;
  bool table_pre = false;
  // banded force phase (populations whose pair rows do not fit, or BDM_RING): rows for a ring of two
  // bands of ring/2 agents (GridDev::rmask = ring - 1); per-band chunk counters; layer starts
  uint32_t ring = 0;
  uint32_t* rwork = nullptr;
  size_t rwork_cap = 0;
  uint32_t* lstart = nullptr;
  uint32_t* lstart_host = nullptr;
  size_t lstart_cap = 0;
  uint32_t ring_band = 0;  // band size of the current step (0: the ring does not hold this grid's reach)
  unsigned long long* scan_state = nullptr;
  uint32_t* scan_ticket = nullptr;
  size_t scan_tiles_cap = 0;
  double* dp = nullptr;
  double* stage = nullptr;  // 4n fp64 staging for host-pointer inputs/outputs (lazily allocated)
  bool have_dp = false;
  const uint32_t* out_ids = nullptr;  // id buffer matching the order of dp / record arrays
  Extents* ext = nullptr;      // device
  Extents* ext_host = nullptr;  // pinned mirror
  bool ext_valid = false;       // ext describes ag[cur]
  ErrDev* err = nullptr;
  ErrDev* err_host = nullptr;
  unsigned long long* maxd_bits = nullptr;
  GridDev grid{};
  bool have_grid = false;
  State state = State::NoGrid;
  bool poisoned = false;
  // BDM_RECORD
  int32_t *r_cand = nullptr, *r_nb = nullptr, *r_ct = nullptr;
  int8_t* r_branch = nullptr;
  unsigned long long *r_nbh = nullptr, *r_cth = nullptr;
  bool have_record = false;
  // timing
  // ragged box table
  int32_t *czlo = nullptr, *czhi = nullptr;
  uint32_t* coff = nullptr;
  size_t col_cap = 0, coff_cap = 0;
  int4* colrec = nullptr;  // packed column records (czlo, czhi, coff) of the current grid (coff_cap)
  // next build's column z-ranges, accumulated by the half-shell sum pass (fused column pass):
  // frame [nlo[0], nlo[0]+nnx) x [nlo[1], nlo[1]+nny) = tight extents of the step start +- 1 box
  int32_t *czlo2 = nullptr, *czhi2 = nullptr;
  size_t col2_cap = 0;
  bool cols_next = false;
  int32_t nlo[2] = {0, 0}, nnx = 0, nny = 0;
  int32_t tlo[3] = {0, 0, 0}, thi[3] = {0, 0, 0};  // tight extents of the last build (reported)
  uint32_t* pbox = nullptr;  // packed new boxes of the last step (sum pass), read by the next key pass
  size_t pbox_cap = 0;
  bool pbox_next = false;
  int32_t pb_z0 = 0, pb_zbits = 0;
  bool defer_ok = false;  // this build may be deferred (not the last step of a bdm_mech_step call)
  int defer_max = g_defer;  // at most this many consecutive deferred builds (bdm_set_defer)
  int deferred = 0;       // consecutive deferred builds
  int scan_blocks_per_sm = 0;
  // x-slab mode (multi-GPU)
  bool slab = false;
  int64_t cap = 0;            // capacity of owned + ghost agents
  uint32_t* dp_ids = nullptr;  // ids in the order of dp (slab mode)
  int64_t n_dp = 0;
  uint32_t* cnt = nullptr;     // pack counters (device)
  uint32_t* cnt_host = nullptr;
  // cell growth and division (NEXT-2): dynamic population up to cap agents
  bool growth_on = false;
  double growth = 0.0, div_diam = 0.0;
  uint64_t gseed = 0;
  uint64_t step_count = 0;   // mechanics steps since init / set_agents (division hash)
  uint32_t* gflag = nullptr;  // id-indexed division flags -> ranks (cap + 1)
  // soma clustering (NEXT-3): two substance fields on a lattice, agent types by id
  bool fields_on = false;
  FieldDev fd{};
  double* field[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};  // [substance][buffer]
  int fcur = 0;
  uint32_t* fcnt = nullptr;  // 2 x nn secretion counts
  int8_t* type_by_id = nullptr;
  // neurite elements (NEXT-4): by element id; element grid in a sub-handle over element centres
  int64_t n_el = 0;
  double4* eq[2] = {nullptr, nullptr};  // distal point + diameter (Jacobi double buffer)
  double4* ea = nullptr;                // anchor + resting length
  int4* et = nullptr;                   // mother, daughter1, daughter2
  double* edq = nullptr;                // distal displacements of the last step
  double* cpos = nullptr;               // element centres (3E) and extents len + d (E)
  ElGeo* geo = nullptr;                 // element geometry of the current step (E)
  double* cdiam = nullptr;
  double* fss = nullptr;                // sphere-sphere forces of the force-only pass (3 cap)
  uint32_t* scnt = nullptr;             // sphere-element contact rows (neurites): counts ...
  uint32_t* srow = nullptr;             // ... and SCAP element sorted indices per sphere
  size_t sc_cap = 0;
  int eqc = 0;
  double k_spring = 0.0;
  double sphere_L = 0.0;  // O1 box edge of the spheres alone
  bdm_ctx* el = nullptr;
  // stationary-region skip (BDM_SKIP_STATIONARY, NEXT-1)
  unsigned long long* hist[2] = {nullptr, nullptr};
  uint8_t* hot = nullptr;  // one hot flag per box-table entry
  size_t hot_cap = 0;
  bool skip_valid = false;   // hist describes the last step
  bool skip_active = false;  // the pending force kernel uses hot flags
  uint32_t last_moved = 0, last_searched = 0;
  bool timing = false;
  // half-shell force path (k_half_search + k_half_sum): pair rows, sized to cap
  uint32_t *h_fwd = nullptr, *h_bwd = nullptr, *h_bcnt = nullptr;
  uint32_t* h_slow = nullptr;  // sum pass: agents whose pair rows overflowed (k_half_slow)
  uint8_t* h_fcnt = nullptr;
  int64_t h_cap = 0;
  bool half_off = false;  // the rows could not be allocated: k_force only
  int force_path = BDM_PATH_AUTO;  // bdm_set_force_path
  bool last_half = false;  // the last step used the half-shell path
  bool split_pending = false;  // slab: bdm_slab_split ran, bdm_slab_commit not yet
  int64_t n_dead = 0;          // slab: committed emigrants still in ag[cur][0..n) (D < 0), dropped by the next sort
  int64_t fused_n0 = 0;        // slab: agents whose next columns the last step accumulated (ag[cur][0..fused_n0))
  uint32_t last_n_lo = 0;      // slab: lower ghosts of the last step (sorted first)
  int32_t split_xb = 0, split_xe = 0;
  int sm_count = 0, force_blocks_per_sm = 0, half_a_blocks_per_sm = 0, half_b_blocks_per_sm = 0, tile_blocks_per_sm = 0;
  cudaStream_t s2 = nullptr;          // banded force phase: the sum passes' stream
  cudaEvent_t bev[33] = {};           // ... and its events (search of band k done; all sums done)
  uint32_t* bwork = nullptr;          // ... chunk-ticket counters of every band's two passes
  int64_t launches = 0;  // kernels of this library launched by mech_step / grid_build (since bdm_get_timing)
  int64_t launches_total = 0;  // launches before the last bdm_get_timing reset
  int64_t host_syncs = 0;      // host synchronisations with the device (bdm_get_stats)
  uint64_t steps_total = 0;    // mechanical steps since init
  DistGroup* dist = nullptr;   // distributed handle (bdm_init_dist): the local slabs, communicator
  std::vector<TimedStep> timed;
  std::string error;
};

namespace {

void dist_destroy(DistGroup* G);
int dist_mech_step(bdm_ctx* H, int32_t n_steps);
void dist_set_timing(DistGroup* G, bool on);
int dist_sync(bdm_ctx* H);
int dist_get_timing(bdm_ctx* H, double* out6);

int fail(bdm_ctx* h, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (h)
    h->error = buf;
  g_tls_error = buf;
  return code;
}

#define CU(h, call)                                                                           \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess) {                                                                  \
      (void)cudaGetLastError();                                                               \
      return fail((h), e_ == cudaErrorMemoryAllocation ? BDM_ENOMEM : BDM_ECUDA, "%s: %s (%s:%d)", \
                  #call, cudaGetErrorString(e_), __FILE__, __LINE__);                         \
    }                                                                                         \
  } while (0)

// BDM_DEBUG=1: synchronise after a launch and name the kernel that failed.
#define DBG(h, name)                                                                                   \
  do {                                                                                                 \
    if (g_debug) {                                                                                     \
      cudaError_t e_ = cudaStreamSynchronize((h)->stream);                                             \
      if (e_ == cudaSuccess) e_ = cudaGetLastError();                                                  \
      if (e_ != cudaSuccess)                                                                           \
        return fail((h), BDM_ECUDA, "%s (n=%lld cap=%lld step=%llu): %s", name, (long long)(h)->n,     \
                    (long long)(h)->cap, (unsigned long long)(h)->step_count, cudaGetErrorString(e_)); \
    }                                                                                                  \
  } while (0)

template <typename T>
int dalloc(bdm_ctx* h, T** p, size_t count) {
  if (count == 0) count = 1;
  CU(h, cudaMalloc(reinterpret_cast<void**>(p), count * sizeof(T)));
  return BDM_OK;
}

unsigned blocks(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

// Launch of a kernel of the step's chain with programmatic stream serialisation (PDL): it may be
// scheduled while its predecessor drains and waits in pdl_wait() (bdm_kernels.cuh) for that grid's
// completion.  Only kernels that call pdl_wait() before any memory access go through here.
template <typename... KArgs, typename... Args>
cudaError_t lx(void (*k)(KArgs...), unsigned grid, unsigned block, size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

bool params_ok(const bdm_params* p) {
  auto fin = [](double v) { return std::isfinite(v); };
  return p && p->eta > 0.0 && p->max_disp > 0.0 && fin(p->eta) && fin(p->max_disp) && p->k_rep >= 0.0 &&
         fin(p->k_rep) && p->gamma_att >= 0.0 && fin(p->gamma_att) && p->adherence >= 0.0 && fin(p->adherence) &&
         p->dt >= 0.0 && fin(p->dt) && p->box_edge_min >= 0.0 && fin(p->box_edge_min);
}

ParamsDev params_dev(const bdm_params& p) {
  ParamsDev d;
  d.k_rep = p.k_rep;
  d.gamma_att = p.gamma_att;
  d.adherence = p.adherence;
  d.c = p.dt / p.eta;
  d.max_disp = p.max_disp;
  return d;
}

// Collect asynchronous device errors (after a stream sync).
int check_async(bdm_ctx* h) {
  CU(h, cudaMemcpyAsync(h->err_host, h->err, sizeof(ErrDev), cudaMemcpyDeviceToHost, h->stream));
  CU(h, cudaStreamSynchronize(h->stream));
  ++h->host_syncs;
  if (h->err_host->code) {
    h->poisoned = true;
    const uint32_t first = (uint32_t)(h->err_host->bad >> 32);
    if (h->err_host->code == 1u)
      return fail(h, BDM_EINVAL, "invalid agent %u: diameter must be > 0 and finite, positions finite", first);
    if (h->err_host->code == 6u) {  // the offending pair (partner located by k_locate_nonfinite)
      const uint32_t j = h->err_host->second;
      if (j < 0xfffffffeu)
        return fail(h, BDM_ENONFINITE, "non-finite force or displacement on agent %u from its pair (%u, %u)", first,
                    first, j);
      return fail(h, BDM_ENONFINITE, "non-finite force or displacement on agent %u", first);
    }
    if (h->err_host->code == 7u)
      return fail(h, BDM_ERANGE, "agent at input position %u left the grid of a deferred build", first);
    return fail(h, BDM_ECUDA, "device error code %u", h->err_host->code);
  }
  return BDM_OK;
}

int ensure_table(bdm_ctx* h, size_t entries, size_t min_scan_items) {
  if (entries > h->table_cap) {
    if (h->table) CU(h, cudaFree(h->table));
    h->table = nullptr;
    if (h->table2) CU(h, cudaFree(h->table2));  // (reallocated on demand with the new capacity)
    h->table2 = nullptr;
    h->table_pre = false;
    size_t cap = entries + entries / 4 + (1u << 20);  // generous: no reallocation as extents drift
    CU(h, cudaMalloc(&h->table, cap * sizeof(uint32_t)));
    h->table_cap = cap;
  }
  size_t tiles = (std::max(entries, min_scan_items) + SCAN_TILE - 1) / SCAN_TILE;
  if (tiles > h->scan_tiles_cap) {
    if (h->scan_state) CU(h, cudaFree(h->scan_state));
    h->scan_state = nullptr;
    size_t cap = tiles + tiles / 4 + 256;
    CU(h, cudaMalloc(&h->scan_state, cap * sizeof(unsigned long long)));
    h->scan_tiles_cap = cap;
  }
  return BDM_OK;
}

// Column arrays for `entries` columns: z-range pair czlo/czhi (second: the next build's pair
// czlo2/czhi2, filled by the fused column pass) and the offsets coff (own capacity: the pairs swap).
int ensure_columns(bdm_ctx* h, size_t entries, bool second = false) {
  int32_t** lo = second ? &h->czlo2 : &h->czlo;
  int32_t** hi = second ? &h->czhi2 : &h->czhi;
  size_t* capp = second ? &h->col2_cap : &h->col_cap;
  const size_t cap = entries + entries / 4 + (1u << 16);
  if (entries > *capp) {
    for (void* p : {(void*)*lo, (void*)*hi})
      if (p) CU(h, cudaFree(p));
    *lo = *hi = nullptr;
    CU(h, cudaMalloc(lo, cap * sizeof(int32_t)));
    CU(h, cudaMalloc(hi, cap * sizeof(int32_t)));
    *capp = cap;
  }
  if (!second && entries > h->coff_cap) {
    if (h->coff) CU(h, cudaFree(h->coff));
    if (h->colrec) CU(h, cudaFree(h->colrec));
    h->coff = nullptr;
    h->colrec = nullptr;
    CU(h, cudaMalloc(&h->coff, cap * sizeof(uint32_t)));
    CU(h, cudaMalloc(&h->colrec, cap * sizeof(int4)));
    h->coff_cap = cap;
  }
  return BDM_OK;
}

void init_device_info(bdm_ctx* h) {
  if (h->sm_count) return;
  cudaDeviceGetAttribute(&h->sm_count, cudaDevAttrMultiProcessorCount, h->device);
  cudaFuncSetAttribute(k_force<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FORCE_SMEM_BYTES);
  cudaFuncSetAttribute(k_force<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FORCE_SMEM_BYTES);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_force<false>, FORCE_THREADS, FORCE_SMEM_BYTES);
  h->force_blocks_per_sm = per_sm > 0 ? per_sm : 1;
  per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_scan, SCAN_THREADS, 0);
  h->scan_blocks_per_sm = per_sm > 0 ? per_sm : 1;
  cudaFuncSetAttribute(k_half_search, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)HA_SMEM_BYTES);
  cudaFuncSetAttribute(k_half_sum<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)HB_SMEM_BYTES);
  cudaFuncSetAttribute(k_half_sum<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)HB_SMEM_BYTES);
  cudaFuncSetAttribute(k_half_sum<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)HB_SMEM_BYTES);
#ifndef BDM_NO_CARVEOUT
  {  // shared memory only as large as the resident blocks need: the rest stays L1 for the gathers
    int smem_sm = 0;
    cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, h->device);
    auto pct = [&](size_t per_block, int blocks_per_sm) {
      const double need = (double)blocks_per_sm * (per_block + 1024);
      return smem_sm > 0 ? std::min(100, (int)std::ceil(100.0 * need / smem_sm) + 1) : -1;
    };
    cudaFuncSetAttribute(k_half_search, cudaFuncAttributePreferredSharedMemoryCarveout, pct(HA_SMEM_BYTES, HA_MIN_BLOCKS));
    cudaFuncSetAttribute(k_half_sum<false>, cudaFuncAttributePreferredSharedMemoryCarveout, pct(HB_SMEM_BYTES, HB_MIN_BLOCKS));
    cudaFuncSetAttribute(k_half_sum<true>, cudaFuncAttributePreferredSharedMemoryCarveout, pct(HB_SMEM_BYTES, HB_MIN_BLOCKS));
    cudaFuncSetAttribute(k_half_sum<false, true>, cudaFuncAttributePreferredSharedMemoryCarveout,
                         pct(HB_SMEM_BYTES, HB_MIN_BLOCKS));
    (void)cudaGetLastError();
  }
#endif
  per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_half_search, HA_THREADS, HA_SMEM_BYTES);
  h->half_a_blocks_per_sm = per_sm > 0 ? per_sm : 1;
  cudaFuncSetAttribute(k_half_search_tile, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TILE_SMEM_BYTES);
  cudaFuncSetAttribute(k_half_search_tile, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_half_search_tile, TILE_THREADS, TILE_SMEM_BYTES);
  h->tile_blocks_per_sm = per_sm > 0 ? per_sm : 1;
  (void)cudaGetLastError();
  per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_half_sum<false>, FORCE_THREADS, HB_SMEM_BYTES);
  h->half_b_blocks_per_sm = per_sm > 0 ? per_sm : 1;
}

// Pair rows of the half-shell path for cap agents (one merged row of 16 u32 + counter + slow-list
// slot: 72 B/agent; 133 B/agent with separate rows, BDM_MROW=0).  An
// allocation failure is not an error: the handle falls back to k_force (no rows needed).
bool ensure_half(bdm_ctx* h) {
  if (h->half_off || h->force_path == BDM_PATH_SINGLE) return false;
  if (h->h_cap >= h->cap && h->h_fwd) return true;
  for (void* q : {(void*)h->h_fwd, (void*)h->h_bwd, (void*)h->h_bcnt, (void*)h->h_fcnt, (void*)h->h_slow})
    if (q) cudaFree(q);
  h->h_fwd = h->h_bwd = h->h_bcnt = h->h_slow = nullptr;
  h->h_fcnt = nullptr;
  h->ring = 0;
  const size_t N = (size_t)std::max<int64_t>(h->cap, 1);
  const size_t Nsep = BDM_MROW ? 1 : N;  // (merged rows: no separate backward rows / forward counts)
  // the banded phase (single handle, merged rows): rows for a ring of R agents when all N rows do not
  // fit beside the state (or BDM_RING asks for it); the overflow list keeps one entry per agent
  size_t free_b = 0, total_b = 0;
  (void)cudaMemGetInfo(&free_b, &total_b);
  const bool want_ring = BDM_MROW && !h->slab && !g_htile &&
                         (g_ring_log > 0 || N * (HFC * 4 + 8) + (size_t)(4ull << 30) > free_b);
  if (want_ring) {
    const size_t R = (size_t)1 << (g_ring_log > 0 ? std::min(g_ring_log, 30) : 25);
    if (cudaMalloc(&h->h_fwd, R * HFC * sizeof(uint32_t)) == cudaSuccess &&
        cudaMalloc(&h->h_bwd, sizeof(uint32_t) * HBC) == cudaSuccess &&
        cudaMalloc(&h->h_bcnt, R * sizeof(uint32_t)) == cudaSuccess && cudaMalloc(&h->h_fcnt, 1) == cudaSuccess &&
        cudaMalloc(&h->h_slow, N * sizeof(uint32_t)) == cudaSuccess) {
      h->ring = (uint32_t)R;
      h->h_cap = h->cap;
      return true;
    }
    (void)cudaGetLastError();
    for (void* q : {(void*)h->h_fwd, (void*)h->h_bwd, (void*)h->h_bcnt, (void*)h->h_fcnt, (void*)h->h_slow})
      if (q) cudaFree(q);
    h->h_fwd = h->h_bwd = h->h_bcnt = h->h_slow = nullptr;
    h->h_fcnt = nullptr;
    h->half_off = true;
    return false;
  }
  if (cudaMalloc(&h->h_fwd, N * HFC * sizeof(uint32_t)) != cudaSuccess ||
      cudaMalloc(&h->h_bwd, Nsep * HBC * sizeof(uint32_t)) != cudaSuccess ||
      cudaMalloc(&h->h_bcnt, N * sizeof(uint32_t)) != cudaSuccess || cudaMalloc(&h->h_fcnt, Nsep) != cudaSuccess ||
      cudaMalloc(&h->h_slow, N * sizeof(uint32_t)) != cudaSuccess) {
    (void)cudaGetLastError();
    for (void* q : {(void*)h->h_fwd, (void*)h->h_bwd, (void*)h->h_bcnt, (void*)h->h_fcnt, (void*)h->h_slow})
      if (q) cudaFree(q);
    h->h_fwd = h->h_bwd = h->h_bcnt = h->h_slow = nullptr;
    h->h_fcnt = nullptr;
    h->half_off = true;
    return false;
  }
  h->h_cap = h->cap;
  return true;
}

// Banded phase: the band size for this grid -- half the ring, if that is no smaller than the largest
// sorted span of two consecutive box-x layers (an agent's forward partners lie before the end of the
// next layer, so the rows written while a band is searched belong to it or to the next band).
// One small device-to-host read per step.  0: the ring cannot hold this grid (the step takes k_force).
int ring_band(bdm_ctx* h, uint32_t n, uint32_t* band) {
  *band = 0;
  const GridDev& g = h->grid;
  const uint32_t nx = (uint32_t)(g.hi[0] - g.lo[0] + 1);
  if ((size_t)nx + 1 > h->lstart_cap) {
    if (h->lstart) CU(h, cudaFree(h->lstart));
    if (h->lstart_host) CU(h, cudaFreeHost(h->lstart_host));
    h->lstart = nullptr;
    h->lstart_host = nullptr;
    h->lstart_cap = (size_t)nx + 1 + 1024;
    CU(h, cudaMalloc(&h->lstart, h->lstart_cap * sizeof(uint32_t)));
    CU(h, cudaMallocHost(&h->lstart_host, h->lstart_cap * sizeof(uint32_t)));
  }
  k_layer_starts<<<std::max(1u, std::min(148u * 4u, (nx + 256u) / 256u)), 256, 0, h->stream>>>(g, nx, n, h->lstart);
  CU(h, cudaMemcpyAsync(h->lstart_host, h->lstart, ((size_t)nx + 1) * sizeof(uint32_t), cudaMemcpyDeviceToHost,
                        h->stream));
  CU(h, cudaStreamSynchronize(h->stream));
  ++h->host_syncs;
  uint32_t span = 0;
  for (uint32_t x = 0; x < nx; ++x) span = std::max(span, h->lstart_host[std::min(x + 2, nx)] - h->lstart_host[x]);
  // the largest band the ring holds (fewer launches and persistent-grid tails), if it covers the span
  const uint32_t b = h->ring / 2;
  if (b >= span && b >= 32u) *band = b;
  return BDM_OK;
}

// Half-shell force step over the owned sorted range [a_begin, a_end) of ag[src]; pass A searches
// from s_begin (slab mode: the lower ghost layer searches too, its pairs with owned agents are
// forward pairs of the ghost).
// frame4 (x lo, y lo, nx, ny) of the fused column pass; nullptr: this step's tight extents +- 1 box.
int half_force(bdm_ctx* h, int src, uint32_t s_begin, uint32_t a_begin, uint32_t a_end, uint32_t n_all,
               const ParamsDev& pd, double4* ag_out, uint32_t* id_out, double* dp, uint32_t* dp_ids,
               bool fuse_cols = false, const int32_t* frame4 = nullptr, unsigned long long* hist_out = nullptr,
               double* force_only = nullptr, int ext_mode = -1) {
  cudaStream_t s = h->stream;
  ColNext cn{0, 0, 0, 0, nullptr, nullptr, nullptr, 0, 0};
  size_t nc2 = 0;
  h->cols_next = false;
  if (fuse_cols) {  // next build's frame: this step's tight extents +- 1 box (|dp| < L)
    cn.lo0 = frame4 ? frame4[0] : h->tlo[0] - 1;
    cn.lo1 = frame4 ? frame4[1] : h->tlo[1] - 1;
    cn.nx = frame4 ? frame4[2] : h->thi[0] - h->tlo[0] + 3;
    cn.ny = frame4 ? frame4[3] : h->thi[1] - h->tlo[1] + 3;
    nc2 = (size_t)cn.nx * (size_t)cn.ny;
    int rc = ensure_columns(h, nc2 + 1, true);
    if (rc) return rc;
    cn.czlo = h->czlo2;
    cn.czhi = h->czhi2;
    h->nlo[0] = cn.lo0;
    h->nlo[1] = cn.lo1;
    h->nnx = cn.nx;
    h->nny = cn.ny;
    // single handle: the new boxes packed as (frame column << zbits | z - z0), z in this grid's
    // z-range +- 1 box, when that fits 32 bits
    h->pbox_next = false;
    if (!frame4 && !h->slab && g_pbox) {
      const int32_t z0 = h->grid.lo[2] - 1, zspan = h->grid.hi[2] - h->grid.lo[2] + 3;
      int zbits = 1;
      while ((1 << zbits) < zspan) ++zbits;
      if (zbits < 31 && (uint64_t)nc2 <= (0xffffffffull >> zbits)) {
        if ((size_t)a_end > h->pbox_cap) {
          if (h->pbox) CU(h, cudaFree(h->pbox));
          h->pbox = nullptr;
          h->pbox_cap = (size_t)a_end + a_end / 4 + 1024;
          CU(h, cudaMalloc(&h->pbox, h->pbox_cap * sizeof(uint32_t)));
        }
        cn.pbox = h->pbox;
        cn.z0 = z0;
        cn.zbits = zbits;
        h->pbox_next = true;
        h->pb_z0 = z0;
        h->pb_zbits = zbits;
      }
    }
  }
  // the next build's histogram buffer, zeroed on a side stream during this force phase (the current
  // table is in use until its end): k_table_zero_tma, joined before half_force returns
  bool tz = false;
  if (fuse_cols && !frame4 && !h->slab && g_tzero && !force_only && h->table_cap >= 8) {
    if (!h->table2) CU(h, cudaMalloc(&h->table2, h->table_cap * sizeof(uint32_t)));
    if (!h->s2) {
      CU(h, cudaStreamCreateWithFlags(&h->s2, cudaStreamNonBlocking));
      for (int k = 0; k < 33; ++k) CU(h, cudaEventCreateWithFlags(&h->bev[k], cudaEventDisableTiming));
      CU(h, cudaMalloc(&h->bwork, 64 * sizeof(uint32_t)));
    }
    tz = true;
  }
  auto fork_zero = [&]() -> int {
    CU(h, cudaEventRecord(h->bev[31], s));
    CU(h, cudaStreamWaitEvent(h->s2, h->bev[31], 0));
    k_table_zero_tma<<<h->sm_count, 32, 0, h->s2>>>(h->table2, h->coff, h->grid.n_cols,
                                                    (uint32_t)std::min<size_t>((h->table_cap - 4) & ~(size_t)3, 0xfffffff0u),
                                                    &h->ext->zeroed);
    CU(h, cudaEventRecord(h->bev[32], h->s2));
    h->launches += 1;
    return BDM_OK;
  };
  if (tz) {  // (overlapping the search: during the latency-bound sum pass it cost 0.12 ms)
    int rc = fork_zero();
    if (rc) return rc;
  }
  {  // one launch: the extents reset (ext_mode >= 0), the next build's column ranges, the pair counters
    const uint64_t w = std::max<uint64_t>(nc2, (uint64_t)n_all / 4 + 1);
    const unsigned gr = (unsigned)std::min<uint64_t>((w + 255) / 256, 148u * 16u);
    CU(h, lx(k_force_reset, gr, 256, 0, s, h->ext, ext_mode, fuse_cols ? h->czlo2 : nullptr, h->czhi2, (uint32_t)nc2,
             h->h_bcnt, h->ring ? h->ring : std::max<uint32_t>(n_all, 1)));
    h->launches += 1;
  }
  // banded force phase: bands of >= 2^20 agents each
  const int nb = force_only || h->ring ? 1 : (int)std::min<int64_t>(g_bands, std::max<int64_t>(1, ((int64_t)a_end - a_begin) >> 20));
  if (nb > 1) {
    if (tz) CU(h, cudaStreamWaitEvent(s, h->bev[32], 0));  // (the bands reuse the side stream's events)
    tz = false;
    if (!h->s2) {
      CU(h, cudaStreamCreateWithFlags(&h->s2, cudaStreamNonBlocking));
      for (int k = 0; k < 33; ++k) CU(h, cudaEventCreateWithFlags(&h->bev[k], cudaEventDisableTiming));
      CU(h, cudaMalloc(&h->bwork, 64 * sizeof(uint32_t)));
    }
    CU(h, cudaMemsetAsync(h->bwork, 0, 64 * sizeof(uint32_t), s));
    const uint32_t bs = (uint32_t)(((((uint64_t)a_end - a_begin) / nb) + 31) / 32 * 32);
    auto cut = [&](int k) { return k == 0 ? a_begin : (k >= nb ? a_end : std::min<uint32_t>(a_end, a_begin + (uint32_t)k * bs)); };
    for (int k = 0; k < nb; ++k) {
      const uint32_t sb = k == 0 ? s_begin : cut(k), se = cut(k + 1);
      const unsigned ga = (unsigned)std::min<uint64_t>((uint64_t)h->sm_count * h->half_a_blocks_per_sm,
                                                       std::max<uint64_t>(1, (se - sb + HA_THREADS - 1) / HA_THREADS));
      k_half_search<<<ga, HA_THREADS, HA_SMEM_BYTES, s>>>(h->ag[src], h->agf, sb, se, h->grid, h->h_fwd, h->h_fcnt,
                                                           h->h_bwd, h->h_bcnt, h->ext, hist_out != nullptr && k == 0,
                                                           nullptr, h->bwork + k);
      CU(h, cudaEventRecord(h->bev[k], s));
    }
    if (h->timing && !h->timed.empty() && !h->timed.back().e3) {
      CU(h, cudaEventCreate(&h->timed.back().e3));
      CU(h, cudaEventRecord(h->timed.back().e3, s));
    }
    for (int k = 0; k < nb; ++k) {  // band k's rows are complete once the searches of bands 0..k are
      CU(h, cudaStreamWaitEvent(h->s2, h->bev[k], 0));
      const uint32_t ab = cut(k), ae = cut(k + 1);
      const unsigned gb = (unsigned)std::min<uint64_t>((uint64_t)h->sm_count * h->half_b_blocks_per_sm,
                                                       std::max<uint64_t>(1, (ae - ab + FORCE_THREADS - 1) / FORCE_THREADS));
      k_half_sum<false><<<gb, FORCE_THREADS, HB_SMEM_BYTES, h->s2>>>(
          h->ag[src], h->id[src], ab, ae, h->grid, pd, ag_out, id_out, dp, dp_ids, h->ext, h->err, h->h_fwd, h->h_fcnt,
          h->h_bwd, h->h_bcnt, cn, hist_out, h->h_slow, nullptr, h->bwork + 32 + k, (int64_t)a_begin);
    }
    CU(h, cudaEventRecord(h->bev[nb], h->s2));
    CU(h, cudaStreamWaitEvent(s, h->bev[nb], 0));
    const unsigned gs = (unsigned)h->sm_count * 4;
    k_half_slow<false><<<gs, 128, 0, s>>>(h->ag[src], h->id[src], a_begin, h->grid, pd, ag_out, id_out, dp, dp_ids,
                                          h->ext, h->err, cn, hist_out, h->h_slow);
    k_locate_nonfinite<<<1, 32, 0, s>>>(h->ag[src], h->id[src], h->grid, pd, h->err);
    CU(h, cudaGetLastError());
    h->launches += 2 * nb + 2;
    h->cols_next = fuse_cols;
    return BDM_OK;
  }
  if (h->ring) {  // banded phase over a ring of pair rows (populations whose rows do not fit)
    const uint32_t B = h->ring_band;
    if (!B || force_only || frame4 || h->slab || s_begin != a_begin) return fail(h, BDM_ESTATE, "ring phase misuse");
    const uint32_t nbands = (a_end - a_begin + B - 1) / B;
    if (2 * (size_t)nbands > h->rwork_cap) {
      if (h->rwork) CU(h, cudaFree(h->rwork));
      h->rwork = nullptr;
      h->rwork_cap = 2 * (size_t)nbands + 64;
      CU(h, cudaMalloc(&h->rwork, h->rwork_cap * sizeof(uint32_t)));
    }
    CU(h, cudaMemsetAsync(h->rwork, 0, 2 * (size_t)nbands * sizeof(uint32_t), s));
    GridDev gr = h->grid;
    gr.rmask = 2u * B - 1u;
    for (uint32_t k = 0; k < nbands; ++k) {
      const uint32_t lo = a_begin + k * B, hi = std::min<uint32_t>(a_end, lo + B);
      const unsigned ga = (unsigned)std::min<uint64_t>((uint64_t)h->sm_count * h->half_a_blocks_per_sm,
                                                       std::max<uint64_t>(1, (hi - lo + HA_THREADS - 1) / HA_THREADS));
      CU(h, lx(k_half_search, ga, HA_THREADS, HA_SMEM_BYTES, s, h->ag[src], h->agf, lo, hi, gr, h->h_fwd, h->h_fcnt,
               h->h_bwd, h->h_bcnt, h->ext, hist_out != nullptr, nullptr, h->rwork + 2 * k));
      const unsigned gb = (unsigned)std::min<uint64_t>((uint64_t)h->sm_count * h->half_b_blocks_per_sm,
                                                       std::max<uint64_t>(1, (hi - lo + FORCE_THREADS - 1) / FORCE_THREADS));
      CU(h, lx(k_half_sum<false, true>, gb, FORCE_THREADS, HB_SMEM_BYTES, s, h->ag[src], h->id[src], lo, hi, gr, pd,
               ag_out, id_out, dp, dp_ids, h->ext, h->err, h->h_fwd, h->h_fcnt, h->h_bwd, h->h_bcnt, cn, hist_out,
               h->h_slow, nullptr, h->rwork + 2 * k + 1, (int64_t)a_begin));
      if (k + 2 < nbands) {  // band k's ring slot is band k+2's: its counts zeroed before search k+1 writes there
        const unsigned gz = (unsigned)std::min<uint64_t>((B / 4 + 255) / 256, 148u * 16u);
        CU(h, lx(k_force_reset, gz, 256, 0, s, h->ext, -1, (int32_t*)nullptr, (int32_t*)nullptr, 0u,
                 h->h_bcnt + (size_t)(k & 1u) * B, B));
      }
    }
    h->launches += 3 * nbands;
    const unsigned gs = (unsigned)h->sm_count * 4;
    CU(h, lx(k_half_slow<false>, gs, 128, 0, s, h->ag[src], h->id[src], a_begin, h->grid, pd, ag_out, id_out, dp,
             dp_ids, h->ext, h->err, cn, hist_out, h->h_slow, nullptr));
    CU(h, lx(k_locate_nonfinite, 1, 32, 0, s, h->ag[src], h->id[src], h->grid, pd, h->err));
    if (tz) {
      CU(h, cudaStreamWaitEvent(s, h->bev[32], 0));
      h->table_pre = true;
    }
    CU(h, cudaGetLastError());
    h->launches += 2;
    h->cols_next = fuse_cols;
    return BDM_OK;
  }
  if (g_htile) {  // staged neighbourhood
    const unsigned gt = (unsigned)std::min<uint64_t>((uint64_t)h->sm_count * h->tile_blocks_per_sm,
                                                     std::max<uint64_t>(1, (a_end - s_begin + TILE_AG - 1) / TILE_AG));
    k_half_search_tile<<<gt, TILE_THREADS, TILE_SMEM_BYTES, s>>>(h->ag[src], h->agf, s_begin, a_end, h->grid, h->h_fwd,
                                                             h->h_fcnt, h->h_bwd, h->h_bcnt, h->ext,
                                                             hist_out != nullptr);
  } else {
    const unsigned ga = (unsigned)std::min<uint64_t>((uint64_t)h->sm_count * h->half_a_blocks_per_sm,
                                                     std::max<uint64_t>(1, (a_end - s_begin + HA_THREADS - 1) / HA_THREADS));
    CU(h, lx(k_half_search, ga, HA_THREADS, HA_SMEM_BYTES, s, h->ag[src], h->agf, s_begin, a_end, h->grid, h->h_fwd,
             h->h_fcnt, h->h_bwd, h->h_bcnt, h->ext, hist_out != nullptr, nullptr, nullptr));
  }
  DBG(h, "k_half_search");
  const unsigned gb = (unsigned)std::min<uint64_t>((uint64_t)h->sm_count * h->half_b_blocks_per_sm,
                                                   std::max<uint64_t>(1, (a_end - a_begin + FORCE_THREADS - 1) / FORCE_THREADS));
  if (h->timing && !h->timed.empty() && !h->timed.back().e3) {
    CU(h, cudaEventCreate(&h->timed.back().e3));
    CU(h, cudaEventRecord(h->timed.back().e3, s));
  }
  const unsigned gs = (unsigned)h->sm_count * 4;  // the overflow list is short: a small persistent grid
  if (force_only) {  // (sphere-sphere sums only: the neurite step adds the element terms, O6 and O7)
    k_half_sum<true><<<gb, FORCE_THREADS, HB_SMEM_BYTES, s>>>(h->ag[src], h->id[src], a_begin, a_end, h->grid, pd,
                                                               nullptr, nullptr, force_only, nullptr, h->ext, h->err,
                                                               h->h_fwd, h->h_fcnt, h->h_bwd, h->h_bcnt, cn, nullptr,
                                                               h->h_slow);
    k_half_slow<true><<<gs, 128, 0, s>>>(h->ag[src], h->id[src], a_begin, h->grid, pd, nullptr, nullptr, force_only,
                                         nullptr, h->ext, h->err, cn, nullptr, h->h_slow);
  } else {
    CU(h, lx(k_half_sum<false>, gb, FORCE_THREADS, HB_SMEM_BYTES, s, h->ag[src], h->id[src], a_begin, a_end, h->grid,
             pd, ag_out, id_out, dp, dp_ids, h->ext, h->err, h->h_fwd, h->h_fcnt, h->h_bwd, h->h_bcnt, cn, hist_out,
             h->h_slow, nullptr, nullptr, (int64_t)-1));
    CU(h, lx(k_half_slow<false>, gs, 128, 0, s, h->ag[src], h->id[src], a_begin, h->grid, pd, ag_out, id_out, dp,
             dp_ids, h->ext, h->err, cn, hist_out, h->h_slow, nullptr));
  }
  DBG(h, "k_half_slow");
  DBG(h, "k_half_sum");
  CU(h, lx(k_locate_nonfinite, 1, 32, 0, s, h->ag[src], h->id[src], h->grid, pd, h->err));
  if (tz) {  // join the side stream's zeroing
    CU(h, cudaStreamWaitEvent(s, h->bev[32], 0));
    h->table_pre = true;
  }
  CU(h, cudaGetLastError());
  h->launches += 4;
  h->cols_next = fuse_cols;
  return BDM_OK;
}

// In-place exclusive scan of data[0 .. items) -- items given on the host, or read on the device as
// *n_dev + 1 (persistent decoupled look-back, grid = resident capacity).
// Tile states for a host-sized scan of `items` (column offsets, division ranks may need more slots).
int scan_reserve(bdm_ctx* h, uint64_t items) {
  const size_t tiles = (items + SCAN_TILE - 1) / SCAN_TILE;
  if (tiles > h->scan_tiles_cap) {
    if (h->scan_state) CU(h, cudaFree(h->scan_state));
    h->scan_state = nullptr;
    const size_t cap = tiles + tiles / 4 + 256;
    CU(h, cudaMalloc(&h->scan_state, cap * sizeof(unsigned long long)));
    h->scan_tiles_cap = cap;
  }
  return BDM_OK;
}

// prezeroed: the tile states and the ticket were zeroed by the preceding kernel (k_col_len,
// k_table_zero), so the launch chain has no memset node.
int scan(bdm_ctx* h, uint32_t* data, uint64_t items, const uint32_t* n_dev, bool prezeroed = false) {
  init_device_info(h);
  if (items) {
    int rc = scan_reserve(h, items);
    if (rc) return rc;
  }
  size_t tiles_bound = h->scan_tiles_cap;
  uint64_t want = items ? (items + SCAN_TILE - 1) / SCAN_TILE : tiles_bound;
  if (!prezeroed) {
    CU(h, cudaMemsetAsync(h->scan_state, 0, std::min<uint64_t>(want, tiles_bound) * sizeof(unsigned long long),
                          h->stream));
    CU(h, cudaMemsetAsync(h->scan_ticket, 0, sizeof(uint32_t), h->stream));
  }
  const uint64_t cap = (uint64_t)h->sm_count * h->scan_blocks_per_sm;
  const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min(want, cap));
  CU(h, lx(k_scan, grid, SCAN_THREADS, 0, h->stream, data, n_dev, items, h->scan_state, h->scan_ticket));
  DBG(h, "k_scan");
  CU(h, cudaGetLastError());
  return BDM_OK;
}

// Grid parameters from the (already reduced) extents of ag[cur]; one small D2H per build.
int compute_extents(bdm_ctx* h) {
  uint32_t n = (uint32_t)h->n;
  GridDev& g = h->grid;
  // Deferred build (no host round trip): the last step fused this build's columns over its frame,
  // which holds every agent by construction (|dp| < L), so the grid is that frame in x/y and the
  // last grid's z-range +- 1 box, no tighter than needed for correctness.  Its flags (range,
  // frame) stay on the device and are checked at the next synchronised build: at least every
  // BDM_DEFER builds and for the last step of every bdm_mech_step call (whose grid info is tight).
  if (h->defer_ok && h->cols_next && h->deferred < h->defer_max && h->ext_valid && !h->slab && !h->hist[0] &&
      !(h->prm.flags & BDM_RECORD)) {
    g.lo[0] = h->tlo[0] = h->nlo[0];
    g.lo[1] = h->tlo[1] = h->nlo[1];
    g.hi[0] = h->thi[0] = h->nlo[0] + h->nnx - 1;
    g.hi[1] = h->thi[1] = h->nlo[1] + h->nny - 1;
    g.lo[2] = h->tlo[2] = g.lo[2] - 1;
    g.hi[2] = h->thi[2] = g.hi[2] + 1;
    int64_t nb = 1;
    for (int a = 0; a < 3; ++a) nb *= (int64_t)g.hi[a] - g.lo[a] + 1;
    if (nb < (int64_t)0xffffffffll && g.hi[2] < (1 << 20) && g.lo[2] > -(1 << 20)) {
      g.ny = g.hi[1] - g.lo[1] + 1;
      g.nz = g.hi[2] - g.lo[2] + 1;
      g.n_boxes = (uint32_t)nb;
      ++h->deferred;
      return BDM_OK;
    }
    h->cols_next = false;  // (frame grown too large: synchronise and start tight again)
  }
  h->deferred = 0;
  if (!h->ext_valid) {
    k_ext_reset<<<1, 32, 0, h->stream>>>(h->ext, 0);
    k_extents<<<blocks(n, 256), 256, 0, h->stream>>>(h->ag[h->cur], n, h->grid.inv, h->ext);
    DBG(h, "k_extents");
    CU(h, cudaGetLastError());
    h->launches += 2;
  }
  CU(h, cudaMemcpyAsync(h->ext_host, h->ext, sizeof(Extents), cudaMemcpyDeviceToHost, h->stream));
  int rc = check_async(h);  // synchronises
  if (rc) return rc;
  if (h->ext_host->range_err || (h->ext_host->sticky & 1u)) {
    h->poisoned = true;
    return fail(h, BDM_ERANGE, "an agent lies >= 2^20 boxes from the origin (|p*inv| >= 2^20, DESIGN.md R9)");
  }
  if (h->ext_host->sticky & 2u) {  // a deferred build's frame missed an agent: cannot happen (|dp| < L)
    h->poisoned = true;
    return fail(h, BDM_ERANGE, "an agent left the frame of a deferred build");
  }
  h->last_moved = h->ext_host->moved;
  h->last_searched = h->ext_host->searched;
  int64_t dims[3];
  for (int a = 0; a < 3; ++a) {
    g.lo[a] = h->tlo[a] = h->ext_host->lo[a];
    g.hi[a] = h->thi[a] = h->ext_host->hi[a];
  }
  // fused column pass of the last step: its frame (tight extents of that step's start +- 1 box)
  // becomes this grid's x/y frame; it contains every box by construction (|dp| < L), verified
  if (h->cols_next) {
    const bool inside = h->ext_host->col_bad == 0u && g.lo[0] >= h->nlo[0] && g.lo[1] >= h->nlo[1] &&
                        g.hi[0] < h->nlo[0] + h->nnx && g.hi[1] < h->nlo[1] + h->nny;
    if (inside) {
      g.lo[0] = h->nlo[0];
      g.lo[1] = h->nlo[1];
      g.hi[0] = h->nlo[0] + h->nnx - 1;
      g.hi[1] = h->nlo[1] + h->nny - 1;
    } else {
      h->cols_next = false;
    }
  }
  for (int a = 0; a < 3; ++a) dims[a] = (int64_t)g.hi[a] - g.lo[a] + 1;
  int64_t nb = dims[0] * dims[1] * dims[2];
  if (nb >= (int64_t)0xffffffffll) return fail(h, BDM_ERANGE, "n_boxes = %lld >= 2^32", (long long)nb);
  g.ny = (int32_t)dims[1];
  g.nz = (int32_t)dims[2];
  g.n_boxes = (uint32_t)nb;
  h->ext_valid = true;
  return BDM_OK;
}

// Counting sort of ag[cur][0..n) by (box key under h->grid, id) into ag[1-cur]:
//   column pass (occupied z-range per (bx, by) column) -> column offsets (scan) -> table zero ->
//   key + histogram -> table scan (box starts) -> scatter -> in-box id order + payload gather.
// The ragged table size T lives on the device (coff[nc]); no host round trip inside the build.
// cur flips to the sorted buffer.
// n input agents of ag[cur], of which n_dead are marked dead (slab emigrants, D < 0) and dropped.
int sort_into(bdm_ctx* h, uint32_t n, uint32_t n_dead = 0) {
  GridDev& g = h->grid;
  const uint64_t nc = (uint64_t)(g.hi[0] - g.lo[0] + 1) * (uint64_t)g.ny;
  if (nc >= 0xffffffffull) return fail(h, BDM_ERANGE, "%llu grid columns >= 2^32", (unsigned long long)nc);
  g.n_cols = (uint32_t)nc;
  int rc = ensure_columns(h, nc + 1);
  if (rc) return rc;
  rc = ensure_table(h, (size_t)g.n_boxes + 1, nc + 1);
  if (rc) return rc;
  g.czlo = h->czlo;
  g.czhi = h->czhi;
  g.coff = h->coff;
  g.table = h->table;
  g.col = h->colrec;
  {  // fp32 prefilter margin from the largest coordinate magnitude of this grid
    double P = 0.0;
    for (int a = 0; a < 3; ++a)
      P = std::max(P, std::max(std::fabs((double)g.lo[a]), std::fabs((double)g.hi[a] + 1.0)) * g.L * (1.0 + 0x1p-20));
    const double ulp32 = P > 0.0 ? std::ldexp(1.0, std::ilogb(P) - 23) : 0x1p-149;
    g.m32 = 2.0 * ulp32 + 0x1p-18 + g.L * 0x1p-20;
  }
  cudaStream_t s = h->stream;
  const int src = h->cur, dst = 1 - h->cur;
  init_device_info(h);
  const unsigned gs = (unsigned)std::min<uint64_t>((nc + 256) / 256, 148u * 16u);
  const bool packed = h->cols_next && h->pbox_next && n_dead == 0;
  h->pbox_next = false;
  if (h->cols_next) {  // z-ranges already accumulated by the last step's sum pass
    std::swap(h->czlo, h->czlo2);
    std::swap(h->czhi, h->czhi2);
    std::swap(h->col_cap, h->col2_cap);
    h->cols_next = false;
    rc = ensure_columns(h, nc + 1);  // no-op for the swapped pair (sized for this frame by force_step)
    if (rc) return rc;
    g.czlo = h->czlo;
    g.czhi = h->czhi;
    g.coff = h->coff;
  } else {
    CU(h, lx(k_col_reset, gs, 256, 0, s, h->czlo, h->czhi, g.n_cols));
    DBG(h, "k_col_reset");
    if (n > 0) CU(h, lx(k_col_ext, blocks(n, 512), 256, 0, s, h->ag[src], n, g, h->czlo, h->czhi, nullptr));
    DBG(h, "k_col_ext");
    h->launches += n > 0 ? 2 : 1;
  }
  // the histogram buffer the last sum pass zeroed (ensure_table above cleared the flag if it had to
  // reallocate); k_table_zero then zeroes only what lies beyond ext->zeroed
  const bool pre = h->table_pre && h->table2;
  if (pre) {
    std::swap(h->table, h->table2);
    g.table = h->table;
    h->table_pre = false;
  }
  // (k_col_len zeroes the offset scan's tile states, k_table_zero the table scan's)
  rc = scan_reserve(h, nc + 1);
  if (rc) return rc;
  CU(h, lx(k_col_len, gs, 256, 0, s, h->czlo, h->czhi, g.n_cols, h->coff, h->scan_state,
           (uint32_t)((nc + 1 + SCAN_TILE - 1) / SCAN_TILE), h->scan_ticket));
  DBG(h, "k_col_len");
  rc = scan(h, h->coff, nc + 1, nullptr, true);  // exclusive: coff[c] = table offset, coff[nc] = T
  if (rc) return rc;
  CU(h, lx(k_table_zero, h->sm_count * 8, 256, 0, s, h->table, h->coff, g.n_cols, h->czlo, h->czhi, h->colrec,
           h->scan_state, (uint32_t)h->scan_tiles_cap, h->scan_ticket, pre ? &h->ext->zeroed : nullptr));
  DBG(h, "k_table_zero");
  if (n > 0 && packed) {  // boxes from the last sum pass (4 B/agent instead of the state)
    CU(h, lx(h->deferred > 0 ? k_key_hist_packed<true> : k_key_hist_packed<false>, blocks(n, 256 * KHP), 256, 0, s,
             h->pbox, n, g, h->pb_z0, h->pb_zbits, h->key, h->slot, h->table, h->err, nullptr));
  } else if (n > 0) {
    CU(h, lx(h->deferred > 0 ? k_key_hist<true> : k_key_hist<false>, blocks(n, 512), 256, 0, s, h->ag[src], n, g,
             h->key, h->slot, h->table, h->err, nullptr, nullptr));
  }
  DBG(h, "k_key_hist");
  rc = scan(h, h->table, 0, h->coff + nc, true);  // T + 1 items: table[k] = first agent of box k, table[T] = n
  if (rc) return rc;
  if (n > 0) {
    CU(h, lx(k_scatter, blocks(n, 256 * KSC), 256, 0, s, h->key, h->slot, h->id[src], h->table, n, h->tsrc, h->tid,
             h->tkey, nullptr));
    DBG(h, "k_scatter");
    const bool perm_hist = h->hist[0] && h->skip_valid && !h->slab;
    CU(h, lx(k_place, blocks(n - n_dead, PLACE_T), PLACE_T, 0, s, h->tsrc, h->tid, h->tkey, h->table, h->ag[src],
             n - n_dead, h->ag[dst], h->id[dst], h->agf, perm_hist ? h->hist[src] : nullptr,
             perm_hist ? h->hist[dst] : nullptr, nullptr, nullptr, nullptr));
    DBG(h, "k_place");
  }
  CU(h, cudaGetLastError());
  h->launches += n > 0 ? 7 : 4;
  h->cur = dst;
  return BDM_OK;
}

int grid_build(bdm_ctx* h) {
  if (h->poisoned) return fail(h, BDM_ESTATE, "handle poisoned by an earlier error: %s", h->error.c_str());
  if (h->state == State::Fresh) return BDM_OK;  // positions unchanged since the last build
  if (h->n == 0) {
    h->state = State::Fresh;
    h->have_grid = true;
    return BDM_OK;
  }
  int rc = compute_extents(h);
  if (rc) return rc;
  rc = sort_into(h, (uint32_t)h->n);
  if (rc) return rc;
  // NEXT-1: mark agents near a moving agent; skip only while few agents move (else it costs more
  // than it saves) and never in RECORD mode (statistics count every candidate)
  h->skip_active = false;
  if (h->hist[0] && h->skip_valid && !(h->prm.flags & BDM_RECORD) && (uint64_t)h->last_moved * 2 <= (uint64_t)h->n) {
    if (h->hot_cap < h->table_cap + 4) {  // one flag byte per box-table entry
      if (h->hot) CU(h, cudaFree(h->hot));
      h->hot = nullptr;
      CU(h, cudaMalloc(&h->hot, h->table_cap + 4));
      h->hot_cap = h->table_cap + 4;
    }
    k_flag_zero<<<h->sm_count * 4, 256, 0, h->stream>>>(h->hot, h->coff, h->grid.n_cols);
    k_mark_hot<<<blocks(h->n, 256), 256, 0, h->stream>>>(h->ag[h->cur], h->hist[h->cur], (uint32_t)h->n, h->grid,
                                                         h->hot);
    DBG(h, "k_mark_hot");
    CU(h, cudaGetLastError());
    h->launches += 2;
    h->skip_active = true;
  }
  h->state = State::Fresh;
  h->have_grid = true;
  return BDM_OK;
}

// Persistent grid: resident blocks per SM x SMs, no more than the work needs.
unsigned force_grid(bdm_ctx* h, uint32_t n) {
  init_device_info(h);
  unsigned want = (n + FORCE_THREADS - 1) / FORCE_THREADS;
  unsigned cap = (unsigned)(h->sm_count * h->force_blocks_per_sm);
  return want < cap ? (want ? want : 1) : cap;
}

int force_step(bdm_ctx* h, bool want_dp) {
  const uint32_t n = (uint32_t)h->n;
  cudaStream_t s = h->stream;
  const int src = h->cur, dst = 1 - h->cur;
  const int ext_mode = h->deferred > 0 ? 2 : 1;
  RecordDev rec{h->r_cand, h->r_nb, h->r_ct, h->r_branch, h->r_nbh, h->r_cth};
  ParamsDev pd = params_dev(h->prm);
  double* dp = want_dp ? h->dp : nullptr;
  const unsigned grid = force_grid(h, n);
  // the single-pass k_force serves the stationary-region skip (it skips the whole search of quiet
  // agents); otherwise the half-shell path, which also keeps the skip statistics (hist) current
  h->last_half = !(h->prm.flags & BDM_RECORD) && !h->skip_active && n > 0 && ensure_half(h);
  h->ring_band = 0;
  if (h->last_half && h->ring) {  // banded phase: the bands must hold two layers' span
    int rc = ring_band(h, n, &h->ring_band);
    if (rc) return rc;
    if (!h->ring_band) h->last_half = false;
  }
  h->cols_next = false;
  if (h->last_half) {
    // fuse the next build's column pass when nothing moves agents between this step and that build
    // and one step moves an agent by less than a box (|dp| <= max_disp (1 + 4u) < L)
    const bool fuse = g_fuse && !h->growth_on && !h->fields_on && h->n_el == 0 && !h->slab &&
                      h->prm.max_disp < h->grid.L * (1.0 - 0x1p-20);
    int rc = half_force(h, src, 0u, 0u, n, n, pd, h->ag[dst], nullptr, dp, nullptr, fuse, nullptr,
                        h->hist[0] ? h->hist[dst] : nullptr, nullptr, ext_mode);  // (k_force_reset resets ext)
    if (rc) return rc;
  } else {
    k_ext_reset<<<1, 32, 0, s>>>(h->ext, ext_mode);
    if (h->prm.flags & BDM_RECORD)
      k_force<true><<<grid, FORCE_THREADS, FORCE_SMEM_BYTES, s>>>(h->ag[src], h->agf, h->id[src], 0u, n, h->grid, pd,
                                                                  h->ag[dst], nullptr, dp, nullptr, h->ext, h->err, rec,
                                                                  nullptr, h->hist[0] ? h->hist[dst] : nullptr, nullptr);
    else
      k_force<false><<<grid, FORCE_THREADS, FORCE_SMEM_BYTES, s>>>(h->ag[src], h->agf, h->id[src], 0u, n, h->grid, pd,
                                                                   h->ag[dst], nullptr, dp, nullptr, h->ext, h->err, rec,
                                                                   h->skip_active ? h->hot : nullptr,
                                                                   h->hist[0] ? h->hist[dst] : nullptr, nullptr);
    k_locate_nonfinite<<<1, 32, 0, s>>>(h->ag[src], h->id[src], h->grid, pd, h->err);
    h->launches += 3;  // (the half-shell path counts its own launches)
  }
  CU(h, cudaGetLastError());
  DBG(h, "k_force");
  // The stepped positions keep the sorted order, so they keep the sorted id buffer: swap the id
  // pointers (the kernel already captured its arguments) instead of copying.
  h->out_ids = h->id[src];
  std::swap(h->id[src], h->id[dst]);
  h->cur = dst;
  if (h->hist[0]) h->skip_valid = true;
  h->skip_active = false;
  h->ext_valid = true;
  h->state = State::Stepped;
  if (want_dp) {
    h->have_dp = true;
    h->n_dp = h->n;
  }
  if (h->prm.flags & BDM_RECORD) h->have_record = true;
  return BDM_OK;
}

// Reallocate every per-agent buffer of a single handle for new_cap agents, keeping the live data
// (agents and ids of both buffers, displacements / statistics of the last step).
template <typename T>
int regrow(bdm_ctx* h, T** p, size_t keep, size_t new_count) {
  if (!*p) return BDM_OK;
  T* q = nullptr;
  CU(h, cudaMalloc(&q, std::max<size_t>(new_count, 1) * sizeof(T)));
  if (keep) CU(h, cudaMemcpyAsync(q, *p, keep * sizeof(T), cudaMemcpyDeviceToDevice, h->stream));
  CU(h, cudaStreamSynchronize(h->stream));
  CU(h, cudaFree(*p));
  *p = q;
  return BDM_OK;
}

// The padding agent after the fp32 copy's capacity N: agf[N] = (+inf, +inf, +inf, 0), which fails
// every prefilter test (pass A's slots past a lane's last candidate read it; GridDev::pad).
int set_agf_pad(bdm_ctx* h, size_t N) {
  const float inf = __builtin_huge_valf();
  const float4 pad = make_float4(inf, inf, inf, 0.f);
  CU(h, cudaMemcpy(h->agf + N, &pad, sizeof pad, cudaMemcpyHostToDevice));
  h->grid.pad = (uint32_t)N;
  return BDM_OK;
}

int grow_capacity(bdm_ctx* h, int64_t new_cap) {
  if (new_cap <= h->cap) return BDM_OK;
  if (new_cap >= (int64_t)0xffffffffll) return fail(h, BDM_ERANGE, "population would exceed 2^32 - 1 agents");
  const size_t N = (size_t)new_cap, n = (size_t)h->n, nd = (size_t)h->n_dp;
  const int oi = h->out_ids == h->id[0] ? 0 : (h->out_ids == h->id[1] ? 1 : -1);
  int rc;
  if ((rc = regrow(h, &h->ag[0], n, N)) || (rc = regrow(h, &h->ag[1], n, N)) || (rc = regrow(h, &h->agf, 0, N + 1)) ||
      (rc = regrow(h, &h->id[0], n, N)) || (rc = regrow(h, &h->id[1], n, N)) || (rc = regrow(h, &h->key, 0, N)) ||
      (rc = regrow(h, &h->slot, 0, N)) || (rc = regrow(h, &h->tsrc, 0, N)) || (rc = regrow(h, &h->tid, 0, N)) ||
      (rc = regrow(h, &h->tkey, 0, N)) || (rc = regrow(h, &h->dp, 3 * nd, 3 * N)) ||
      (rc = regrow(h, &h->r_cand, nd, N)) || (rc = regrow(h, &h->r_nb, nd, N)) || (rc = regrow(h, &h->r_ct, nd, N)) ||
      (rc = regrow(h, &h->r_branch, nd, N)) || (rc = regrow(h, &h->r_nbh, nd, N)) ||
      (rc = regrow(h, &h->r_cth, nd, N)) || (rc = regrow(h, &h->hist[0], 0, N)) ||
      (rc = regrow(h, &h->hist[1], 0, N)) || (rc = regrow(h, &h->gflag, n + 1, N + 1)))
    return rc;
  if (oi >= 0) h->out_ids = h->id[oi];
  if ((rc = set_agf_pad(h, N))) return rc;
  if (h->stage) {
    CU(h, cudaFree(h->stage));
    h->stage = nullptr;
  }
  h->cap = new_cap;
  return BDM_OK;
}

// NEXT-3: secretion + diffusion of both substances, then chemotaxis of every agent (S1-S3,
// DESIGN.md §12), on the current positions before the step's grid build.
int fields_step(bdm_ctx* h) {
  const uint32_t n = (uint32_t)h->n;
  cudaStream_t s = h->stream;
  const FieldDev& f = h->fd;
  CU(h, cudaMemsetAsync(h->fcnt, 0, 2 * (size_t)f.nn * sizeof(uint32_t), s));
  if (n) k_secrete<<<blocks(n, 256), 256, 0, s>>>(h->ag[h->cur], h->id[h->cur], n, h->type_by_id, f, h->fcnt);
  DBG(h, "k_secrete");
  const int src = h->fcur, dst = 1 - h->fcur;
  for (int t = 0; t < 2; ++t) {
    k_diffuse<<<blocks(f.nn, 256), 256, 0, s>>>(h->field[t][src], h->fcnt + (size_t)t * f.nn, h->field[t][dst], f);
    DBG(h, "k_diffuse");
  }
  h->fcur = dst;
  if (n) {
    k_chemotaxis<<<blocks(n, 256), 256, 0, s>>>(h->ag[h->cur], h->id[h->cur], n, h->type_by_id, f, h->field[0][dst],
                                                h->field[1][dst]);
    DBG(h, "k_chemotaxis");
  }
  CU(h, cudaGetLastError());
  h->launches += 3 + (n ? 2 : 0);
  // the agents moved: new extents and a fresh grid are needed
  h->ext_valid = false;
  h->cols_next = false;
  h->skip_valid = false;
  if (h->state == State::Fresh) h->state = State::Stepped;
  return BDM_OK;
}

// NEXT-2: growth + division after the mechanics of a step (G1-G3).
int grow_divide_step(bdm_ctx* h) {
  const uint32_t n = (uint32_t)h->n;
  if (!h->gflag) CU(h, cudaMalloc(&h->gflag, ((size_t)h->cap + 1) * sizeof(uint32_t)));
  cudaStream_t s = h->stream;
  const int cur = h->cur;  // stepped buffer, sorted order of the step, ids in id[cur]
  // G1 + division flags + the new max D (k_grow knows every final diameter), then the ranks; one
  // round trip reads the births and max D, and the capacity grows only if the births need it
  CU(h, cudaMemsetAsync(h->maxd_bits, 0, sizeof(unsigned long long), s));
  k_grow<<<blocks(n, 256), 256, 0, s>>>(h->ag[cur], h->id[cur], n, h->growth, h->div_diam, h->gflag, h->maxd_bits);
  DBG(h, "k_grow");
  CU(h, cudaMemsetAsync(h->gflag + n, 0, sizeof(uint32_t), s));
  int rc = scan(h, h->gflag, (uint64_t)n + 1, nullptr);
  if (rc) return rc;
  uint32_t* hostbuf = reinterpret_cast<uint32_t*>(h->ext_host);  // pinned scratch: total, then max D
  CU(h, cudaMemcpyAsync(hostbuf, h->gflag + n, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  CU(h, cudaMemcpyAsync(hostbuf + 2, h->maxd_bits, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  rc = check_async(h);
  if (rc) return rc;
  if ((uint64_t)h->cap < (uint64_t)n + hostbuf[0]) {  // (keeps the agents and the ranks)
    rc = grow_capacity(h, std::max<int64_t>((int64_t)n + hostbuf[0], h->cap + h->cap / 2));
    if (rc) return rc;
  }
  k_divide<<<blocks(n, 256), 256, 0, s>>>(h->ag[cur], h->id[cur], n, h->div_diam, h->gseed, h->step_count, h->gflag);
  DBG(h, "k_divide");
  CU(h, cudaGetLastError());
  h->launches += 3;
  const uint32_t born = hostbuf[0];
  double maxd;
  std::memcpy(&maxd, hostbuf + 2, sizeof maxd);
  h->n += born;
  // O1 for the new population: the box edge follows the largest diameter
  const double L = std::max(maxd, h->prm.box_edge_min);
  h->grid.L = L;
  h->grid.L2 = L * L;
  h->grid.inv = 1.0 / (L * (1.0 + 0x1p-30));
  h->grid.thr_pad = 0.5 * L;
  h->ext_valid = false;  // extents were reduced with the old box edge
  h->cols_next = false;
  h->skip_valid = false;
  return BDM_OK;
}

// NEXT-4 step (N1-N6): element geometry -> element grid (sub-handle) with the common box edge ->
// sphere grid -> sphere-sphere forces (force-only pass) -> spheres + element terms, O6/O7 ->
// distal points (springs + reactions), O6.  Called instead of grid_build + force_step.
void set_box_edge(GridDev& g, double L) {
  g.L = L;
  g.L2 = L * L;
  g.inv = 1.0 / (L * (1.0 + 0x1p-30));
  g.thr_pad = 0.5 * L;
}

int upload(bdm_ctx* h, const double* pos, const double* diam);

int neurite_step(bdm_ctx* h, bool want_dp) {
  const uint32_t n = (uint32_t)h->n, E = (uint32_t)h->n_el;
  cudaStream_t s = h->stream;
  const int ec = h->eqc;
  k_el_geom<<<blocks(E, 256), 256, 0, s>>>(h->eq[ec], h->ea, h->et, E, h->cpos, h->cdiam, h->geo, h->k_spring);
  CU(h, cudaGetLastError());
  DBG(h, "k_el_geom");
  bdm_ctx* el = h->el;
  int rc = upload(el, h->cpos, h->cdiam);  // re-bin the elements (synchronises; L of the elements)
  if (rc) return fail(h, rc, "element grid: %s", el->error.c_str());
  const double L = std::max(h->sphere_L, el->grid.L);  // N2: one box edge for both grids
  set_box_edge(el->grid, L);
  if (h->grid.L != L) {
    set_box_edge(h->grid, L);
    h->ext_valid = false;
    h->cols_next = false;
    if (h->state == State::Fresh) h->state = State::Stepped;
  }
  if ((rc = grid_build(el))) return fail(h, rc, "element grid: %s", el->error.c_str());
  if (h->state != State::Fresh && (rc = grid_build(h))) return rc;
  const int src = h->cur, dst = 1 - h->cur;
  k_ext_reset<<<1, 32, 0, s>>>(h->ext);
  RecordDev rec{};
  ParamsDev pd = params_dev(h->prm);
  if (n > 0) {  // sphere-sphere sums (half-shell passes when the pair rows fit, else k_force)
    if (!(h->prm.flags & BDM_RECORD) && ensure_half(h) && !h->ring) {  // (no force-only ring phase: k_force)
      rc = half_force(h, src, 0u, 0u, n, n, pd, nullptr, nullptr, nullptr, nullptr, false, nullptr, nullptr, h->fss);
      if (rc) return rc;
    } else {
      k_force<false><<<force_grid(h, n), FORCE_THREADS, FORCE_SMEM_BYTES, s>>>(
          h->ag[src], h->agf, h->id[src], 0u, n, h->grid, pd, h->ag[dst], nullptr, nullptr, nullptr, h->ext, h->err,
          rec, nullptr, nullptr, h->fss);
      DBG(h, "k_force (force-only)");
    }
  }
  if (n > 0 && (size_t)n > h->sc_cap) {  // sphere-element contact rows (k_el_update -> k_sc_rows)
    if (h->scnt) CU(h, cudaFree(h->scnt));
    if (h->srow) CU(h, cudaFree(h->srow));
    h->scnt = nullptr;
    h->srow = nullptr;
    h->sc_cap = (size_t)n + (size_t)n / 4;
    CU(h, cudaMalloc(&h->scnt, h->sc_cap * sizeof(uint32_t)));
    CU(h, cudaMalloc(&h->srow, h->sc_cap * SCAP * sizeof(uint32_t)));
  }
  if (n > 0) CU(h, cudaMemsetAsync(h->scnt, 0, (size_t)n * sizeof(uint32_t), s));
  GridDev gs = h->grid;
  if (n == 0) gs.table = nullptr;
  k_el_update<<<blocks(E, 256), 256, 0, s>>>(h->eq[ec], h->geo, h->et, E, el->id[el->cur], h->ag[src], h->agf, gs,
                                             el->grid.m32, pd, h->eq[1 - ec], h->edq, h->scnt, h->srow);
  CU(h, cudaGetLastError());
  DBG(h, "k_el_update");
  if (n > 0) {
    k_sc_rows<<<blocks(n, 256), 256, 0, s>>>(h->ag[src], h->agf, h->fss, n, h->grid, el->grid, el->agf,
                                             el->id[el->cur], h->geo, h->scnt, h->srow, pd,
                                             h->ag[dst], want_dp ? h->dp : nullptr, h->ext);
    CU(h, cudaGetLastError());
    DBG(h, "k_sc_rows");
  }
  h->launches += 5;
  h->eqc = 1 - ec;
  h->out_ids = h->id[src];
  std::swap(h->id[src], h->id[dst]);
  h->cur = dst;
  h->ext_valid = true;
  h->state = State::Stepped;
  if (want_dp) {
    h->have_dp = true;
    h->n_dp = h->n;
  }
  return BDM_OK;
}

int copy_out(bdm_ctx* h, void* dst, const void* dev_src, size_t bytes) {
  if (h->prm.flags & BDM_DEVICE_PTRS) {
    CU(h, cudaMemcpyAsync(dst, dev_src, bytes, cudaMemcpyDeviceToDevice, h->stream));
    return BDM_OK;
  }
  CU(h, cudaMemcpyAsync(dst, dev_src, bytes, cudaMemcpyDeviceToHost, h->stream));
  return check_async(h);  // synchronises and surfaces device-side errors
}

// Scratch device buffer for id-order outputs when the caller passed host pointers.
struct Scratch {
  void* p = nullptr;
  ~Scratch() {
    if (p) cudaFree(p);
  }
};

int staging(bdm_ctx* h) {  // sized for the capacity, so it stays valid while the population grows
  if (!h->stage) return dalloc(h, &h->stage, 4 * (size_t)std::max(h->n, h->cap));
  return BDM_OK;
}

// Copy (or adopt) the population, validate it on the device and derive the box edge (O1).
int upload(bdm_ctx* h, const double* pos, const double* diam) {
  const int64_t n = h->n;
  const size_t N = (size_t)n;
  h->have_dp = false;
  h->have_record = false;
  h->ext_valid = false;
  h->cols_next = false;
  h->skip_valid = false;
  h->step_count = 0;
  h->n_dp = 0;
  h->state = State::NoGrid;
  h->have_grid = false;
  h->cur = 0;
  if (n > 0) {
    const double *dpos = pos, *ddiam = diam;
    if (!(h->prm.flags & BDM_DEVICE_PTRS)) {
      int rc = staging(h);
      if (rc) return rc;
      CU(h, cudaMemcpyAsync(h->stage, pos, 3 * N * sizeof(double), cudaMemcpyHostToDevice, h->stream));
      CU(h, cudaMemcpyAsync(h->stage + 3 * N, diam, N * sizeof(double), cudaMemcpyHostToDevice, h->stream));
      dpos = h->stage;
      ddiam = h->stage + 3 * N;
    }
    CU(h, cudaMemsetAsync(h->maxd_bits, 0, sizeof(unsigned long long), h->stream));
    k_pack<<<blocks(n, 256), 256, 0, h->stream>>>(dpos, ddiam, (uint32_t)n, h->ag[0], h->id[0], h->maxd_bits,
                                                  h->err);
    CU(h, cudaGetLastError());
    CU(h, cudaMemcpyAsync(h->ext_host, h->maxd_bits, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                          h->stream));
    int rc = check_async(h);  // synchronises (the scratch copies are freed after)
    if (rc) return rc;
    double maxd;
    std::memcpy(&maxd, h->ext_host, sizeof maxd);
    // O1: L = max(max D, box_edge_min); inv = 1/(L*(1+2^-30))
    double L = std::max(maxd, h->prm.box_edge_min);
    h->sphere_L = L;
    h->grid.L = L;
    h->grid.L2 = L * L;
    h->grid.inv = 1.0 / (L * (1.0 + 0x1p-30));
    h->grid.thr_pad = 0.5 * L;
  } else {
    double L = h->prm.box_edge_min;
    h->grid.L = L;
    h->grid.L2 = L * L;
    h->grid.inv = L > 0 ? 1.0 / (L * (1.0 + 0x1p-30)) : 0.0;
  }
  return BDM_OK;
}

}  // namespace

extern "C" {

int bdm_abi_version(void) { return BDM_ABI_VERSION; }

int bdm_params_default(bdm_params* p) {
  if (!p) return fail(nullptr, BDM_EINVAL, "bdm_params_default: NULL");
  p->k_rep = 10.0;
  p->gamma_att = 4.0;
  p->adherence = 0.1;
  p->dt = 1.0;
  p->eta = 1.0;
  p->max_disp = 3.0;
  p->box_edge_min = 0.0;
  p->flags = 0;
  p->device = -1;
  return BDM_OK;
}

const char* bdm_last_error(bdm_handle h) { return h ? h->error.c_str() : g_tls_error.c_str(); }

void bdm_destroy(bdm_handle h) {
  if (!h) return;
  if (h->dist) {
    dist_destroy(h->dist);
    h->dist = nullptr;
  }
  if (h->el) bdm_destroy(h->el);
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(h->device);
  cudaStreamSynchronize(h->stream);
  if (h->s2) {
    cudaStreamSynchronize(h->s2);
    cudaStreamDestroy(h->s2);
    for (auto& e : h->bev)
      if (e) cudaEventDestroy(e);
    cudaFree(h->bwork);
  }
  for (auto& t : h->timed) {
    cudaEventDestroy(t.e0);
    cudaEventDestroy(t.e1);
    cudaEventDestroy(t.e2);
    if (t.e3) cudaEventDestroy(t.e3);
  }
  void* ptrs[] = {h->ag[0], h->ag[1], h->agf, h->id[0], h->id[1], h->key, h->slot, h->tsrc, h->tid, h->tkey, h->table, h->table2,
                  h->scan_state, h->scan_ticket, h->dp, h->stage, h->dp_ids, h->cnt, h->czlo, h->czhi, h->coff, h->hist[0], h->hist[1], h->hot, h->gflag, h->field[0][0], h->field[0][1], h->field[1][0], h->field[1][1], h->fcnt, h->type_by_id, h->eq[0], h->eq[1], h->ea, h->et, h->edq, h->cpos, h->cdiam, h->fss, h->scnt, h->srow, h->geo, h->pbox, h->colrec, h->ext, h->err, h->maxd_bits, h->r_cand, h->r_nb, h->r_ct,
                  h->r_branch, h->r_nbh, h->r_cth, h->h_fwd, h->h_bwd, h->h_bcnt, h->h_fcnt, h->h_slow, h->czlo2, h->czhi2, h->rwork, h->lstart};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (h->ext_host) cudaFreeHost(h->ext_host);
  if (h->lstart_host) cudaFreeHost(h->lstart_host);
  if (h->err_host) cudaFreeHost(h->err_host);
  if (h->cnt_host) cudaFreeHost(h->cnt_host);
  cudaSetDevice(prev);
  delete h;
}

int bdm_init(bdm_handle* out, int64_t n, const double* pos, const double* diam, const bdm_params* p) {
  if (!out) return fail(nullptr, BDM_EINVAL, "bdm_init: handle pointer is NULL");
  *out = nullptr;
  if (n < 0) return fail(nullptr, BDM_EINVAL, "bdm_init: n = %lld < 0", (long long)n);
  if (n > 0 && (!pos || !diam)) return fail(nullptr, BDM_EINVAL, "bdm_init: NULL array with n > 0");
  if (!params_ok(p)) return fail(nullptr, BDM_EINVAL, "bdm_init: invalid params (eta, max_disp must be > 0; all finite, >= 0)");
  if (n >= (int64_t)0xffffffffll) return fail(nullptr, BDM_ERANGE, "bdm_init: n >= 2^32 - 1 agents per handle");
  bdm_ctx* h = new (std::nothrow) bdm_ctx();
  if (!h) return fail(nullptr, BDM_ENOMEM, "bdm_init: host allocation");
  h->prm = *p;
  h->n = n;
  h->cap = n;
  int dev = p->device;
  if (dev < 0) {
    if (cudaGetDevice(&dev) != cudaSuccess) {
      (void)cudaGetLastError();
      delete h;
      return fail(nullptr, BDM_ECUDA, "bdm_init: no CUDA device");
    }
  }
  h->device = dev;
  int rc = BDM_OK;
#define TRY(x)                   \
  do {                           \
    rc = (x);                    \
    if (rc) {                    \
      g_tls_error = h->error;    \
      bdm_destroy(h);            \
      return rc;                 \
    }                            \
  } while (0)
  if (cudaSetDevice(dev) != cudaSuccess) {
    (void)cudaGetLastError();
    delete h;
    return fail(nullptr, BDM_ECUDA, "bdm_init: cudaSetDevice(%d) failed", dev);
  }
  h->stream = nullptr;  // legacy default stream until bdm_set_stream
  const size_t N = (size_t)n;
  TRY(dalloc(h, &h->ag[0], N));
  TRY(dalloc(h, &h->ag[1], N));
  TRY(dalloc(h, &h->agf, N + 1));
  TRY(set_agf_pad(h, N));
  TRY(dalloc(h, &h->id[0], N));
  TRY(dalloc(h, &h->id[1], N));
  TRY(dalloc(h, &h->key, N));
  TRY(dalloc(h, &h->slot, N));
  TRY(dalloc(h, &h->tsrc, N));
  TRY(dalloc(h, &h->tid, N));
  TRY(dalloc(h, &h->tkey, N));
  TRY(dalloc(h, &h->dp, 3 * N));
  TRY(dalloc(h, &h->ext, 1));
  TRY(dalloc(h, &h->err, 1));
  TRY(dalloc(h, &h->maxd_bits, 1));
  TRY(dalloc(h, &h->scan_ticket, 1));
  if (p->flags & BDM_SKIP_STATIONARY) {
    TRY(dalloc(h, &h->hist[0], N));
    TRY(dalloc(h, &h->hist[1], N));
  }
  if (p->flags & BDM_RECORD) {
    TRY(dalloc(h, &h->r_cand, N));
    TRY(dalloc(h, &h->r_nb, N));
    TRY(dalloc(h, &h->r_ct, N));
    TRY(dalloc(h, &h->r_branch, N));
    TRY(dalloc(h, &h->r_nbh, N));
    TRY(dalloc(h, &h->r_cth, N));
  }
  if (cudaMallocHost(&h->ext_host, sizeof(Extents)) != cudaSuccess ||
      cudaMallocHost(&h->err_host, sizeof(ErrDev)) != cudaSuccess) {
    (void)cudaGetLastError();
    TRY(fail(h, BDM_ENOMEM, "bdm_init: pinned host allocation"));
  }
  ErrDev e0{0u, 0xffffffffu, ERR_NONE};
  if (cudaMemcpy(h->err, &e0, sizeof e0, cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemset(h->maxd_bits, 0, sizeof(unsigned long long)) != cudaSuccess) {
    (void)cudaGetLastError();
    TRY(fail(h, BDM_ECUDA, "bdm_init: device initialisation"));
  }
  TRY(upload(h, pos, diam));
#undef TRY
  h->cur = 0;
  h->state = State::NoGrid;
  *out = h;
  return BDM_OK;
}

int bdm_set_agents(bdm_handle h, const double* pos, const double* diam) {
  if (h && h->dist) return fail(h, BDM_ESTATE, "bdm_set_agents: not for distributed handles (bdm_get_local, bdm_set_agents_dist)");
  if (!h) return fail(nullptr, BDM_EINVAL, "bdm_set_agents: NULL handle");
  if (h->n > 0 && (!pos || !diam)) return fail(h, BDM_EINVAL, "bdm_set_agents: NULL array with n > 0");
  CU(h, cudaSetDevice(h->device));
  if (h->poisoned) {  // a fresh population clears an earlier data error
    ErrDev e0{0u, 0xffffffffu, ERR_NONE};
    CU(h, cudaMemcpyAsync(h->err, &e0, sizeof e0, cudaMemcpyHostToDevice, h->stream));
    CU(h, cudaStreamSynchronize(h->stream));
    h->poisoned = false;
  }
  int rc = upload(h, pos, diam);
  if (rc) h->poisoned = true;
  return rc;
}

int bdm_set_stream(bdm_handle h, void* stream) {
  if (!h) return fail(nullptr, BDM_EINVAL, "bdm_set_stream: NULL handle");
  h->stream = static_cast<cudaStream_t>(stream);
  return BDM_OK;
}

int bdm_sync(bdm_handle h) {
  if (!h) return fail(nullptr, BDM_EINVAL, "bdm_sync: NULL handle");
  CU(h, cudaSetDevice(h->device));
  if (h->dist) return dist_sync(h);
  return check_async(h);
}

int bdm_grid_build(bdm_handle h) {
  if (h && h->dist) return fail(h, BDM_ESTATE, "bdm_grid_build: not for distributed handles (bdm_get_local, bdm_set_agents_dist)");
  if (!h) return fail(nullptr, BDM_EINVAL, "bdm_grid_build: NULL handle");
  CU(h, cudaSetDevice(h->device));
  return grid_build(h);
}

int bdm_mech_step(bdm_handle h, int32_t n_steps) {
  if (!h) return fail(nullptr, BDM_EINVAL, "bdm_mech_step: NULL handle");
  if (n_steps < 0) return fail(h, BDM_EINVAL, "bdm_mech_step: n_steps = %d < 0", n_steps);
  if (h->poisoned) return fail(h, BDM_ESTATE, "handle poisoned by an earlier error: %s", h->error.c_str());
  CU(h, cudaSetDevice(h->device));
  if (h->dist) return dist_mech_step(h, n_steps);
  if (h->n == 0 && h->n_el == 0) {
    if (n_steps > 0) h->have_dp = true;
    return BDM_OK;
  }
  for (int32_t s = 0; s < n_steps; ++s) {
    TimedStep ts{};
    if (h->timing) {
      CU(h, cudaEventCreate(&ts.e0));
      CU(h, cudaEventCreate(&ts.e1));
      CU(h, cudaEventCreate(&ts.e2));
      h->timed.push_back(ts);
      CU(h, cudaEventRecord(ts.e0, h->stream));
    }
    if (h->fields_on) {
      int rc = fields_step(h);
      if (rc) return rc;
    }
    if (h->n_el > 0) {  // NEXT-4: spheres + neurite elements
      if (h->timing) CU(h, cudaEventRecord(ts.e1, h->stream));
      int rc = neurite_step(h, s == n_steps - 1);
      if (rc) return rc;
      ++h->step_count;
      ++h->steps_total;
      if (h->timing) CU(h, cudaEventRecord(ts.e2, h->stream));
      continue;
    }
    if (h->state != State::Fresh) {
      h->defer_ok = s < n_steps - 1;
      int rc = grid_build(h);
      h->defer_ok = false;
      if (rc) return rc;
    }
    if (h->timing) CU(h, cudaEventRecord(ts.e1, h->stream));
    int rc = force_step(h, s == n_steps - 1);
    if (rc) return rc;
    if (h->growth_on) {
      rc = grow_divide_step(h);
      if (rc) return rc;
    }
    ++h->step_count;
    ++h->steps_total;
    if (h->timing) CU(h, cudaEventRecord(ts.e2, h->stream));
  }
  return BDM_OK;
}

int bdm_set_growth(bdm_handle h, double growth, double div_diam, uint64_t seed) {
  if (h && h->dist) return fail(h, BDM_ESTATE, "bdm_set_growth: not for distributed handles (bdm_get_local, bdm_set_agents_dist)");
  if (!h) return fail(nullptr, BDM_EINVAL, "bdm_set_growth: NULL handle");
  if (h->slab || h->fields_on || h->n_el) return fail(h, BDM_EINVAL, "bdm_set_growth: not available with slabs, fields or neurites");
  if (!(growth >= 0.0) || !std::isfinite(growth) || !(div_diam > 0.0))
    return fail(h, BDM_EINVAL, "bdm_set_growth: need growth >= 0 (finite) and div_diam > 0");
  h->growth_on = std::isfinite(div_diam) || growth > 0.0;
  h->growth = growth;
  h->div_diam = div_diam;
  h->gseed = seed;
  return BDM_OK;
}

int bdm_set_fields(bdm_handle h, const bdm_field_params* fp, const int8_t* types) {
  if (h && h->dist) return fail(h, BDM_ESTATE, "bdm_set_fields: not for distributed handles (bdm_get_local, bdm_set_agents_dist)");
  if (!h || !fp) return fail(h, BDM_EINVAL, "bdm_set_fields: NULL argument");
  if (h->slab || h->growth_on) return fail(h, BDM_EINVAL, "bdm_set_fields: not available with slabs or growth");
  const double h_ = fp->h;
  if (!(h_ > 0.0) || !std::isfinite(h_) || fp->dims[0] < 1 || fp->dims[1] < 1 || fp->dims[2] < 1 ||
      !(fp->diff >= 0.0) || !(fp->decay >= 0.0) || !(fp->dt >= 0.0) || !std::isfinite(fp->secretion) ||
      !(fp->speed >= 0.0) || !std::isfinite(fp->speed))
    return fail(h, BDM_EINVAL, "bdm_set_fields: bad field parameters");
  if (fp->diff * fp->dt / (h_ * h_) > 1.0 / 6.0)
    return fail(h, BDM_EINVAL, "bdm_set_fields: explicit Euler unstable, need D dt / h^2 <= 1/6 (SPEC.md:266), got %g",
                fp->diff * fp->dt / (h_ * h_));
  const uint64_t nn = (uint64_t)fp->dims[0] * fp->dims[1] * fp->dims[2];
  if (2 * nn >= 0xffffffffull) return fail(h, BDM_ERANGE, "bdm_set_fields: lattice too large");
  if (h->n > 0 && !types) return fail(h, BDM_EINVAL, "bdm_set_fields: NULL types");
  CU(h, cudaSetDevice(h->device));
  FieldDev& f = h->fd;
  f.h = h_;
  f.invh = 1.0 / h_;
  f.ih2 = 1.0 / (h_ * h_);
  f.gh1 = 1.0 / h_;
  f.gh2 = 0.5 / h_;
  f.ox = fp->origin[0];
  f.oy = fp->origin[1];
  f.oz = fp->origin[2];
  f.nx = fp->dims[0];
  f.ny = fp->dims[1];
  f.nz = fp->dims[2];
  f.nn = (uint32_t)nn;
  f.diff = fp->diff;
  f.decay = fp->decay;
  f.dt = fp->dt;
  f.secretion = fp->secretion;
  f.speed = fp->speed;
  for (int t = 0; t < 2; ++t)
    for (int b = 0; b < 2; ++b) {
      if (h->field[t][b]) CU(h, cudaFree(h->field[t][b]));
      CU(h, cudaMalloc(&h->field[t][b], nn * sizeof(double)));
      CU(h, cudaMemsetAsync(h->field[t][b], 0, nn * sizeof(double), h->stream));
    }
  h->fcur = 0;
  if (h->fcnt) CU(h, cudaFree(h->fcnt));
  CU(h, cudaMalloc(&h->fcnt, 2 * nn * sizeof(uint32_t)));
  if (h->type_by_id) CU(h, cudaFree(h->type_by_id));
  CU(h, cudaMalloc(&h->type_by_id, std::max<size_t>(1, (size_t)h->n)));
  if (h->n > 0)
    CU(h, cudaMemcpyAsync(h->type_by_id, types, (size_t)h->n,
                          (h->prm.flags & BDM_DEVICE_PTRS) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                          h->stream));
  CU(h, cudaStreamSynchronize(h->stream));
  h->fields_on = true;
  return BDM_OK;
}

int bdm_get_field(bdm_handle h, int which, double* out) {
  if (h && h->dist) return fail(h, BDM_ESTATE, "bdm_get_field: not for distributed handles (bdm_get_local, bdm_set_agents_dist)");
  if (!h || !out || (which != 0 && which != 1)) return fail(h, BDM_EINVAL, "bdm_get_field: bad arguments");
  if (!h->fields_on) return fail(h, BDM_ESTATE, "bdm_get_field: no fields (bdm_set_fields)");
  CU(h, cudaSetDevice(h->device));
  const size_t bytes = (size_t)h->fd.nn * sizeof(double);
  CU(h, cudaMemcpyAsync(out, h->field[which][h->fcur], bytes,
                        (h->prm.flags & BDM_DEVICE_PTRS) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, h->stream));
  return check_async(h);
}

int bdm_set_neurites(bdm_handle h, int64_t n_el, const double* distal, const double* diam, const double* rest_len,
                     const double* anchor, const int64_t* mother, const int64_t* daughters, double k_spring) {
  if (h && h->dist) return fail(h, BDM_ESTATE, "bdm_set_neurites: not for distributed handles (bdm_get_local, bdm_set_agents_dist)");
  if (!h) return fail(nullptr, BDM_EINVAL, "bdm_set_neurites: NULL handle");
  if (h->slab || h->growth_on || h->fields_on)
    return fail(h, BDM_EINVAL, "bdm_set_neurites: not available with slabs, growth or fields");
  if (n_el < 0 || n_el >= (int64_t)0x7fffffff || !(k_spring >= 0.0) || !std::isfinite(k_spring))
    return fail(h, BDM_EINVAL, "bdm_set_neurites: bad count or spring constant");
  if (n_el > 0 && (!distal || !diam || !rest_len || !anchor || !mother || !daughters))
    return fail(h, BDM_EINVAL, "bdm_set_neurites: NULL array");
  const size_t E = (size_t)n_el;
  std::vector<double4> q(E), a(E);
  std::vector<int4> t(E);
  for (size_t e = 0; e < E; ++e) {
    int64_t m = mother[e], d1 = daughters[2 * e], d2 = daughters[2 * e + 1];
    if (!(diam[e] > 0.0) || !std::isfinite(diam[e]) || !(rest_len[e] > 0.0) || !std::isfinite(rest_len[e]) ||
        m < -1 || m >= n_el || m == (int64_t)e || d1 < -1 || d1 >= n_el || d2 < -1 || d2 >= n_el)
      return fail(h, BDM_EINVAL, "bdm_set_neurites: bad element %zu (diameter, resting length > 0; indices)", e);
    for (int k = 0; k < 3; ++k)
      if (!std::isfinite(distal[3 * e + k]) || !std::isfinite(anchor[3 * e + k]))
        return fail(h, BDM_EINVAL, "bdm_set_neurites: non-finite coordinate of element %zu", e);
    if (d1 >= 0 && d2 >= 0 && d2 < d1) std::swap(d1, d2);
    if (d1 < 0 && d2 >= 0) std::swap(d1, d2);
    q[e] = make_double4(distal[3 * e], distal[3 * e + 1], distal[3 * e + 2], diam[e]);
    a[e] = make_double4(anchor[3 * e], anchor[3 * e + 1], anchor[3 * e + 2], rest_len[e]);
    t[e] = make_int4((int)m, (int)d1, (int)d2, 0);
  }
  CU(h, cudaSetDevice(h->device));
  auto fr = [](void* p) {
    if (p) cudaFree(p);
  };
  fr(h->eq[0]); fr(h->eq[1]); fr(h->ea); fr(h->et); fr(h->edq); fr(h->cpos); fr(h->cdiam); fr(h->fss); fr(h->geo);
  h->geo = nullptr;
  h->eq[0] = h->eq[1] = h->ea = nullptr;
  h->et = nullptr;
  h->edq = h->cpos = h->cdiam = h->fss = nullptr;
  if (h->el) {
    bdm_destroy(h->el);
    h->el = nullptr;
  }
  h->n_el = n_el;
  if (n_el == 0) return BDM_OK;
  int rc;
  if ((rc = dalloc(h, &h->eq[0], E)) || (rc = dalloc(h, &h->eq[1], E)) || (rc = dalloc(h, &h->ea, E)) ||
      (rc = dalloc(h, &h->et, E)) || (rc = dalloc(h, &h->edq, 3 * E)) || (rc = dalloc(h, &h->cpos, 3 * E)) ||
      (rc = dalloc(h, &h->cdiam, E)) || (rc = dalloc(h, &h->fss, 3 * (size_t)std::max<int64_t>(h->cap, 1))) ||
      (rc = dalloc(h, &h->geo, E)))
    return rc;
  CU(h, cudaMemcpy(h->eq[0], q.data(), E * sizeof(double4), cudaMemcpyHostToDevice));
  CU(h, cudaMemcpy(h->ea, a.data(), E * sizeof(double4), cudaMemcpyHostToDevice));
  CU(h, cudaMemcpy(h->et, t.data(), E * sizeof(int4), cudaMemcpyHostToDevice));
  CU(h, cudaMemset(h->edq, 0, 3 * E * sizeof(double)));
  h->eqc = 0;
  h->k_spring = k_spring;
  k_el_geom<<<blocks(E, 256), 256, 0, h->stream>>>(h->eq[0], h->ea, h->et, (uint32_t)E, h->cpos, h->cdiam, nullptr,
                                                    0.0);
  CU(h, cudaGetLastError());
  CU(h, cudaStreamSynchronize(h->stream));
  bdm_params ep = h->prm;
  ep.flags = BDM_DEVICE_PTRS;
  ep.device = h->device;
  bdm_ctx* el = nullptr;
  rc = bdm_init(&el, n_el, h->cpos, h->cdiam, &ep);
  if (rc) return fail(h, rc, "bdm_set_neurites: element grid: %s", bdm_last_error(nullptr));
  el->stream = h->stream;
  h->el = el;
  h->state = State::NoGrid;
  h->ext_valid = false;
  h->cols_next = false;
  return BDM_OK;
}

int bdm_get_neurites(bdm_handle h, double* distal, double* ddistal) {
  if (h && h->dist) return fail(h, BDM_ESTATE, "bdm_get_neurites: not for distributed handles (bdm_get_local, bdm_set_agents_dist)");
  if (!h) return fail(nullptr, BDM_EINVAL, "bdm_get_neurites: NULL handle");
  if (h->n_el == 0) return BDM_OK;
  CU(h, cudaSetDevice(h->device));
  const size_t E = (size_t)h->n_el;
  if (distal) {
    std::vector<double4> q(E);
    CU(h, cudaMemcpyAsync(q.data(), h->eq[h->eqc], E * sizeof(double4), cudaMemcpyDeviceToHost, h->stream));
    CU(h, cudaStreamSynchronize(h->stream));
    for (size_t e = 0; e < E; ++e) {
      distal[3 * e] = q[e].x;
      distal[3 * e + 1] = q[e].y;
      distal[3 * e + 2] = q[e].z;
    }
  }
  if (ddistal) {
    CU(h, cudaMemcpyAsync(ddistal, h->edq, 3 * E * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
    CU(h, cudaStreamSynchronize(h->stream));
  }
  return check_async(h);
}

int bdm_reserve(bdm_handle h, int64_t capacity) {
  if (h && h->dist) return fail(h, BDM_ESTATE, "bdm_reserve: not for distributed handles (bdm_get_local, bdm_set_agents_dist)");
  if (!h) return fail(nullptr, BDM_EINVAL, "bdm_reserve: NULL handle");
  if (h->slab) return fail(h, BDM_EINVAL, "bdm_reserve: not available in slab mode");
  CU(h, cudaSetDevice(h->device));
  return grow_capacity(h, capacity);
}

int bdm_get_count(bdm_handle h, int64_t* out2) {
  if (!h || !out2) return fail(h, BDM_EINVAL, "bdm_get_count: NULL argument");
  out2[0] = h->n;
  out2[1] = h->n_dp;
  return BDM_OK;
}

int bdm_set_force_path(bdm_handle h, int path) {
  if (h && h->dist) return fail(h, BDM_ESTATE, "bdm_set_force_path: not for distributed handles (bdm_get_local, bdm_set_agents_dist)");
  if (!h) return fail(nullptr, BDM_EINVAL, "bdm_set_force_path: NULL handle");
  if (path != BDM_PATH_AUTO && path != BDM_PATH_SINGLE) return fail(h, BDM_EINVAL, "bdm_set_force_path: bad path %d", path);
  h->force_path = path;
  return BDM_OK;
}

int bdm_set_defer(bdm_handle h, int max_deferred) {
  if (h && h->dist) return fail(h, BDM_ESTATE, "bdm_set_defer: not for distributed handles (bdm_get_local, bdm_set_agents_dist)");
  if (!h || max_deferred < 0) return fail(h, BDM_EINVAL, "bdm_set_defer: NULL handle or negative count");
  h->defer_max = max_deferred;
  return BDM_OK;
}

int bdm_set_timing(bdm_handle h, int enabled) {
  if (!h) return fail(nullptr, BDM_EINVAL, "bdm_set_timing: NULL handle");
  h->timing = enabled != 0;
  if (h->dist) dist_set_timing(h->dist, h->timing);
  return BDM_OK;
}

int bdm_get_timing_ex(bdm_handle h, double* out6) {
  if (!h || !out6) return fail(h, BDM_EINVAL, "bdm_get_timing_ex: NULL argument");
  CU(h, cudaSetDevice(h->device));
  if (h->dist) return dist_get_timing(h, out6);
  CU(h, cudaStreamSynchronize(h->stream));
  double grid = 0.0, force = 0.0, search = 0.0, sum = 0.0;
  for (auto& t : h->timed) {
    float a = 0.f, b = 0.f, c = 0.f;
    CU(h, cudaEventElapsedTime(&a, t.e0, t.e1));
    CU(h, cudaEventElapsedTime(&b, t.e1, t.e2));
    grid += a;
    force += b;
    if (t.e3) {
      CU(h, cudaEventElapsedTime(&c, t.e1, t.e3));
      search += c;
      sum += b - c;
      cudaEventDestroy(t.e3);
    }
    cudaEventDestroy(t.e0);
    cudaEventDestroy(t.e1);
    cudaEventDestroy(t.e2);
  }
  out6[0] = grid;
  out6[1] = force;
  out6[2] = (double)h->timed.size();
  out6[3] = (double)h->launches;
  out6[4] = search;
  out6[5] = sum;
  h->timed.clear();
  h->launches_total += h->launches;
  h->launches = 0;
  return BDM_OK;
}

int bdm_get_timing(bdm_handle h, double* out4) {
  if (!out4) return fail(h, BDM_EINVAL, "bdm_get_timing: NULL argument");
  double o[6];
  int rc = bdm_get_timing_ex(h, o);
  for (int k = 0; k < 4; ++k) out4[k] = rc ? 0.0 : o[k];
  return rc;
}

int bdm_get_displacements(bdm_handle h, double* out) {
  if (h && h->dist) return fail(h, BDM_ESTATE, "bdm_get_displacements: not for distributed handles (bdm_get_local, bdm_set_agents_dist)");
  if (!h) return fail(nullptr, BDM_EINVAL, "bdm_get_displacements: NULL handle");
  if (!h->have_dp) return fail(h, BDM_ESTATE, "bdm_get_displacements: no step has been run");
  if (h->n_dp == 0) return BDM_OK;
  if (!out) return fail(h, BDM_EINVAL, "bdm_get_displacements: NULL output");
  CU(h, cudaSetDevice(h->device));
  const uint32_t n = (uint32_t)h->n_dp;
  const size_t bytes = 3 * (size_t)n * sizeof(double);
  double* dst = out;
  if (!(h->prm.flags & BDM_DEVICE_PTRS)) {
    int rc = staging(h);
    if (rc) return rc;
    dst = h->stage;
  }
  // dp is stored in the order of the buffer that was stepped into; ids of that order are id[cur]
  k_unpermute3<<<blocks(n, 256), 256, 0, h->stream>>>(h->dp, h->out_ids, n, dst);
  CU(h, cudaGetLastError());
  if (dst != static_cast<void*>(out)) return copy_out(h, out, dst, bytes);
  return BDM_OK;
}

int bdm_get_positions(bdm_handle h, double* out) {
  if (h && h->dist) return fail(h, BDM_ESTATE, "bdm_get_positions: not for distributed handles (bdm_get_local, bdm_set_agents_dist)");
  if (!h) return fail(nullptr, BDM_EINVAL, "bdm_get_positions: NULL handle");
  if (h->n == 0) return BDM_OK;
  if (!out) return fail(h, BDM_EINVAL, "bdm_get_positions: NULL output");
  CU(h, cudaSetDevice(h->device));
  const uint32_t n = (uint32_t)h->n;
  const size_t bytes = 3 * (size_t)n * sizeof(double);
  double* dst = out;
  if (!(h->prm.flags & BDM_DEVICE_PTRS)) {
    int rc = staging(h);
    if (rc) return rc;
    dst = h->stage;
  }
  k_unpermute_pos<<<blocks(n, 256), 256, 0, h->stream>>>(h->ag[h->cur], h->id[h->cur], n, dst);
  CU(h, cudaGetLastError());
  if (dst != static_cast<void*>(out)) return copy_out(h, out, dst, bytes);
  return BDM_OK;
}

int bdm_get_diameters(bdm_handle h, double* out) {
  if (h && h->dist) return fail(h, BDM_ESTATE, "bdm_get_diameters: not for distributed handles (bdm_get_local, bdm_set_agents_dist)");
  if (!h) return fail(nullptr, BDM_EINVAL, "bdm_get_diameters: NULL handle");
  if (h->n == 0) return BDM_OK;
  if (!out) return fail(h, BDM_EINVAL, "bdm_get_diameters: NULL output");
  CU(h, cudaSetDevice(h->device));
  const uint32_t n = (uint32_t)h->n;
  const size_t bytes = (size_t)n * sizeof(double);
  double* dst = out;
  if (!(h->prm.flags & BDM_DEVICE_PTRS)) {
    int rc = staging(h);
    if (rc) return rc;
    dst = h->stage;
  }
  k_unpermute_diam<<<blocks(n, 256), 256, 0, h->stream>>>(h->ag[h->cur], h->id[h->cur], n, dst);
  CU(h, cudaGetLastError());
  if (dst != out) return copy_out(h, out, dst, bytes);
  return BDM_OK;
}

int bdm_get_box_coords(bdm_handle h, int32_t* out) {
  if (h && h->dist) return fail(h, BDM_ESTATE, "bdm_get_box_coords: not for distributed handles (bdm_get_local, bdm_set_agents_dist)");
  if (!h) return fail(nullptr, BDM_EINVAL, "bdm_get_box_coords: NULL handle");
  if (h->n == 0) return BDM_OK;
  if (!out) return fail(h, BDM_EINVAL, "bdm_get_box_coords: NULL output");
  CU(h, cudaSetDevice(h->device));
  if (h->state != State::Fresh) {
    int rc = grid_build(h);
    if (rc) return rc;
  }
  const uint32_t n = (uint32_t)h->n;
  const size_t bytes = 3 * (size_t)n * sizeof(int32_t);
  int32_t* dst = out;
  if (!(h->prm.flags & BDM_DEVICE_PTRS)) {
    int rc = staging(h);
    if (rc) return rc;
    dst = reinterpret_cast<int32_t*>(h->stage);
  }
  k_box_coords<<<blocks(n, 256), 256, 0, h->stream>>>(h->ag[h->cur], h->id[h->cur], n, h->grid.inv, dst);
  CU(h, cudaGetLastError());
  if (dst != static_cast<void*>(out)) return copy_out(h, out, dst, bytes);
  return BDM_OK;
}

int bdm_get_grid_info(bdm_handle h, bdm_grid_info* out) {
  if (h && h->dist) return fail(h, BDM_ESTATE, "bdm_get_grid_info: not for distributed handles (bdm_get_local, bdm_set_agents_dist)");
  if (!h || !out) return fail(h, BDM_EINVAL, "bdm_get_grid_info: NULL argument");
  if (!h->have_grid) return fail(h, BDM_ESTATE, "bdm_get_grid_info: no grid built yet");
  out->L = h->grid.L;
  out->L2 = h->grid.L2;
  out->inv = h->grid.inv;
  int64_t nb = h->n ? 1 : 1;
  for (int a = 0; a < 3; ++a) {  // tight extents (a fused build's x/y frame is one box wider)
    out->lo[a] = h->n ? (h->slab ? h->grid.lo[a] : h->tlo[a]) : 0;
    out->hi[a] = h->n ? (h->slab ? h->grid.hi[a] : h->thi[a]) : 0;
    nb *= (int64_t)out->hi[a] - out->lo[a] + 1;
  }
  out->n_boxes = nb;
  out->n_agents = h->n;
  return BDM_OK;
}

int bdm_get_agent_stats(bdm_handle h, const bdm_agent_stats* out) {
  if (h && h->dist) return fail(h, BDM_ESTATE, "bdm_get_agent_stats: not for distributed handles (bdm_get_local, bdm_set_agents_dist)");
  if (!h || !out) return fail(h, BDM_EINVAL, "bdm_get_agent_stats: NULL argument");
  if (!(h->prm.flags & BDM_RECORD) || !h->have_record)
    return fail(h, BDM_ESTATE, "bdm_get_agent_stats: needs BDM_RECORD at init and one step");
  if (h->n_dp == 0 && h->n == 0) return BDM_OK;
  CU(h, cudaSetDevice(h->device));
  const uint32_t n = (uint32_t)(h->n_dp ? h->n_dp : h->n);
  const uint32_t* ids = h->out_ids;
  const bool dev = h->prm.flags & BDM_DEVICE_PTRS;
  auto one = [&](auto* src, auto* dst) -> int {
    using T = std::remove_pointer_t<decltype(src)>;
    if (!dst) return BDM_OK;
    Scratch sc;
    T* d = reinterpret_cast<T*>(dst);
    if (!dev) {
      CU(h, cudaMalloc(&sc.p, n * sizeof(T)));
      d = static_cast<T*>(sc.p);
    }
    k_unpermute1<T><<<blocks(n, 256), 256, 0, h->stream>>>(src, ids, n, d);
    CU(h, cudaGetLastError());
    if (!dev) return copy_out(h, dst, sc.p, n * sizeof(T));
    return BDM_OK;
  };
  int rc;
  if ((rc = one(h->r_cand, out->n_cand))) return rc;
  if ((rc = one(h->r_nb, out->n_nb))) return rc;
  if ((rc = one(h->r_ct, out->n_ct))) return rc;
  if ((rc = one(h->r_branch, out->branch))) return rc;
  if ((rc = one(h->r_nbh, reinterpret_cast<unsigned long long*>(out->nb_hash)))) return rc;
  if ((rc = one(h->r_cth, reinterpret_cast<unsigned long long*>(out->ct_hash)))) return rc;
  return check_async(h);
}

int bdm_get_pairs(bdm_handle h, int kind, int64_t* n_pairs, int64_t* out, int64_t cap) {
  if (h && h->dist) return fail(h, BDM_ESTATE, "bdm_get_pairs: not for distributed handles (bdm_get_local, bdm_set_agents_dist)");
  if (!h || !n_pairs) return fail(h, BDM_EINVAL, "bdm_get_pairs: NULL argument");
  if (kind != BDM_NEIGHBOR && kind != BDM_CONTACT) return fail(h, BDM_EINVAL, "bdm_get_pairs: bad kind %d", kind);
  if (cap < 0 || (cap > 0 && !out)) return fail(h, BDM_EINVAL, "bdm_get_pairs: bad output buffer");
  *n_pairs = 0;
  if (h->n == 0) return BDM_OK;
  CU(h, cudaSetDevice(h->device));
  if (h->state != State::Fresh) {
    int rc = grid_build(h);
    if (rc) return rc;
  }
  const uint32_t n = (uint32_t)h->n;
  ParamsDev pd = params_dev(h->prm);
  Scratch sc_counts, sc_off, sc_out;
  CU(h, cudaMalloc(&sc_counts.p, n * sizeof(uint32_t)));
  k_pairs<<<blocks(n, 128), 128, 0, h->stream>>>(h->ag[h->cur], h->id[h->cur], n, h->grid, pd, kind,
                                                 static_cast<uint32_t*>(sc_counts.p), nullptr, nullptr);
  CU(h, cudaGetLastError());
  std::vector<uint32_t> counts(n);
  CU(h, cudaMemcpyAsync(counts.data(), sc_counts.p, n * sizeof(uint32_t), cudaMemcpyDeviceToHost, h->stream));
  CU(h, cudaStreamSynchronize(h->stream));
  std::vector<unsigned long long> off(n);
  unsigned long long total = 0;
  for (uint32_t i = 0; i < n; ++i) {
    off[i] = total;
    total += counts[i];
  }
  *n_pairs = (int64_t)total;
  if ((int64_t)total > cap) return fail(h, BDM_ETRUNC, "bdm_get_pairs: %llu pairs > cap %lld", total, (long long)cap);
  if (total == 0) return BDM_OK;
  CU(h, cudaMalloc(&sc_off.p, n * sizeof(unsigned long long)));
  CU(h, cudaMalloc(&sc_out.p, 2 * total * sizeof(long long)));
  CU(h, cudaMemcpyAsync(sc_off.p, off.data(), n * sizeof(unsigned long long), cudaMemcpyHostToDevice, h->stream));
  k_pairs<<<blocks(n, 128), 128, 0, h->stream>>>(h->ag[h->cur], h->id[h->cur], n, h->grid, pd, kind,
                                                 nullptr, static_cast<unsigned long long*>(sc_off.p),
                                                 static_cast<long long*>(sc_out.p));
  CU(h, cudaGetLastError());
  CU(h, cudaMemcpyAsync(out, sc_out.p, 2 * total * sizeof(long long), cudaMemcpyDeviceToHost, h->stream));
  CU(h, cudaStreamSynchronize(h->stream));
  struct P {
    int64_t a, b;
  };
  P* pp = reinterpret_cast<P*>(out);
  std::sort(pp, pp + total, [](const P& x, const P& y) { return x.a != y.a ? x.a < y.a : x.b < y.b; });
  return BDM_OK;
}

// ---------------------------------------------------------------------------------- x-slab mode
// DESIGN.md §7.  The caller (paper_2006_06775_b200/dist.py) owns the exchange (torch.distributed);
// these calls are the device-side halves: pack / unpack records, build the slab-local grid over
// owned + ghost agents, run the force on the owned range only, and split off migrants.

namespace {

int slab_check(bdm_ctx* h, const char* fn) {
  if (!h) return fail(nullptr, BDM_EINVAL, "%s: NULL handle", fn);
  if (!h->slab) return fail(h, BDM_ESTATE, "%s: handle was not created by bdm_slab_init", fn);
  if (h->poisoned) return fail(h, BDM_ESTATE, "%s: handle poisoned by an earlier error: %s", fn, h->error.c_str());
  CU(h, cudaSetDevice(h->device));
  return BDM_OK;
}

int read_counts(bdm_ctx* h) {
  CU(h, cudaMemcpyAsync(h->cnt_host, h->cnt, 4 * sizeof(uint32_t), cudaMemcpyDeviceToHost, h->stream));
  return check_async(h);
}

}  // namespace

int bdm_slab_init(bdm_handle* out, int64_t n_local, int64_t capacity, const uint32_t* ids, const double* pos,
                  const double* diam, const bdm_params* p) {
  if (!out) return fail(nullptr, BDM_EINVAL, "bdm_slab_init: handle pointer is NULL");
  *out = nullptr;
  if (!params_ok(p)) return fail(nullptr, BDM_EINVAL, "bdm_slab_init: invalid params");
  if (!(p->flags & BDM_DEVICE_PTRS)) return fail(nullptr, BDM_EINVAL, "bdm_slab_init: slab mode needs BDM_DEVICE_PTRS");
  if (n_local < 0 || capacity < n_local || capacity >= (int64_t)0xffffffffll)
    return fail(nullptr, BDM_EINVAL, "bdm_slab_init: need 0 <= n_local <= capacity < 2^32");
  if (n_local > 0 && (!pos || !diam || !ids)) return fail(nullptr, BDM_EINVAL, "bdm_slab_init: NULL array");
  bdm_ctx* h = new (std::nothrow) bdm_ctx();
  if (!h) return fail(nullptr, BDM_ENOMEM, "bdm_slab_init: host allocation");
  h->prm = *p;
  h->slab = true;
  h->n = n_local;
  h->cap = capacity;
  int dev = p->device;
  if (dev < 0 && cudaGetDevice(&dev) != cudaSuccess) {
    (void)cudaGetLastError();
    delete h;
    return fail(nullptr, BDM_ECUDA, "bdm_slab_init: no CUDA device");
  }
  h->device = dev;
  int rc = BDM_OK;
#define TRY(x)                \
  do {                        \
    rc = (x);                 \
    if (rc) {                 \
      g_tls_error = h->error; \
      bdm_destroy(h);         \
      return rc;              \
    }                         \
  } while (0)
  if (cudaSetDevice(dev) != cudaSuccess) {
    (void)cudaGetLastError();
    delete h;
    return fail(nullptr, BDM_ECUDA, "bdm_slab_init: cudaSetDevice(%d) failed", dev);
  }
  const size_t N = (size_t)capacity;
  TRY(dalloc(h, &h->ag[0], N));
  TRY(dalloc(h, &h->ag[1], N));
  TRY(dalloc(h, &h->agf, N + 1));
  TRY(set_agf_pad(h, N));
  TRY(dalloc(h, &h->id[0], N));
  TRY(dalloc(h, &h->id[1], N));
  TRY(dalloc(h, &h->key, N));
  TRY(dalloc(h, &h->slot, N));
  TRY(dalloc(h, &h->tsrc, N));
  TRY(dalloc(h, &h->tid, N));
  TRY(dalloc(h, &h->tkey, N));
  TRY(dalloc(h, &h->dp, 3 * N));
  TRY(dalloc(h, &h->dp_ids, N));
  TRY(dalloc(h, &h->ext, 1));
  TRY(dalloc(h, &h->err, 1));
  TRY(dalloc(h, &h->maxd_bits, 1));
  TRY(dalloc(h, &h->scan_ticket, 1));
  TRY(dalloc(h, &h->cnt, 8));
  if (cudaMallocHost(&h->ext_host, sizeof(Extents)) != cudaSuccess ||
      cudaMallocHost(&h->err_host, sizeof(ErrDev)) != cudaSuccess ||
      cudaMallocHost(&h->cnt_host, 4 * sizeof(uint32_t)) != cudaSuccess) {
    (void)cudaGetLastError();
    TRY(fail(h, BDM_ENOMEM, "bdm_slab_init: pinned host allocation"));
  }
  ErrDev e0{0u, 0xffffffffu, ERR_NONE};
  if (cudaMemcpy(h->err, &e0, sizeof e0, cudaMemcpyHostToDevice) != cudaSuccess) {
    (void)cudaGetLastError();
    TRY(fail(h, BDM_ECUDA, "bdm_slab_init: device initialisation"));
  }
  if (n_local > 0) {
    CU(h, cudaMemsetAsync(h->maxd_bits, 0, sizeof(unsigned long long), h->stream));
    k_pack<<<blocks(n_local, 256), 256, 0, h->stream>>>(pos, diam, (uint32_t)n_local, h->ag[0], h->id[0],
                                                        h->maxd_bits, h->err);
    if (cudaGetLastError() != cudaSuccess) TRY(fail(h, BDM_ECUDA, "bdm_slab_init: k_pack launch"));
    if (cudaMemcpyAsync(h->id[0], ids, (size_t)n_local * sizeof(uint32_t), cudaMemcpyDeviceToDevice, h->stream) !=
        cudaSuccess)
      TRY(fail(h, BDM_ECUDA, "bdm_slab_init: id copy"));
    TRY(check_async(h));
  }
#undef TRY
  h->cur = 0;
  h->state = State::NoGrid;
  *out = h;
  return BDM_OK;
}

int bdm_slab_load(bdm_handle h, int64_t n_local, const uint32_t* ids, const double* pos, const double* diam) {
  int rc = slab_check(h, "bdm_slab_load");
  if (rc) return rc;
  if (n_local < 0 || n_local > h->cap || (n_local > 0 && (!ids || !pos || !diam)))
    return fail(h, BDM_EINVAL, "bdm_slab_load: need 0 <= n_local <= capacity and non-NULL arrays");
  if (n_local > 0) {
    k_pack<<<blocks(n_local, 256), 256, 0, h->stream>>>(pos, diam, (uint32_t)n_local, h->ag[0], h->id[0],
                                                        h->maxd_bits, h->err);
    CU(h, cudaGetLastError());
    CU(h, cudaMemcpyAsync(h->id[0], ids, (size_t)n_local * sizeof(uint32_t), cudaMemcpyDeviceToDevice, h->stream));
    h->launches += 1;
  }
  h->cur = 0;
  h->n = n_local;
  h->n_dead = 0;
  h->split_pending = false;
  h->ext_valid = false;
  h->cols_next = false;
  h->have_dp = false;
  h->n_dp = 0;
  h->state = State::NoGrid;
  return BDM_OK;
}

int bdm_slab_local_maxd(bdm_handle h, double* maxd) {
  int rc = slab_check(h, "bdm_slab_local_maxd");
  if (rc) return rc;
  if (h->n_dead) return fail(h, BDM_ESTATE, "bdm_slab_local_maxd: emigrants of the last split are pending (run a step)");
  if (!maxd) return fail(h, BDM_EINVAL, "bdm_slab_local_maxd: NULL output");
  CU(h, cudaMemsetAsync(h->maxd_bits, 0, sizeof(unsigned long long), h->stream));
  if (h->n > 0) k_maxd<<<blocks(h->n, 256), 256, 0, h->stream>>>(h->ag[h->cur], (uint32_t)h->n, h->maxd_bits);
  CU(h, cudaGetLastError());
  CU(h, cudaMemcpyAsync(h->ext_host, h->maxd_bits, sizeof(unsigned long long), cudaMemcpyDeviceToHost, h->stream));
  rc = check_async(h);
  if (rc) return rc;
  std::memcpy(maxd, h->ext_host, sizeof(double));
  return BDM_OK;
}

int bdm_slab_set_box_edge(bdm_handle h, double L) {
  int rc = slab_check(h, "bdm_slab_set_box_edge");
  if (rc) return rc;
  L = std::max(L, h->prm.box_edge_min);
  if (!(L > 0.0) || !std::isfinite(L)) return fail(h, BDM_EINVAL, "bdm_slab_set_box_edge: L must be > 0 and finite");
  h->grid.L = L;
  h->grid.L2 = L * L;
  h->grid.inv = 1.0 / (L * (1.0 + 0x1p-30));
  h->grid.thr_pad = 0.5 * L;
  h->ext_valid = false;
  h->cols_next = false;
  h->have_grid = true;
  return BDM_OK;
}

int bdm_slab_local_extents(bdm_handle h, int32_t* lohi6) {
  int rc = slab_check(h, "bdm_slab_local_extents");
  if (rc) return rc;
  if (h->n_dead) return fail(h, BDM_ESTATE, "bdm_slab_local_extents: emigrants of the last split are pending (run a step)");
  if (!lohi6) return fail(h, BDM_EINVAL, "bdm_slab_local_extents: NULL output");
  if (!(h->grid.inv > 0.0)) return fail(h, BDM_ESTATE, "bdm_slab_local_extents: call bdm_slab_set_box_edge first");
  if (!h->ext_valid) {
    k_ext_reset<<<1, 32, 0, h->stream>>>(h->ext);
    if (h->n > 0) k_extents<<<blocks(h->n, 256), 256, 0, h->stream>>>(h->ag[h->cur], (uint32_t)h->n, h->grid.inv, h->ext);
    DBG(h, "k_extents");
    CU(h, cudaGetLastError());
    h->ext_valid = true;
  }
  CU(h, cudaMemcpyAsync(h->ext_host, h->ext, sizeof(Extents), cudaMemcpyDeviceToHost, h->stream));
  rc = check_async(h);
  if (rc) return rc;
  if (h->ext_host->range_err) {
    h->poisoned = true;
    return fail(h, BDM_ERANGE, "an agent lies >= 2^20 boxes from the origin (DESIGN.md R9)");
  }
  for (int a = 0; a < 3; ++a) {
    lohi6[a] = h->ext_host->lo[a];
    lohi6[3 + a] = h->ext_host->hi[a];
  }
  return BDM_OK;
}

int bdm_slab_pack(bdm_handle h, int what, int32_t x_begin, int32_t x_end, double* send_lo, double* send_hi,
                  int64_t cap, int64_t* n_lo, int64_t* n_hi) {
  int rc = slab_check(h, "bdm_slab_pack");
  if (rc) return rc;
  if (h->n_dead) return fail(h, BDM_ESTATE, "bdm_slab_pack: emigrants of the last split are pending (run a step)");
  if ((what != BDM_HALO && what != BDM_MIGRANTS) || !n_lo || !n_hi || cap < 0 || (cap > 0 && (!send_lo || !send_hi)))
    return fail(h, BDM_EINVAL, "bdm_slab_pack: bad arguments");
  if (x_begin >= x_end) return fail(h, BDM_EINVAL, "bdm_slab_pack: empty slab [%d, %d)", x_begin, x_end);
  CU(h, cudaMemsetAsync(h->cnt, 0, 4 * sizeof(uint32_t), h->stream));
  const uint32_t n = (uint32_t)h->n;
  if (n > 0)
    k_slab_pack<<<blocks(n, 256), 256, 0, h->stream>>>(h->ag[h->cur], h->id[h->cur], n, h->grid.inv,
                                                        what == BDM_HALO ? 0 : 1, x_begin, x_end, send_lo, send_hi,
                                                        (uint64_t)cap, h->cnt, h->ag[1 - h->cur], h->id[1 - h->cur]);
  CU(h, cudaGetLastError());
  h->launches += n > 0;
  rc = read_counts(h);
  if (rc) return rc;
  *n_lo = h->cnt_host[0];
  *n_hi = h->cnt_host[1];
  if (*n_lo > cap || *n_hi > cap)
    return fail(h, BDM_ETRUNC, "bdm_slab_pack: %lld / %lld records > cap %lld", (long long)*n_lo, (long long)*n_hi,
                (long long)cap);
  if (what == BDM_MIGRANTS) {  // commit the compaction of the agents that stay
    h->cur = 1 - h->cur;
    h->n = h->cnt_host[2];
    h->fused_n0 = std::min<int64_t>(h->fused_n0, h->n);  // agents appended from here on need their columns
  }
  return BDM_OK;
}

int bdm_slab_split(bdm_handle h, int32_t x_begin, int32_t x_end, double* send_lo, double* send_hi, int64_t cap,
                   int64_t* info) {
  int rc = slab_check(h, "bdm_slab_split");
  if (rc) return rc;
  if (!info || cap < 0 || (cap > 0 && (!send_lo || !send_hi)) || x_begin >= x_end)
    return fail(h, BDM_EINVAL, "bdm_slab_split: bad arguments");
  if (h->split_pending) return fail(h, BDM_ESTATE, "bdm_slab_split: the previous split was not committed");
  if (h->n_dead) return fail(h, BDM_ESTATE, "bdm_slab_split: run a step after the last commit");
  CU(h, cudaMemsetAsync(h->cnt, 0, 8 * sizeof(uint32_t), h->stream));
  const uint32_t n = (uint32_t)h->n;
  init_device_info(h);
  if (h->state == State::Stepped && h->have_grid) {  // boundary layers of the step's sorted order
    k_layer_bounds<<<1, 32, 0, h->stream>>>(h->grid, x_begin, x_end, h->last_n_lo, n, h->cnt + 4);
  } else {  // no step since the last load / add: the whole array
    const uint32_t r2[2] = {n, n};
    CU(h, cudaMemcpyAsync(h->cnt + 4, r2, sizeof r2, cudaMemcpyHostToDevice, h->stream));
  }
  if (!h->ext_valid) {  // extents of the owned agents now
    k_ext_reset<<<1, 32, 0, h->stream>>>(h->ext);
    if (n > 0) k_extents<<<blocks(n, 256), 256, 0, h->stream>>>(h->ag[h->cur], n, h->grid.inv, h->ext);
    h->launches += 1 + (n > 0);
    h->ext_valid = true;
  }
  if (n > 0)
    k_slab_split<<<h->sm_count * 4, 256, 0, h->stream>>>(h->ag[h->cur], h->id[h->cur], n, h->cnt + 4, h->grid.inv,
                                                          x_begin, x_end, send_lo, send_hi, (uint64_t)cap, h->cnt);
  k_split_info<<<1, 32, 0, h->stream>>>(h->cnt, h->ext, (uint64_t)cap, n, info);
  CU(h, cudaGetLastError());
  h->launches += 2 + (n > 0);
  h->split_pending = true;
  h->split_xb = x_begin;
  h->split_xe = x_end;
  return BDM_OK;
}

int bdm_slab_commit(bdm_handle h, int64_t n_stay) {
  int rc = slab_check(h, "bdm_slab_commit");
  if (rc) return rc;
  if (!h->split_pending) return fail(h, BDM_ESTATE, "bdm_slab_commit: no split to commit");
  if (n_stay < 0) {  // cancel: the owned agents are unchanged (the split only wrote other buffers)
    h->split_pending = false;
    return BDM_OK;
  }
  if (n_stay > h->n) return fail(h, BDM_EINVAL, "bdm_slab_commit: n_stay = %lld", (long long)n_stay);
  // mark the emigrants dead in place (boundary ranges only); the next sort drops them
  if (n_stay < h->n)
    k_slab_mark_dead<<<h->sm_count * 4, 256, 0, h->stream>>>(h->ag[h->cur], (uint32_t)h->n, h->cnt + 4, h->grid.inv,
                                                              h->split_xb, h->split_xe);
  CU(h, cudaGetLastError());
  h->launches += n_stay < h->n;
  h->n_dead = h->n - n_stay;  // (the fused next columns stay valid: they cover a superset)
  h->split_pending = false;
  h->ext_valid = false;
  return BDM_OK;
}

int bdm_slab_add(bdm_handle h, const double* recv_lo, int64_t n_lo, const double* recv_hi, int64_t n_hi) {
  int rc = slab_check(h, "bdm_slab_add");
  if (rc) return rc;
  if (n_lo < 0 || n_hi < 0 || (n_lo && !recv_lo) || (n_hi && !recv_hi))
    return fail(h, BDM_EINVAL, "bdm_slab_add: bad arguments");
  if (h->n + n_lo + n_hi > h->cap)
    return fail(h, BDM_ERANGE, "bdm_slab_add: %lld agents exceed the slab capacity %lld", (long long)(h->n + n_lo + n_hi),
                (long long)h->cap);
  uint32_t off = (uint32_t)h->n;
  if (n_lo) k_unpack<<<blocks(n_lo, 256), 256, 0, h->stream>>>(recv_lo, (uint32_t)n_lo, h->ag[h->cur], h->id[h->cur], off);
  if (n_hi)
    k_unpack<<<blocks(n_hi, 256), 256, 0, h->stream>>>(recv_hi, (uint32_t)n_hi, h->ag[h->cur], h->id[h->cur],
                                                       off + (uint32_t)n_lo);
  CU(h, cudaGetLastError());
  h->launches += (n_lo > 0) + (n_hi > 0);
  h->n += n_lo + n_hi;
  return BDM_OK;
}

int bdm_slab_step(bdm_handle h, const int32_t* glo3, const int32_t* ghi3, int32_t x_begin, int32_t x_end,
                  const double* recv_lo, int64_t n_lo, const double* recv_hi, int64_t n_hi, int want_dp) {
  int rc = slab_check(h, "bdm_slab_step");
  if (rc) return rc;
  if (!glo3 || !ghi3 || n_lo < 0 || n_hi < 0 || (n_lo && !recv_lo) || (n_hi && !recv_hi) || x_begin >= x_end)
    return fail(h, BDM_EINVAL, "bdm_slab_step: bad arguments");
  if (!(h->grid.inv > 0.0)) return fail(h, BDM_ESTATE, "bdm_slab_step: call bdm_slab_set_box_edge first");
  const int64_t n_own = h->n, n_tot = n_own + n_lo + n_hi, n_dead = h->n_dead;  // n_own counts dead entries
  if (n_tot > h->cap)
    return fail(h, BDM_ERANGE, "bdm_slab_step: %lld owned + ghost agents exceed the capacity %lld", (long long)n_tot,
                (long long)h->cap);
  cudaStream_t s = h->stream;
  TimedStep ts{};
  if (h->timing) {
    CU(h, cudaEventCreate(&ts.e0));
    CU(h, cudaEventCreate(&ts.e1));
    CU(h, cudaEventCreate(&ts.e2));
    h->timed.push_back(ts);
    CU(h, cudaEventRecord(ts.e0, s));
  }
  // ghosts after the owned agents
  if (n_lo) k_unpack<<<blocks(n_lo, 256), 256, 0, s>>>(recv_lo, (uint32_t)n_lo, h->ag[h->cur], h->id[h->cur], (uint32_t)n_own);
  if (n_hi)
    k_unpack<<<blocks(n_hi, 256), 256, 0, s>>>(recv_hi, (uint32_t)n_hi, h->ag[h->cur], h->id[h->cur],
                                               (uint32_t)(n_own + n_lo));
  CU(h, cudaGetLastError());
  h->launches += (n_lo > 0) + (n_hi > 0);
  // slab-local grid: box-x [x_begin-1, x_end] clipped to the global extents; y, z global
  GridDev& g = h->grid;
  const int64_t lox = std::max<int64_t>((int64_t)x_begin - 1, glo3[0]);
  const int64_t hix = std::min<int64_t>((int64_t)x_end, ghi3[0]);
  k_ext_reset<<<1, 32, 0, s>>>(h->ext);
  h->launches += 1;
  if (n_tot == 0 || lox > hix) {
    if (n_tot) return fail(h, BDM_ESTATE, "bdm_slab_step: agents present but the slab lies outside the extents");
    h->ext_valid = true;
    h->n_dp = 0;
    h->state = State::Stepped;
    return BDM_OK;
  }
  g.lo[0] = (int32_t)lox;
  g.hi[0] = (int32_t)hix;
  for (int a = 1; a < 3; ++a) {
    g.lo[a] = glo3[a];
    g.hi[a] = ghi3[a];
  }
  // fused column pass of the last step: its frame becomes this grid's x/y frame if it contains this
  // step's (it does when every agent moved less than a box); the agents appended since (immigrants,
  // ghosts) add their columns first
  if (h->cols_next && g.lo[0] >= h->nlo[0] && g.hi[0] < h->nlo[0] + h->nnx && g.lo[1] >= h->nlo[1] &&
      g.hi[1] < h->nlo[1] + h->nny && h->fused_n0 <= n_own) {
    g.lo[0] = h->nlo[0];
    g.lo[1] = h->nlo[1];
    g.hi[0] = h->nlo[0] + h->nnx - 1;
    g.hi[1] = h->nlo[1] + h->nny - 1;
    g.ny = h->nny;
    g.n_cols = (uint32_t)((int64_t)h->nnx * h->nny);  // (the column count of this frame, before its pass)
    const int64_t m = n_tot - h->fused_n0;
    if (m > 0) {
      k_col_ext<<<blocks(m, 512), 256, 0, s>>>(h->ag[h->cur] + h->fused_n0, (uint32_t)m, g, h->czlo2, h->czhi2);
      h->launches += 1;
    }
  } else {
    h->cols_next = false;
  }
  const int64_t nb = ((int64_t)g.hi[0] - g.lo[0] + 1) * ((int64_t)g.hi[1] - g.lo[1] + 1) * ((int64_t)g.hi[2] - g.lo[2] + 1);
  if (nb >= (int64_t)0xffffffffll) return fail(h, BDM_ERANGE, "bdm_slab_step: n_boxes = %lld >= 2^32", (long long)nb);
  g.ny = g.hi[1] - g.lo[1] + 1;
  g.nz = g.hi[2] - g.lo[2] + 1;
  g.n_boxes = (uint32_t)nb;
  rc = sort_into(h, (uint32_t)n_tot, (uint32_t)n_dead);  // cur -> sorted live owned + ghosts (dead dropped)
  if (rc) return rc;
  if (h->timing) CU(h, cudaEventRecord(ts.e1, s));
  // ghosts_lo (box-x = x_begin-1) sort first, ghosts_hi (box-x = x_end) last: the owned agents are
  // the contiguous range [n_lo, n_sorted - n_hi) of the sorted array
  const int src = h->cur, dst = 1 - h->cur;
  const int64_t n_live = n_own - n_dead, n_sorted = n_tot - n_dead;
  h->last_n_lo = (uint32_t)n_lo;
  RecordDev rec{h->r_cand, h->r_nb, h->r_ct, h->r_branch, h->r_nbh, h->r_cth};
  ParamsDev pd = params_dev(h->prm);
  const unsigned grid = force_grid(h, (uint32_t)n_live);
  h->last_half = n_live > 0 && ensure_half(h);
  if (h->last_half) {
    // pass A from the first lower ghost (their forward pairs with owned agents are the owned
    // agents' backward pairs); owned agents' forward runs reach into the upper ghosts.  The sum
    // pass accumulates the next step's columns in the frame [x_begin-1, x_end] x [ylo-1, yhi+1]
    // (clipped to the extents +- 1): every agent of the next step lies in it (|dp| < L)
    const bool fuse = h->prm.max_disp < h->grid.L * (1.0 - 0x1p-20);
    const int64_t fx0 = std::max<int64_t>((int64_t)x_begin - 1, (int64_t)glo3[0] - 1);
    const int64_t fx1 = std::min<int64_t>((int64_t)x_end, (int64_t)ghi3[0] + 1);
    const int32_t frame4[4] = {(int32_t)fx0, glo3[1] - 1, (int32_t)(fx1 - fx0 + 1), ghi3[1] - glo3[1] + 3};
    rc = half_force(h, src, 0u, (uint32_t)n_lo, (uint32_t)(n_sorted - n_hi), (uint32_t)n_sorted, pd, h->ag[dst], h->id[dst],
                    want_dp ? h->dp : nullptr, want_dp ? h->dp_ids : nullptr, fuse, frame4);
    if (rc) return rc;
  } else if (n_live > 0) {
    k_force<false><<<grid, FORCE_THREADS, FORCE_SMEM_BYTES, s>>>(h->ag[src], h->agf, h->id[src], (uint32_t)n_lo,
                                                 (uint32_t)(n_sorted - n_hi), g, pd, h->ag[dst], h->id[dst],
                                                 want_dp ? h->dp : nullptr, want_dp ? h->dp_ids : nullptr, h->ext,
                                                 h->err, rec, nullptr, nullptr, nullptr);
    k_locate_nonfinite<<<1, 32, 0, s>>>(h->ag[src], h->id[src], g, pd, h->err);
    CU(h, cudaGetLastError());
    h->launches += 2;
  }
  if (h->timing) CU(h, cudaEventRecord(ts.e2, s));
  h->cur = dst;
  h->n = n_live;
  h->n_dead = 0;
  h->fused_n0 = n_live;
  h->ext_valid = true;
  if (want_dp) {
    h->n_dp = n_live;
    h->have_dp = true;
  }
  h->state = State::Stepped;
  return BDM_OK;
}

int bdm_slab_get(bdm_handle h, int what, int64_t* n, uint32_t* ids, double* vals) {
  int rc = slab_check(h, "bdm_slab_get");
  if (rc) return rc;
  if (h->n_dead) return fail(h, BDM_ESTATE, "bdm_slab_get: emigrants of the last split are pending (run a step)");
  if (!n || (what != BDM_OWNED_POSITIONS && what != BDM_LAST_DISPLACEMENTS))
    return fail(h, BDM_EINVAL, "bdm_slab_get: bad arguments");
  if (what == BDM_LAST_DISPLACEMENTS && !h->have_dp) return fail(h, BDM_ESTATE, "bdm_slab_get: no displacements yet");
  const int64_t m = what == BDM_OWNED_POSITIONS ? h->n : h->n_dp;
  *n = m;
  if (m == 0 || (!ids && !vals)) return check_async(h);
  if (what == BDM_OWNED_POSITIONS) {
    if (ids) CU(h, cudaMemcpyAsync(ids, h->id[h->cur], m * sizeof(uint32_t), cudaMemcpyDeviceToDevice, h->stream));
    if (vals) {
      CU(h, cudaMemcpy2DAsync(vals, 3 * sizeof(double), h->ag[h->cur], sizeof(double4), 3 * sizeof(double), m,
                              cudaMemcpyDeviceToDevice, h->stream));
    }
  } else {
    if (ids) CU(h, cudaMemcpyAsync(ids, h->dp_ids, m * sizeof(uint32_t), cudaMemcpyDeviceToDevice, h->stream));
    if (vals) CU(h, cudaMemcpyAsync(vals, h->dp, 3 * m * sizeof(double), cudaMemcpyDeviceToDevice, h->stream));
  }
  return check_async(h);
}

int bdm_get_skip_stats(bdm_handle h, int64_t* out3) {
  if (h && h->dist) return fail(h, BDM_ESTATE, "bdm_get_skip_stats: not for distributed handles (bdm_get_local, bdm_set_agents_dist)");
  if (!h || !out3) return fail(h, BDM_EINVAL, "bdm_get_skip_stats: NULL argument");
  CU(h, cudaSetDevice(h->device));
  if (!h->ext_valid || h->state != State::Stepped) {
    out3[0] = out3[1] = out3[2] = -1;
    return BDM_OK;
  }
  CU(h, cudaMemcpyAsync(h->ext_host, h->ext, sizeof(Extents), cudaMemcpyDeviceToHost, h->stream));
  int rc = check_async(h);
  if (rc) return rc;
  out3[0] = h->hist[0] ? (int64_t)h->ext_host->moved : -1;
  out3[1] = h->hist[0] ? (int64_t)h->ext_host->searched : -1;
  out3[2] = h->n;
  return BDM_OK;
}

int bdm_get_path_stats(bdm_handle h, int64_t* out2) {
  if (h && h->dist) return fail(h, BDM_ESTATE, "bdm_get_path_stats: not for distributed handles (bdm_get_local, bdm_set_agents_dist)");
  if (!h || !out2) return fail(h, BDM_EINVAL, "bdm_get_path_stats: NULL argument");
  CU(h, cudaSetDevice(h->device));
  if (!h->ext_valid || h->state != State::Stepped) {
    out2[0] = out2[1] = -1;
    return BDM_OK;
  }
  CU(h, cudaMemcpyAsync(h->ext_host, h->ext, sizeof(Extents), cudaMemcpyDeviceToHost, h->stream));
  int rc = check_async(h);
  if (rc) return rc;
  out2[0] = h->last_half ? (h->ring_band ? 2 : 1) : 0;
  out2[1] = h->last_half ? (int64_t)h->ext_host->slow : 0;
  return BDM_OK;
}

int bdm_generate_uniform(uint64_t seed, int64_t id0, int64_t n, const double* lo3, const double* hi3, double dlo,
                         double dhi, double* pos, double* diam, void* stream) {
  if (n < 0 || id0 < 0 || !lo3 || !hi3 || (n > 0 && (!pos || !diam)))
    return fail(nullptr, BDM_EINVAL, "bdm_generate_uniform: bad arguments");
  if (n == 0) return BDM_OK;
  unsigned nb = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 64);
  k_gen_uniform<<<nb, 256, 0, static_cast<cudaStream_t>(stream)>>>(seed, id0, n, lo3[0], lo3[1], lo3[2], hi3[0],
                                                                   hi3[1], hi3[2], dlo, dhi, pos, diam);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(nullptr, BDM_ECUDA, "bdm_generate_uniform: %s", cudaGetErrorString(e));
  return BDM_OK;
}

}  // extern "C"

#include "bdm_dist.cuh"
