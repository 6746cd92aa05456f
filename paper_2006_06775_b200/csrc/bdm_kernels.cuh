// bdm_kernels.cuh -- sm_100a kernels of the mechanical-interaction step.
//
// Compiled with -fmad=false: every fp64 +,-,* on the method's path is a separately rounded IEEE
// operation, so per-pair arithmetic is bit-identical to the reading in DESIGN.md §3 (O3-O6);
// sqrt() and '/' on doubles are correctly rounded.  No tensor cores: nothing here is a dense
// contraction (north_star).  Kernels of the step chain start with pdl_wait() (programmatic
// dependent launch).
//
//   K0 k_gen_uniform     counter-hash synthetic agents (bench / cfg4-5 utility)
//   K1 k_pack            n x 3 positions + diameters -> double4 agents, validation, max D
//      k_extents         min/max integer box coordinate per axis (first build only; later fused in K6)
//   build:
//      k_col_len / k_table_zero   ragged table layout from the column z-ranges (+ scan tile states)
//   K2 k_key_hist(_packed)       box key (x slowest) + per-box histogram with warp-aggregated atomics
//   K3 k_scan            single-pass decoupled look-back exclusive scan -> box start table
//   K4 k_scatter         counting-sort scatter into box segments
//      k_place           ascending-id order inside each box + payload gather (deterministic sort)
//      k_table_zero_tma  the next build's histogram zeroed by TMA bulk stores (side stream)
//   force phase (the default step):
//      k_force_reset     extents / counters / next-frame columns / pair counters, one launch
//      k_half_search     pass A: forward half of the 27 boxes, fp32 prefilter -> pair rows
//      k_half_sum        pass B: canonical-order contact sums -> adherence/clamp -> p' = p + dp,
//                        fused with the next build's extents, column ranges and packed boxes
//      k_half_slow       agents whose rows overflowed: full canonical search, warp per agent
//      k_layer_starts    band sizes of the ring phase (populations whose rows do not fit)
//   K6 k_force           single pass: 27-box search -> force -> ... (RECORD, skip, neurites)
//   K7 k_unpermute_*     sorted order -> id order for the getters
//   K8 k_pairs_*         neighbour / contact pair export (tests)
#pragma once
#include <cassert>
#include <cstdint>
#include <cuda_runtime.h>

// BDM_CHECK=1 (tools/build_variant.sh checked -DBDM_CHECK=1): device-side bounds assertions on the index
// computations of the hot kernels (table keys, scatter / place destinations, column indices, z-runs,
// row partners, distributed ingest) -- the substitute for compute-sanitizer, which is closed on this
// pool.  Off in the product build.
#ifndef BDM_CHECK
#define BDM_CHECK 0
#endif
#if BDM_CHECK
#define BDM_ASSERT(c) assert(c)
#else
#define BDM_ASSERT(c) ((void)0)
#endif

namespace bdm {

constexpr unsigned FULL = 0xffffffffu;

// Grid parameters of one build, passed by value to kernels.
//
// Box table layout ("ragged" by column): a column is one (bx, by) pair; column c of the frame
// [lo_x, hi_x] x [lo_y, hi_y] stores only its occupied z-range [czlo[c], czhi[c]], at table offset
// coff[c].  Box (bx, by, bz) has key coff[c] + (bz - czlo[c]); keys keep x slowest, then y, then z,
// so a slab is a contiguous key range and the 3 boxes (bx, by, bz-1..bz+1) are one contiguous range
// of the sorted agents.  table[key] = first sorted agent of the box, table[T] = N.  For the
// Gaussian cfg3 this is 3.8e7 entries instead of the 3.1e8 of the dense box lattice.
struct GridDev {
  double L, L2, inv;
  double thr_pad;  // (L/2) used for the conservative contact prefilter
  double m32;      // fp32 prefilter margin: 2 ulp32(max |coord|) + 2^-18 + 2^-20 L
  int32_t lo[3], hi[3];
  int32_t ny, nz;
  uint32_t n_boxes;  // dense lattice size (reported; the table itself is ragged)
  uint32_t n_cols;   // nx * ny
  const int32_t* czlo;
  const int32_t* czhi;
  const uint32_t* coff;  // n_cols + 1
  const uint32_t* table;
  const int4* col;       // per column (czlo, czhi, coff, 0): one 16-byte load per column lookup
  uint32_t pad;          // index of the padding agent agf[pad] = (+inf, +inf, +inf, 0) (capacity; pass A's
                         // slots past the end of a lane's candidates read it and fail the filter)
  uint32_t rmask = 0xffffffffu;  // pair rows / counts of agent j at index j & rmask (a ring of two bands
                                 // in the banded force phase of very large populations; else all ones)
};

struct ParamsDev {
  double k_rep, gamma_att, adherence, c /* dt/eta */, max_disp;
};

// Box extents (reduced with atomics) + asynchronous error reporting.
struct Extents {
  int32_t lo[3], hi[3];
  int32_t range_err;  // 1 if some |p*inv| >= 2^20
  uint32_t work;      // chunk counter of the persistent force kernel
  uint32_t moved;     // agents with dp != 0 in the step that produced these extents (skip mode)
  uint32_t searched;  // agents whose neighbourhood was searched in that step (skip mode)
  uint32_t work_a;    // chunk counter of the half-shell search pass (k_half_search)
  uint32_t slow;      // agents of the half-shell sum pass whose pair rows overflowed (full search)
  uint32_t col_bad;   // fused column pass: some agent's new box left its frame (columns invalid)
  uint32_t sticky;    // range_err (bit 0) / col_bad (bit 1) of earlier steps (deferred builds)
  uint32_t zeroed;    // entries of the next build's histogram buffer the last sum pass zeroed (ColNext::zbuf)
};

// Fused column pass (k_half_sum): occupied z-range of every column (bx, by) of the NEXT build's
// frame [lo0, lo0+nx) x [lo1, lo1+ny), accumulated from the stepped positions (czlo = nullptr: off).
struct ColNext {
  int32_t lo0, lo1, nx, ny;
  int32_t* czlo;
  int32_t* czhi;
  uint32_t* pbox;  // (optional) per stepped agent: its new column in the frame << zbits | (bz - z0)
  int32_t z0, zbits;
};

struct ErrDev {
  uint32_t code;            // 0 ok, else |BDM_E*|
  uint32_t second;          // ENONFINITE: partner id located by k_locate_nonfinite (0xffffffff = not yet)
  unsigned long long bad;   // (id of the first offending agent << 32) | aux, min over reports; aux =
                            // the agent's sorted index in the force phase's state (ENONFINITE)
};
constexpr unsigned long long ERR_NONE = ~0ull;

struct RecordDev {
  int32_t *n_cand, *n_nb, *n_ct;
  int8_t* branch;
  unsigned long long *nb_hash, *ct_hash;
};

__device__ __forceinline__ unsigned long long pack2(float lo, float hi) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// First error wins the code; the reported (id, aux) pair is the one with the smallest id (one 64-bit
// atomicMin keeps id and aux consistent).
__device__ __forceinline__ void report(ErrDev* e, uint32_t code, uint32_t id, uint32_t aux) {
  atomicCAS(&e->code, 0u, code);
  atomicMin(&e->bad, ((unsigned long long)id << 32) | aux);
}

// ------------------------------------------------------------------------------------------ K0
__global__ void k_gen_uniform(uint64_t seed, int64_t id0, int64_t n, double lx, double ly, double lz, double hx,
                              double hy, double hz, double dlo, double dhi, double* __restrict__ pos,
                              double* __restrict__ diam) {
  const uint64_t base = seed * 0x9E3779B97F4A7C15ull;
  const double lo[3] = {lx, ly, lz};
  const double wd[3] = {hx - lx, hy - ly, hz - lz};
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    uint64_t id = (uint64_t)(id0 + t);
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      double u = (double)(mix64(base + 4ull * id + (uint64_t)a) >> 11) * 0x1p-53;
      pos[3 * t + a] = lo[a] + wd[a] * u;
    }
    double u = (double)(mix64(base + 4ull * id + 3ull) >> 11) * 0x1p-53;
    diam[t] = dlo + (dhi - dlo) * u;
  }
}

// ------------------------------------------------------------------------------------------ K1
// Packs AoS xyz + D into double4 agents, sets id = index, validates (finite, D > 0) and reduces
// max D (positive doubles order like their bit patterns).
__global__ void k_pack(const double* __restrict__ pos, const double* __restrict__ diam, uint32_t n,
                       double4* __restrict__ ag, uint32_t* __restrict__ ids, unsigned long long* maxd_bits,
                       ErrDev* err) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  double D = 0.0;
  if (i < n) {
    double x = pos[3 * (size_t)i], y = pos[3 * (size_t)i + 1], z = pos[3 * (size_t)i + 2];
    D = diam[i];
    bool ok = isfinite(x) && isfinite(y) && isfinite(z) && isfinite(D) && D > 0.0;
    if (!ok) {
      report(err, 1u /*EINVAL*/, i, i);
      D = 0.0;
    }
    ag[i] = make_double4(x, y, z, D);
    ids[i] = i;
  }
  unsigned long long b = __double_as_longlong(D);
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long v = __shfl_xor_sync(FULL, b, o);
    b = v > b ? v : b;
  }
  if ((threadIdx.x & 31) == 0 && b) atomicMax(maxd_bits, b);
}

// Block-level min/max of integer box coordinates, then at most 6 atomics per block, each issued
// only if it can still change the global value (ld.cg read of the current extent): a same-address
// atomic per warp serialises at one L2 slice and cost milliseconds at 2e7 agents.
// Must be called by every thread of the block.
__device__ __forceinline__ void block_minmax_atomic(Extents* ext, const int b[3], bool valid) {
  __shared__ int s_red[32][6];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    int lo = __reduce_min_sync(FULL, valid ? b[a] : INT32_MAX);
    int hi = __reduce_max_sync(FULL, valid ? b[a] : INT32_MIN);
    if (lane == 0) {
      s_red[warp][a] = lo;
      s_red[warp][3 + a] = hi;
    }
  }
  __syncthreads();
  if (threadIdx.x < 6) {
    const int a = threadIdx.x;
    int v = s_red[0][a];
    for (int w = 1; w < nwarps; ++w) v = a < 3 ? min(v, s_red[w][a]) : max(v, s_red[w][a]);
    if (a < 3) {
      if (v != INT32_MAX && v < __ldcg(&ext->lo[a])) atomicMin(&ext->lo[a], v);
    } else {
      if (v != INT32_MIN && v > __ldcg(&ext->hi[a - 3])) atomicMax(&ext->hi[a - 3], v);
    }
  }
}

// Programmatic dependent launch (the step's kernels are launched with programmatic stream
// serialisation, so a kernel's launch and block scheduling overlap its predecessor's drain): every
// kernel of the chain waits here, before touching anything its predecessor reads or writes, for the
// predecessor grid to complete and its memory to be visible; then it lets its own successor launch
// (whose blocks take the SMs this grid's tail frees and wait in turn -- the trigger fires only once
// every block of this grid has started, so they never displace one of its blocks).  A no-op for
// ordinary launches.
__device__ __forceinline__ void pdl_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
#ifndef BDM_SCAN_ITEMS
#define BDM_SCAN_ITEMS 16
#endif
constexpr uint32_t SCAN_TILE_C = 256u * BDM_SCAN_ITEMS;  // items per scan tile (= SCAN_TILE, below)

// integer box coordinate of one component; flags |q| >= 2^20 (R9)

__device__ __forceinline__ int box_coord(double p, double inv, bool& bad) {
  double q = p * inv;
  bad |= !(fabs(q) < 1048576.0);
  return (int)floor(q);
}

__global__ void k_extents(const double4* __restrict__ ag, uint32_t n, double inv, Extents* ext) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  bool valid = i < n, bad = false;
  int b[3] = {0, 0, 0};
  if (valid) {
    double4 p = ag[i];
    b[0] = box_coord(p.x, inv, bad);
    b[1] = box_coord(p.y, inv, bad);
    b[2] = box_coord(p.z, inv, bad);
  }
  if (__any_sync(FULL, bad) && (threadIdx.x & 31) == 0) ext->range_err = 1;
  block_minmax_atomic(ext, b, valid);
}

#ifndef BDM_V256
#define BDM_V256 1  // 256-bit loads/stores of the 32-byte state (one LSU instruction and one request per sector)
#endif
// The state is double4 in 32-byte aligned arrays (cudaMalloc'd): one 256-bit access per lane.
__device__ __forceinline__ double4 ld_state(const double4* p) {
#if BDM_V256
  double4 v;
  asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
  return v;
#else
  return *p;
#endif
}
__device__ __forceinline__ void st_state(double4* p, double4 v) {
#if BDM_V256
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(v.x), "d"(v.y), "d"(v.z), "d"(v.w) : "memory");
#else
  *p = v;
#endif
}

// mode 0: also clear the sticky flags; 1: the range flag of the last step becomes sticky first; 2: so
// does its frame flag (the build just made was deferred: its frame had to hold every agent)
__global__ void k_ext_reset(Extents* ext, int mode = 1) {
  pdl_wait();
  if (threadIdx.x == 0)
    ext->sticky = mode == 0 ? 0u
                            : ext->sticky | (ext->range_err ? 1u : 0u) | (mode == 2 && ext->col_bad ? 2u : 0u);
  __syncwarp();
  if (threadIdx.x < 3) {
    ext->lo[threadIdx.x] = INT32_MAX;
    ext->hi[threadIdx.x] = INT32_MIN;
  }
  if (threadIdx.x == 3) ext->range_err = 0;
  if (threadIdx.x == 4) ext->work = 0u;
  if (threadIdx.x == 5) ext->moved = 0u;
  if (threadIdx.x == 6) ext->searched = 0u;
  if (threadIdx.x == 7) ext->work_a = 0u;
  if (threadIdx.x == 8) ext->slow = 0u;
  if (threadIdx.x == 9) ext->col_bad = 0u;
}

__device__ __forceinline__ uint32_t col_of(const GridDev& g, int bx, int by) {
  return (uint32_t)(bx - g.lo[0]) * (uint32_t)g.ny + (uint32_t)(by - g.lo[1]);
}

// key of an occupied box (the agent's own box)
__device__ __forceinline__ uint32_t box_key(const GridDev& g, int bx, int by, int bz) {
  const uint32_t c = col_of(g, bx, by);
  const int4 ci = __ldg(&g.col[c]);
  return (uint32_t)ci.z + (uint32_t)(bz - ci.x);
}

// Sorted-agent range [b, e) of the boxes (cx, cy, z0..z1) (O3's z-run of one column); false if empty.
__device__ __forceinline__ bool zrun(const GridDev& g, int cx, int cy, int z0, int z1, uint32_t& b, uint32_t& e) {
  if (cx < g.lo[0] || cx > g.hi[0] || cy < g.lo[1] || cy > g.hi[1]) return false;
  const uint32_t c = col_of(g, cx, cy);
  BDM_ASSERT(c < g.n_cols);
  const int4 ci = __ldg(&g.col[c]);
  const int zl = ci.x, zh = ci.y;
  const int a = z0 > zl ? z0 : zl, d = z1 < zh ? z1 : zh;
  if (a > d) return false;
  const uint32_t o = (uint32_t)ci.z;
  BDM_ASSERT(o + (uint32_t)(d - zl) + 1u <= __ldg(&g.coff[g.n_cols]));
  b = __ldg(&g.table[o + (uint32_t)(a - zl)]);
  e = __ldg(&g.table[o + (uint32_t)(d - zl) + 1u]);
  BDM_ASSERT(b <= e);
  return true;
}

// The 9 z-runs (z in [bz-1, bz+1]) of the columns around (bx, by), in canonical column order; empty
// runs as b = e.  All table loads of one level are issued together (two dependent levels instead of
// 9 x 3 for successive zrun calls).
__device__ __forceinline__ void zrun9(const GridDev& g, int bx, int by, int bz, uint32_t rb[9], uint32_t re[9]) {
  int zl[9], zh[9];
  uint32_t o[9];
  bool ok[9];
#pragma unroll
  for (int col = 0; col < 9; ++col) {
    const int cx = bx + col / 3 - 1, cy = by + col % 3 - 1;
    ok[col] = cx >= g.lo[0] && cx <= g.hi[0] && cy >= g.lo[1] && cy <= g.hi[1];
    const uint32_t c = ok[col] ? col_of(g, cx, cy) : 0u;
    const int4 ci = ok[col] ? __ldg(&g.col[c]) : make_int4(1, 0, 0, 0);
    zl[col] = ci.x;
    zh[col] = ci.y;
    o[col] = (uint32_t)ci.z;
  }
#pragma unroll
  for (int col = 0; col < 9; ++col) {
    const int a = bz - 1 > zl[col] ? bz - 1 : zl[col], d = bz + 1 < zh[col] ? bz + 1 : zh[col];
    const bool live = ok[col] && a <= d;
    rb[col] = live ? __ldg(&g.table[o[col] + (uint32_t)(a - zl[col])]) : 0u;
    re[col] = live ? __ldg(&g.table[o[col] + (uint32_t)(d - zl[col]) + 1u]) : 0u;
  }
}

// Warp aggregation of histogram atomics over runs of equal keys in consecutive lanes (the agents
// arrive in the last step's sorted order, so a box's agents are mostly adjacent): one shuffle and
// one ballot per element instead of __match_any_sync (which kept the key passes MIO-throttled).
// Returns the run's first lane; *len the run length.  Equal keys in separate runs get separate
// atomics (correct, just not merged).
__device__ __forceinline__ int key_run(uint32_t k, int lane, uint32_t& len) {
  const uint32_t prev = __shfl_up_sync(FULL, k, 1);
  const unsigned heads = __ballot_sync(FULL, lane == 0 || prev != k);
  const unsigned upto = lane == 31 ? FULL : ((2u << lane) - 1u);  // lanes 0..lane
  const int start = 31 - __clz(heads & upto);
  const unsigned above = heads & ~upto;
  const int end = above ? __ffs(above) - 1 : 32;
  len = (uint32_t)(end - start);
  return start;
}

// Start of a half-shell force phase, one launch: the extents / counters reset of k_ext_reset (block 0),
// the next build's column ranges of the fused pass (czlo2 / czhi2, nc2 columns) and the pair counters
// (nb agents).
__global__ void k_force_reset(Extents* ext, int ext_mode, int32_t* __restrict__ czlo2, int32_t* __restrict__ czhi2,
                              uint32_t nc2, uint32_t* __restrict__ bcnt, uint32_t nb) {
  pdl_wait();
  if (blockIdx.x == 0 && threadIdx.x < 32 && ext_mode >= 0) {
    if (threadIdx.x == 0)
      ext->sticky = ext_mode == 0 ? 0u
                                  : ext->sticky | (ext->range_err ? 1u : 0u) | (ext_mode == 2 && ext->col_bad ? 2u : 0u);
    __syncwarp();
    if (threadIdx.x < 3) {
      ext->lo[threadIdx.x] = INT32_MAX;
      ext->hi[threadIdx.x] = INT32_MIN;
    }
    if (threadIdx.x == 3) ext->range_err = 0;
    if (threadIdx.x == 4) ext->work = 0u;
    if (threadIdx.x == 5) ext->moved = 0u;
    if (threadIdx.x == 6) ext->searched = 0u;
    if (threadIdx.x == 7) ext->work_a = 0u;
    if (threadIdx.x == 8) ext->slow = 0u;
    if (threadIdx.x == 9) ext->col_bad = 0u;
  }
  const uint32_t t0 = blockIdx.x * blockDim.x + threadIdx.x, stride = gridDim.x * blockDim.x;
  if (czlo2)
    for (uint32_t c = t0; c < nc2; c += stride) {
      czlo2[c] = INT32_MAX;
      czhi2[c] = INT32_MIN;
    }
  const uint32_t n4 = nb / 4;
  uint4* b4 = reinterpret_cast<uint4*>(bcnt);
  for (uint32_t k = t0; k < n4; k += stride) b4[k] = make_uint4(0u, 0u, 0u, 0u);
  for (uint32_t k = 4 * n4 + t0; k < nb; k += stride) bcnt[k] = 0u;
}

// ---- column pass: occupied z-range of every column, then lengths for the offset scan
__global__ void k_col_reset(int32_t* __restrict__ czlo, int32_t* __restrict__ czhi, uint32_t nc) {
  pdl_wait();
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < nc; c += gridDim.x * blockDim.x) {
    czlo[c] = INT32_MAX;
    czhi[c] = INT32_MIN;
  }
}

// rng (distributed steps, device counts): the agents [rng[0], rng[1]) of ag instead of [0, n), block-
// strided over a small grid (the range is often short: the records appended since the last step)
__global__ void k_col_ext(const double4* __restrict__ ag, uint32_t n, GridDev g, int32_t* __restrict__ czlo,
                          int32_t* __restrict__ czhi, const uint32_t* __restrict__ rng = nullptr) {
  pdl_wait();
  uint32_t b0 = 0u;
  if (rng) {
    b0 = __ldg(&rng[0]);
    n = __ldg(&rng[1]) - b0;
    ag += b0;
  }
  for (uint32_t blk = blockIdx.x; blk * (2 * blockDim.x) < n; blk += rng ? gridDim.x : 0xffffffffu) {
  const uint32_t i0 = blk * (2 * blockDim.x) + threadIdx.x;
  const uint32_t ia[2] = {i0, i0 + blockDim.x};
  double4 pa[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) pa[u] = ia[u] < n ? ag[ia[u]] : make_double4(0.0, 0.0, 0.0, 0.0);
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const bool valid = ia[u] < n;
    uint32_t c = 0xffffffffu;
    int bz = 0;
    if (valid && pa[u].w >= 0.0) {  // (slab mode: emigrants are marked dead by D < 0 until the sort)
      const int bx = (int)floor(pa[u].x * g.inv), by = (int)floor(pa[u].y * g.inv);
      bz = (int)floor(pa[u].z * g.inv);
      // distributed steps (rng): the frame is fixed for a chunk; an agent outside it is left to the
      // guarded key pass (which reports it) instead of indexing outside the column arrays
      if (!rng || (bx >= g.lo[0] && bx <= g.hi[0] && by >= g.lo[1] && by <= g.hi[1])) c = col_of(g, bx, by);
      BDM_ASSERT(c == 0xffffffffu || c < g.n_cols);
    }
    // warp-aggregated: agents arrive mostly in box order, so a warp touches few columns; each group
    // of lanes with the same column reduces with redux.sync over its own member mask
    unsigned peers;
    {  // lanes with the same column: a run of consecutive lanes (the agents arrive nearly sorted)
      uint32_t len;
      const int r0 = key_run(c, lane, len);
      peers = (len == 32u ? FULL : ((1u << len) - 1u)) << r0;
    }
    const int zmin = __reduce_min_sync(peers, bz);
    const int zmax = __reduce_max_sync(peers, bz);
    if (c != 0xffffffffu && lane == __ffs(peers) - 1) {
      if (zmin < __ldcg(&czlo[c])) atomicMin(&czlo[c], zmin);
      if (zmax > __ldcg(&czhi[c])) atomicMax(&czhi[c], zmax);
    }
  }
  if (!rng) break;
  }
}

// (st / st_n / ticket: the next scan's tile states and ticket are zeroed here, so that no memset node
// interrupts the launch chain)
__global__ void k_col_len(const int32_t* __restrict__ czlo, const int32_t* __restrict__ czhi, uint32_t nc,
                          uint32_t* __restrict__ len, unsigned long long* __restrict__ st = nullptr, uint32_t st_n = 0,
                          uint32_t* __restrict__ ticket = nullptr) {
  pdl_wait();
  if (st)
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < st_n; t += gridDim.x * blockDim.x) st[t] = 0ull;
  if (ticket && blockIdx.x == 0 && threadIdx.x == 0) *ticket = 0u;
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c <= nc; c += gridDim.x * blockDim.x)
    len[c] = c < nc && czhi[c] >= czlo[c] ? (uint32_t)(czhi[c] - czlo[c] + 1) : 0u;
}

// zero table[0 .. T] with T = coff[nc] read on the device (no host round trip); also packs the
// column records (czlo, czhi, coff) for the lookups
__global__ void k_table_zero(uint32_t* __restrict__ table, const uint32_t* __restrict__ coff, uint32_t nc,
                             const int32_t* __restrict__ czlo, const int32_t* __restrict__ czhi,
                             int4* __restrict__ col, unsigned long long* __restrict__ st = nullptr,
                             uint32_t st_cap = 0, uint32_t* __restrict__ ticket = nullptr,
                             const uint32_t* __restrict__ zeroed = nullptr) {
  pdl_wait();
  if (st) {  // the table scan's tile states (T + 1 items) and ticket (see k_col_len)
    const uint32_t tiles = min(st_cap, (__ldg(&coff[nc]) + 1u + (uint32_t)SCAN_TILE_C - 1u) / (uint32_t)SCAN_TILE_C);
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < tiles; t += gridDim.x * blockDim.x) st[t] = 0ull;
    if (ticket && blockIdx.x == 0 && threadIdx.x == 0) *ticket = 0u;
  }
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < nc; c += gridDim.x * blockDim.x)
    col[c] = make_int4(czlo[c], czhi[c], (int)coff[c], 0);
  const uint32_t T = coff[nc];
  // 16-byte stores (the table is 256-byte aligned), then the last T+1 mod 4 entries; entries the last
  // sum pass already zeroed (a multiple of 4) are skipped
  const uint32_t n4 = (T + 1) / 4;
  const uint32_t z4 = zeroed ? min(*zeroed / 4u, n4) : 0u;
  uint4* t4 = reinterpret_cast<uint4*>(table);
  for (uint32_t k = z4 + blockIdx.x * blockDim.x + threadIdx.x; k < n4; k += gridDim.x * blockDim.x)
    t4[k] = make_uint4(0u, 0u, 0u, 0u);
  const uint32_t k = 4 * n4 + blockIdx.x * blockDim.x + threadIdx.x;
  if (k <= T) table[k] = 0u;
}

// The next build's histogram buffer zeroed while the force phase runs (a side stream; the search is
// bound by the L1 data pipe and leaves HBM idle): TMA bulk stores from a zeroed shared-memory block
// (async proxy: no LSU wavefronts), one CTA per SM with a contiguous slice each.  Zeroes the first
// min(cap4, T + T/8 + 4096) entries (T: the current grid's table size, a multiple of 4) and records
// the count in *zdone for k_table_zero.
constexpr int ZT_BYTES = 4096;
__global__ void __launch_bounds__(32) k_table_zero_tma(uint32_t* __restrict__ table2, const uint32_t* __restrict__ coff,
                                                       uint32_t nc, uint32_t cap4, uint32_t* __restrict__ zdone) {
  __shared__ __align__(128) uint4 zbuf[ZT_BYTES / 16];
  for (int k = threadIdx.x; k < ZT_BYTES / 16; k += blockDim.x) zbuf[k] = make_uint4(0u, 0u, 0u, 0u);
  const uint32_t T = __ldg(&coff[nc]);
  const uint32_t zn = min(cap4, (T + T / 8u + 4096u) & ~3u);
  if (blockIdx.x == 0 && threadIdx.x == 0) *zdone = zn;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  if (threadIdx.x != 0) return;
  const uint64_t bytes = (uint64_t)zn * 4u, per = ((bytes / gridDim.x) + 15u) & ~15ull;
  const uint64_t b0 = per * blockIdx.x, b1 = min(bytes, b0 + per);
  const uint32_t src = (uint32_t)__cvta_generic_to_shared(zbuf);
  for (uint64_t o = b0; o < b1; o += ZT_BYTES) {
    const uint32_t len = (uint32_t)(b1 - o < (uint64_t)ZT_BYTES ? b1 - o : (uint64_t)ZT_BYTES);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                     reinterpret_cast<char*>(table2) + o), "r"(src), "r"(len) : "memory");
  }
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// Sorted-order start of every box-x layer of the grid (out[x] for x in [0, nx), out[nx] = n): the
// banded force phase of very large populations sizes its bands from the largest two-layer span.
__global__ void k_layer_starts(GridDev g, uint32_t nx, uint32_t n, uint32_t* __restrict__ out) {
  pdl_wait();
  for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x <= nx; x += gridDim.x * blockDim.x)
    out[x] = x < nx ? __ldg(&g.table[__ldg(&g.coff[x * (uint32_t)g.ny])]) : n;
}

// ------------------------------------------------------------------------------------------ K2
// Two agents per thread (block-strided, both loads coalesced and in flight together).
// GUARD (deferred builds, whose extents were not checked on the host): an agent whose box lies
// outside the grid (a non-finite or out-of-range position) is counted in box 0 and reported (code 7)
// instead of indexing outside the table.
// n_dev (distributed steps): the agent count is read on the device (n is the launch bound)
template <bool GUARD>
__global__ void k_key_hist(const double4* __restrict__ ag, uint32_t n, GridDev g, uint32_t* __restrict__ key,
                           uint32_t* __restrict__ slot, uint32_t* __restrict__ count, ErrDev* err,
                           const uint32_t* __restrict__ n_dev = nullptr, const uint32_t* __restrict__ b0_dev = nullptr) {
  pdl_wait();
  if (n_dev) n = __ldg(n_dev);
  if (b0_dev) {  // (the agents [*b0_dev, n) only: the records appended after the packed ones)
    const uint32_t b0 = __ldg(b0_dev);
    n = n > b0 ? n - b0 : 0u;
    ag += b0;
    key += b0;
    slot += b0;
  }
  if (blockIdx.x * (2 * blockDim.x) >= n) return;  // (whole blocks only: the warps aggregate below)
  const uint32_t i0 = blockIdx.x * (2 * blockDim.x) + threadIdx.x;
  const uint32_t ia[2] = {i0, i0 + blockDim.x};
  double4 pa[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) pa[u] = ia[u] < n ? ag[ia[u]] : make_double4(0.0, 0.0, 0.0, 0.0);
  const int lane = threadIdx.x & 31;
  uint32_t kk[2], peers[2], base[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const bool valid = ia[u] < n;
    uint32_t k = 0xffffffffu;
    if (valid && pa[u].w >= 0.0) {  // dead (slab emigrant, D < 0): dropped by the sort
      const double4 p = pa[u];
      const int bx = (int)floor(p.x * g.inv), by = (int)floor(p.y * g.inv), bz = (int)floor(p.z * g.inv);
      if (GUARD) {  // column inside the frame and key inside the table (T = coff[n_cols])
        const bool okxy = bx >= g.lo[0] && bx <= g.hi[0] && by >= g.lo[1] && by <= g.hi[1];
        const uint32_t c = okxy ? col_of(g, bx, by) : 0u;
        const int4 ci = __ldg(&g.col[c]);
        k = (uint32_t)ci.z + (uint32_t)(bz - ci.x);
        if (!okxy || k >= __ldg(&g.coff[g.n_cols])) {
          k = 0u;
          report(err, 7u, ia[u], 0u);
        }
      } else {
        k = box_key(g, bx, by, bz);
      }
    }
    kk[u] = k;
  }
  // warp-aggregated histogram (one atomic per run of equal keys), both atomics in flight
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    uint32_t len;
    peers[u] = (uint32_t)key_run(kk[u], lane, len);  // (the run's first lane)
    base[u] = 0u;
    if (kk[u] != 0xffffffffu && lane == (int)peers[u])
      base[u] = (BDM_ASSERT(kk[u] < __ldg(&g.coff[g.n_cols])), atomicAdd(&count[kk[u]], len));
  }
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const uint32_t b = __shfl_sync(FULL, base[u], (int)peers[u]);
    if (ia[u] < n) {
      key[ia[u]] = kk[u];
      slot[ia[u]] = b + (uint32_t)(lane - (int)peers[u]);
    }
  }
}

#ifndef BDM_KHP
#define BDM_KHP 4  // agents per thread in k_key_hist_packed (all loads and atomics of a level in flight)
#endif
constexpr int KHP = BDM_KHP;
// K2 from the packed boxes the last step's sum pass wrote (column << zbits | z - z0): 4 bytes per
// agent instead of the 32-byte state.  GUARD as in k_key_hist.
template <bool GUARD>
__global__ void k_key_hist_packed(const uint32_t* __restrict__ pbox, uint32_t n, GridDev g, int32_t z0, int32_t zbits,
                                  uint32_t* __restrict__ key, uint32_t* __restrict__ slot,
                                  uint32_t* __restrict__ count, ErrDev* err, const uint32_t* __restrict__ n_dev = nullptr) {
  pdl_wait();
  if (n_dev) n = __ldg(n_dev);  // (distributed steps: dead emigrants carry pbox 0xffffffff and are dropped)
  const uint32_t i0 = blockIdx.x * (KHP * blockDim.x) + threadIdx.x;
  uint32_t pa[KHP];
#pragma unroll
  for (int u = 0; u < KHP; ++u) pa[u] = i0 + u * blockDim.x < n ? __ldg(&pbox[i0 + u * blockDim.x]) : 0u;
  const int lane = threadIdx.x & 31;
  const uint32_t T = GUARD ? __ldg(&g.coff[g.n_cols]) : 0u;
  uint32_t k[KHP], peers[KHP], base[KHP];
#pragma unroll
  for (int u = 0; u < KHP; ++u) {
    const uint32_t i = i0 + u * blockDim.x;
    k[u] = 0xffffffffu;
    if (i < n && pa[u] != 0xffffffffu) {
      uint32_t c = pa[u] >> zbits;
      const int bz = z0 + (int)(pa[u] & ((1u << zbits) - 1u));
      const bool okc = !GUARD || c < g.n_cols;
      c = okc ? c : 0u;
      const int4 ci = __ldg(&g.col[c]);
      k[u] = (uint32_t)ci.z + (uint32_t)(bz - ci.x);
      if (GUARD && (!okc || k[u] >= T)) {
        k[u] = 0u;
        report(err, 7u, i, 0u);
      }
    }
  }
  // the four warp-aggregated atomics (one per run of equal keys) in flight together, then their bases
  // broadcast
#pragma unroll
  for (int u = 0; u < KHP; ++u) {
    uint32_t len;
    peers[u] = (uint32_t)key_run(k[u], lane, len);  // (the run's first lane)
    base[u] = 0u;
    if (k[u] != 0xffffffffu && lane == (int)peers[u]) {
      BDM_ASSERT(k[u] < __ldg(&g.coff[g.n_cols]));
      base[u] = atomicAdd(&count[k[u]], len);
    }
  }
#pragma unroll
  for (int u = 0; u < KHP; ++u) {
    const uint32_t i = i0 + u * blockDim.x;
    const uint32_t b = __shfl_sync(FULL, base[u], (int)peers[u]);
    if (i < n) {
      key[i] = k[u];
      slot[i] = b + (uint32_t)(lane - (int)peers[u]);
    }
  }
}

// ------------------------------------------------------------------------------------------ K3
constexpr int SCAN_THREADS = 256;
constexpr int SCAN_ITEMS = BDM_SCAN_ITEMS;  // per thread
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v) {
  int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t t = __shfl_up_sync(FULL, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

__device__ __forceinline__ uint32_t warp_sum(uint32_t v) { return __reduce_add_sync(FULL, v); }

// In-place exclusive scan of data[0..n_items) (the last input is 0 so that data[n_items-1] becomes
// the total).  n_items = n_items_host, or *n_dev + 1 read on the device when n_items_host == 0.
// Persistent blocks take tiles from an atomic ticket, so every predecessor of a tile is held by a
// running block and the decoupled look-back cannot deadlock (the grid never exceeds the resident
// capacity).
__global__ void __launch_bounds__(SCAN_THREADS) k_scan(uint32_t* __restrict__ data, const uint32_t* __restrict__ n_dev,
                                                       uint64_t n_items_host, unsigned long long* __restrict__ state,
                                                       uint32_t* __restrict__ ticket) {
  pdl_wait();
  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_warp[SCAN_THREADS / 32];
  __shared__ uint32_t s_prefix;
  const uint64_t n_items = n_items_host ? n_items_host : (uint64_t)(*n_dev) + 1;
  const uint64_t n_tiles = (n_items + SCAN_TILE - 1) / SCAN_TILE;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  while (true) {
    __syncthreads();
    if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    if (tile >= n_tiles) return;
    const uint64_t base = (uint64_t)tile * SCAN_TILE + (uint64_t)threadIdx.x * SCAN_ITEMS;
    uint32_t v[SCAN_ITEMS];
    if (base + SCAN_ITEMS <= n_items) {
      const uint4* src = reinterpret_cast<const uint4*>(data + base);
#pragma unroll
      for (int q = 0; q < SCAN_ITEMS / 4; ++q) {
        uint4 w = src[q];
        v[4 * q] = w.x;
        v[4 * q + 1] = w.y;
        v[4 * q + 2] = w.z;
        v[4 * q + 3] = w.w;
      }
    } else {
#pragma unroll
      for (int q = 0; q < SCAN_ITEMS; ++q) v[q] = base + q < n_items ? data[base + q] : 0u;
    }
    uint32_t tsum = 0;
#pragma unroll
    for (int q = 0; q < SCAN_ITEMS; ++q) tsum += v[q];
    uint32_t incl = warp_incl_scan(tsum);
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      uint32_t ws = lane < SCAN_THREADS / 32 ? s_warp[lane] : 0u;
      uint32_t wi = warp_incl_scan(ws);
      if (lane < SCAN_THREADS / 32) s_warp[lane] = wi - ws;  // exclusive warp offsets
      uint32_t agg = __shfl_sync(FULL, wi, SCAN_THREADS / 32 - 1);
      uint32_t excl = 0;
      if (tile == 0) {
        if (lane == 0) atomicExch(&state[0], (2ull << 32) | agg);
      } else {
        if (lane == 0) atomicExch(&state[tile], (1ull << 32) | agg);
        int64_t pred = (int64_t)tile - 1;
        while (true) {
          int64_t idx = pred - lane;
          unsigned long long st = idx >= 0 ? atomicAdd(&state[idx], 0ull) : (2ull << 32);
          uint32_t status = (uint32_t)(st >> 32);
          if (__any_sync(FULL, status == 0u)) continue;
          unsigned incl_mask = __ballot_sync(FULL, status == 2u);
          if (incl_mask) {
            int first = __ffs(incl_mask) - 1;
            excl += warp_sum(lane <= first ? (uint32_t)st : 0u);
            break;
          }
          excl += warp_sum((uint32_t)st);
          pred -= 32;
        }
        if (lane == 0) atomicExch(&state[tile], (2ull << 32) | (uint32_t)(excl + agg));
      }
      if (lane == 0) s_prefix = excl;
    }
    __syncthreads();
    uint32_t run = s_prefix + s_warp[warp] + (incl - tsum);
    uint32_t o[SCAN_ITEMS];
#pragma unroll
    for (int q = 0; q < SCAN_ITEMS; ++q) {
      o[q] = run;
      run += v[q];
    }
    if (base + SCAN_ITEMS <= n_items) {
      uint4* dst = reinterpret_cast<uint4*>(data + base);
#pragma unroll
      for (int q = 0; q < SCAN_ITEMS / 4; ++q) dst[q] = make_uint4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
    } else {
#pragma unroll
      for (int q = 0; q < SCAN_ITEMS; ++q)
        if (base + q < n_items) data[base + q] = o[q];
    }
  }
}

// ------------------------------------------------------------------------------------------ K4
// (KSC agents per thread, all loads of a level in flight together: the pass is latency-bound)
#ifndef BDM_KSC
#define BDM_KSC 2  // agents per thread in k_scatter
#endif
constexpr int KSC = BDM_KSC;
__global__ void k_scatter(const uint32_t* __restrict__ key, const uint32_t* __restrict__ slot,
                          const uint32_t* __restrict__ ids, const uint32_t* __restrict__ start, uint32_t n,
                          uint32_t* __restrict__ tsrc, uint32_t* __restrict__ tid, uint32_t* __restrict__ tkey,
                          const uint32_t* __restrict__ n_dev = nullptr) {
  pdl_wait();
  if (n_dev) n = __ldg(n_dev);
  if (blockIdx.x * (KSC * blockDim.x) >= n) return;
  const uint32_t i0 = blockIdx.x * (KSC * blockDim.x) + threadIdx.x;
  uint32_t k[KSC], sl[KSC], id[KSC], st[KSC];
#pragma unroll
  for (int u = 0; u < KSC; ++u) {
    const uint32_t i = i0 + u * blockDim.x;
    k[u] = i < n ? __ldg(&key[i]) : 0xffffffffu;
    sl[u] = i < n ? __ldg(&slot[i]) : 0u;
    id[u] = i < n ? __ldg(&ids[i]) : 0u;
  }
#pragma unroll
  for (int u = 0; u < KSC; ++u) st[u] = k[u] != 0xffffffffu ? __ldg(&start[k[u]]) : 0u;  // (dead: dropped)
#pragma unroll
  for (int u = 0; u < KSC; ++u) {
    if (k[u] == 0xffffffffu) continue;
    const uint32_t d = st[u] + sl[u];
    BDM_ASSERT(d < n);
    tsrc[d] = i0 + u * blockDim.x;
    tid[d] = id[u];
    tkey[d] = k[u];
  }
}

#ifndef BDM_PLACE_T
#define BDM_PLACE_T 256
#endif
constexpr int PLACE_T = BDM_PLACE_T;  // threads per k_place block
// Rank inside the box by id (boxes hold a handful of agents), then gather the payload.
__global__ void k_place(const uint32_t* __restrict__ tsrc, const uint32_t* __restrict__ tid,
                        const uint32_t* __restrict__ tkey, const uint32_t* __restrict__ start,
                        const double4* __restrict__ ag_in, uint32_t n, double4* __restrict__ ag_out,
                        uint32_t* __restrict__ ids_out, float4* __restrict__ agf_out,
                        const unsigned long long* __restrict__ hist_in, unsigned long long* __restrict__ hist_out,
                        const uint32_t* __restrict__ n_dev = nullptr, uint32_t* __restrict__ ids_owned = nullptr,
                        const uint32_t* __restrict__ ab_dev = nullptr) {
  pdl_wait();
  uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  if (n_dev) n = __ldg(n_dev);
  if (q >= n) return;
  const uint32_t k = tkey[q], id = tid[q], src = tsrc[q];
  const double4 p = ld_state(&ag_in[src]);  // (the gather is in flight during the rank loop)
  const uint32_t b = start[k], e = start[k + 1];
  uint32_t rank = 0;
#pragma unroll 4
  for (uint32_t t = b; t < e; ++t) rank += tid[t] < id;
  const uint32_t dst = b + rank;
  BDM_ASSERT(b <= q && q < e && dst < e);
  st_state(&ag_out[dst], p);
  ids_out[dst] = id;
  // distributed steps: the owned range [A_BEGIN, A_END) of this order is what the force phase steps;
  // its ids go straight to the stepped state's id buffer (compacted), so the sum pass need not copy them
  if (ids_owned) {
    const uint32_t ab = __ldg(&ab_dev[0]), ae = __ldg(&ab_dev[1]);
    if (dst >= ab && dst < ae) ids_owned[dst - ab] = id;
  }
  if (hist_out) hist_out[dst] = hist_in[src];
  // fp32 copy of the position for the force kernel's conservative candidate filter
  agf_out[dst] = make_float4(__double2float_rn(p.x), __double2float_rn(p.y), __double2float_rn(p.z),
                             -__double2float_rn(0.5 * p.w));  // -r: (z, -r) pairs with (z_i, r_i) in one FADD2
}

// ------------------------------------------------------------------------------------------ NEXT-1
// Stationary-region skip (§2.3(iv)).  Per agent the previous
// step leaves hist = moved-bit (bit 63, dp != 0) | packed box of the position before that step.
// A box is hot if some moved agent's new or old box lies within Chebyshev distance 1 of it.  An
// agent in a quiet box had no moving agent in its 27-box neighbourhood before or after the last
// step, so its candidate set, pair terms and canonical order are unchanged, and since it did not
// move its displacement was and stays exactly 0: the force kernel skips it, bit-identically.
constexpr int HB = 21;  // bits per packed box coordinate (|b| < 2^20)

__device__ __forceinline__ unsigned long long pack_box(int bx, int by, int bz) {
  const unsigned long long m = (1ull << HB) - 1ull;
  return ((unsigned long long)(bx + (1 << 20)) & m) | (((unsigned long long)(by + (1 << 20)) & m) << HB) |
         (((unsigned long long)(bz + (1 << 20)) & m) << (2 * HB));
}

__device__ __forceinline__ void unpack_box(unsigned long long v, int& bx, int& by, int& bz) {
  const unsigned long long m = (1ull << HB) - 1ull;
  bx = (int)(v & m) - (1 << 20);
  by = (int)((v >> HB) & m) - (1 << 20);
  bz = (int)((v >> (2 * HB)) & m) - (1 << 20);
}

// Warp per 32 sorted agents: the bounding region of the warp's movers' new and old boxes, grown by
// one box, is marked hot (conservative superset of every mover's two 3x3x3 neighbourhoods).
// Only boxes inside their column's occupied z-range exist (and only they can hold agents).
__global__ void k_mark_hot(const double4* __restrict__ ag, const unsigned long long* __restrict__ hist, uint32_t n,
                           GridDev g, uint8_t* __restrict__ bflag, int radius = 1, uint8_t value = 1) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const unsigned long long h = i < n ? hist[i] : 0ull;
  const bool moved = (h >> 63) != 0;
  if (!__any_sync(FULL, moved)) return;
  int lo[3] = {INT32_MAX, INT32_MAX, INT32_MAX}, hi[3] = {INT32_MIN, INT32_MIN, INT32_MIN};
  if (moved) {
    const double4 p = ag[i];
    const int nb[3] = {(int)floor(p.x * g.inv), (int)floor(p.y * g.inv), (int)floor(p.z * g.inv)};
    int ob[3];
    unpack_box(h & ~(1ull << 63), ob[0], ob[1], ob[2]);
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      lo[a] = min(nb[a], ob[a]) - radius;
      hi[a] = max(nb[a], ob[a]) + radius;
    }
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    lo[a] = __reduce_min_sync(FULL, lo[a]);
    hi[a] = __reduce_max_sync(FULL, hi[a]);
  }
  lo[0] = max(lo[0], g.lo[0]);
  hi[0] = min(hi[0], g.hi[0]);
  lo[1] = max(lo[1], g.lo[1]);
  hi[1] = min(hi[1], g.hi[1]);
  for (int cx = lo[0]; cx <= hi[0]; ++cx)
    for (int cy = lo[1]; cy <= hi[1]; ++cy) {
      const uint32_t c = col_of(g, cx, cy);
      const int zl = __ldg(&g.czlo[c]), zh = __ldg(&g.czhi[c]);
      const int a = max(lo[2], zl), d = min(hi[2], zh);
      if (a > d) continue;
      const uint32_t o = __ldg(&g.coff[c]) + (uint32_t)(a - zl);
      for (int t = lane; t <= d - a; t += 32) bflag[o + t] = value;
    }
}

// zero box flags [0 .. T] (T = coff[nc] on the device)
__global__ void k_flag_zero(uint8_t* __restrict__ bflag, const uint32_t* __restrict__ coff, uint32_t nc) {
  const uint32_t T = coff[nc];
  uint32_t* w = reinterpret_cast<uint32_t*>(bflag);
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k <= T / 4; k += gridDim.x * blockDim.x) w[k] = 0u;
}

// ------------------------------------------------------------------------------------------ K6
#ifndef BDM_TICKET
#define BDM_TICKET 4
#endif
// Chunk tickets of the persistent kernels: a warp takes BDM_TICKET consecutive 32-agent chunks per
// atomic on the (single, same-address) work counter -- one atomic per chunk serialises in L2.
// Small populations keep one chunk per ticket while a warp would get fewer than 8 tickets (tail balance).
struct Tickets {
  uint32_t next = 0, left = 0, per = 1;
  __device__ __forceinline__ explicit Tickets(uint64_t n_agents) {
    const uint64_t chunks = (n_agents + 31) / 32, warps = (uint64_t)gridDim.x * (blockDim.x / 32);
    const uint64_t k = chunks / (warps * 8 + 1);
    per = k < 1 ? 1u : (k > (uint64_t)BDM_TICKET ? (uint32_t)BDM_TICKET : (uint32_t)k);
  }
  __device__ __forceinline__ uint32_t take(uint32_t* work, int lane) {
    if (left == 0) {
      uint32_t t = 0;
      if (lane == 0) t = atomicAdd(work, 1u);
      next = __shfl_sync(0xffffffffu, t, 0) * per;
      left = per;
    }
    --left;
    return next++;
  }
};

constexpr int FORCE_THREADS = 256;
constexpr int FORCE_WARPS = FORCE_THREADS / 32;
#ifndef BDM_FORCE_MIN_BLOCKS
#define BDM_FORCE_MIN_BLOCKS 3
#endif
constexpr int FORCE_MIN_BLOCKS = BDM_FORCE_MIN_BLOCKS;  // 3: 24 resident warps per SM
#ifndef BDM_NSLOT
#define BDM_NSLOT 3  // candidate slots per iteration of the candidate loops (k_force, pass A)
#endif
constexpr int NSLOT = BDM_NSLOT;
#ifndef BDM_CURSOR
#define BDM_CURSOR 0  // candidate cursor of k_force: 0 flattened per slot, 1 range-granular
#endif
constexpr int LCAP = 16;             // per-lane survivor list capacity (flushed before overflow)

#ifndef BDM_PTSPEC
#define BDM_PTSPEC 1
#endif
// One contact candidate of agent i (O4), returns false if delta <= 0.
// i, j are sorted indices; ids[] is read only for coincident centres (the R8 tie-break, rare).
__device__ __forceinline__ bool pair_term(double xi, double yi, double zi, double ri, uint32_t i, const double4& o,
                                          const uint32_t* __restrict__ ids, uint32_t j, const ParamsDev& p, double& tx,
                                          double& ty, double& tz, double& fabs_out) {
  double dx = xi - o.x;
  double dy = yi - o.y;
  double dz = zi - o.z;
  double d2 = (dx * dx + dy * dy) + dz * dz;
  double rj = 0.5 * o.w;
  double s = ri + rj;
#if BDM_PTSPEC
  // (the reduced radius first: its division then overlaps the square root instead of following the
  // contact test -- nearly every candidate that reaches here is a contact)
  double r = (ri * rj) / s;
  double d = sqrt(d2);
  double delta = s - d;
  if (!(delta > 0.0)) return false;
#else
  double d = sqrt(d2);
  double delta = s - d;
  if (!(delta > 0.0)) return false;
  double r = (ri * rj) / s;
#endif
  double f = p.k_rep * delta - p.gamma_att * sqrt(r * delta);
  fabs_out = fabs(f);
  if (d2 == 0.0) {  // coincident centres (R8)
    tx = __ldg(&ids[i]) > __ldg(&ids[j]) ? f : -f;
    ty = 0.0;
    tz = 0.0;
    return true;
  }
  double m = f / d;
  tx = m * dx;
  ty = m * dy;
  tz = m * dz;
  return true;
}

constexpr int TSPAN = 40;  // box-start window per neighbour column staged by a single-column chunk

struct ForceSmem {
  uint32_t list[LCAP][32];  // survivors per lane (sorted index of the candidate), candidate order
  double term[3][32];       // contact terms of one compacted batch
  uint32_t cidx[32];        // candidate id of the batch entry, 0xffffffff = not a contact
  uint32_t rb[9][32], re[9][32];
  uint32_t tab[9][TSPAN];   // box starts start(c, z) for z in [zf-1, zl+2] of the 9 neighbour columns
};
constexpr size_t FORCE_SMEM_BYTES = sizeof(ForceSmem) * FORCE_WARPS;

// Contact phase over the survivors of the warp (DESIGN.md §6.3 step 3).  The survivors of all lanes
// are enumerated as one flat sequence (lane-major, candidate order inside a lane); each batch of 32
// is evaluated with one entry per lane (owner found by a shuffle binary search over the inclusive
// prefix of list lengths), then every owner adds its own entries of the batch in order -- so each
// agent's force is summed in O5's canonical order.
template <bool RECORD, class Smem>
__device__ __forceinline__ void flush_contacts(Smem& sm, int lane, int& cnt, double xi, double yi, double zi,
                                               double ri, uint32_t ii, const double4* __restrict__ ag,
                                               const uint32_t* __restrict__ ids, const ParamsDev& p, double& Fx,
                                               double& Fy, double& Fz, int32_t& n_ct,
                                               unsigned long long& ct_hash) {
  const int incl = warp_incl_scan((uint32_t)cnt);
  const int excl = incl - cnt;
  const int total = __shfl_sync(FULL, incl, 31);
  for (int b0 = 0; b0 < total; b0 += 32) {
    const int e = b0 + lane;
    int owner = 0;
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) {
      int v = __shfl_sync(FULL, incl, owner + s - 1);
      if (v <= e) owner += s;
    }
    owner = owner > 31 ? 31 : owner;
    const int oexcl = __shfl_sync(FULL, excl, owner);
    const double ox = __shfl_sync(FULL, xi, owner);
    const double oy = __shfl_sync(FULL, yi, owner);
    const double oz = __shfl_sync(FULL, zi, owner);
    const double orr = __shfl_sync(FULL, ri, owner);
    const uint32_t oidx = __shfl_sync(FULL, ii, owner);
    uint32_t flag = 0xffffffffu;
    if (e < total) {
      const uint32_t j = sm.list[e - oexcl][owner];
      const double4 o = ld_state(&ag[j]);
      double tx, ty, tz, fa;
      if (pair_term(ox, oy, oz, orr, oidx, o, ids, j, p, tx, ty, tz, fa)) {
        sm.term[0][lane] = tx;
        sm.term[1][lane] = ty;
        sm.term[2][lane] = tz;
        flag = RECORD ? ids[j] : 0u;  // id for the contact digest; any value != ~0 marks a contact
      }
    }
    // which batch entries are contacts: a ballot (the id for the RECORD digest goes through cidx)
    const unsigned cmask = __ballot_sync(FULL, flag != 0xffffffffu);
    if (RECORD) sm.cidx[lane] = flag;
    __syncwarp();
    const int lo = excl > b0 ? excl : b0;
    const int hi = incl < b0 + 32 ? incl : b0 + 32;
    for (int x = lo; x < hi; ++x) {
      const int t = x - b0;
      const uint32_t fl = RECORD ? sm.cidx[t] : 0u;
      if ((cmask >> t) & 1u) {
        Fx = Fx + sm.term[0][t];
        Fy = Fy + sm.term[1][t];
        Fz = Fz + sm.term[2][t];
        if (RECORD) {
          ++n_ct;
          ct_hash += mix64(fl);
        }
      }
    }
    __syncwarp();
  }
  cnt = 0;
}

// K6.  Persistent warps take chunks of 32 consecutive sorted agents from an atomic counter
// (load balance without block barriers).  Lane = agent.  Candidate phase: warp-uniform loop over
// the 9 columns (dx, dy) lexicographic; inside a column each lane walks its own z-run
// [start(bz-1), start(bz+2)) two candidates per iteration (independent loads and d2 chains), and
// keeps candidates passing the conservative bound d2 <= (r_i + L/2)^2 (1 + 2^-50) (contact implies
// d2 < (r_i + r_j)^2 <= (r_i + L/2)^2).  Agents [a_begin, a_end) of the sorted array are updated
// (the whole array is the environment, so slab ghosts are read but not moved); p' goes to
// ag_out[i - a_begin] (and ids to id_out if given).
template <bool RECORD>
__global__ void __launch_bounds__(FORCE_THREADS, FORCE_MIN_BLOCKS)
    k_force(const double4* __restrict__ ag, const float4* __restrict__ agf, const uint32_t* __restrict__ ids,
            uint32_t a_begin, uint32_t a_end, GridDev g, ParamsDev p, double4* __restrict__ ag_out,
            uint32_t* __restrict__ id_out, double* __restrict__ dp_out, uint32_t* __restrict__ dp_id_out,
            Extents* ext_next, ErrDev* err, RecordDev rec, const uint8_t* __restrict__ hot,
            unsigned long long* __restrict__ hist_out, double* __restrict__ f_out) {
  extern __shared__ __align__(16) unsigned char s_raw[];  // FORCE_WARPS x ForceSmem (dynamic)
  ForceSmem* s_all = reinterpret_cast<ForceSmem*>(s_raw);
  const int lane = threadIdx.x & 31;
  ForceSmem& sm = s_all[threadIdx.x >> 5];
  int elo[3] = {INT32_MAX, INT32_MAX, INT32_MAX}, ehi[3] = {INT32_MIN, INT32_MIN, INT32_MIN};
  bool ebad = false;
  uint32_t n_moved = 0, n_searched = 0;  // skip statistics of this warp

  Tickets tk(a_end - a_begin);
  while (true) {
    const uint32_t chunk = tk.take(&ext_next->work, lane);
    const uint64_t base = (uint64_t)a_begin + 32ull * chunk;
    if (base >= a_end) break;
    const uint32_t i = (uint32_t)base + lane;
    const bool valid = i < a_end;
    const double4 me = valid ? ld_state(&ag[i]) : make_double4(0.0, 0.0, 0.0, 0.0);
    const uint32_t myid = valid ? ids[i] : 0u;
    const double ri = 0.5 * me.w;
    const int bx = (int)floor(me.x * g.inv), by = (int)floor(me.y * g.inv), bz = (int)floor(me.z * g.inv);
    // skip mode: quiet agents (no moving agent around them, NEXT-1) do not search: F = 0 exactly
    const bool search = valid && (hot == nullptr || hot[box_key(g, bx, by, bz)] != 0);
    double thr = (ri + g.thr_pad) * (ri + g.thr_pad);
    thr = thr + thr * 0x1p-50;
    // fp32 bound: (r_i + L/2 + m32)^2 (1 + 2^-20), rounded up
    const double rp = (ri + g.thr_pad + g.m32) * (1.0 + 0x1p-20);
    const float thr32 = __double2float_ru(rp * rp);
    const float4 mf = valid ? __ldg(&agf[i]) : make_float4(0.f, 0.f, 0.f, 0.f);
    // Box culling (product kernel only): a neighbour box can hold a contact only if its region
    // comes within R_i = r_i + L/2 of p_i (contact => d < r_i + r_j <= R_i).  fx/gx are the
    // distances from p_i to the lower/upper x faces of its own box (clamped at 0 against rounding of
    // floor(x*inv)); the bound is padded by the fp32 margin (>= 2^-18 um >> fp64 rounding here).
    // RECORD counts all 27-box candidates (O3) and does not cull.
    const double Lb = 1.0 / g.inv;
    const double fx = fmax(me.x - bx * Lb, 0.0), gx = fmax((bx + 1) * Lb - me.x, 0.0);
    const double fy = fmax(me.y - by * Lb, 0.0), gy = fmax((by + 1) * Lb - me.y, 0.0);
    const double fz = fmax(me.z - bz * Lb, 0.0), gz = fmax((bz + 1) * Lb - me.z, 0.0);
    const double Rc = rp + g.m32;
    const double Rc2 = Rc * Rc;
    int nr = 0;  // non-empty ranges of this lane, compacted in canonical (dx, dy) order
    // Chunks whose agents all sit in one column (bx, by) -- most chunks in dense regions -- look
    // the 9 neighbour columns up once per warp: lane c < 9 reads column c's descriptor, then the
    // warp stages start(c, z) for z in [zf-1, zl+2] with coalesced loads; lanes then read their
    // z-runs from shared memory instead of 9 dependent global lookups each.
    const unsigned smask = __ballot_sync(FULL, search);
    const int src0 = smask ? __ffs(smask) - 1 : 0;
    const int bx0 = __shfl_sync(FULL, bx, src0), by0 = __shfl_sync(FULL, by, src0);
    const int zf = __reduce_min_sync(FULL, search ? bz : INT32_MAX);
    const int zl = __reduce_max_sync(FULL, search ? bz : INT32_MIN);
    const bool coop = !RECORD && __any_sync(FULL, search) &&
                      __all_sync(FULL, !search || (bx == bx0 && by == by0)) && zl - zf + 4 <= TSPAN;
    if (coop) {
      int czl = 0, cze = 0;  // column descriptor: first occupied z, number of occupied z
      uint32_t cof = 0;
      if (lane < 9) {
        const int cx = bx0 + lane / 3 - 1, cy = by0 + lane % 3 - 1;
        if (cx >= g.lo[0] && cx <= g.hi[0] && cy >= g.lo[1] && cy <= g.hi[1]) {
          const uint32_t cc = col_of(g, cx, cy);
          czl = __ldg(&g.czlo[cc]);
          const int czh = __ldg(&g.czhi[cc]);
          cof = __ldg(&g.coff[cc]);
          cze = czh >= czl ? czh - czl + 1 : 0;
        } else {
          cof = 0xffffffffu;  // outside the grid: no agents
        }
      }
      const int span = zl - zf + 4;
      // stage start(c, z) = table[coff + clamp(z - zlo, 0, ext)] for all 9 x span entries at once
      // (flattened so that every lane has its loads in flight together)
      const int total = 9 * span;
#pragma unroll 2
      for (int t0 = 0; t0 < total; t0 += 32) {
        const int t = t0 + lane;
        const int c = t / span < 8 ? t / span : 8;
        const int zlo_c = __shfl_sync(FULL, czl, c), ext_c = __shfl_sync(FULL, cze, c);
        const uint32_t off_c = __shfl_sync(FULL, cof, c);
        if (t < total) {
          uint32_t v = 0u;
          const int tt = t - c * span;
          if (off_c != 0xffffffffu) {
            int k = zf - 1 + tt - zlo_c;
            k = k < 0 ? 0 : (k > ext_c ? ext_c : k);
            v = __ldg(&g.table[off_c + (uint32_t)k]);
          }
          sm.tab[c][tt] = v;
        }
      }
      __syncwarp();
    }
#pragma unroll
    for (int c = 0; c < 9; ++c) {
      const int ddx = c / 3 - 1, ddy = c % 3 - 1;
      uint32_t b = 0, e = 0;
      if (search) {
        int z0 = bz - 1, z1 = bz + 1;
        bool keep = true;
        if (!RECORD) {
          const double ex = ddx < 0 ? fx : (ddx > 0 ? gx : 0.0);
          const double ey = ddy < 0 ? fy : (ddy > 0 ? gy : 0.0);
          const double exy2 = ex * ex + ey * ey;
          keep = exy2 <= Rc2;
          if (exy2 + fz * fz > Rc2) z0 = bz;
          if (exy2 + gz * gz > Rc2) z1 = bz;
        }
        if (keep) {
          if (coop) {
            b = sm.tab[c][z0 - zf + 1];
            e = sm.tab[c][z1 - zf + 2];
          } else {
            zrun(g, bx + ddx, by + ddy, z0, z1, b, e);
          }
        }
      }
      if (RECORD) {
        sm.rb[c][lane] = b;
        sm.re[c][lane] = e;
      } else if (b < e) {
        sm.rb[nr][lane] = b;
        sm.re[nr][lane] = e;
        ++nr;
      }
    }
    __syncwarp();
    double Fx = 0.0, Fy = 0.0, Fz = 0.0;
    int cnt = 0;
    int32_t n_cand = 0, n_nb = 0, n_ct = 0;
    unsigned long long nb_hash = 0, ct_hash = 0;
    if (RECORD) {
      for (int c = 0; c < 9; ++c) {
        uint32_t q = sm.rb[c][lane];
        const uint32_t e = sm.re[c][lane];
        while (__any_sync(FULL, q < e)) {
          const bool a0 = q < e && q != i;
          const bool a1 = q + 1 < e && q + 1 != i;
          // exact fp64 test of every candidate: the per-agent neighbour statistics need d2 <= L2
          double3 o0 = make_double3(0.0, 0.0, 0.0), o1 = make_double3(0.0, 0.0, 0.0);
          if (a0) {
            const double2 xy = __ldg(reinterpret_cast<const double2*>(ag + q));
            o0 = make_double3(xy.x, xy.y, __ldg(&ag[q].z));
          }
          if (a1) {
            const double2 xy = __ldg(reinterpret_cast<const double2*>(ag + q + 1));
            o1 = make_double3(xy.x, xy.y, __ldg(&ag[q + 1].z));
          }
          const double dx0 = me.x - o0.x, dy0 = me.y - o0.y, dz0 = me.z - o0.z;
          const double dx1 = me.x - o1.x, dy1 = me.y - o1.y, dz1 = me.z - o1.z;
          const double d20 = (dx0 * dx0 + dy0 * dy0) + dz0 * dz0;
          const double d21 = (dx1 * dx1 + dy1 * dy1) + dz1 * dz1;
          n_cand += (int)a0 + (int)a1;
          if (a0 && d20 <= g.L2) {
            ++n_nb;
            nb_hash += mix64(ids[q]);
          }
          if (a1 && d21 <= g.L2) {
            ++n_nb;
            nb_hash += mix64(ids[q + 1]);
          }
          if (a0 && d20 <= thr) sm.list[cnt++][lane] = q;
          if (a1 && d21 <= thr) sm.list[cnt++][lane] = q + 1;
          q += 2;
          if (__any_sync(FULL, cnt > LCAP - 2))
            flush_contacts<RECORD, ForceSmem>(sm, lane, cnt, me.x, me.y, me.z, ri, i, ag, ids, p, Fx, Fy, Fz, n_ct, ct_hash);
        }
      }
    } else {
      // Flattened cursor over this lane's culled non-empty ranges (canonical order), four candidate
      // slots per iteration: the warp iterates max over lanes of the lane's TOTAL work rather than
      // the sum over columns of per-column maxima.  Conservative fp32 test against the pair bound
      // (r_i + r_j + m32)^2 (1 + 2^-20): only candidates that can be contacts reach
      // the exact fp64 evaluation.
      const float ri32 = __double2float_ru(ri + g.m32);
      const unsigned long long mxy = pack2(mf.x, mf.y), mzr = pack2(mf.z, ri32);
      int k = 0;
      bool live = nr > 0;
      uint32_t q = live ? sm.rb[0][lane] : 0u, e = live ? sm.re[0][lane] : 0u;
      while (__any_sync(FULL, live)) {
        uint32_t qs[NSLOT];
        bool as[NSLOT];
#if BDM_CURSOR == 0
#pragma unroll
        for (int t = 0; t < NSLOT; ++t) {
          as[t] = live && q != i;
          qs[t] = live ? q : i;
          if (live && ++q == e) {
            ++k;
            live = k < nr;
            if (live) {
              q = sm.rb[k][lane];
              e = sm.re[k][lane];
            }
          }
        }
#else
        // range-granular cursor: the NSLOT slots come from the current range only (slots past its end
        // idle); one range switch per iteration at most
#pragma unroll
        for (int t = 0; t < NSLOT; ++t) {
          const uint32_t qt = q + (uint32_t)t;
          as[t] = live && qt < e && qt != i;
          qs[t] = as[t] ? qt : i;
        }
        q += (uint32_t)NSLOT;
        if (live && q >= e) {
          ++k;
          live = k < nr;
          if (live) {
            q = sm.rb[k][lane];
            e = sm.re[k][lane];
          }
        }
#endif
        float4 o[NSLOT];
#pragma unroll
        for (int t = 0; t < NSLOT; ++t) o[t] = __ldg(&agf[qs[t]]);
#pragma unroll
        for (int t = 0; t < NSLOT; ++t) {
          // packed fp32x2 (FADD2/FMUL2): (dx, dy) = (x_i, y_i) - (x_j, y_j); (dz, s) = (z_i, r_i) - (z_j, -r_j)
          float2 dxy, dzs;
          asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(*reinterpret_cast<unsigned long long*>(&dxy))
              : "l"(mxy), "l"(pack2(o[t].x, o[t].y)));
          asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(*reinterpret_cast<unsigned long long*>(&dzs))
              : "l"(mzr), "l"(pack2(o[t].z, o[t].w)));
          float2 sq, qz;
          asm("mul.rn.f32x2 %0, %1, %1;" : "=l"(*reinterpret_cast<unsigned long long*>(&sq))
              : "l"(*reinterpret_cast<unsigned long long*>(&dxy)));
          asm("mul.rn.f32x2 %0, %1, %1;" : "=l"(*reinterpret_cast<unsigned long long*>(&qz))
              : "l"(*reinterpret_cast<unsigned long long*>(&dzs)));
          const float d2 = (sq.x + sq.y) + qz.x;
          if (as[t] && d2 <= __fmaf_rn(qz.y, 0x1p-20f, qz.y)) sm.list[cnt++][lane] = qs[t];
        }
        if (__any_sync(FULL, cnt > LCAP - NSLOT))
          flush_contacts<RECORD, ForceSmem>(sm, lane, cnt, me.x, me.y, me.z, ri, i, ag, ids, p, Fx, Fy, Fz, n_ct, ct_hash);
      }
    }
    if (__any_sync(FULL, cnt > 0))
      flush_contacts<RECORD, ForceSmem>(sm, lane, cnt, me.x, me.y, me.z, ri, i, ag, ids, p, Fx, Fy, Fz, n_ct, ct_hash);

    if (f_out) {  // force-only mode (NEXT-4): the sphere-sphere sum goes to a later kernel
      if (valid) {
        const uint32_t o = i - a_begin;
        f_out[3 * (size_t)o] = Fx;
        f_out[3 * (size_t)o + 1] = Fy;
        f_out[3 * (size_t)o + 2] = Fz;
      }
      continue;
    }
    // O6 displacement, O7 update
    double dpx = 0.0, dpy = 0.0, dpz = 0.0;
    int branch = 0;
    const double fn = sqrt((Fx * Fx + Fy * Fy) + Fz * Fz);
    if (fn <= p.adherence) {
      branch = 0;
    } else if (fn * p.c > p.max_disp) {
      const double scale = p.max_disp / fn;
      dpx = Fx * scale;
      dpy = Fy * scale;
      dpz = Fz * scale;
      branch = 1;
    } else {
      dpx = Fx * p.c;
      dpy = Fy * p.c;
      dpz = Fz * p.c;
      branch = 2;
    }
    if (valid) {
      if (!(isfinite(Fx) && isfinite(Fy) && isfinite(Fz) && isfinite(fn))) report(err, 6u /*ENONFINITE*/, myid, i);
      const double4 np = make_double4(me.x + dpx, me.y + dpy, me.z + dpz, me.w);
      const uint32_t o = i - a_begin;
      st_state(&ag_out[o], np);
      if (hist_out) {
        const bool moved = dpx != 0.0 || dpy != 0.0 || dpz != 0.0;
        hist_out[o] = ((unsigned long long)moved << 63) | pack_box(bx, by, bz);
      }
      if (id_out) id_out[o] = myid;
      if (dp_out) {
        dp_out[3 * (size_t)o] = dpx;
        dp_out[3 * (size_t)o + 1] = dpy;
        dp_out[3 * (size_t)o + 2] = dpz;
        if (dp_id_out) dp_id_out[o] = myid;
      }
      const int nb3[3] = {box_coord(np.x, g.inv, ebad), box_coord(np.y, g.inv, ebad), box_coord(np.z, g.inv, ebad)};
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        elo[a] = min(elo[a], nb3[a]);
        ehi[a] = max(ehi[a], nb3[a]);
      }
      if (RECORD) {
        rec.n_cand[o] = n_cand;
        rec.n_nb[o] = n_nb;
        rec.n_ct[o] = n_ct;
        rec.branch[o] = (int8_t)branch;
        rec.nb_hash[o] = nb_hash;
        rec.ct_hash[o] = ct_hash;
      }
    }
    if (hist_out) {  // counted per warp, added once at the end (a same-address atomic per chunk serialises)
      n_moved += __popc(__ballot_sync(FULL, valid && (dpx != 0.0 || dpy != 0.0 || dpz != 0.0)));
      n_searched += __popc(__ballot_sync(FULL, search));
    }
  }
  if (hist_out && lane == 0) {
    if (n_moved) atomicAdd(&ext_next->moved, n_moved);
    if (n_searched) atomicAdd(&ext_next->searched, n_searched);
  }
  // next step's extents: one guarded atomic set per warp (a few thousand warps per launch)
  if (__any_sync(FULL, ebad) && lane == 0) ext_next->range_err = 1;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const int lo = __reduce_min_sync(FULL, elo[a]);
    const int hi = __reduce_max_sync(FULL, ehi[a]);
    if (lane == 0) {
      if (lo != INT32_MAX && lo < __ldcg(&ext_next->lo[a])) atomicMin(&ext_next->lo[a], lo);
      if (hi != INT32_MIN && hi > __ldcg(&ext_next->hi[a])) atomicMax(&ext_next->hi[a], hi);
    }
  }
}

// ------------------------------------------------------------------------------------------ K6h
// Half-shell force path, used for plain steps (no statistics, no stationary-region
// skip, no neurites).  Newton's third law (R2: F_ji = -F_ij bit-exactly) lets each candidate pair
// be TESTED once instead of twice:
//   pass A, k_half_search: agent i walks only the half of its 27-box neighbourhood that follows it in
//     the sorted order (the rest of its own box after i, the box above in its column, and the 13
//     boxes of larger key: columns (0,+1), (+1,-1), (+1,0), (+1,+1)), with the conservative fp32
//     filter of k_force.  A surviving pair (i, j), i < j in sorted order, goes to i's forward row
//     (ascending j: the walk is in sorted order) and, through an atomic slot, to j's backward row;
//   pass B, k_half_sum: agent i evaluates the exact fp64 term (O4) of every pair of its backward row
//     (sorted ascending first) then of its forward row -- i.e. of all its contacts in ascending
//     sorted order = O5's canonical order (boxes in key order, ascending id inside a box) -- with
//     the balanced contact phase of k_force, then O6/O7.  So Δp is bit-identical to k_force's.
// Rows hold HFC / HBC entries; an agent whose row overflowed takes a slow path in pass B (a full
// 27-box canonical search of its own), so the result does not depend on the capacities.
#ifndef BDM_HROW
#define BDM_HROW 16
#endif
constexpr int HFC = BDM_HROW;  // forward row capacity (entries per agent; merged rows: all its entries)
constexpr int HBC = BDM_HROW;  // backward row capacity
#ifndef BDM_HLA
#define BDM_HLA 16
#endif
constexpr int HLA = BDM_HLA;  // pass A survivor buffer per lane (shared memory)
#ifndef BDM_HBCNT
#define BDM_HBCNT 1  // pass B loads the next chunk's pair counts one chunk ahead
#endif
#ifndef BDM_HAPF
#define BDM_HAPF 1  // pass A loads the next chunk's fp32 agents one chunk ahead
#endif
#ifndef BDM_HA32
#define BDM_HA32 1  // pass A takes boxes and radii from the fp32 copy (fp64 position only near box faces)
#endif
#ifndef BDM_HA_THREADS
#define BDM_HA_THREADS 256
#endif
constexpr int HA_THREADS = BDM_HA_THREADS;
#ifndef BDM_HA_MIN_BLOCKS
#define BDM_HA_MIN_BLOCKS 5
#endif
#ifndef BDM_HB_MIN_BLOCKS
#define BDM_HB_MIN_BLOCKS 4
#endif
constexpr int HA_MIN_BLOCKS = BDM_HA_MIN_BLOCKS;  // pass A: 5 x 8 resident warps per SM (48 registers)
constexpr int HB_MIN_BLOCKS = BDM_HB_MIN_BLOCKS;  // pass B

#ifndef BDM_HMAP
#define BDM_HMAP 0  // pass A cursor: 0 shared-memory run list with predicated refills, 1 closed-form map
#endif
#ifndef BDM_HSTAGE
#define BDM_HSTAGE 0  // 1: pass A single-column chunks read candidates from a TMA-staged shared copy (measured slower)
#endif
#ifndef BDM_HPCAP
#define BDM_HPCAP 256
#endif
constexpr int HPCAP = BDM_HPCAP;  // staged candidates (float4) per warp

#define HA_RR (!BDM_HMAP || BDM_HSTAGE)  // the shared-memory run list (cursor with refills)
#ifndef BDM_HDEF
#define BDM_HDEF 1  // pass A: a chunk's row stores deferred to the next chunk (the atomics' latency hidden)
#endif
#ifndef BDM_HLST
#define BDM_HLST 1  // pass A: survivor appends through a precomputed shared address
#endif
#ifndef BDM_HBATCH
#define BDM_HBATCH 1  // pass A: the z-run lookups of the 5 forward columns batched in two load levels
#endif
#ifndef BDM_HCOOP
#define BDM_HCOOP BDM_HSTAGE  // single-column chunks stage their box starts cooperatively (needed by BDM_HSTAGE;
                              // per-lane lookups are slightly faster otherwise)
#endif
struct HalfASmem {
#if BDM_HSTAGE
  float4 buf[HPCAP];        // fp32 candidates of the 5 forward columns' union z-runs (staged chunks)
  unsigned long long bar;   // mbarrier of the bulk copies into buf
  uint32_t off[6];          // buffer offset of each column's union run (off[5] = total)
  uint32_t ub[5];           // global sorted index of each union run's first agent
  uint32_t pad_;
#endif
  uint32_t list[HLA][32];  // survivors (sorted index j, or staged buffer index) of this lane, ascending
  uint2 rr[7][32];         // this lane's non-empty forward z-runs [b, e), then the sentinel
  uint32_t tab[5][BDM_HCOOP ? TSPAN : 1];  // box starts of the 5 forward columns (cooperative lookups only:
                                           // otherwise the shared memory goes to L1)
};

// ---- TMA bulk copies (cp.async.bulk, async proxy) completing on a per-warp mbarrier
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
constexpr size_t HA_SMEM_BYTES = sizeof(HalfASmem) * (HA_THREADS / 32);

#ifndef BDM_MROW
#define BDM_MROW 1  // one merged pair row per agent (forward and backward entries under one counter)
#endif
#ifndef BDM_HRPF
#define BDM_HRPF 0  // pass B: counts two chunks ahead, first row vector one chunk ahead (merged rows; spills: slower)
#endif
#ifndef BDM_HDIRECT
#define BDM_HDIRECT 0  // pass B: each lane evaluates its own contacts (instead of the balanced contact phase)
#endif
#ifndef BDM_HNPF
#define BDM_HNPF 2  // pass B: prefetch the next chunk's row (1: measured slower) and / or state (2) into L1
#endif
#ifndef BDM_HNET
#define BDM_HNET 1  // pass B: rows of <= 4 entries sorted by a register sorting network (else insertion sort)
#endif
#ifndef BDM_HPPF
#define BDM_HPPF 1  // pass B: partner states prefetched into L1 as soon as the row is read
#endif
// BDM_MROW: agent j's row fwd[j * HFC ..] holds all its pair candidates, forward (found by its own
// search) and backward (found by partners' searches), packed from the front in arrival order through
// one atomic counter bcnt[j]; the sum pass sorts the row.  A typical agent's entries then share one
// 32-byte sector (instead of one sector in each of two rows): the sum pass reads half the row bytes.
// Otherwise: a forward row written by the owner and a backward row (bwd, bcnt) filled by partners.
__device__ __forceinline__ void bw_put(uint32_t* __restrict__ fwd, uint32_t* __restrict__ bwd,
                                       uint32_t j, uint32_t slot, uint32_t i, uint32_t rm) {
  if (slot < (uint32_t)HBC) (BDM_MROW ? fwd : bwd)[(size_t)(j & rm) * HBC + slot] = i;
}

// End of a chunk (lane of agent i, cnt survivors in its list, extra beyond it): the forward entries
// of i and one backward entry per pair through an atomic slot of the partner.  Separate rows: the
// forward row as whole 32-byte sectors (entries past cnt are don't-care; full sectors avoid
// read-modify-write of partially written sectors in DRAM).
__device__ __forceinline__ void half_emit(HalfASmem& sm, int lane, int cnt, uint32_t extra, uint32_t i,
                                          uint32_t* __restrict__ fwd, uint32_t* __restrict__ bwd,
                                          uint32_t* __restrict__ bcnt, uint32_t rm) {
#if BDM_MROW
  // own entries: a base slot for all of them (the overflow beyond the list counts, so a row that
  // cannot hold everything is recognised by its count); its round trip overlaps the partners' atomics
  // (survivors beyond the list were not kept: push the count past the row so the sum pass takes the
  // exact full search for i)
  const uint32_t nf = (uint32_t)cnt + extra + (extra ? (uint32_t)HFC : 0u);
  const uint32_t base = nf ? atomicAdd(&bcnt[i & rm], nf) : 0u;
#elif BDM_V256
  uint32_t* frow = fwd + (size_t)(i & rm) * HFC;  // 64-byte rows: one 256-bit store per used sector
#pragma unroll
  for (int v = 0; v < HFC / 8; ++v)
    if (cnt > 8 * v) {
      const uint32_t* l = &sm.list[8 * v][lane];
      asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(frow + 8 * v), "r"(l[0]),
                   "r"(l[32]), "r"(l[64]), "r"(l[96]), "r"(l[128]), "r"(l[160]), "r"(l[192]), "r"(l[224])
                   : "memory");
    }
#else
  uint4* frow = reinterpret_cast<uint4*>(fwd + (size_t)(i & rm) * HFC);
#pragma unroll
  for (int v = 0; v < HFC / 4; ++v)
    if (cnt > 8 * (v / 2))
      frow[v] = make_uint4(sm.list[4 * v][lane], sm.list[4 * v + 1][lane], sm.list[4 * v + 2][lane],
                           sm.list[4 * v + 3][lane]);
#endif
  for (int x0 = 0; x0 < cnt; x0 += 4) {
    uint32_t j[4], slot[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      j[u] = x0 + u < cnt ? sm.list[x0 + u][lane] : 0u;
      if (x0 + u < cnt) slot[u] = atomicAdd(&bcnt[j[u] & rm], 1u);  // four atomics in flight
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (x0 + u < cnt) {
        BDM_ASSERT(j[u] > i);  // forward partners only (the half-shell order)
        bw_put(fwd, bwd, j[u], slot[u], i, rm);
      }
  }
#if BDM_MROW
  uint32_t* row = fwd + (size_t)(i & rm) * HFC;
  for (int k = 0; k < cnt; ++k)
    if (base + (uint32_t)k < (uint32_t)HFC) row[base + k] = sm.list[k][lane];
#endif
}

#if BDM_MROW
// BDM_HDEF: half_emit in two halves.  At a chunk's end the atomics are issued (the owner's base slot,
// a slot in each of the first four partners' rows; a fifth survivor onwards is emitted at once, rare);
// the stores that need their results are done at the next chunk, after its set-up, so the atomics'
// round trip hides behind that chunk's dependent loads.  sm.list still holds the survivors then.
struct HalfPending {
  uint32_t i, base, cnt;  // cnt = 0: nothing pending
  uint32_t slot[4];
};
__device__ __forceinline__ void half_emit_issue(HalfASmem& sm, int lane, int cnt, uint32_t extra, uint32_t i,
                                                uint32_t* __restrict__ fwd, uint32_t* __restrict__ bcnt,
                                                HalfPending& pd, uint32_t rm) {
  const uint32_t nf = (uint32_t)cnt + extra + (extra ? (uint32_t)HFC : 0u);
  pd.base = nf ? atomicAdd(&bcnt[i & rm], nf) : 0u;
  pd.i = i;
  pd.cnt = (uint32_t)cnt;
#pragma unroll
  for (int u = 0; u < 4; ++u)
    if (u < cnt) pd.slot[u] = atomicAdd(&bcnt[sm.list[u][lane] & rm], 1u);
  for (int x = 4; x < cnt; ++x) {  // (rare)
    const uint32_t j = sm.list[x][lane];
    bw_put(fwd, fwd, j, atomicAdd(&bcnt[j & rm], 1u), i, rm);
  }
}
__device__ __forceinline__ void half_emit_finish(HalfASmem& sm, int lane, uint32_t* __restrict__ fwd,
                                                 HalfPending& pd, uint32_t rm) {
  if (pd.cnt == 0u) return;
#pragma unroll
  for (int u = 0; u < 4; ++u)
    if ((uint32_t)u < pd.cnt) {
      BDM_ASSERT(sm.list[u][lane] > pd.i);
      bw_put(fwd, fwd, sm.list[u][lane], pd.slot[u], pd.i, rm);
    }
  uint32_t* row = fwd + (size_t)(pd.i & rm) * HFC;
  for (uint32_t k = 0; k < pd.cnt; ++k)
    if (pd.base + k < (uint32_t)HFC) row[pd.base + k] = sm.list[k][lane];
  pd.cnt = 0u;
}
#endif

// Candidate loop of pass A over this lane's runs rr[] (flattened, branch-free run switch): fp32
// conservative filter of k_force; survivors to the lane's list (STAGED: runs and survivors are
// buffer indices of sm.buf).  A survivor beyond the list (rare) gets its backward entry at once.
template <bool STAGED>
__device__ __forceinline__ void half_scan(HalfASmem& sm, const float4* __restrict__ agf, uint32_t rr_base,
                                          uint32_t wmax, uint32_t w, uint32_t i, unsigned long long mxy,
                                          unsigned long long mzr, int& cnt, uint32_t& extra,
                                          uint32_t* __restrict__ fwd_rows, uint32_t* __restrict__ bwd,
                                          uint32_t* __restrict__ bcnt, uint32_t pad, uint32_t rm) {
  const int lane = threadIdx.x & 31;
  uint2 cur = sm.rr[0][lane];
  uint32_t q = cur.x, e = cur.y;
  uint2 nx = sm.rr[1][lane];
  uint32_t kaddr = rr_base + 2u * 256u;  // address of the run after nx
#if BDM_HLST
  // shared address of this lane's list column, from the run list's (the generic -> shared address of
  // sm.list would otherwise be rematerialised at every append under the register cap)
  // (through an opaque move: the compiler cannot rematerialise it and keeps it in a register)
  uint32_t laddr;
  asm volatile("mov.u32 %0, %1;"
               : "=r"(laddr)
               : "r"(rr_base + (uint32_t)(offsetof(HalfASmem, list) - offsetof(HalfASmem, rr)) - 4u * (uint32_t)lane));
#endif
  for (uint32_t s0 = 0; s0 < wmax; s0 += NSLOT) {
    uint32_t qs[NSLOT];
    bool ok[NSLOT];
#pragma unroll
    for (int t = 0; t < NSLOT; ++t) {
      // unstaged: past its last run a lane walks the sentinel run (pad, ~0): every slot reads the
      // padding agent, which fails the filter, so no per-slot bound test
      ok[t] = STAGED ? s0 + t < w : true;
      qs[t] = STAGED ? (ok[t] ? q : 0u) : min(q, pad);
      ++q;
      const uint32_t sw = q == e;
      q = sw ? nx.x : q;
      e = sw ? nx.y : e;
      // predicated refill of the next run (no branch): nx = rr[k], k advanced on a switch
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p ld.shared.v2.u32 {%0, %1}, [%3];\n\t}"
                   : "+r"(nx.x), "+r"(nx.y) : "r"(sw), "r"(kaddr));
      kaddr += sw * 256u;
    }
    float4 o[NSLOT];
#pragma unroll
    for (int t = 0; t < NSLOT; ++t) {
#if BDM_HSTAGE
      if (STAGED)
        o[t] = sm.buf[qs[t]];
      else
#endif
        o[t] = __ldg(&agf[qs[t]]);
    }
#pragma unroll
    for (int t = 0; t < NSLOT; ++t) {
      float2 dxy, dzs;
      asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(*reinterpret_cast<unsigned long long*>(&dxy))
          : "l"(mxy), "l"(pack2(o[t].x, o[t].y)));
      asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(*reinterpret_cast<unsigned long long*>(&dzs))
          : "l"(mzr), "l"(pack2(o[t].z, o[t].w)));
      float2 sq, qz;
      asm("mul.rn.f32x2 %0, %1, %1;" : "=l"(*reinterpret_cast<unsigned long long*>(&sq))
          : "l"(*reinterpret_cast<unsigned long long*>(&dxy)));
      asm("mul.rn.f32x2 %0, %1, %1;" : "=l"(*reinterpret_cast<unsigned long long*>(&qz))
          : "l"(*reinterpret_cast<unsigned long long*>(&dzs)));
      const float d2 = (sq.x + sq.y) + qz.x;
      if (ok[t] && d2 <= __fmaf_rn(qz.y, 0x1p-20f, qz.y)) {
        if (cnt < HLA) {
#if BDM_HLST
          asm volatile("st.shared.u32 [%0], %1;" ::"r"(laddr + 128u * (uint32_t)cnt), "r"(qs[t]) : "memory");
          ++cnt;
#else
          sm.list[cnt++][lane] = qs[t];
#endif
        } else {  // rare: the partner still gets its backward entry
          uint32_t j = qs[t];
#if BDM_HSTAGE
          if (STAGED) {
            uint32_t c = 0;
#pragma unroll
            for (int u = 1; u < 5; ++u) c += j >= sm.off[u] ? 1u : 0u;
            j = j - sm.off[c] + sm.ub[c];
          }
#endif
          bw_put(fwd_rows, bwd, j, atomicAdd(&bcnt[j & rm], 1u), i, rm);
          ++extra;
        }
      }
    }
  }
}

// BDM_HMAP: the candidate loop with the closed-form cursor -- no shared-memory run refills and no
// serial dependency between the slots of an iteration.
__device__ __forceinline__ void half_scan_map(HalfASmem& sm, const float4* __restrict__ agf, const uint32_t S[5],
                                              const uint32_t A[5], uint32_t wmax, uint32_t w, uint32_t i,
                                              unsigned long long mxy, unsigned long long mzr, int& cnt,
                                              uint32_t& extra, uint32_t* __restrict__ fwd_rows,
                                              uint32_t* __restrict__ bwd, uint32_t* __restrict__ bcnt, uint32_t pad,
                                              uint32_t laddr, uint32_t rm) {
  const int lane = threadIdx.x & 31;
  for (uint32_t s0 = 0; s0 < wmax; s0 += NSLOT) {
    uint32_t qs[NSLOT];
    bool ok[NSLOT];
#pragma unroll
    for (int t = 0; t < NSLOT; ++t) {
      const uint32_t k = s0 + t;
      uint32_t a = A[0];
#pragma unroll
      for (int q = 1; q < 5; ++q) a = k >= S[q] ? A[q] : a;
      ok[t] = true;  // (slots past w read the padding agent, which fails the filter)
      qs[t] = k < w ? k + a : pad;
    }
    float4 o[NSLOT];
#pragma unroll
    for (int t = 0; t < NSLOT; ++t) o[t] = __ldg(&agf[qs[t]]);
#pragma unroll
    for (int t = 0; t < NSLOT; ++t) {
      float2 dxy, dzs;
      asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(*reinterpret_cast<unsigned long long*>(&dxy))
          : "l"(mxy), "l"(pack2(o[t].x, o[t].y)));
      asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(*reinterpret_cast<unsigned long long*>(&dzs))
          : "l"(mzr), "l"(pack2(o[t].z, o[t].w)));
      float2 sq, qz;
      asm("mul.rn.f32x2 %0, %1, %1;" : "=l"(*reinterpret_cast<unsigned long long*>(&sq))
          : "l"(*reinterpret_cast<unsigned long long*>(&dxy)));
      asm("mul.rn.f32x2 %0, %1, %1;" : "=l"(*reinterpret_cast<unsigned long long*>(&qz))
          : "l"(*reinterpret_cast<unsigned long long*>(&dzs)));
      const float d2 = (sq.x + sq.y) + qz.x;
      if (ok[t] && d2 <= __fmaf_rn(qz.y, 0x1p-20f, qz.y)) {
        if (cnt < HLA) {
          asm volatile("st.shared.u32 [%0], %1;" ::"r"(laddr + 128u * (uint32_t)cnt), "r"(qs[t]) : "memory");
          ++cnt;
        } else {  // rare: the partner still gets its backward entry
          bw_put(fwd_rows, bwd, qs[t], atomicAdd(&bcnt[qs[t] & rm], 1u), i, rm);
          ++extra;
        }
      }
    }
  }
}

// The forward z-runs [rb[q], re[q]) of the 5 forward columns q of agent i in box (bx, by, bz) with
// culling bits `cull` (empty: rb >= re): the 5 column records first, then the 9 box starts (own
// column: its run starts at i + 1), each level's loads all in flight together -- two dependent
// levels instead of five zrun chains.
__device__ __forceinline__ void forward_runs(const GridDev& g, int bx, int by, int bz, uint32_t i, uint32_t cull,
                                             uint32_t rb[5], uint32_t re[5]) {
  int4 ci[5];
#pragma unroll
  for (int q = 0; q < 5; ++q) {
    const int cx = bx + (q >= 2 ? 1 : 0), cy = by + (q == 1 || q == 4 ? 1 : (q == 2 ? -1 : 0));
    const bool in = ((cull >> q) & 1u) && cx >= g.lo[0] && cx <= g.hi[0] && cy >= g.lo[1] && cy <= g.hi[1];
    BDM_ASSERT(!in || col_of(g, cx, cy) < g.n_cols);
    ci[q] = in ? __ldg(&g.col[col_of(g, cx, cy)]) : make_int4(1, 0, 0, 0);  // (empty: zl > zh)
  }
#pragma unroll
  for (int q = 0; q < 5; ++q) {
    const int z0 = q == 0 ? bz : bz - 1 + (int)((cull >> (8 + q)) & 1u);
    const int z1 = bz + 1 - (int)((cull >> (16 + q)) & 1u);
    const int a = z0 > ci[q].x ? z0 : ci[q].x, d = z1 < ci[q].y ? z1 : ci[q].y;
    rb[q] = q == 0 ? i + 1 : 0u;
    re[q] = 0u;
    if (a <= d) {
      BDM_ASSERT((uint32_t)ci[q].z + (uint32_t)(d - ci[q].x) + 1u <= __ldg(&g.coff[g.n_cols]));
      if (q != 0) rb[q] = __ldg(&g.table[(uint32_t)ci[q].z + (uint32_t)(a - ci[q].x)]);
      re[q] = __ldg(&g.table[(uint32_t)ci[q].z + (uint32_t)(d - ci[q].x) + 1u]);
    }
  }
}

__global__ void __launch_bounds__(HA_THREADS, HA_MIN_BLOCKS)
    k_half_search(const double4* __restrict__ ag, const float4* __restrict__ agf, uint32_t s_begin, uint32_t s_end,
                  GridDev g, uint32_t* __restrict__ fwd, uint8_t* __restrict__ fcnt, uint32_t* __restrict__ bwd,
                  uint32_t* __restrict__ bcnt, Extents* ext, bool count_searched,
                  const uint32_t* __restrict__ s_end_dev = nullptr, uint32_t* __restrict__ work = nullptr) {
  pdl_wait();
  if (s_end_dev) s_end = __ldg(s_end_dev);
  if (!work) work = &ext->work_a;  // (banded launches: the band's own counter)
  extern __shared__ __align__(16) unsigned char s_raw[];
  HalfASmem& sm = reinterpret_cast<HalfASmem*>(s_raw)[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
#if HA_RR
  const uint32_t rr_base = (uint32_t)__cvta_generic_to_shared(&sm.rr[0][lane]);
#endif
#if BDM_HMAP
  uint32_t la_base;  // shared address of this lane's list column (opaque: kept in a register)
  asm volatile("mov.u32 %0, %1;" : "=r"(la_base) : "r"((uint32_t)__cvta_generic_to_shared(&sm.list[0][lane])));
#endif
  // statistics of the stationary-region skip mode (bdm_get_skip_stats): this path searches everyone
  if (count_searched && blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&ext->searched, s_end - s_begin);
#if BDM_HSTAGE
  uint32_t phase = 0;  // parity of this warp's staging mbarrier
  if (lane == 0) mbar_init(&sm.bar);
  __syncwarp();
#endif
  Tickets tk(s_end - s_begin);
#if BDM_HDEF && BDM_MROW && !BDM_HSTAGE
  HalfPending pd;
  pd.cnt = 0u;
#endif
#if BDM_HAPF
  // the next chunk's fp32 agents are loaded one chunk ahead (four registers)
  uint32_t chunk = tk.take(work, lane);
  float4 mf_next = make_float4(0.f, 0.f, 0.f, 0.f);
  {
    const uint64_t i1 = (uint64_t)s_begin + 32ull * chunk + lane;
    if (i1 < s_end) mf_next = __ldg(&agf[i1]);
  }
#endif
  while (true) {
#if !BDM_HAPF
    const uint32_t chunk = tk.take(work, lane);
#endif
    const uint64_t base = (uint64_t)s_begin + 32ull * chunk;
    if (base >= s_end) break;
    const uint32_t i = (uint32_t)base + lane;
    const bool valid = i < s_end;
#if BDM_HAPF
    const float4 mf = mf_next;
    chunk = tk.take(work, lane);
    {
      const uint64_t i1 = (uint64_t)s_begin + 32ull * chunk + lane;
      mf_next = i1 < s_end ? __ldg(&agf[i1]) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#else
    const float4 mf = valid ? __ldg(&agf[i]) : make_float4(0.f, 0.f, 0.f, 0.f);
#endif
#if BDM_HA32
    // O2's box from the fp32 copy: t = x32 * inv32 is within 3 * 2^-24 |t| of x * inv, so floor(t)
    // is O2's box unless t lies within |t| 2^-21 + 2^-30 of an integer; such lanes (about 1e-3 of
    // the agents) load the fp64 position.  r_i from the fp32 copy too, rounded up with a relative
    // 2^-20 (the filter bound only has to be an upper bound)
    int bx, by, bz;
    {
      const float inv32 = (float)g.inv;
      const float t[3] = {mf.x * inv32, mf.y * inv32, mf.z * inv32};
      int b3[3];
      bool amb = false;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const float fl = floorf(t[a]);
        const float tol = fabsf(t[a]) * 0x1p-21f + 0x1p-30f;
        amb |= t[a] - fl <= tol || fl + 1.0f - t[a] <= tol;
        b3[a] = (int)fl;
      }
      if (valid && amb) {
        const double4 me = ag[i];
        b3[0] = (int)floor(me.x * g.inv);
        b3[1] = (int)floor(me.y * g.inv);
        b3[2] = (int)floor(me.z * g.inv);
      }
      bx = b3[0];
      by = b3[1];
      bz = b3[2];
    }
    const double ri = (double)__fmul_ru(-mf.w, 1.0f + 0x1p-20f);
#else
    const double4 me = valid ? ag[i] : make_double4(0.0, 0.0, 0.0, 0.0);
    const double ri = 0.5 * me.w;
    const int bx = (int)floor(me.x * g.inv), by = (int)floor(me.y * g.inv), bz = (int)floor(me.z * g.inv);
#endif
    // box culling of k_force, for the 5 forward columns q = 0..4 <-> (dx, dy) = (0,0), (0,+1),
    // (+1,-1), (+1,0), (+1,+1): bit q kept, bit 8+q z-1 box culled, bit 16+q z+1 box culled
    uint32_t cull = 0u;
    {
      // in fp32 from the fp32 copy: the face distances are off by a few ulp32(max |coordinate|) at
      // most (< m32), so the bound carries two extra margins m32 and a relative
      // 2^-18: a box is culled only if it truly cannot hold a contact (conservative)
      const float m = (float)g.m32;
      const float rp = (-mf.w + (float)g.thr_pad + m) * (1.0f + 0x1p-19f);
      const float Rc = rp + 3.0f * m;
      const float Rc2 = Rc * Rc * (1.0f + 0x1p-18f);
      const float Lb = (float)(1.0 / g.inv);
      const float fy = fmaxf(mf.y - (float)by * Lb, 0.f), gy = fmaxf((float)(by + 1) * Lb - mf.y, 0.f);
      const float gx = fmaxf((float)(bx + 1) * Lb - mf.x, 0.f);
      const float fz = fmaxf(mf.z - (float)bz * Lb, 0.f), gz = fmaxf((float)(bz + 1) * Lb - mf.z, 0.f);
#pragma unroll
      for (int q = 0; q < 5; ++q) {
        const float ex = q >= 2 ? gx : 0.f;
        const float ey = q == 1 || q == 4 ? gy : (q == 2 ? fy : 0.f);
        const float exy2 = ex * ex + ey * ey;
        cull |= (uint32_t)(exy2 <= Rc2) << q;
        cull |= (uint32_t)(exy2 + fz * fz > Rc2) << (8 + q);
        cull |= (uint32_t)(exy2 + gz * gz > Rc2) << (16 + q);
      }
    }
    // single-column chunks stage the box starts of the 5 forward columns (as k_force does for 9)
    const int bx0 = __shfl_sync(FULL, bx, 0), by0 = __shfl_sync(FULL, by, 0);
    const int zf = __reduce_min_sync(FULL, valid ? bz : INT32_MAX);
    const int zl = __reduce_max_sync(FULL, valid ? bz : INT32_MIN);

    const bool coop = BDM_HCOOP && __all_sync(FULL, !valid || (bx == bx0 && by == by0)) && zl - zf + 4 <= TSPAN;
    const int span = zl - zf + 4;
    if (coop) {
      int czl = 0, cze = 0;
      uint32_t cof = 0xffffffffu;
      if (lane < 5) {
        const int cx = bx0 + (lane >= 2 ? 1 : 0);
        const int cy = by0 + (lane == 1 || lane == 4 ? 1 : (lane == 2 ? -1 : 0));
        if (cx >= g.lo[0] && cx <= g.hi[0] && cy >= g.lo[1] && cy <= g.hi[1]) {
          const uint32_t cc = col_of(g, cx, cy);
          czl = __ldg(&g.czlo[cc]);
          const int czh = __ldg(&g.czhi[cc]);
          cof = __ldg(&g.coff[cc]);
          cze = czh >= czl ? czh - czl + 1 : 0;
        }
      }
#pragma unroll
      for (int c = 0; c < 5; ++c) {  // box starts of column c, z in [zf-1, zl+2], one lane per z
        const int zlo_c = __shfl_sync(FULL, czl, c), ext_c = __shfl_sync(FULL, cze, c);
        const uint32_t off_c = __shfl_sync(FULL, cof, c);
        for (int tt = lane; tt < span; tt += 32) {
          uint32_t v = 0u;
          if (off_c != 0xffffffffu) {
            int k = zf - 1 + tt - zlo_c;
            k = k < 0 ? 0 : (k > ext_c ? ext_c : k);
            v = __ldg(&g.table[off_c + (uint32_t)k]);
          }
          sm.tab[c][tt] = v;
        }
      }
      __syncwarp();
    }
    bool staged = false;
#if BDM_HSTAGE
    uint32_t stage_ub[5] = {0u, 0u, 0u, 0u, 0u}, stage_off[5] = {0u, 0u, 0u, 0u, 0u};
    if (coop) {
      // union runs of the 5 forward columns over the chunk: own column from box zf (the agents
      // before a lane are never its candidates, but the union is simpler), the others from zf-1,
      // all to the end of box zl+1.  If they fit, one lane copies them into sm.buf (TMA bulk
      // copies, completing on the warp's mbarrier) while the lanes set up their runs.
      uint32_t ub[5], off[6];
      off[0] = 0u;
#pragma unroll
      for (int q = 0; q < 5; ++q) {
        ub[q] = sm.tab[q][q == 0 ? 1 : 0];
        off[q + 1] = off[q] + (sm.tab[q][span - 1] - ub[q]);
      }
      staged = off[5] > 0u && off[5] <= (uint32_t)HPCAP;
#pragma unroll
      for (int q = 0; q < 5; ++q) {
        stage_ub[q] = ub[q];
        stage_off[q] = off[q];
      }
      if (staged && lane == 0) {
#pragma unroll
        for (int q = 0; q < 5; ++q) {
          sm.off[q] = off[q];
          sm.ub[q] = ub[q];
        }
        sm.off[5] = off[5];
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&sm.bar, off[5] * 16u);
#pragma unroll
        for (int q = 0; q < 5; ++q)
          if (off[q + 1] > off[q]) bulk_g2s(&sm.buf[off[q]], agf + ub[q], (off[q + 1] - off[q]) * 16u, &sm.bar);
      }
    }
#endif
    // this lane's forward z-runs in canonical (= ascending sorted) order
    int nr = 0;
    uint32_t w = 0;
#if BDM_HMAP
    // closed-form cursor (BDM_HMAP): run q occupies flattened positions [S[q], S[q+1]); position k
    // maps to k + A[q] (empty runs are skipped by the compare chain)
    uint32_t S[5], A[5];
#if BDM_HBATCH
    if (valid && !coop) {
      uint32_t rb[5], re[5];
      forward_runs(g, bx, by, bz, i, cull, rb, re);
#pragma unroll
      for (int q = 0; q < 5; ++q) {
        const uint32_t b = rb[q] < re[q] ? rb[q] : 0u, e = rb[q] < re[q] ? re[q] : 0u;
        S[q] = w;
        A[q] = b - w;
        w += e - b;
      }
    } else
#endif
#pragma unroll
    for (int q = 0; q < 5; ++q) {
      uint32_t b = 0, e = 0;
      if (valid && ((cull >> q) & 1u)) {
        const int z0 = q == 0 ? bz : bz - 1 + (int)((cull >> (8 + q)) & 1u);
        const int z1 = bz + 1 - (int)((cull >> (16 + q)) & 1u);
        if (coop) {
          b = sm.tab[q][z0 - zf + 1];
          e = sm.tab[q][z1 - zf + 2];
        } else {
          const int cx = bx + (q >= 2 ? 1 : 0), cy = by + (q == 1 || q == 4 ? 1 : (q == 2 ? -1 : 0));
          zrun(g, cx, cy, z0, z1, b, e);
        }
        if (q == 0) b = i + 1;  // own box: only the agents after i
        if (b >= e) b = e = 0;
      }
      S[q] = w;
      A[q] = b - w;
      w += e - b;
    }
#endif
#if HA_RR
    uint32_t wr = 0;  // total length of the run list (staged path, or BDM_HMAP=0)
#if BDM_HBATCH
    if (valid && !coop) {
      uint32_t rb[5], re[5];
      forward_runs(g, bx, by, bz, i, cull, rb, re);
#pragma unroll
      for (int q = 0; q < 5; ++q)
        if (rb[q] < re[q]) {
          sm.rr[nr][lane] = make_uint2(rb[q], re[q]);
          wr += re[q] - rb[q];
          ++nr;
        }
    } else
#endif
    if (valid) {
#pragma unroll
      for (int q = 0; q < 5; ++q) {
        if (!((cull >> q) & 1u)) continue;
        const int z0 = q == 0 ? bz : bz - 1 + (int)((cull >> (8 + q)) & 1u);
        const int z1 = bz + 1 - (int)((cull >> (16 + q)) & 1u);
        uint32_t b = 0, e = 0;
        if (coop) {
          b = sm.tab[q][z0 - zf + 1];
          e = sm.tab[q][z1 - zf + 2];
        } else {
          const int cx = bx + (q >= 2 ? 1 : 0), cy = by + (q == 1 || q == 4 ? 1 : (q == 2 ? -1 : 0));
          zrun(g, cx, cy, z0, z1, b, e);
        }
        if (q == 0) b = i + 1;  // own box: only the agents after i
        if (b < e) {
#if BDM_HSTAGE
          if (staged) {  // the run in buffer indices of its column's union run
            const uint32_t d = stage_ub[q] - stage_off[q];
            b -= d;
            e -= d;
          }
#endif
          sm.rr[nr][lane] = make_uint2(b, e);
          wr += e - b;
          ++nr;
        }
      }
    }
    // sentinel: after the last run q never meets e again (unstaged: the padding run, see half_scan)
    sm.rr[nr][lane] = staged ? make_uint2(0u, 0u) : make_uint2(g.pad, 0xffffffffu);
#if !BDM_HMAP
    w = wr;
#endif
#endif
    __syncwarp();
    const uint32_t wmax = __reduce_max_sync(FULL, w);
    const float ri32 = __double2float_ru(ri + g.m32);
    const unsigned long long mxy = pack2(mf.x, mf.y), mzr = pack2(mf.z, ri32);
    int cnt = 0;
    uint32_t extra = 0;  // survivors beyond the buffer (forward row overflow: pass B's slow path)
#if BDM_HSTAGE
    if (staged) {
      mbar_wait(&sm.bar, phase);
      phase ^= 1u;
      half_scan<true>(sm, agf, rr_base, wmax, w, i, mxy, mzr, cnt, extra, fwd, bwd, bcnt, g.pad, g.rmask);
      // buffer index -> global sorted index (each union run is contiguous in both)
      for (int x = 0; x < cnt; ++x) {
        const uint32_t v = sm.list[x][lane];
        uint32_t c = 0;
#pragma unroll
        for (int q = 1; q < 5; ++q) c += v >= sm.off[q] ? 1u : 0u;
        sm.list[x][lane] = v - sm.off[c] + sm.ub[c];
      }
      __syncwarp();  // every lane is done with buf before the next chunk's copies overwrite it
    } else
#endif
#if BDM_HMAP
    {
#if BDM_HDEF && BDM_MROW && !BDM_HSTAGE
      half_emit_finish(sm, lane, fwd, pd, g.rmask);  // the last chunk's stores (before the list is overwritten)
#endif
      half_scan_map(sm, agf, S, A, wmax, w, i, mxy, mzr, cnt, extra, fwd, bwd, bcnt, g.pad, la_base, g.rmask);
    }
#else
    {
#if BDM_HDEF && BDM_MROW && !BDM_HSTAGE
      half_emit_finish(sm, lane, fwd, pd, g.rmask);  // the last chunk's stores (before the list is overwritten)
#endif
      half_scan<false>(sm, agf, rr_base, wmax, w, i, mxy, mzr, cnt, extra, fwd, bwd, bcnt, g.pad, g.rmask);
    }
#endif
    if (valid) {
#if BDM_HDEF && BDM_MROW && !BDM_HSTAGE
      half_emit_issue(sm, lane, cnt, extra, i, fwd, bcnt, pd, g.rmask);
#else
      half_emit(sm, lane, cnt, extra, i, fwd, bwd, bcnt, g.rmask);
#endif
      if (!BDM_MROW) {
        const uint32_t nf = (uint32_t)cnt + extra;
        fcnt[i] = (uint8_t)(nf > 255u ? 255u : nf);
      }
    }
    __syncwarp();
  }
#if BDM_HDEF && BDM_MROW && !BDM_HSTAGE
  half_emit_finish(sm, lane, fwd, pd, g.rmask);
#endif
}

// ---- Pass A with the neighbourhood staged in shared memory (north_star: "a force kernel that stages
// each 3x3x3 neighbourhood of sorted agents in shared memory (or uses TMA bulk copies)").
// Warp-specialised, persistent CTAs: one producer warp and TILE_W consumer warps.  The producer takes
// tiles of TILE_AG = 32 TILE_W consecutive sorted agents; for a tile whose agents lie in at most TMAXC
// columns it stages the forward half of their 3x3x3 neighbourhood -- for every own column c and
// forward column q (0,0), (0,+1), (+1,-1), (+1,0), (+1,+1) the agents of the boxes
// [zmin_c - 1, zmax_c + 1] (own column: from zmin_c), each one contiguous run of the sorted fp32
// copy -- into shared memory with TMA bulk copies (cp.async.bulk completing on the slot's "full"
// mbarrier), two slots deep: it prepares tile k+1 (columns, box starts of every run, copies) while
// the consumers search tile k and releases nothing until they arrive on the slot's "empty"
// mbarrier.  Consumers (one 32-agent chunk per warp) read candidates with LDS instead of L1/L2
// gathers; culling, flattened cursor, fp32 filter and rows are pass A's.  Tiles spanning more
// columns (sparse regions) or whose neighbourhood exceeds the buffer are searched from global memory.
#ifndef BDM_TILE_NOSTAGE
#define BDM_TILE_NOSTAGE 0  // experiment: the producer never stages (the pipeline without the shared copies)
#endif
#ifndef BDM_TILE_W
#define BDM_TILE_W 4
#endif
constexpr int TILE_W = BDM_TILE_W;          // consumer warps (one chunk each)
constexpr int TILE_AG = 32 * TILE_W;        // agents per tile
constexpr int TILE_THREADS = 32 * (TILE_W + 1);
constexpr int TMAXC = 3;                    // own columns of a staged tile
constexpr int TRUNS = 5 * TMAXC;
constexpr int TZS = 48;                     // box starts per staged run (z-span + 4)
#ifndef BDM_TCAP
#define BDM_TCAP (TILE_W == 4 ? 768 : 1152)
#endif
constexpr int TCAP = BDM_TCAP;              // staged candidates (float4) per slot
#ifndef BDM_TILE_MIN_BLOCKS
#define BDM_TILE_MIN_BLOCKS (TILE_W == 4 ? 4 : 2)
#endif
constexpr int TILE_MIN_BLOCKS = BDM_TILE_MIN_BLOCKS;

struct TileMeta {
  uint32_t t0;        // first sorted agent of the tile (>= s_end: no more tiles)
  int32_t staged;     // 1 if the runs below are in the buffer
  int32_t ncol;       // own columns (staged tiles)
  int32_t cx[TMAXC], cy[TMAXC], zb[TMAXC];  // own column (bx, by) and its first staged box z (zmin - 1)
  uint32_t ub[TRUNS + 1];                   // global sorted index of each staged run's first agent
  uint32_t off[TRUNS + 1];                  // buffer offset of each run (off[5 ncol] = total)
};

struct TileSmem {
  float4 buf[2][TCAP];
  uint32_t tab[2][TRUNS][TZS];  // box starts of each (own column, forward column) run
  TileMeta meta[2];
  unsigned long long full[2], empty[2];
};
constexpr size_t TILE_SMEM_BYTES = sizeof(TileSmem) + sizeof(HalfASmem) * TILE_W;

__device__ __forceinline__ void mbar_init_n(unsigned long long* bar, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Producer (one warp): the tile at t0 -> meta[slot], tab[slot], bulk copies into buf[slot]; arrives on
// full[slot] (with the copies' byte count when staged).  Boxes as pass A computes them (fp32 copy,
// fp64 position near box faces).  Loads of one level are issued together (latency-bound warp).
__device__ void tile_produce(TileSmem& ts, int slot, uint32_t t0, uint32_t s_end, const double4* __restrict__ ag,
                             const float4* __restrict__ agf, const GridDev& g) {
  const int lane = threadIdx.x & 31;
  TileMeta& m = ts.meta[slot];
  bool staged = false;
  int ncol = 0;
  uint32_t total = 0;
  if (t0 < s_end) {
    const float inv32 = (float)g.inv;
    float4 mf[TILE_W];
#pragma unroll
    for (int w = 0; w < TILE_W; ++w) {
      const uint32_t i = t0 + 32u * w + lane;
      mf[w] = i < s_end ? __ldg(&agf[i]) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    int cxs[TMAXC], cys[TMAXC], zlo[TMAXC], zhi[TMAXC];
    bool ok = true;
#pragma unroll
    for (int w = 0; w < TILE_W; ++w) {
      const uint32_t i = t0 + 32u * w + lane;
      const bool valid = i < s_end;
      int b3[3];
      const float t[3] = {mf[w].x * inv32, mf[w].y * inv32, mf[w].z * inv32};
      bool amb = false;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const float fl = floorf(t[a]);
        const float tol = fabsf(t[a]) * 0x1p-21f + 0x1p-30f;
        amb |= t[a] - fl <= tol || fl + 1.0f - t[a] <= tol;
        b3[a] = (int)fl;
      }
      if (valid && amb) {
        const double4 me = ag[i];
        b3[0] = (int)floor(me.x * g.inv);
        b3[1] = (int)floor(me.y * g.inv);
        b3[2] = (int)floor(me.z * g.inv);
      }
      // distinct columns in order (the agents are sorted by column, then z)
      unsigned left = __ballot_sync(FULL, valid);
      while (left && ok) {
        const int src = __ffs(left) - 1;
        const int cx = __shfl_sync(FULL, b3[0], src), cy = __shfl_sync(FULL, b3[1], src);
        const bool same = valid && b3[0] == cx && b3[1] == cy;
        left &= ~__ballot_sync(FULL, same);
        const int zl = __reduce_min_sync(FULL, same ? b3[2] : INT32_MAX);
        const int zh = __reduce_max_sync(FULL, same ? b3[2] : INT32_MIN);
        if (ncol > 0 && cxs[ncol - 1] == cx && cys[ncol - 1] == cy) {
          zlo[ncol - 1] = min(zlo[ncol - 1], zl);
          zhi[ncol - 1] = max(zhi[ncol - 1], zh);
        } else if (ncol < TMAXC) {
          cxs[ncol] = cx;
          cys[ncol] = cy;
          zlo[ncol] = zl;
          zhi[ncol] = zh;
          ++ncol;
        } else {
          ok = false;
        }
      }
    }
    for (int c = 0; c < ncol; ++c) ok &= zhi[c] - zlo[c] + 4 <= TZS;
    if (ok && ncol > 0) {
      // lane r < 5 ncol: run r = 5 c + q -> its neighbour column's record (one load level)
      const int nrun = 5 * ncol;
      int czl = 1, czh = 0, zb = 0, span = 0;
      uint32_t cof = 0;
      bool inside = false;
      if (lane < nrun) {
        const int c = lane / 5, q = lane % 5;
        int cxv = cxs[0], cyv = cys[0], zlv = zlo[0], zhv = zhi[0];
#pragma unroll
        for (int u = 1; u < TMAXC; ++u)
          if (c == u) {
            cxv = cxs[u];
            cyv = cys[u];
            zlv = zlo[u];
            zhv = zhi[u];
          }
        const int nx = cxv + (q >= 2 ? 1 : 0), ny = cyv + (q == 1 || q == 4 ? 1 : (q == 2 ? -1 : 0));
        zb = zlv - 1;
        span = zhv - zlv + 3;  // entries 0..span: starts of boxes zb .. zhi + 2
        inside = nx >= g.lo[0] && nx <= g.hi[0] && ny >= g.lo[1] && ny <= g.hi[1];
        if (inside) {
          const int4 ci = __ldg(&g.col[col_of(g, nx, ny)]);
          czl = ci.x;
          czh = ci.y;
          cof = (uint32_t)ci.z;
        }
      }
      // every box start of every run (second load level: all loads issued, then stored)
      constexpr int PER = (TRUNS * TZS + 31) / 32;
      uint32_t v[PER];
#pragma unroll
      for (int k = 0; k < PER; ++k) {
        const int e = lane + 32 * k;
        const int r = e / TZS, tt = e % TZS;
        const int rs = r < nrun ? r : 0;
        const int zl_r = __shfl_sync(FULL, czl, rs), zh_r = __shfl_sync(FULL, czh, rs);
        const int zb_r = __shfl_sync(FULL, zb, rs), sp_r = __shfl_sync(FULL, span, rs);
        const uint32_t of_r = __shfl_sync(FULL, cof, rs);
        const bool in_r = __shfl_sync(FULL, inside, rs);
        v[k] = 0u;
        const int ext = zh_r >= zl_r ? zh_r - zl_r + 1 : 0;
        if (r < nrun && tt <= sp_r && in_r && ext > 0) {
          int kk = zb_r + tt - zl_r;
          kk = kk < 0 ? 0 : (kk > ext ? ext : kk);
          v[k] = __ldg(&g.table[of_r + (uint32_t)kk]);
        }
      }
#pragma unroll
      for (int k = 0; k < PER; ++k) {
        const int e = lane + 32 * k;
        if (e < TRUNS * TZS) (&ts.tab[slot][0][0])[e] = v[k];
      }
      __syncwarp();
      // run lengths -> buffer offsets (warp scan over the runs)
      uint32_t ub = 0, len = 0;
      if (lane < nrun) {
        ub = ts.tab[slot][lane][lane % 5 == 0 ? 1 : 0];
        const uint32_t ue = ts.tab[slot][lane][span];
        len = ue > ub ? ue - ub : 0u;
      }
      const uint32_t incl = warp_incl_scan(len);
      total = __shfl_sync(FULL, incl, 31);
      if (lane < nrun) {
        m.ub[lane] = ub;
        m.off[lane] = incl - len;
      }
      if (lane == 0) {
        m.off[nrun] = total;
        for (int c = 0; c < ncol; ++c) {
          m.cx[c] = cxs[c];
          m.cy[c] = cys[c];
          m.zb[c] = zlo[c] - 1;
        }
      }
      staged = total > 0u && total <= (uint32_t)TCAP && !BDM_TILE_NOSTAGE;
      __syncwarp();
      if (staged) {
        if (lane == 0) {
          m.t0 = t0;
          m.staged = 1;
          m.ncol = ncol;
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          mbar_expect_tx(&ts.full[slot], total * 16u);  // (the producer's arrival, with the byte count)
        }
        __syncwarp();
        if (lane < nrun && len) bulk_g2s(&ts.buf[slot][incl - len], agf + ub, len * 16u, &ts.full[slot]);
        return;
      }
    }
  }
  if (lane == 0) {
    m.t0 = t0;
    m.staged = 0;
    m.ncol = 0;
    mbar_arrive(&ts.full[slot]);
  }
}

// Candidate loop over runs of buffer indices (a staged tile): half_scan reading shared memory.
__device__ __forceinline__ void tile_scan(HalfASmem& sm, const float4* __restrict__ sbuf, const TileMeta& m,
                                          uint32_t rr_base, uint32_t wmax, uint32_t w, uint32_t i,
                                          unsigned long long mxy, unsigned long long mzr, int& cnt, uint32_t& extra,
                                          uint32_t* __restrict__ fwd_rows, uint32_t* __restrict__ bwd,
                                          uint32_t* __restrict__ bcnt, uint32_t rm) {
  const int lane = threadIdx.x & 31;
  uint2 cur = sm.rr[0][lane];
  uint32_t q = cur.x, e = cur.y;
  uint2 nx = sm.rr[1][lane];
  uint32_t kaddr = rr_base + 2u * 256u;
  for (uint32_t s0 = 0; s0 < wmax; s0 += NSLOT) {
    uint32_t qs[NSLOT];
    bool ok[NSLOT];
#pragma unroll
    for (int t = 0; t < NSLOT; ++t) {
      ok[t] = s0 + t < w;
      qs[t] = ok[t] ? q : 0u;
      ++q;
      const uint32_t sw = q == e;
      q = sw ? nx.x : q;
      e = sw ? nx.y : e;
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p ld.shared.v2.u32 {%0, %1}, [%3];\n\t}"
                   : "+r"(nx.x), "+r"(nx.y) : "r"(sw), "r"(kaddr));
      kaddr += sw * 256u;
    }
    float4 o[NSLOT];
#pragma unroll
    for (int t = 0; t < NSLOT; ++t) o[t] = sbuf[qs[t]];
#pragma unroll
    for (int t = 0; t < NSLOT; ++t) {
      float2 dxy, dzs;
      asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(*reinterpret_cast<unsigned long long*>(&dxy))
          : "l"(mxy), "l"(pack2(o[t].x, o[t].y)));
      asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(*reinterpret_cast<unsigned long long*>(&dzs))
          : "l"(mzr), "l"(pack2(o[t].z, o[t].w)));
      float2 sq, qz;
      asm("mul.rn.f32x2 %0, %1, %1;" : "=l"(*reinterpret_cast<unsigned long long*>(&sq))
          : "l"(*reinterpret_cast<unsigned long long*>(&dxy)));
      asm("mul.rn.f32x2 %0, %1, %1;" : "=l"(*reinterpret_cast<unsigned long long*>(&qz))
          : "l"(*reinterpret_cast<unsigned long long*>(&dzs)));
      const float d2 = (sq.x + sq.y) + qz.x;
      if (ok[t] && d2 <= __fmaf_rn(qz.y, 0x1p-20f, qz.y)) {
        if (cnt < HLA) {
          sm.list[cnt++][lane] = qs[t];
        } else {  // rare: the partner (global index) still gets its backward entry
          uint32_t r = 0;
          while (r + 1 < (uint32_t)(5 * m.ncol) && qs[t] >= m.off[r + 1]) ++r;
          const uint32_t j = qs[t] - m.off[r] + m.ub[r];
          bw_put(fwd_rows, bwd, j, atomicAdd(&bcnt[j & rm], 1u), i, rm);
          ++extra;
        }
      }
    }
  }
}

__global__ void __launch_bounds__(TILE_THREADS, TILE_MIN_BLOCKS)
    k_half_search_tile(const double4* __restrict__ ag, const float4* __restrict__ agf, uint32_t s_begin,
                       uint32_t s_end, GridDev g, uint32_t* __restrict__ fwd, uint8_t* __restrict__ fcnt,
                       uint32_t* __restrict__ bwd, uint32_t* __restrict__ bcnt, Extents* ext, bool count_searched,
                       const uint32_t* __restrict__ s_end_dev = nullptr) {
  if (s_end_dev) s_end = __ldg(s_end_dev);
  extern __shared__ __align__(128) unsigned char s_raw[];
  TileSmem& ts = *reinterpret_cast<TileSmem*>(s_raw);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (count_searched && blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&ext->searched, s_end - s_begin);
  if (threadIdx.x == 0) {
    for (int k = 0; k < 2; ++k) {
      mbar_init_n(&ts.full[k], 1u);
      mbar_init_n(&ts.empty[k], (uint32_t)TILE_W);
    }
  }
  __syncthreads();
  if (warp == TILE_W) {  // ---- producer
    uint32_t tnext = 0;  // the next tile's ticket, taken one tile ahead (the atomic's round trip overlaps)
    if (lane == 0) tnext = atomicAdd(&ext->work_a, 1u);
    for (uint32_t k = 0;; ++k) {
      const int slot = (int)(k & 1u);
      uint32_t t = __shfl_sync(FULL, tnext, 0);
      if (lane == 0) tnext = atomicAdd(&ext->work_a, 1u);
      if (k >= 2) mbar_wait(&ts.empty[slot], ((k >> 1) - 1u) & 1u);  // the consumers released the slot
      const uint64_t a = (uint64_t)s_begin + (uint64_t)TILE_AG * t;
      const uint32_t t0 = a < s_end ? (uint32_t)a : s_end;
      tile_produce(ts, slot, t0, s_end, ag, agf, g);
      if (t0 >= s_end) break;
    }
    return;
  }
  // ---- consumers
  HalfASmem& sm = reinterpret_cast<HalfASmem*>(s_raw + sizeof(TileSmem))[warp];
  const uint32_t rr_base = (uint32_t)__cvta_generic_to_shared(&sm.rr[0][lane]);
  for (uint32_t k = 0;; ++k) {
    const int slot = (int)(k & 1u);
    mbar_wait(&ts.full[slot], (k >> 1) & 1u);
    const TileMeta& m = ts.meta[slot];
    const uint32_t t0 = m.t0;
    if (t0 >= s_end) break;
    const bool staged = m.staged != 0;
    const uint32_t i = t0 + 32u * warp + lane;
    const bool valid = i < s_end;
    if (__any_sync(FULL, valid)) {
      const float4 mf = valid ? __ldg(&agf[i]) : make_float4(0.f, 0.f, 0.f, 0.f);
      int bx, by, bz;
      {
        const float inv32 = (float)g.inv;
        const float t[3] = {mf.x * inv32, mf.y * inv32, mf.z * inv32};
        int b3[3];
        bool amb = false;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          const float fl = floorf(t[a]);
          const float tol = fabsf(t[a]) * 0x1p-21f + 0x1p-30f;
          amb |= t[a] - fl <= tol || fl + 1.0f - t[a] <= tol;
          b3[a] = (int)fl;
        }
        if (valid && amb) {
          const double4 me = ag[i];
          b3[0] = (int)floor(me.x * g.inv);
          b3[1] = (int)floor(me.y * g.inv);
          b3[2] = (int)floor(me.z * g.inv);
        }
        bx = b3[0];
        by = b3[1];
        bz = b3[2];
      }
      const double ri = (double)__fmul_ru(-mf.w, 1.0f + 0x1p-20f);
      uint32_t cull = 0u;
      {
        const float mm = (float)g.m32;
        const float rp = (-mf.w + (float)g.thr_pad + mm) * (1.0f + 0x1p-19f);
        const float Rc = rp + 3.0f * mm;
        const float Rc2 = Rc * Rc * (1.0f + 0x1p-18f);
        const float Lb = (float)(1.0 / g.inv);
        const float fy = fmaxf(mf.y - (float)by * Lb, 0.f), gy = fmaxf((float)(by + 1) * Lb - mf.y, 0.f);
        const float gx = fmaxf((float)(bx + 1) * Lb - mf.x, 0.f);
        const float fz = fmaxf(mf.z - (float)bz * Lb, 0.f), gz = fmaxf((float)(bz + 1) * Lb - mf.z, 0.f);
#pragma unroll
        for (int q = 0; q < 5; ++q) {
          const float ex = q >= 2 ? gx : 0.f;
          const float ey = q == 1 || q == 4 ? gy : (q == 2 ? fy : 0.f);
          const float exy2 = ex * ex + ey * ey;
          cull |= (uint32_t)(exy2 <= Rc2) << q;
          cull |= (uint32_t)(exy2 + fz * fz > Rc2) << (8 + q);
          cull |= (uint32_t)(exy2 + gz * gz > Rc2) << (16 + q);
        }
      }
      // this lane's forward z-runs in canonical (= ascending sorted) order; staged: buffer indices
      int nr = 0;
      uint32_t w = 0;
      int c = 0;
      if (staged)
        while (c + 1 < m.ncol && !(m.cx[c] == bx && m.cy[c] == by)) ++c;
      if (valid) {
#pragma unroll
        for (int q = 0; q < 5; ++q) {
          if (!((cull >> q) & 1u)) continue;
          const int z0 = q == 0 ? bz : bz - 1 + (int)((cull >> (8 + q)) & 1u);
          const int z1 = bz + 1 - (int)((cull >> (16 + q)) & 1u);
          uint32_t b = 0, e = 0;
          if (staged) {
            const int r = 5 * c + q;
            b = ts.tab[slot][r][z0 - m.zb[c]];
            e = ts.tab[slot][r][z1 - m.zb[c] + 1];
            if (q == 0) b = i + 1;
            if (b < e) {
              const uint32_t d = m.ub[r] - m.off[r];
              b -= d;
              e -= d;
            }
          } else {
            const int cx = bx + (q >= 2 ? 1 : 0), cy = by + (q == 1 || q == 4 ? 1 : (q == 2 ? -1 : 0));
            zrun(g, cx, cy, z0, z1, b, e);
            if (q == 0) b = i + 1;
          }
          if (b < e) {
            sm.rr[nr][lane] = make_uint2(b, e);
            w += e - b;
            ++nr;
          }
        }
      }
      sm.rr[nr][lane] = staged ? make_uint2(0u, 0u) : make_uint2(g.pad, 0xffffffffu);
      __syncwarp();
      const uint32_t wmax = __reduce_max_sync(FULL, w);
      const float ri32 = __double2float_ru(ri + g.m32);
      const unsigned long long mxy = pack2(mf.x, mf.y), mzr = pack2(mf.z, ri32);
      int cnt = 0;
      uint32_t extra = 0;
      if (staged) {
        tile_scan(sm, ts.buf[slot], m, rr_base, wmax, w, i, mxy, mzr, cnt, extra, fwd, bwd, bcnt, g.rmask);
        for (int x = 0; x < cnt; ++x) {  // buffer index -> global sorted index
          const uint32_t vv = sm.list[x][lane];
          uint32_t r = 0;
          while (r + 1 < (uint32_t)(5 * m.ncol) && vv >= m.off[r + 1]) ++r;
          sm.list[x][lane] = vv - m.off[r] + m.ub[r];
        }
      } else {
        half_scan<false>(sm, agf, rr_base, wmax, w, i, mxy, mzr, cnt, extra, fwd, bwd, bcnt, g.pad, g.rmask);
      }
      if (valid) {
        half_emit(sm, lane, cnt, extra, i, fwd, bwd, bcnt, g.rmask);
        if (!BDM_MROW) {
          const uint32_t nf = (uint32_t)cnt + extra;
          fcnt[i] = (uint8_t)(nf > 255u ? 255u : nf);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&ts.empty[slot]);  // this warp is done with the slot
  }
}

struct HalfBSmem {
  uint32_t list[HFC + HBC][32];  // all contact candidates of this lane, ascending sorted index
  double term[3][32];
  uint32_t cidx[32];
  int ext[8];  // this warp's running next-step extents lo[3], hi[3] and range flag (lane 0)
};
constexpr size_t HB_SMEM_BYTES = sizeof(HalfBSmem) * FORCE_WARPS;

// Full canonical 27-box sum of agent i (O3-O5 as written) by one warp -- the overflow path of pass B.
// All lanes call it and all return the sum: the lanes evaluate 32 candidates of a z-run at a time,
// then every lane adds the batch's contact terms in candidate order (shuffled from their lanes), the
// same sequence of separately rounded additions as a sequential walk, without one thread walking a
// dense neighbourhood alone (a lone overflow agent of a cfg3 step took ~40 us that way).
__device__ __forceinline__ double3 full_force_warp(const GridDev& g, const double4* __restrict__ ag,
                                                   const uint32_t* __restrict__ ids, const ParamsDev& p, uint32_t i,
                                                   double4 me, int lane) {
  const double ri = 0.5 * me.w;
  const int bx = (int)floor(me.x * g.inv), by = (int)floor(me.y * g.inv), bz = (int)floor(me.z * g.inv);
  double Fx = 0.0, Fy = 0.0, Fz = 0.0;
  for (int c = 0; c < 9; ++c) {
    uint32_t b = 0, e = 0;
    if (!zrun(g, bx + c / 3 - 1, by + c % 3 - 1, bz - 1, bz + 1, b, e)) continue;
    for (uint32_t j0 = b; j0 < e; j0 += 32) {
      const uint32_t j = j0 + (uint32_t)lane;
      double tx = 0.0, ty = 0.0, tz = 0.0, fa;
      const bool hit = j < e && j != i && pair_term(me.x, me.y, me.z, ri, i, ag[j], ids, j, p, tx, ty, tz, fa);
      for (unsigned m = __ballot_sync(FULL, hit); m; m &= m - 1u) {
        const int src = __ffs(m) - 1;
        Fx = Fx + __shfl_sync(FULL, tx, src);
        Fy = Fy + __shfl_sync(FULL, ty, src);
        Fz = Fz + __shfl_sync(FULL, tz, src);
      }
    }
  }
  return make_double3(Fx, Fy, Fz);
}

// ENONFINITE diagnosis ("abort ... with the offending pair"): after a force phase that
// reported a non-finite sum, one thread re-walks the reported agent's 27 boxes in canonical order
// (O3-O5 as written) and names the first partner whose term, or the partial sum / its norm after
// adding it, is not finite.  Returns at once when nothing was reported (one load).
__global__ void k_locate_nonfinite(const double4* __restrict__ ag, const uint32_t* __restrict__ ids, GridDev g,
                                   ParamsDev p, ErrDev* err) {
  pdl_wait();
  if (threadIdx.x != 0 || __ldcg(&err->code) != 6u || __ldcg(&err->second) != 0xffffffffu) return;
  const uint32_t i = (uint32_t)(__ldcg(&err->bad) & 0xffffffffull);
  const double4 me = ag[i];
  const double ri = 0.5 * me.w;
  const int bx = (int)floor(me.x * g.inv), by = (int)floor(me.y * g.inv), bz = (int)floor(me.z * g.inv);
  double Fx = 0.0, Fy = 0.0, Fz = 0.0;
  for (int c = 0; c < 9; ++c) {
    uint32_t b = 0, e = 0;
    if (!zrun(g, bx + c / 3 - 1, by + c % 3 - 1, bz - 1, bz + 1, b, e)) continue;
    for (uint32_t j = b; j < e; ++j) {
      if (j == i) continue;
      double tx, ty, tz, fa;
      if (!pair_term(me.x, me.y, me.z, ri, i, ag[j], ids, j, p, tx, ty, tz, fa)) continue;
      Fx = Fx + tx;
      Fy = Fy + ty;
      Fz = Fz + tz;
      const double fn = sqrt((Fx * Fx + Fy * Fy) + Fz * Fz);
      if (!(isfinite(tx) && isfinite(ty) && isfinite(tz) && isfinite(fn))) {
        err->second = ids[j];
        return;
      }
    }
  }
  err->second = 0xfffffffeu;  // (no single pair: cannot happen for a sum that the force phase found non-finite)
}

// FONLY (neurite steps): the sphere-sphere sums F go to dp_out (3 per agent, the force-only output
// fss of k_force), the displacement rule and everything after it are left to k_sc_rows.
template <bool FONLY, bool RING = false>
__global__ void __launch_bounds__(FORCE_THREADS, HB_MIN_BLOCKS)
    k_half_sum(const double4* __restrict__ ag, const uint32_t* __restrict__ ids, uint32_t a_begin, uint32_t a_end,
               GridDev g, ParamsDev p, double4* __restrict__ ag_out, uint32_t* __restrict__ id_out,
               double* __restrict__ dp_out, uint32_t* __restrict__ dp_id_out, Extents* ext_next, ErrDev* err,
               const uint32_t* __restrict__ fwd, const uint8_t* __restrict__ fcnt, const uint32_t* __restrict__ bwd,
               const uint32_t* __restrict__ bcnt, ColNext cn, unsigned long long* __restrict__ hist_out,
               uint32_t* __restrict__ slow_list, const uint32_t* __restrict__ ab_dev = nullptr,
               uint32_t* __restrict__ work = nullptr, int64_t o_base = -1) {
  pdl_wait();
  const uint32_t rmk = RING ? g.rmask : 0xffffffffu;  // (the ring of rows of the banded phase: RING only)
  if (ab_dev) {  // distributed steps: the owned range [a_begin, a_end) read on the device
    a_begin = __ldg(&ab_dev[0]);
    a_end = __ldg(&ab_dev[1]);
  }
  // banded launches: this launch sums [a_begin, a_end), outputs are indexed from the
  // whole owned range's first agent o_base, chunk tickets come from the band's own counter
  const uint32_t ob = o_base >= 0 ? (uint32_t)o_base : a_begin;
  if (!work) work = &ext_next->work;
  extern __shared__ __align__(16) unsigned char s_raw[];
  HalfBSmem& sm = reinterpret_cast<HalfBSmem*>(s_raw)[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
  // next-step extents: reduced per chunk, kept per warp in shared memory (not in registers across
  // the chunk loop), one guarded atomic set per warp at the end
  if (lane < 8) sm.ext[lane] = lane < 3 ? INT32_MAX : (lane < 6 ? INT32_MIN : 0);
  __syncwarp();
  uint32_t n_moved = 0;
  Tickets tk(a_end - a_begin);
#if BDM_HRPF
  // merged rows: the pair counts are loaded two chunks ahead and the first vector of each row one
  // chunk ahead (the count is there by then), so a chunk's dependent chain starts at its partners
  uint32_t chunk = tk.take(work, lane);
  uint32_t chunk_n = tk.take(work, lane);
  uint32_t nb_n = 0u, nb_nn = 0u;
  uint4 r4_n = make_uint4(0u, 0u, 0u, 0u);
  {
    const uint64_t i1 = (uint64_t)a_begin + 32ull * chunk + lane;
    nb_n = i1 < a_end ? bcnt[i1 & rmk] : 0u;
    if (nb_n) r4_n = __ldg(reinterpret_cast<const uint4*>(fwd + (size_t)(i1 & rmk) * HBC));
    const uint64_t i2 = (uint64_t)a_begin + 32ull * chunk_n + lane;
    nb_nn = i2 < a_end ? bcnt[i2 & rmk] : 0u;
  }
#elif BDM_HBCNT
  // the next chunk's pair counts are loaded one chunk ahead (two registers): a chunk's dependent
  // chain then starts at its rows
  uint32_t chunk = tk.take(work, lane);
  uint32_t nf_n = 0u, nb_n = 0u;
  {
    const uint64_t i1 = (uint64_t)a_begin + 32ull * chunk + lane;
    if (i1 < a_end) {
      nf_n = BDM_MROW ? 0u : fcnt[i1];  // (merged rows: bcnt counts every entry of the one row)
      nb_n = bcnt[i1 & rmk];
    }
  }
#endif
  while (true) {
#if !BDM_HBCNT && !BDM_HRPF
    const uint32_t chunk = tk.take(work, lane);
#endif
    const uint64_t base = (uint64_t)a_begin + 32ull * chunk;
    if (base >= a_end) break;
    const uint32_t i = (uint32_t)base + lane;
    const bool valid = i < a_end;
    // the agent and both counts, then the first 4 entries of each non-empty row (one vector load;
    // entries past a count are stale and ignored)
    const uint4* brow = reinterpret_cast<const uint4*>((BDM_MROW ? fwd : bwd) + (size_t)(i & rmk) * HBC);
    const uint4* frow = reinterpret_cast<const uint4*>(fwd + (size_t)(i & rmk) * HFC);
    const double4 me = valid ? ld_state(&ag[i]) : make_double4(0.0, 0.0, 0.0, 0.0);
#if BDM_HRPF
    const uint32_t nf = 0u, nb = nb_n;
    const uint4 r4 = r4_n;
    {  // rotate: next chunk's first row vector (its count arrived during this chunk's predecessor),
       // the count of the chunk after it
      chunk = chunk_n;
      chunk_n = tk.take(work, lane);
      const uint64_t i1 = (uint64_t)a_begin + 32ull * chunk + lane;
      nb_n = nb_nn;
      r4_n = nb_n ? __ldg(reinterpret_cast<const uint4*>(fwd + (size_t)(i1 & rmk) * HBC)) : make_uint4(0u, 0u, 0u, 0u);
      const uint64_t i2 = (uint64_t)a_begin + 32ull * chunk_n + lane;
      nb_nn = i2 < a_end ? bcnt[i2 & rmk] : 0u;
    }
#elif BDM_HBCNT
    const uint32_t nf = nf_n, nb = nb_n;
    chunk = tk.take(work, lane);
    {
      const uint64_t i1 = (uint64_t)a_begin + 32ull * chunk + lane;
      nf_n = i1 < a_end && !BDM_MROW ? fcnt[i1] : 0u;
      nb_n = i1 < a_end ? bcnt[i1 & rmk] : 0u;
#if BDM_HNPF
      if (i1 < a_end) {  // the next chunk's row (and state) toward L1 while this chunk runs
        if (BDM_HNPF & 1) asm volatile("prefetch.global.L1 [%0];" ::"l"(fwd + (size_t)(i1 & rmk) * HBC));
        if (BDM_HNPF & 2) asm volatile("prefetch.global.L1 [%0];" ::"l"(ag + i1));
      }
#endif
    }
#else
    const uint32_t nf = valid && !BDM_MROW ? fcnt[i] : 0u;
    const uint32_t nb = valid ? bcnt[i & rmk] : 0u;
#endif
    // (rows are read only where the count says so: a speculative read of every row costs more DRAM
    // traffic than the round trip it saves)
#if BDM_HRPF
    const uint4 b4 = r4;
    const uint4 f4 = make_uint4(0u, 0u, 0u, 0u);
#else
    const uint4 b4 = nb ? __ldg(brow) : make_uint4(0u, 0u, 0u, 0u);
    const uint4 f4 = nf ? __ldg(frow) : make_uint4(0u, 0u, 0u, 0u);
#endif
    const double ri = 0.5 * me.w;
    const bool slow = nf > (uint32_t)HFC || nb > (uint32_t)HBC;
    int cnt = 0;
    if (!slow) {
#if BDM_HPPF
      {  // the partners' states toward L1 while the row is sorted (the contact phase gathers them)
        const uint32_t e4[4] = {b4.x, b4.y, b4.z, b4.w}, g4[4] = {f4.x, f4.y, f4.z, f4.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if ((uint32_t)k < nb) asm volatile("prefetch.global.L1 [%0];" ::"l"(ag + e4[k]));
          if (!BDM_MROW && (uint32_t)k < nf) asm volatile("prefetch.global.L1 [%0];" ::"l"(ag + g4[k]));
        }
      }
#endif
      // backward partners (all < i) sorted ascending, then forward partners (all > i, ascending)
      uint32_t* col = &sm.list[0][lane];
#if BDM_HNET
      if (nb <= 4u) {  // (the common case) a 4-input sorting network in registers, missing entries as ~0
        uint32_t a0 = b4.x, a1 = nb > 1u ? b4.y : ~0u, a2 = nb > 2u ? b4.z : ~0u, a3 = nb > 3u ? b4.w : ~0u, t;
        t = min(a0, a1); a1 = max(a0, a1); a0 = t;
        t = min(a2, a3); a3 = max(a2, a3); a2 = t;
        t = min(a0, a2); a2 = max(a0, a2); a0 = t;
        t = min(a1, a3); a3 = max(a1, a3); a1 = t;
        t = min(a1, a2); a2 = max(a1, a2); a1 = t;
        col[0] = a0;
        col[32] = a1;
        col[64] = a2;
        col[96] = a3;
      } else
#endif
      {
      col[0] = b4.x;
      col[32] = b4.y;
      col[64] = b4.z;
      col[96] = b4.w;
      for (uint32_t v = 1; 4 * v < nb; ++v) {
        const uint4 t4 = __ldg(brow + v);
        col[32 * (4 * v)] = t4.x;
        col[32 * (4 * v + 1)] = t4.y;
        col[32 * (4 * v + 2)] = t4.z;
        col[32 * (4 * v + 3)] = t4.w;
      }
      for (uint32_t t = 1; t < nb; ++t) {  // insertion sort (rows hold a handful of entries)
        const uint32_t v = col[32 * t];
        int x = (int)t;
        while (x > 0 && col[32 * (x - 1)] > v) {
          col[32 * x] = col[32 * (x - 1)];
          --x;
        }
        col[32 * x] = v;
      }
      }
      uint32_t* fc = col + 32 * nb;
      if (nf > 0) fc[0] = f4.x;
      if (nf > 1) fc[32] = f4.y;
      if (nf > 2) fc[64] = f4.z;
      if (nf > 3) fc[96] = f4.w;
      for (uint32_t v = 1; 4 * v < nf; ++v) {
        const uint4 t4 = __ldg(frow + v);
        const uint32_t u[4] = {t4.x, t4.y, t4.z, t4.w};
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (4 * v + k < nf) fc[32 * (4 * v + k)] = u[k];
      }
      cnt = (int)(nb + nf);
#if BDM_CHECK
      for (int t = 0; t < cnt; ++t) {  // canonical order: backward partners ascending below i, then forward above
        const uint32_t j = col[32 * t];
        BDM_ASSERT(BDM_MROW ? j != i : (t < (int)nb ? j < i : j > i));
        BDM_ASSERT(t == 0 || col[32 * (t - 1)] < j);
      }
#endif
    }
    __syncwarp();
    double Fx = 0.0, Fy = 0.0, Fz = 0.0;
    int32_t n_ct = 0;
    unsigned long long ct_hash = 0;
#if BDM_HDIRECT
    {  // each lane its own candidates, in canonical order (a divergent loop: lanes of one chunk have
       // similar counts)
      const uint32_t* col = &sm.list[0][lane];
      for (int t = 0; t < cnt; ++t) {
        const uint32_t j = col[32 * t];
        double tx, ty, tz, fa;
        if (pair_term(me.x, me.y, me.z, ri, i, ld_state(&ag[j]), ids, j, p, tx, ty, tz, fa)) {
          Fx = Fx + tx;
          Fy = Fy + ty;
          Fz = Fz + tz;
        }
      }
      cnt = 0;
    }
#else
    if (__any_sync(FULL, cnt > 0))
      flush_contacts<false, HalfBSmem>(sm, lane, cnt, me.x, me.y, me.z, ri, i, ag, ids, p, Fx, Fy, Fz, n_ct,
                                       ct_hash);
#endif
    {  // overflowing agents go to the slow list: k_half_slow sums and steps them (keeping the full
       // search out of this kernel keeps its registers and stack small)
      const unsigned sm_ = __ballot_sync(FULL, slow);
      if (sm_) {
        uint32_t b0 = 0;
        if (lane == 0) b0 = atomicAdd(&ext_next->slow, (uint32_t)__popc(sm_));
        b0 = __shfl_sync(FULL, b0, 0);
        if (slow) slow_list[b0 + __popc(sm_ & ((1u << lane) - 1u))] = i;
      }
    }
    const bool live = valid && !slow;
    if (FONLY) {
      if (live) {
        if (!(isfinite(Fx) && isfinite(Fy) && isfinite(Fz))) report(err, 6u /*ENONFINITE*/, ids[i], i);
        const size_t o = 3 * (size_t)(i - ob);
        dp_out[o] = Fx;
        dp_out[o + 1] = Fy;
        dp_out[o + 2] = Fz;
      }
      continue;
    }

    // O6 displacement, O7 update (as k_force)
    double dpx = 0.0, dpy = 0.0, dpz = 0.0;
    const double fn = sqrt((Fx * Fx + Fy * Fy) + Fz * Fz);
    if (fn <= p.adherence) {
    } else if (fn * p.c > p.max_disp) {
      const double scale = p.max_disp / fn;
      dpx = Fx * scale;
      dpy = Fy * scale;
      dpz = Fz * scale;
    } else {
      dpx = Fx * p.c;
      dpy = Fy * p.c;
      dpz = Fz * p.c;
    }
    int nb3[3] = {INT32_MAX, INT32_MAX, INT32_MAX};  // box of p'
    bool ebad = false;
    if (live) {
      if (!(isfinite(Fx) && isfinite(Fy) && isfinite(Fz) && isfinite(fn))) report(err, 6u /*ENONFINITE*/, ids[i], i);
      const double4 np = make_double4(me.x + dpx, me.y + dpy, me.z + dpz, me.w);
      const uint32_t o = i - ob;
      st_state(&ag_out[o], np);
      if (hist_out) {
        const bool moved = dpx != 0.0 || dpy != 0.0 || dpz != 0.0;
        hist_out[o] = ((unsigned long long)moved << 63) |
                      pack_box((int)floor(me.x * g.inv), (int)floor(me.y * g.inv), (int)floor(me.z * g.inv));
      }
      if (id_out) id_out[o] = ids[i];
      if (dp_out) {
        dp_out[3 * (size_t)o] = dpx;
        dp_out[3 * (size_t)o + 1] = dpy;
        dp_out[3 * (size_t)o + 2] = dpz;
        if (dp_id_out) dp_id_out[o] = ids[i];
      }
      nb3[0] = box_coord(np.x, g.inv, ebad);
      nb3[1] = box_coord(np.y, g.inv, ebad);
      nb3[2] = box_coord(np.z, g.inv, ebad);
    }
    {
      int lo3[3], hi3[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        lo3[a] = __reduce_min_sync(FULL, nb3[a]);
        hi3[a] = __reduce_max_sync(FULL, live ? nb3[a] : INT32_MIN);
      }
      const bool anybad = __any_sync(FULL, ebad);
      if (lane == 0) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          sm.ext[a] = min(sm.ext[a], lo3[a]);
          sm.ext[3 + a] = max(sm.ext[3 + a], hi3[a]);
        }
        if (anybad) sm.ext[6] = 1;
      }
    }
    if (hist_out)  // movers of this step (the skip heuristic of the next build), added once per warp
      n_moved += __popc(__ballot_sync(FULL, live && (dpx != 0.0 || dpy != 0.0 || dpz != 0.0)));
    if (cn.czlo) {  // fused column pass (warp-aggregated: a chunk touches one or two columns)
      uint32_t c = 0xffffffffu;
      bool out = false;
      if (live) {
        const int ux = nb3[0] - cn.lo0, uy = nb3[1] - cn.lo1;
        if (ux >= 0 && ux < cn.nx && uy >= 0 && uy < cn.ny)
          c = (uint32_t)ux * (uint32_t)cn.ny + (uint32_t)uy;
        else
          out = true;
        if (cn.pbox) {  // the next build's column and z, so its key pass need not re-read the state
          const uint32_t uz = (uint32_t)(nb3[2] - cn.z0);
          out |= uz >> cn.zbits != 0u;
          cn.pbox[i - ob] = (c << cn.zbits) | uz;
        }
      }
      const unsigned peers = __match_any_sync(FULL, c);  // (a run-based mask here measured slower: 0.77 ms)
      const int zmin = __reduce_min_sync(peers, live ? nb3[2] : INT32_MAX);
      const int zmax = __reduce_max_sync(peers, live ? nb3[2] : INT32_MIN);
      if (c != 0xffffffffu && lane == __ffs(peers) - 1) {  // fire-and-forget reductions (RED)
        atomicMin(&cn.czlo[c], zmin);
        atomicMax(&cn.czhi[c], zmax);
      }
      if (__any_sync(FULL, out) && lane == 0) ext_next->col_bad = 1u;
    }
  }
  if (hist_out && lane == 0 && n_moved) atomicAdd(&ext_next->moved, n_moved);
  __syncwarp();
  if (lane == 0) {
    if (sm.ext[6]) ext_next->range_err = 1;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const int lo = sm.ext[a], hi = sm.ext[3 + a];
      if (lo != INT32_MAX && lo < __ldcg(&ext_next->lo[a])) atomicMin(&ext_next->lo[a], lo);
      if (hi != INT32_MIN && hi > __ldcg(&ext_next->hi[a])) atomicMax(&ext_next->hi[a], hi);
    }
  }
}


// The agents of the sum pass whose pair rows overflowed (slow_list[0 .. ext->slow)): the full
// canonical 27-box sum (full_force, O3-O5 as written), then exactly the sum pass's per-agent
// epilogue with global atomics in place of the warp reductions.  Grid-stride over the list.
template <bool FONLY>
__global__ void __launch_bounds__(128) k_half_slow(const double4* __restrict__ ag, const uint32_t* __restrict__ ids,
                                                   uint32_t a_begin, GridDev g, ParamsDev p,
                                                   double4* __restrict__ ag_out, uint32_t* __restrict__ id_out,
                                                   double* __restrict__ dp_out, uint32_t* __restrict__ dp_id_out,
                                                   Extents* ext_next, ErrDev* err, ColNext cn,
                                                   unsigned long long* __restrict__ hist_out,
                                                   const uint32_t* __restrict__ slow_list,
                                                   const uint32_t* __restrict__ ab_dev = nullptr) {
  pdl_wait();
  if (ab_dev) a_begin = __ldg(&ab_dev[0]);
  const uint32_t n_slow = __ldcg(&ext_next->slow);
  const int lane = threadIdx.x & 31;
  const uint32_t warps = gridDim.x * (blockDim.x >> 5);
  for (uint32_t k = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); k < n_slow; k += warps) {  // warp per agent
    const uint32_t i = slow_list[k];
    const double4 me = ag[i];
    const double3 f = full_force_warp(g, ag, ids, p, i, me, lane);
    if (lane != 0) continue;  // (lane 0 writes the agent's results)
    const double Fx = f.x, Fy = f.y, Fz = f.z;
    const uint32_t o = i - a_begin;
    if (FONLY) {
      if (!(isfinite(Fx) && isfinite(Fy) && isfinite(Fz))) report(err, 6u /*ENONFINITE*/, ids[i], i);
      dp_out[3 * (size_t)o] = Fx;
      dp_out[3 * (size_t)o + 1] = Fy;
      dp_out[3 * (size_t)o + 2] = Fz;
      continue;
    }
    double dpx = 0.0, dpy = 0.0, dpz = 0.0;
    const double fn = sqrt((Fx * Fx + Fy * Fy) + Fz * Fz);
    if (fn <= p.adherence) {
    } else if (fn * p.c > p.max_disp) {
      const double scale = p.max_disp / fn;
      dpx = Fx * scale;
      dpy = Fy * scale;
      dpz = Fz * scale;
    } else {
      dpx = Fx * p.c;
      dpy = Fy * p.c;
      dpz = Fz * p.c;
    }
    if (!(isfinite(Fx) && isfinite(Fy) && isfinite(Fz) && isfinite(fn))) report(err, 6u /*ENONFINITE*/, ids[i], i);
    const double4 np = make_double4(me.x + dpx, me.y + dpy, me.z + dpz, me.w);
    ag_out[o] = np;
    const bool moved = dpx != 0.0 || dpy != 0.0 || dpz != 0.0;
    if (hist_out) {
      hist_out[o] = ((unsigned long long)moved << 63) |
                    pack_box((int)floor(me.x * g.inv), (int)floor(me.y * g.inv), (int)floor(me.z * g.inv));
      if (moved) atomicAdd(&ext_next->moved, 1u);
    }
    if (id_out) id_out[o] = ids[i];
    if (dp_out) {
      dp_out[3 * (size_t)o] = dpx;
      dp_out[3 * (size_t)o + 1] = dpy;
      dp_out[3 * (size_t)o + 2] = dpz;
      if (dp_id_out) dp_id_out[o] = ids[i];
    }
    bool ebad = false;
    const int nb3[3] = {box_coord(np.x, g.inv, ebad), box_coord(np.y, g.inv, ebad), box_coord(np.z, g.inv, ebad)};
    if (ebad) ext_next->range_err = 1;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      atomicMin(&ext_next->lo[a], nb3[a]);
      atomicMax(&ext_next->hi[a], nb3[a]);
    }
    if (cn.czlo) {
      const int ux = nb3[0] - cn.lo0, uy = nb3[1] - cn.lo1;
      if (ux >= 0 && ux < cn.nx && uy >= 0 && uy < cn.ny) {
        const uint32_t c = (uint32_t)ux * (uint32_t)cn.ny + (uint32_t)uy;
        atomicMin(&cn.czlo[c], nb3[2]);
        atomicMax(&cn.czhi[c], nb3[2]);
        if (cn.pbox) {
          const uint32_t uz = (uint32_t)(nb3[2] - cn.z0);
          if (uz >> cn.zbits != 0u) ext_next->col_bad = 1u;
          cn.pbox[o] = (c << cn.zbits) | uz;
        }
      } else {
        ext_next->col_bad = 1u;
      }
    }
  }
}

// ------------------------------------------------------------------------------------------ K5/K9
// x-slab exchange records: 5 fp64 per agent (x, y, z, D, id) -- ids < 2^32 are exact in fp64.
constexpr int REC = 5;

// Halo (mode 0): owned agents in the first box-x layer of the slab go to the lower neighbour, those
// in the last layer to the upper one (both when the slab is one box wide).  Migration (mode 1):
// agents whose box-x left [x_begin, x_end) go to the neighbour on that side; the others are
// compacted into keep_ag/keep_id.  Order inside the buffers is irrelevant: the receiver sorts by
// (box, id).  Counters: cnt[0] lo, cnt[1] hi, cnt[2] kept; records past a capacity are dropped
// (the counts still tell the caller how much to allocate, and keep_* is only committed when both
// sends fit).
__global__ void k_slab_pack(const double4* __restrict__ ag, const uint32_t* __restrict__ ids, uint32_t n,
                            double inv, int mode, int32_t x_begin, int32_t x_end, double* __restrict__ send_lo,
                            double* __restrict__ send_hi, uint64_t cap, uint32_t* __restrict__ cnt,
                            double4* __restrict__ keep_ag, uint32_t* __restrict__ keep_id) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = i < n;
  double4 p = valid ? ag[i] : make_double4(0.0, 0.0, 0.0, 0.0);
  const uint32_t id = valid ? ids[i] : 0u;
  const int bx = (int)floor(p.x * inv);
  bool to_lo, to_hi;
  if (mode == 0) {
    to_lo = valid && x_begin != INT32_MIN && bx == x_begin;
    to_hi = valid && x_end != INT32_MAX && bx == x_end - 1;
  } else {
    to_lo = valid && bx < x_begin;
    to_hi = valid && bx >= x_end;
  }
  const bool keep = mode == 1 && valid && !to_lo && !to_hi;
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const unsigned mlo = __ballot_sync(FULL, to_lo), mhi = __ballot_sync(FULL, to_hi), mk = __ballot_sync(FULL, keep);
  uint32_t blo = 0, bhi = 0, bk = 0;
  if (lane == 0) {
    if (mlo) blo = atomicAdd(&cnt[0], (uint32_t)__popc(mlo));
    if (mhi) bhi = atomicAdd(&cnt[1], (uint32_t)__popc(mhi));
    if (mk) bk = atomicAdd(&cnt[2], (uint32_t)__popc(mk));
  }
  blo = __shfl_sync(FULL, blo, 0) + __popc(mlo & lt);
  bhi = __shfl_sync(FULL, bhi, 0) + __popc(mhi & lt);
  bk = __shfl_sync(FULL, bk, 0) + __popc(mk & lt);
  if (to_lo && blo < cap) {
    double* r = send_lo + (size_t)REC * blo;
    r[0] = p.x; r[1] = p.y; r[2] = p.z; r[3] = p.w; r[4] = (double)id;
  }
  if (to_hi && bhi < cap) {
    double* r = send_hi + (size_t)REC * bhi;
    r[0] = p.x; r[1] = p.y; r[2] = p.z; r[3] = p.w; r[4] = (double)id;
  }
  if (keep) {
    keep_ag[bk] = p;
    keep_id[bk] = id;
  }
}

// Post-step split of the owned agents (single-sync protocol).  Only the first two and
// last two box-x layers of the step's sorted order can hold emigrants (a step moves an agent by less
// than a box) or the stayers of the first / last layer (the neighbours' next ghosts): ranges
// [0, r_lo) and [r_hi, n) of the stepped array.  Emigrants (new box-x outside [x_begin, x_end)) go
// to the FRONT of send_lo / send_hi (bdm_slab_commit then marks them dead in place, D < 0, and the
// next sort drops them); the stayers of the first / last layer go to the BACK (record cap-1-k).  The middle of the array
// is not touched.  cnt[0] emigrants lo, [1] halo lo, [2] emigrants hi, [3] halo hi (block-aggregated
// atomics); records past a segment's room are dropped (the counts still tell).
__global__ void k_slab_split(const double4* __restrict__ ag, const uint32_t* __restrict__ ids, uint32_t n,
                             const uint32_t* __restrict__ r2, double inv, int32_t x_begin, int32_t x_end,
                             double* __restrict__ send_lo, double* __restrict__ send_hi, uint64_t cap,
                             uint32_t* __restrict__ cnt, const uint32_t* __restrict__ n_dev = nullptr) {
  pdl_wait();
  __shared__ uint32_t s_cnt[4], s_base[4];
  if (n_dev) n = __ldg(n_dev);
  const uint32_t n_lo_part = r2[0] < n ? r2[0] : n;
  const uint32_t hi0 = r2[1] > n_lo_part ? r2[1] : n_lo_part;  // ranges do not overlap
  const uint64_t total = (uint64_t)n_lo_part + (n - hi0);
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  for (uint64_t t0 = (uint64_t)blockIdx.x * blockDim.x; t0 < total; t0 += (uint64_t)gridDim.x * blockDim.x) {
    if (threadIdx.x < 4) s_cnt[threadIdx.x] = 0u;
    __syncthreads();
    const uint64_t t = t0 + threadIdx.x;
    const bool valid = t < total;
    const uint32_t i = !valid ? 0u : (t < n_lo_part ? (uint32_t)t : hi0 + (uint32_t)(t - n_lo_part));
    double4 p = valid ? ag[i] : make_double4(0.0, 0.0, 0.0, 0.0);
    const int bx = (int)floor(p.x * inv);
    const bool mlo = valid && bx < x_begin, mhi = valid && bx >= x_end;
    const bool keep = valid && !mlo && !mhi;
    const bool hlo = keep && x_begin != INT32_MIN && bx == x_begin;
    const bool hhi = keep && x_end != INT32_MAX && bx == x_end - 1;
    const bool f[4] = {mlo, hlo, mhi, hhi};
    uint32_t loc[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const unsigned m = __ballot_sync(FULL, f[c]);
      uint32_t b = 0;
      if (lane == 0 && m) b = atomicAdd(&s_cnt[c], (uint32_t)__popc(m));
      loc[c] = __shfl_sync(FULL, b, 0) + __popc(m & lt);
    }
    __syncthreads();
    if (threadIdx.x < 4) s_base[threadIdx.x] = s_cnt[threadIdx.x] ? atomicAdd(&cnt[threadIdx.x], s_cnt[threadIdx.x]) : 0u;
    __syncthreads();
    if (valid && (mlo || mhi || hlo || hhi)) {
      const uint32_t id = ids[i];
      auto put = [&](double* buf, uint64_t k) {
        double* r = buf + (size_t)REC * k;
        r[0] = p.x; r[1] = p.y; r[2] = p.z; r[3] = p.w; r[4] = (double)id;
      };
      if (mlo && s_base[0] + loc[0] < cap) put(send_lo, s_base[0] + loc[0]);
      if (mhi && s_base[2] + loc[2] < cap) put(send_hi, s_base[2] + loc[2]);
      if (hlo && s_base[1] + loc[1] < cap) put(send_lo, cap - 1 - (s_base[1] + loc[1]));
      if (hhi && s_base[3] + loc[3] < cap) put(send_hi, cap - 1 - (s_base[3] + loc[3]));
    }
    __syncthreads();
  }
}

// bdm_slab_commit: emigrants of the split (same boundary ranges) are marked dead (D < 0) in place.
__global__ void k_slab_mark_dead(double4* __restrict__ ag, uint32_t n, const uint32_t* __restrict__ r2, double inv,
                                 int32_t x_begin, int32_t x_end, const uint32_t* __restrict__ n_dev = nullptr,
                                 uint32_t* __restrict__ pbox = nullptr) {
  pdl_wait();
  if (n_dev) n = __ldg(n_dev);
  const uint32_t n_lo_part = r2[0] < n ? r2[0] : n;
  const uint32_t hi0 = r2[1] > n_lo_part ? r2[1] : n_lo_part;
  const uint64_t total = (uint64_t)n_lo_part + (n - hi0);
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t i = t < n_lo_part ? (uint32_t)t : hi0 + (uint32_t)(t - n_lo_part);
    const int bx = (int)floor(ag[i].x * inv);
    if (bx < x_begin || bx >= x_end) {
      ag[i].w = -1.0;
      if (pbox) pbox[i] = 0xffffffffu;
    }
  }
}

// First stepped agent of box-x layer X in the slab step's sorted order (owned indexing: the lower
// ghosts, which sort first, are subtracted); X outside the grid clamps.
__global__ void k_layer_bounds(GridDev g, int32_t x_begin, int32_t x_end, uint32_t n_lo, uint32_t n,
                               uint32_t* __restrict__ out2) {
  if (threadIdx.x >= 2) return;
  const int64_t X = threadIdx.x == 0 ? (int64_t)x_begin + 2 : (int64_t)x_end - 2;
  uint32_t r;
  if (threadIdx.x == 0 && x_begin == INT32_MIN) {
    r = 0u;
  } else if (threadIdx.x == 1 && x_end == INT32_MAX) {
    r = n;
  } else if (X <= g.lo[0]) {
    r = 0u;
  } else if (X > g.hi[0]) {
    r = n;
  } else {
    const uint32_t c = (uint32_t)(X - g.lo[0]) * (uint32_t)g.ny;
    const uint32_t k = g.table[g.coff[c]];
    r = k > n_lo ? k - n_lo : 0u;
    r = r < n ? r : n;
  }
  out2[threadIdx.x] = r;
}

// info[0..3] = split counters, info[4] = stayers, info[5..10] = the owned agents' box extents lo[3], hi[3] (from the
// step that produced these positions), info[11] = 1 if a segment overflowed its room.
__global__ void k_split_info(const uint32_t* __restrict__ cnt, const Extents* __restrict__ ext, uint64_t cap,
                             uint32_t n, int64_t* __restrict__ info) {
  const int t = threadIdx.x;
  if (t < 4) info[t] = cnt[t];
  if (t == 4) info[4] = (int64_t)n - cnt[0] - cnt[2];
  if (t < 3) {
    info[5 + t] = ext->lo[t];
    info[8 + t] = ext->hi[t];
  }
  if (t == 0) info[11] = (uint64_t)cnt[0] + cnt[1] > cap || (uint64_t)cnt[2] + cnt[3] > cap ? 1 : 0;
}

// Appends records (ghosts or immigrants) at ag[off..off+m).
__global__ void k_unpack(const double* __restrict__ rec, uint32_t m, double4* __restrict__ ag,
                         uint32_t* __restrict__ ids, uint32_t off) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m) return;
  const double* r = rec + (size_t)REC * t;
  ag[off + t] = make_double4(r[0], r[1], r[2], r[3]);
  ids[off + t] = (uint32_t)r[4];
}

// Max diameter of ag[0..n) (positive doubles order like their bit patterns).
__global__ void k_maxd(const double4* __restrict__ ag, uint32_t n, unsigned long long* maxd_bits) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long b = i < n ? (unsigned long long)__double_as_longlong(ag[i].w) : 0ull;
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long v = __shfl_xor_sync(FULL, b, o);
    b = v > b ? v : b;
  }
  if ((threadIdx.x & 31) == 0 && b && b > __ldcg(maxd_bits)) atomicMax(maxd_bits, b);
}

// ------------------------------------------------------------------------------------------ NEXT-2
// Cell growth and division (G1-G3), after the mechanics of a step, on the stepped
// buffer (sorted order of that step, ids alongside).  Daughters are appended behind the n agents
// (unsorted; the next build sorts them).
__global__ void k_grow(double4* __restrict__ ag, const uint32_t* __restrict__ ids, uint32_t n, double growth,
                       double div_diam, uint32_t* __restrict__ flag_by_id, unsigned long long* maxd_bits) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  double Dfin = 0.0;  // the diameter this agent has after G2 (the new max D of O1 is over these)
  if (i < n) {
    const double D = ag[i].w + growth;  // G1
    ag[i].w = D;
    const bool divides = D >= div_diam;
    flag_by_id[ids[i]] = divides ? 1u : 0u;
    Dfin = divides ? D * 0.79370052598409973737585281963615 : D;  // (k_divide's D', bit for bit)
  }
  unsigned long long b = __double_as_longlong(Dfin);
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long v = __shfl_xor_sync(FULL, b, o);
    b = v > b ? v : b;
  }
  if ((threadIdx.x & 31) == 0 && b && b > __ldcg(maxd_bits)) atomicMax(maxd_bits, b);
}

__device__ __forceinline__ double div_u01(uint64_t seed, uint64_t step, uint64_t id, uint64_t a) {
  return (double)(mix64(seed * 0x9E3779B97F4A7C15ull + ((step << 32) + id) * 4ull + a) >> 11) * 0x1p-53;
}

// G2.  rank_by_id = exclusive scan of the division flags in id order, so the k-th divider in
// ascending id order creates daughter id n + k at position n + k.
__global__ void k_divide(double4* __restrict__ ag, uint32_t* __restrict__ ids, uint32_t n, double div_diam,
                         uint64_t seed, uint64_t step, const uint32_t* __restrict__ rank_by_id) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    double4 p = ag[i];
    if (p.w >= div_diam) {
      const uint32_t id = ids[i];
      const uint32_t d = n + rank_by_id[id];
      double v[3], u[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) v[a] = 2.0 * div_u01(seed, step, id, (uint64_t)a) - 1.0;
      const double norm = sqrt((v[0] * v[0] + v[1] * v[1]) + v[2] * v[2]);
      if (norm == 0.0) {
        u[0] = 1.0;
        u[1] = 0.0;
        u[2] = 0.0;
      } else {
#pragma unroll
        for (int a = 0; a < 3; ++a) u[a] = v[a] / norm;
      }
      const double Dd = p.w * 0.79370052598409973737585281963615;  // 2^(-1/3)
      const double h = 0.5 * Dd;
      const double ox = h * u[0], oy = h * u[1], oz = h * u[2];
      ag[i] = make_double4(p.x - ox, p.y - oy, p.z - oz, Dd);
      ag[d] = make_double4(p.x + ox, p.y + oy, p.z + oz, Dd);
      ids[d] = d;
    }
  }
}

// ------------------------------------------------------------------------------------------ NEXT-3
// Soma clustering (S1-S4): two substances on a regular lattice, secreted by the
// agents of their type, diffused by explicit Euler with the 7-point stencil (closed boundary), and
// followed by chemotaxis before the mechanics.  Arithmetic written exactly as the oracle's.
struct FieldDev {
  double h, invh, ih2, gh1, gh2;  // h, 1/h, 1/(h*h), 1/h (one-sided), 0.5/h (central)
  double ox, oy, oz;
  int32_t nx, ny, nz;
  uint32_t nn;
  double diff, decay, dt, secretion, speed;
};

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

// S1: integer count of secreting agents per nearest node (warp-aggregated atomics)
__global__ void k_secrete(const double4* __restrict__ ag, const uint32_t* __restrict__ ids, uint32_t n,
                          const int8_t* __restrict__ type_by_id, FieldDev f, uint32_t* __restrict__ counts) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t k = 0xffffffffu;
  if (i < n) {
    const double4 p = ag[i];
    const int bx = clampi((int)floor((p.x - f.ox) * f.invh + 0.5), 0, f.nx - 1);
    const int by = clampi((int)floor((p.y - f.oy) * f.invh + 0.5), 0, f.ny - 1);
    const int bz = clampi((int)floor((p.z - f.oz) * f.invh + 0.5), 0, f.nz - 1);
    k = (type_by_id[ids[i]] ? f.nn : 0u) + ((uint32_t)bx * f.ny + by) * f.nz + bz;
  }
  const unsigned peers = __match_any_sync(FULL, k);
  if (i < n && (threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&counts[k], (uint32_t)__popc(peers));
}

__device__ __forceinline__ double secreted(const double* __restrict__ c, const uint32_t* __restrict__ cnt,
                                           uint32_t k, double s) {
  const uint32_t m = cnt[k];
  const double v = c[k];
  return m ? v + (double)m * s : v;
}

// S1 + S2 fused: every stencil value is the secreted value of that node (c + count * s).  One
// thread per node, z fastest (coalesced); neighbours come from L1/L2.
__global__ void k_diffuse(const double* __restrict__ c, const uint32_t* __restrict__ cnt, double* __restrict__ out,
                          FieldDev f) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= f.nn) return;
  const int z = (int)(k % (uint32_t)f.nz);
  const int y = (int)((k / (uint32_t)f.nz) % (uint32_t)f.ny);
  const int x = (int)(k / ((uint32_t)f.nz * (uint32_t)f.ny));
  const uint32_t sx = (uint32_t)f.ny * f.nz, sy = (uint32_t)f.nz;
  const double s = f.secretion;
  const double c0 = secreted(c, cnt, k, s);
  const double xm = secreted(c, cnt, x > 0 ? k - sx : k, s), xp = secreted(c, cnt, x + 1 < f.nx ? k + sx : k, s);
  const double ym = secreted(c, cnt, y > 0 ? k - sy : k, s), yp = secreted(c, cnt, y + 1 < f.ny ? k + sy : k, s);
  const double zm = secreted(c, cnt, z > 0 ? k - 1 : k, s), zp = secreted(c, cnt, z + 1 < f.nz ? k + 1 : k, s);
  const double lap = ((((xm + xp) + (ym + yp)) + (zm + zp)) - 6.0 * c0) * f.ih2;
  const double v = c0 + f.dt * (f.diff * lap - f.decay * c0);
  out[k] = v < 0.0 ? 0.0 : v;  // negative results clamped to 0 (reachable when 6 D dt/h^2 + mu dt > 1)
}

__device__ __forceinline__ double node_grad(const double* __restrict__ c, const FieldDev& f, int x, int y, int z,
                                            int a) {
  int v[3] = {x, y, z}, lo[3] = {x, y, z}, hi[3] = {x, y, z};
  const int dim[3] = {f.nx, f.ny, f.nz};
  if (v[a] > 0) lo[a] = v[a] - 1;
  if (v[a] + 1 < dim[a]) hi[a] = v[a] + 1;
  if (lo[a] == v[a] && hi[a] == v[a]) return 0.0;
  const double cl = c[((uint32_t)lo[0] * f.ny + lo[1]) * f.nz + lo[2]];
  const double ch = c[((uint32_t)hi[0] * f.ny + hi[1]) * f.nz + hi[2]];
  if (lo[a] == v[a] || hi[a] == v[a]) return (ch - cl) * f.gh1;
  return (ch - cl) * f.gh2;
}

// S3: gradient of the own substance at p (trilinear interpolation of node gradients), then
// p <- p + speed * g / |g|.  In place on the agents.
__global__ void k_chemotaxis(double4* __restrict__ ag, const uint32_t* __restrict__ ids, uint32_t n,
                             const int8_t* __restrict__ type_by_id, FieldDev f, const double* __restrict__ c0,
                             const double* __restrict__ c1) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double4 p = ag[i];
  const double* c = type_by_id[ids[i]] ? c1 : c0;
  const double pp[3] = {p.x, p.y, p.z}, org[3] = {f.ox, f.oy, f.oz};
  const int dim[3] = {f.nx, f.ny, f.nz};
  int b[3];
  double w[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double q = (pp[a] - org[a]) * f.invh;
    const double fl = floor(q);
    int i0 = (int)fl;
    double t = q - fl;
    if (i0 < 0) {
      i0 = 0;
      t = 0.0;
    }
    if (i0 > dim[a] - 2) {
      i0 = dim[a] - 2 >= 0 ? dim[a] - 2 : 0;
      t = dim[a] >= 2 ? 1.0 : 0.0;
    }
    b[a] = i0;
    w[a] = t;
  }
  // the 8 corner weights are the same for the three axes (computed once, the same expressions)
  double wk[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int dx = (k >> 2) & 1, dy = (k >> 1) & 1, dz = k & 1;
    const double wxy = (dx ? w[0] : 1.0 - w[0]) * (dy ? w[1] : 1.0 - w[1]);
    wk[k] = wxy * (dz ? w[2] : 1.0 - w[2]);
  }
  double g[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int dx = (k >> 2) & 1, dy = (k >> 1) & 1, dz = k & 1;
      const int x = min(b[0] + dx, f.nx - 1), y = min(b[1] + dy, f.ny - 1), z = min(b[2] + dz, f.nz - 1);
      acc = acc + wk[k] * node_grad(c, f, x, y, z, a);
    }
    g[a] = acc;
  }
  const double gn = sqrt((g[0] * g[0] + g[1] * g[1]) + g[2] * g[2]);
  if (!(gn > 0.0)) return;
  const double sc = f.speed / gn;
  ag[i] = make_double4(p.x + g[0] * sc, p.y + g[1] * sc, p.z + g[2] * sc, p.w);
}

// ------------------------------------------------------------------------------------------ NEXT-4
// Neurite elements (cylinders): sphere-cylinder contacts and spring chains (N1-N6).
// Element e by id: eq[e] = (distal Q, diameter d), ea[e] = (anchor A, resting length l0),
// et[e] = (mother, daughter1, daughter2) with daughter1 < daughter2 when both exist.

__device__ __forceinline__ void el_geom(uint32_t e, const double4* __restrict__ eq, const double4* __restrict__ ea,
                                        const int4* __restrict__ et, double P[3], double v[3], double& len) {
  const double4 q = eq[e];
  const int m = et[e].x;
  const double4 pp = m >= 0 ? eq[m] : ea[e];
  P[0] = pp.x;
  P[1] = pp.y;
  P[2] = pp.z;
  v[0] = q.x - pp.x;
  v[1] = q.y - pp.y;
  v[2] = q.z - pp.z;
  len = sqrt((v[0] * v[0] + v[1] * v[1]) + v[2] * v[2]);
}

// Per-element geometry of a step, computed once (id order) and gathered by the contact kernels:
// a = (P, r_e), b = (v, len), c = (T, 1/len) with T = k_s ((len - l0)/l0) (N1, N3)
struct ElGeo {
  double4 a, b, c;
};

// N1/N2: element centres (for the element grid) and their extent len + d; the geometry records
__global__ void k_el_geom(const double4* __restrict__ eq, const double4* __restrict__ ea, const int4* __restrict__ et,
                          uint32_t E, double* __restrict__ cpos, double* __restrict__ cdiam, ElGeo* __restrict__ geo,
                          double k_spring) {
  const uint32_t e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  double P[3], v[3], len;
  el_geom(e, eq, ea, et, P, v, len);
  const double de = eq[e].w;
  cpos[3 * (size_t)e] = P[0] + 0.5 * v[0];
  cpos[3 * (size_t)e + 1] = P[1] + 0.5 * v[1];
  cpos[3 * (size_t)e + 2] = P[2] + 0.5 * v[2];
  cdiam[e] = len + de;
  if (geo) {
    const double l0 = ea[e].w;
    ElGeo g;
    g.a = make_double4(P[0], P[1], P[2], 0.5 * de);
    g.b = make_double4(v[0], v[1], v[2], len);
    g.c = make_double4(k_spring * ((len - l0) / l0), 1.0 / len, 0.0, 0.0);
    geo[e] = g;
  }
}

// N4: force on the sphere at c (radius rs) from the element (P, v, re); false without contact
__device__ __forceinline__ bool sc_term(const double c[3], double rs, const double P[3], const double v[3], double re,
                                        const ParamsDev& p, double t3[3]) {
  const double cp0 = c[0] - P[0], cp1 = c[1] - P[1], cp2 = c[2] - P[2];
  const double vv = (v[0] * v[0] + v[1] * v[1]) + v[2] * v[2];
  double t = 0.0;
  if (vv > 0.0) {
    t = ((cp0 * v[0] + cp1 * v[1]) + cp2 * v[2]) / vv;
    t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
  }
  const double w0 = c[0] - (P[0] + t * v[0]), w1 = c[1] - (P[1] + t * v[1]), w2 = c[2] - (P[2] + t * v[2]);
  const double d2 = (w0 * w0 + w1 * w1) + w2 * w2;
  if (!(d2 > 0.0)) return false;
  const double d = sqrt(d2);
  const double s = rs + re;
  const double delta = s - d;
  if (!(delta > 0.0)) return false;
  const double r = (rs * re) / s;
  const double f = p.k_rep * delta - p.gamma_att * sqrt(r * delta);
  const double m = f / d;
  t3[0] = m * w0;
  t3[1] = m * w1;
  t3[2] = m * w2;
  return true;
}

__device__ __forceinline__ int disp_rule(double Fx, double Fy, double Fz, const ParamsDev& p, double& dx, double& dy,
                                         double& dz) {
  dx = dy = dz = 0.0;
  const double fn = sqrt((Fx * Fx + Fy * Fy) + Fz * Fz);
  if (fn <= p.adherence) return 0;
  if (fn * p.c > p.max_disp) {
    const double scale = p.max_disp / fn;
    dx = Fx * scale;
    dy = Fy * scale;
    dz = Fz * scale;
    return 1;
  }
  dx = Fx * p.c;
  dy = Fy * p.c;
  dz = Fz * p.c;
  return 2;
}

// N5 (spheres) + O6/O7: sphere-sphere sum from the force-only pass, then the element terms over the
// 27 element boxes (canonical order, ascending element id inside a box).
// Conservative fp32 sphere-element prefilter.  A contact needs d < r_s + r_e with d the distance
// to the segment, and d >= |c - C| - len/2 for the midpoint C, so |c - C| < r_s + h with h = len/2 +
// r_e = 0.5 * (len + d_e), the element grid's half extent (the element agf holds (C, -h) in fp32).
// Both fp32 centres are within their grid's m32 of the fp64 values, the bound is
// rounded up and carries a relative 2^-20 for the fp32 sum of squares: only pairs that can be
// contacts reach the exact fp64 evaluation (sc_term), so the sums are unchanged.
__device__ __forceinline__ bool sc_near(float4 a, float4 b, float rsm, float h) {
  const float dx = a.x - b.x, dy = a.y - b.y, dz = a.z - b.z;
  const float d2 = (dx * dx + dy * dy) + dz * dz;
  const float R = __fadd_ru(rsm, h);
  return d2 <= __fmul_ru(__fmul_ru(R, R), 1.0f + 0x1p-20f);
}

// Sphere-element contact rows: k_el_update finds every contact (it searches the 27 sphere boxes of
// each element anyway) and appends the element's sorted index to the sphere's row; the sphere pass
// evaluates its row's terms in ascending element sorted index, which is N5's canonical order (boxes
// in (dx,dy,dz) lexicographic order = ascending key, ascending id inside a box), with the same
// sc_term arguments as a sphere-side search: the sums are bit-identical to one.
constexpr int SCAP = 16;  // entries per sphere row; more contacts -> the sphere searches itself

// N4 + N5 (one sphere): element terms over the 27 element boxes in canonical order (overflow path)
__device__ __noinline__ double3 sc_full(const double4 me, const float4 mf, double3 F, const GridDev gs,
                                        const GridDev ge, const float4* __restrict__ elf,
                                        const uint32_t* __restrict__ el_ids, const ElGeo* __restrict__ geo,
                                        const ParamsDev p) {
  const double c[3] = {me.x, me.y, me.z};
  const double rs = 0.5 * me.w;
  const float rsm = __double2float_ru(rs + gs.m32 + ge.m32);
  const int bx = (int)floor(me.x * ge.inv), by = (int)floor(me.y * ge.inv), bz = (int)floor(me.z * ge.inv);
  for (int col = 0; col < 9; ++col) {
    uint32_t b, e;
    if (!zrun(ge, bx + col / 3 - 1, by + col % 3 - 1, bz - 1, bz + 1, b, e)) continue;
    for (uint32_t q = b; q < e; ++q) {
      const float4 ef = __ldg(&elf[q]);
      if (!sc_near(mf, ef, rsm, -ef.w)) continue;
      const uint32_t el = el_ids[q];
      const double4 ga = geo[el].a, gb = geo[el].b;
      const double P[3] = {ga.x, ga.y, ga.z}, v[3] = {gb.x, gb.y, gb.z};
      double t3[3];
      if (sc_term(c, rs, P, v, ga.w, p, t3)) {
        F.x = F.x + t3[0];
        F.y = F.y + t3[1];
        F.z = F.z + t3[2];
      }
    }
  }
  return F;
}

// resident blocks of 256 threads per SM for the neurite kernels (they are latency-bound: 64
// registers and 32 warps per SM beat fewer warps without spills, 1.58 -> 1.30 ms per step)
#ifndef BDM_ELU_MINB
#define BDM_ELU_MINB 4
#endif
#ifndef BDM_SCR_MINB
#define BDM_SCR_MINB 4
#endif
// N5 (spheres) + O6/O7: sphere-sphere sums fss plus the element terms of the sphere's contact row
// (sorted by element index; overflowing rows take sc_full), then the displacement rule and update.
__global__ void __launch_bounds__(256, BDM_SCR_MINB) k_sc_rows(const double4* __restrict__ ag, const float4* __restrict__ agf,
                          const double* __restrict__ fss, uint32_t n, GridDev gs, GridDev ge,
                          const float4* __restrict__ elf, const uint32_t* __restrict__ el_ids,
                          const ElGeo* __restrict__ geo, const uint32_t* __restrict__ scnt,
                          const uint32_t* __restrict__ srow, ParamsDev p,
                          double4* __restrict__ ag_out, double* __restrict__ dp_out, Extents* ext_next) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = i < n;
  int nb3[3] = {0, 0, 0};
  bool bad = false;
  if (valid) {
    const double4 me = ag[i];
    double3 F = make_double3(fss[3 * (size_t)i], fss[3 * (size_t)i + 1], fss[3 * (size_t)i + 2]);
    const uint32_t c = scnt[i];
    if (c > (uint32_t)SCAP) {
      F = sc_full(me, agf[i], F, gs, ge, elf, el_ids, geo, p);
    } else if (c > 0) {
      uint32_t r[SCAP];
      const uint32_t* row = srow + (size_t)i * SCAP;
      for (uint32_t k = 0; k < c; ++k) {  // insertion sort (a handful of entries)
        const uint32_t v = row[k];
        uint32_t x = k;
        while (x > 0 && r[x - 1] > v) {
          r[x] = r[x - 1];
          --x;
        }
        r[x] = v;
      }
      const double cc[3] = {me.x, me.y, me.z};
      const double rs = 0.5 * me.w;
      for (uint32_t k = 0; k < c; ++k) {
        const uint32_t el = el_ids[r[k]];
        const double4 ga = geo[el].a, gb = geo[el].b;
        const double P[3] = {ga.x, ga.y, ga.z}, v[3] = {gb.x, gb.y, gb.z};
        double t3[3];
        if (sc_term(cc, rs, P, v, ga.w, p, t3)) {  // (always: the row holds contacts)
          F.x = F.x + t3[0];
          F.y = F.y + t3[1];
          F.z = F.z + t3[2];
        }
      }
    }
    double dx, dy, dz;
    disp_rule(F.x, F.y, F.z, p, dx, dy, dz);
    const double4 np = make_double4(me.x + dx, me.y + dy, me.z + dz, me.w);
    ag_out[i] = np;
    if (dp_out) {
      dp_out[3 * (size_t)i] = dx;
      dp_out[3 * (size_t)i + 1] = dy;
      dp_out[3 * (size_t)i + 2] = dz;
    }
    nb3[0] = box_coord(np.x, gs.inv, bad);
    nb3[1] = box_coord(np.y, gs.inv, bad);
    nb3[2] = box_coord(np.z, gs.inv, bad);
  }
  if (__any_sync(FULL, bad) && (threadIdx.x & 31) == 0) ext_next->range_err = 1;
  block_minmax_atomic(ext_next, nb3, valid);
}

// N3 + N5 (distal points) + O6: own spring, daughters' springs (ascending id), sphere reactions over
// the 27 sphere boxes around box(C_e) (canonical order, ascending sphere id).
// One thread per element in the element grid's sorted order (el_ids: sorted -> id), so the lanes of a
// warp search neighbouring sphere boxes.  Each contact also goes to the sphere's contact row for
// k_sc_rows (the element's sorted index); the row slots are taken after the search, a few atomics in
// flight at once (an atomic whose result feeds a store inside the divergent search loop stalls the
// whole warp for an L2 round trip per contact).
constexpr int EL_PEND = 8;
__device__ __forceinline__ void sc_flush(uint32_t* __restrict__ scnt, uint32_t* __restrict__ srow, const uint32_t* cs,
                                         int nc, uint32_t qe) {
  uint32_t slot[EL_PEND];
#pragma unroll
  for (int k = 0; k < EL_PEND; ++k)
    if (k < nc) slot[k] = atomicAdd(&scnt[cs[k]], 1u);
#pragma unroll
  for (int k = 0; k < EL_PEND; ++k)
    if (k < nc && slot[k] < (uint32_t)SCAP) srow[(size_t)cs[k] * SCAP + slot[k]] = qe;
}

__global__ void __launch_bounds__(256, BDM_ELU_MINB) k_el_update(const double4* __restrict__ eq, const ElGeo* __restrict__ geo,
                            const int4* __restrict__ et, uint32_t E, const uint32_t* __restrict__ el_ids,
                            const double4* __restrict__ ag, const float4* __restrict__ agf, GridDev gs,
                            double m_el, ParamsDev p, double4* __restrict__ eq_out, double* __restrict__ dq_out,
                            uint32_t* __restrict__ scnt, uint32_t* __restrict__ srow) {
  const uint32_t qe = blockIdx.x * blockDim.x + threadIdx.x;
  if (qe >= E) return;
  const uint32_t e = el_ids[qe];
  const ElGeo ge = geo[e];
  const double P[3] = {ge.a.x, ge.a.y, ge.a.z}, v[3] = {ge.b.x, ge.b.y, ge.b.z};
  const double len = ge.b.w, T = ge.c.x, inv = ge.c.y;
  double F[3] = {0.0, 0.0, 0.0};
#pragma unroll
  for (int k = 0; k < 3; ++k) F[k] = F[k] + (-T) * (v[k] * inv);
  const int4 tp = et[e];
  const int ch[2] = {tp.y, tp.z};
  for (int k = 0; k < 2; ++k) {
    if (ch[k] < 0) continue;
    const double4 cb = geo[ch[k]].b, cc = geo[ch[k]].c;
    const double vc[3] = {cb.x, cb.y, cb.z};
    const double Tc = cc.x, ic = cc.y;
#pragma unroll
    for (int j = 0; j < 3; ++j) F[j] = F[j] + Tc * (vc[j] * ic);
  }
  const double re = ge.a.w;
  const double C[3] = {P[0] + 0.5 * v[0], P[1] + 0.5 * v[1], P[2] + 0.5 * v[2]};
  if (gs.table) {
    const int bx = (int)floor(C[0] * gs.inv), by = (int)floor(C[1] * gs.inv), bz = (int)floor(C[2] * gs.inv);
    // fp32 prefilter (sc_near): this element's centre and half extent against each sphere's agf
    const float4 cf = make_float4(__double2float_rn(C[0]), __double2float_rn(C[1]), __double2float_rn(C[2]), 0.f);
    const float hm = __double2float_ru(0.5 * (len + 2.0 * re) + gs.m32 + m_el);
    uint32_t cs[EL_PEND];
    int nc = 0;
    uint32_t rb[9], rn[9];
    zrun9(gs, bx, by, bz, rb, rn);
    for (int col = 0; col < 9; ++col) {
      const uint32_t b = rb[col], en = rn[col];
      for (uint32_t q = b; q < en; ++q) {
        const float4 sf = __ldg(&agf[q]);
        if (!sc_near(cf, sf, hm, -sf.w)) continue;
        const double4 sp = ag[q];
        const double c[3] = {sp.x, sp.y, sp.z};
        double t3[3];
        if (sc_term(c, 0.5 * sp.w, P, v, re, p, t3)) {
          F[0] = F[0] - t3[0];
          F[1] = F[1] - t3[1];
          F[2] = F[2] - t3[2];
          if (nc == EL_PEND) {
            sc_flush(scnt, srow, cs, nc, qe);
            nc = 0;
          }
          cs[nc++] = q;
        }
      }
    }
    sc_flush(scnt, srow, cs, nc, qe);
  }
  double dx, dy, dz;
  disp_rule(F[0], F[1], F[2], p, dx, dy, dz);
  const double4 q = eq[e];
  eq_out[e] = make_double4(q.x + dx, q.y + dy, q.z + dz, q.w);
  dq_out[3 * (size_t)e] = dx;
  dq_out[3 * (size_t)e + 1] = dy;
  dq_out[3 * (size_t)e + 2] = dz;
}

// ------------------------------------------------------------------------------------------ K7
__global__ void k_unpermute_pos(const double4* __restrict__ ag, const uint32_t* __restrict__ ids, uint32_t n,
                                double* __restrict__ out) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double4 p = ag[i];
  size_t d = 3 * (size_t)ids[i];
  out[d] = p.x;
  out[d + 1] = p.y;
  out[d + 2] = p.z;
}

__global__ void k_unpermute3(const double* __restrict__ v, const uint32_t* __restrict__ ids, uint32_t n,
                             double* __restrict__ out) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  size_t d = 3 * (size_t)ids[i];
  out[d] = v[3 * (size_t)i];
  out[d + 1] = v[3 * (size_t)i + 1];
  out[d + 2] = v[3 * (size_t)i + 2];
}

__global__ void k_unpermute_diam(const double4* __restrict__ ag, const uint32_t* __restrict__ ids, uint32_t n,
                                 double* __restrict__ out) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[ids[i]] = ag[i].w;
}

__global__ void k_box_coords(const double4* __restrict__ ag, const uint32_t* __restrict__ ids, uint32_t n,
                             double inv, int32_t* __restrict__ out) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double4 p = ag[i];
  size_t d = 3 * (size_t)ids[i];
  out[d] = (int32_t)floor(p.x * inv);
  out[d + 1] = (int32_t)floor(p.y * inv);
  out[d + 2] = (int32_t)floor(p.z * inv);
}

template <typename T>
__global__ void k_unpermute1(const T* __restrict__ v, const uint32_t* __restrict__ ids, uint32_t n,
                             T* __restrict__ out) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[ids[i]] = v[i];
}

// ------------------------------------------------------------------------------------------ K8
// Pairs (id_i < id_j) per agent in canonical order; pass 0 counts, pass 1 writes at offsets.
__global__ void k_pairs(const double4* __restrict__ ag, const uint32_t* __restrict__ ids, uint32_t n, GridDev g, ParamsDev p, int kind,
                        uint32_t* __restrict__ counts, const unsigned long long* __restrict__ offsets,
                        long long* __restrict__ out) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double4 me = ag[i];
  uint32_t myid = ids[i];
  double ri = 0.5 * me.w;
  int bx = (int)floor(me.x * g.inv), by = (int)floor(me.y * g.inv), bz = (int)floor(me.z * g.inv);
  uint32_t cnt = 0;
  unsigned long long w = offsets ? offsets[i] : 0ull;
  for (int c = 0; c < 9; ++c) {
    int cx = bx + c / 3 - 1, cy = by + c % 3 - 1;
    uint32_t b, e;
    if (!zrun(g, cx, cy, bz - 1, bz + 1, b, e)) continue;
    for (uint32_t q = b; q < e; ++q) {
      uint32_t idj = ids[q];
      if (idj <= myid) continue;
      double4 o = ag[q];
      double dx = me.x - o.x, dy = me.y - o.y, dz = me.z - o.z;
      double d2 = (dx * dx + dy * dy) + dz * dz;
      if (!(d2 <= g.L2)) continue;
      if (kind == 1) {
        double tx, ty, tz, fa;
        if (!pair_term(me.x, me.y, me.z, ri, i, o, ids, q, p, tx, ty, tz, fa)) continue;
      }
      if (out) {
        out[2 * w] = myid;
        out[2 * w + 1] = idj;
        ++w;
      }
      ++cnt;
    }
  }
  if (counts) counts[i] = cnt;
}

}  // namespace bdm
