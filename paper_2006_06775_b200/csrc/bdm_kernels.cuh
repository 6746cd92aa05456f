// bdm_kernels.cuh -- sm_100a kernels of the mechanical-interaction step.
//
// Compiled with -fmad=false: every fp64 +,-,* on the method's path is a separately rounded IEEE
// operation, so per-pair arithmetic is bit-identical to the reading in DESIGN.md §3 (O3-O6);
// sqrt() and '/' on doubles are correctly rounded.  No tensor cores: nothing here is a dense
// contraction (north_star).
//
//   K0 k_gen_uniform     counter-hash synthetic agents (bench / cfg4-5 utility)
//   K1 k_pack            n x 3 positions + diameters -> double4 agents, validation, max D
//      k_extents         min/max integer box coordinate per axis (first build only; later fused in K6)
//   K2 k_key_hist        box key (x slowest) + per-box histogram with warp-aggregated atomics
//   K3 k_scan            single-pass decoupled look-back exclusive scan -> box start table
//   K4 k_scatter         counting-sort scatter into box segments
//      k_place           ascending-id order inside each box + payload gather (deterministic sort)
//   K6 k_force           27-box search -> contact force -> sum -> adherence/clamp -> p' = p + dp,
//                        fused with the next step's box extents
//   K7 k_unpermute_*     sorted order -> id order for the getters
//   K8 k_pairs_*         neighbour / contact pair export (tests)
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace bdm {

constexpr unsigned FULL = 0xffffffffu;

// Grid parameters of one build, passed by value to kernels.
struct GridDev {
  double L, L2, inv;
  double thr_pad;  // (L/2) used for the conservative contact prefilter
  int32_t lo[3], hi[3];
  int32_t ny, nz;
  uint32_t n_boxes;
};

struct ParamsDev {
  double k_rep, gamma_att, adherence, c /* dt/eta */, max_disp;
};

// Box extents (reduced with atomics) + asynchronous error reporting.
struct Extents {
  int32_t lo[3], hi[3];
  int32_t range_err;  // 1 if some |p*inv| >= 2^20
  int32_t pad;
};

struct ErrDev {
  uint32_t code;       // 0 ok, else |BDM_E*|
  uint32_t first_bad;  // id of the first offending agent (min over reports)
  uint32_t second;     // partner id for ENONFINITE
  uint32_t pad;
};

struct RecordDev {
  int32_t *n_cand, *n_nb, *n_ct;
  int8_t* branch;
  unsigned long long *nb_hash, *ct_hash;
};

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ void report(ErrDev* e, uint32_t code, uint32_t id, uint32_t other) {
  atomicCAS(&e->code, 0u, code);
  uint32_t prev = atomicMin(&e->first_bad, id);
  if (id < prev) e->second = other;  // best effort partner id
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

__device__ __forceinline__ void warp_minmax_atomic(Extents* ext, const int b[3], bool valid) {
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    int lo = valid ? b[a] : INT32_MAX;
    int hi = valid ? b[a] : INT32_MIN;
    lo = __reduce_min_sync(FULL, lo);
    hi = __reduce_max_sync(FULL, hi);
    if ((threadIdx.x & 31) == 0 && lo != INT32_MAX) {
      atomicMin(&ext->lo[a], lo);
      atomicMax(&ext->hi[a], hi);
    }
  }
}

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
  warp_minmax_atomic(ext, b, valid);
}

__global__ void k_ext_reset(Extents* ext) {
  if (threadIdx.x < 3) {
    ext->lo[threadIdx.x] = INT32_MAX;
    ext->hi[threadIdx.x] = INT32_MIN;
  }
  if (threadIdx.x == 3) ext->range_err = 0;
}

__device__ __forceinline__ uint32_t box_key(const GridDev& g, int bx, int by, int bz) {
  return ((uint32_t)(bx - g.lo[0]) * (uint32_t)g.ny + (uint32_t)(by - g.lo[1])) * (uint32_t)g.nz +
         (uint32_t)(bz - g.lo[2]);
}

// ------------------------------------------------------------------------------------------ K2
__global__ void k_key_hist(const double4* __restrict__ ag, uint32_t n, GridDev g, uint32_t* __restrict__ key,
                           uint32_t* __restrict__ slot, uint32_t* __restrict__ count) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  bool valid = i < n;
  uint32_t k = 0xffffffffu;
  if (valid) {
    double4 p = ag[i];
    int bx = (int)floor(p.x * g.inv), by = (int)floor(p.y * g.inv), bz = (int)floor(p.z * g.inv);
    k = box_key(g, bx, by, bz);
  }
  // warp-aggregated histogram: one atomic per distinct key in the warp
  unsigned peers = __match_any_sync(FULL, k);
  int leader = __ffs(peers) - 1;
  int lane = threadIdx.x & 31;
  uint32_t base = 0;
  if (valid && lane == leader) base = atomicAdd(&count[k], (uint32_t)__popc(peers));
  base = __shfl_sync(FULL, base, leader);
  if (valid) {
    key[i] = k;
    slot[i] = base + __popc(peers & ((1u << lane) - 1u));
  }
}

// ------------------------------------------------------------------------------------------ K3
constexpr int SCAN_THREADS = 256;
constexpr int SCAN_ITEMS = 16;  // per thread
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

// In-place exclusive scan of data[0..n_items) (n_items = n_boxes + 1, last input 0 so that
// data[n_boxes] becomes the total).  Tile order is taken from an atomic ticket so every
// predecessor of a tile has started: the look-back cannot deadlock.
__global__ void __launch_bounds__(SCAN_THREADS) k_scan(uint32_t* __restrict__ data, uint64_t n_items,
                                                       unsigned long long* __restrict__ state,
                                                       uint32_t* __restrict__ ticket) {
  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_warp[SCAN_THREADS / 32];
  __shared__ uint32_t s_prefix;
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
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
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t incl = warp_incl_scan(tsum);
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    uint32_t ws = lane < SCAN_THREADS / 32 ? s_warp[lane] : 0u;
    uint32_t wi = warp_incl_scan(ws);
    if (lane < SCAN_THREADS / 32) s_warp[lane] = wi - ws;  // exclusive warp offsets
    uint32_t agg = __shfl_sync(FULL, wi, SCAN_THREADS / 32 - 1);
    // decoupled look-back
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

// ------------------------------------------------------------------------------------------ K4
__global__ void k_scatter(const uint32_t* __restrict__ key, const uint32_t* __restrict__ slot,
                          const uint32_t* __restrict__ ids, const uint32_t* __restrict__ start, uint32_t n,
                          uint32_t* __restrict__ tsrc, uint32_t* __restrict__ tid, uint32_t* __restrict__ tkey) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t k = key[i];
  uint32_t d = start[k] + slot[i];
  tsrc[d] = i;
  tid[d] = ids[i];
  tkey[d] = k;
}

// Rank inside the box by id (boxes hold a handful of agents), then gather the payload.
__global__ void k_place(const uint32_t* __restrict__ tsrc, const uint32_t* __restrict__ tid,
                        const uint32_t* __restrict__ tkey, const uint32_t* __restrict__ start,
                        const double4* __restrict__ ag_in, uint32_t n, double4* __restrict__ ag_out,
                        uint32_t* __restrict__ ids_out) {
  uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n) return;
  uint32_t k = tkey[q], id = tid[q];
  uint32_t b = start[k], e = start[k + 1];
  uint32_t rank = 0;
  for (uint32_t t = b; t < e; ++t) rank += tid[t] < id;
  uint32_t dst = b + rank;
  ag_out[dst] = ag_in[tsrc[q]];
  ids_out[dst] = id;
}

// ------------------------------------------------------------------------------------------ K6
constexpr int FORCE_THREADS = 256;
constexpr int FORCE_WARPS = FORCE_THREADS / 32;
constexpr int QCAP = 8;  // per-lane pending-contact FIFO depth (power of two)
constexpr int QTHRESH = 16;

// One contact candidate of agent i (O4), returns false if delta <= 0.
__device__ __forceinline__ bool pair_term(double xi, double yi, double zi, double ri, uint32_t idi, const double4& o,
                                          uint32_t idj, const ParamsDev& p, double& tx, double& ty, double& tz,
                                          double& fabs_out) {
  double dx = xi - o.x;
  double dy = yi - o.y;
  double dz = zi - o.z;
  double d2 = (dx * dx + dy * dy) + dz * dz;
  double rj = 0.5 * o.w;
  double s = ri + rj;
  double d = sqrt(d2);
  double delta = s - d;
  if (!(delta > 0.0)) return false;
  double r = (ri * rj) / s;
  double f = p.k_rep * delta - p.gamma_att * sqrt(r * delta);
  fabs_out = fabs(f);
  if (d2 == 0.0) {  // coincident centres (R8)
    tx = idi > idj ? f : -f;
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

// Lane = agent (sorted order).  Each lane walks its 9 z-runs (27 boxes) in canonical order; the
// cheap candidate test (d2 against a conservative per-lane bound) runs densely and pushes
// possible contacts into a per-lane FIFO in shared memory; the expensive exact contact
// evaluation (2 sqrt, 2 div) runs when at least QTHRESH lanes have work, so it is not paid by
// the whole warp for one lane's contact.  FIFO order = candidate order, so each agent's force
// is summed in the canonical order of DESIGN.md O5.
template <bool RECORD>
__global__ void __launch_bounds__(FORCE_THREADS) k_force(const double4* __restrict__ ag,
                                                         const uint32_t* __restrict__ ids,
                                                         const uint32_t* __restrict__ start, uint32_t n, GridDev g,
                                                         ParamsDev p, double4* __restrict__ ag_out,
                                                         double* __restrict__ dp_out, Extents* ext_next,
                                                         ErrDev* err, RecordDev rec) {
  __shared__ uint32_t s_rb[FORCE_WARPS][9][32];
  __shared__ uint32_t s_re[FORCE_WARPS][9][32];
  __shared__ uint32_t s_q[FORCE_WARPS][QCAP][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t i = blockIdx.x * FORCE_THREADS + threadIdx.x;
  const bool valid = i < n;
  double4 me = valid ? ag[i] : make_double4(0.0, 0.0, 0.0, 0.0);
  const double ri = 0.5 * me.w;
  const int bx = (int)floor(me.x * g.inv), by = (int)floor(me.y * g.inv), bz = (int)floor(me.z * g.inv);
  // conservative bound: contact => d2 < (ri + rj)^2 <= (ri + L/2)^2 (exact reals); pad by 2^-50
  double thr = (ri + g.thr_pad) * (ri + g.thr_pad);
  thr = thr + thr * 0x1p-50;
  const uint32_t myid = valid ? ids[i] : 0u;

  // z-run ranges of the 9 columns, (dx, dy) lexicographic
#pragma unroll
  for (int c = 0; c < 9; ++c) {
    int cx = bx + c / 3 - 1, cy = by + c % 3 - 1;
    uint32_t b = 0, e = 0;
    if (valid && cx >= g.lo[0] && cx <= g.hi[0] && cy >= g.lo[1] && cy <= g.hi[1]) {
      int z0 = bz - 1 < g.lo[2] ? g.lo[2] : bz - 1;
      int z1 = bz + 1 > g.hi[2] ? g.hi[2] : bz + 1;
      b = start[box_key(g, cx, cy, z0)];
      e = start[box_key(g, cx, cy, z1) + 1];
    }
    s_rb[warp][c][lane] = b;
    s_re[warp][c][lane] = e;
  }
  __syncwarp();

  int c = 0;
  uint32_t q = s_rb[warp][0][lane], e = s_re[warp][0][lane];
  while (q >= e && c < 8) {
    ++c;
    q = s_rb[warp][c][lane];
    e = s_re[warp][c][lane];
  }
  bool done = q >= e;
  uint32_t qh = 0, qt = 0;  // FIFO head / tail
  double Fx = 0.0, Fy = 0.0, Fz = 0.0;
  int32_t n_cand = 0, n_nb = 0, n_ct = 0;
  unsigned long long nb_hash = 0, ct_hash = 0;
  double s_abs = 0.0;
  (void)s_abs;

  while (true) {
    if (!done && qt - qh < QCAP) {
      if (q != i) {
        double4 o = ag[q];
        double dx = me.x - o.x;
        double dy = me.y - o.y;
        double dz = me.z - o.z;
        double d2 = (dx * dx + dy * dy) + dz * dz;
        if (RECORD) {
          ++n_cand;
          if (d2 <= g.L2) {
            ++n_nb;
            nb_hash += mix64(ids[q]);
          }
        }
        if (d2 <= thr) {
          s_q[warp][qt & (QCAP - 1)][lane] = q;
          ++qt;
        }
      }
      ++q;
      while (q >= e && c < 8) {
        ++c;
        q = s_rb[warp][c][lane];
        e = s_re[warp][c][lane];
      }
      done = q >= e;
    }
    const unsigned pend = __ballot_sync(FULL, qt != qh);
    const unsigned fetching = __ballot_sync(FULL, !done);
    if (!pend && !fetching) break;
    const unsigned full = __ballot_sync(FULL, qt - qh == QCAP);
    if (__popc(pend) >= QTHRESH || full || !fetching) {
      if (qt != qh) {
        uint32_t j = s_q[warp][qh & (QCAP - 1)][lane];
        ++qh;
        double4 o = ag[j];
        uint32_t idj = ids[j];
        double tx, ty, tz, fa;
        if (pair_term(me.x, me.y, me.z, ri, myid, o, idj, p, tx, ty, tz, fa)) {
          Fx = Fx + tx;
          Fy = Fy + ty;
          Fz = Fz + tz;
          if (RECORD) {
            ++n_ct;
            ct_hash += mix64(idj);
          }
        }
      }
    }
  }

  // O6 displacement, O7 update
  double dpx = 0.0, dpy = 0.0, dpz = 0.0;
  int branch = 0;
  double fn = sqrt((Fx * Fx + Fy * Fy) + Fz * Fz);
  if (fn <= p.adherence) {
    branch = 0;
  } else if (fn * p.c > p.max_disp) {
    double scale = p.max_disp / fn;
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
  bool bad = false;
  int nb3[3] = {0, 0, 0};
  if (valid) {
    if (!(isfinite(Fx) && isfinite(Fy) && isfinite(Fz) && isfinite(fn))) report(err, 6u /*ENONFINITE*/, myid, myid);
    double4 np = make_double4(me.x + dpx, me.y + dpy, me.z + dpz, me.w);
    ag_out[i] = np;
    if (dp_out) {
      dp_out[3 * (size_t)i] = dpx;
      dp_out[3 * (size_t)i + 1] = dpy;
      dp_out[3 * (size_t)i + 2] = dpz;
    }
    nb3[0] = box_coord(np.x, g.inv, bad);
    nb3[1] = box_coord(np.y, g.inv, bad);
    nb3[2] = box_coord(np.z, g.inv, bad);
    if (RECORD) {
      rec.n_cand[i] = n_cand;
      rec.n_nb[i] = n_nb;
      rec.n_ct[i] = n_ct;
      rec.branch[i] = (int8_t)branch;
      rec.nb_hash[i] = nb_hash;
      rec.ct_hash[i] = ct_hash;
    }
  }
  if (__any_sync(FULL, bad) && lane == 0) ext_next->range_err = 1;
  warp_minmax_atomic(ext_next, nb3, valid);
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
__global__ void k_pairs(const double4* __restrict__ ag, const uint32_t* __restrict__ ids,
                        const uint32_t* __restrict__ start, uint32_t n, GridDev g, ParamsDev p, int kind,
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
    if (cx < g.lo[0] || cx > g.hi[0] || cy < g.lo[1] || cy > g.hi[1]) continue;
    int z0 = bz - 1 < g.lo[2] ? g.lo[2] : bz - 1;
    int z1 = bz + 1 > g.hi[2] ? g.hi[2] : bz + 1;
    uint32_t b = start[box_key(g, cx, cy, z0)], e = start[box_key(g, cx, cy, z1) + 1];
    for (uint32_t q = b; q < e; ++q) {
      uint32_t idj = ids[q];
      if (idj <= myid) continue;
      double4 o = ag[q];
      double dx = me.x - o.x, dy = me.y - o.y, dz = me.z - o.z;
      double d2 = (dx * dx + dy * dy) + dz * dz;
      if (!(d2 <= g.L2)) continue;
      if (kind == 1) {
        double tx, ty, tz, fa;
        if (!pair_term(me.x, me.y, me.z, ri, myid, o, idj, p, tx, ty, tz, fa)) continue;
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
