// bdm_dist.cuh -- distributed x-slab runtime behind bdm_nccl_unique_id / bdm_init_dist.
// Included at the end of bdm_capi.cu (one translation unit: it drives the slab machinery there).
//
// north_star: "Across the 8 GPUs of one box the domain is split into x-slabs.  Each step does a halo
// exchange of boundary-box agents and migrates agents that cross slab boundaries, using NCCL
// send/recv over NVLink."  SURVEY §8(b) (the distributed entry points), §8(e) (partition, exchanges).
//
// One process per GPU ("rank"); a rank owns the agents whose integer box-x lies in
// [cut[r], cut[r+1]).  Setup (bdm_init_dist, host round trips allowed): global box edge (allreduce
// max D, O1), global extents, per-layer histogram (allreduce) -> count-balanced cuts -> all-to-all
// redistribution -> per-layer work from each rank's own grid (sum n_b + sum n_b^2 / mean) ->
// work-balanced cuts -> redistribution (cut by work, not count).
//
// Steps (bdm_mech_step) run in chunks of at most DIST_CHUNK steps with NO host synchronisation
// inside a chunk: every message has a fixed capacity agreed by all ranks (its header carries the
// counts), every count lives on the device (DistSlab::dc) and the kernels read it there; the grid
// frame is fixed for the chunk (global extents at the chunk start +- (chunk + 1) boxes: a step moves
// an agent by less than one box).  One step of one rank:
//   prep (owned count, boundary-layer ranges) -> split (emigrants + boundary stayers into the two
//   send messages) -> header -> NCCL group { send lo, send hi, recv lo, recv hi } -> mark emigrants
//   dead -> ingest (immigrants appended as owned, neighbours' boundary stayers + own emigrants as
//   ghosts) -> slab-local grid build -> half-shell force phase on the owned range.
// At the end of a chunk: one host round trip reads the counts and flags; the extents, flags and
// the largest message need are all-reduced; a chunk in which any message or buffer overflowed is
// re-run from a device checkpoint taken at its start with larger buffers (exact, never silent).
// Ghosts carry global ids and sort in canonical in-box order, so every owned agent's force is summed
// in the single-GPU order: results are bit-identical to one GPU (tests/test_gpu_dist.py).
//
// NCCL is loaded with dlopen (libnccl.so.2: the copy torch already loaded, else the system one), so
// single-GPU use of libbdm.so needs no NCCL.  Virtual mode (bdm_init_dist_local): G ranks of one
// process on one GPU over a 1-rank communicator, every message a self send/recv -- the same data
// plane and protocol, for tests on a single GPU (the kernels never wait on each other).
#include <dlfcn.h>
#include <nccl.h>

namespace {

// ------------------------------------------------------------------------------------ NCCL (dlopen)
struct NcclApi {
  void* lib = nullptr;
  decltype(&::ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&::ncclCommInitRank) commInitRank = nullptr;
  decltype(&::ncclCommDestroy) commDestroy = nullptr;
  decltype(&::ncclSend) send = nullptr;
  decltype(&::ncclRecv) recv = nullptr;
  decltype(&::ncclGroupStart) groupStart = nullptr;
  decltype(&::ncclGroupEnd) groupEnd = nullptr;
  decltype(&::ncclAllReduce) allReduce = nullptr;
  decltype(&::ncclAllGather) allGather = nullptr;
  decltype(&::ncclGetErrorString) errStr = nullptr;
  std::string load_error;
};

NcclApi* nccl_api() {
  static NcclApi api;
  static bool tried = false;
  if (tried) return api.lib ? &api : nullptr;
  tried = true;
  const char* names[] = {"libnccl.so.2", "libnccl.so"};
  for (const char* nm : names) {
    api.lib = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
    if (api.lib) break;
  }
  if (!api.lib) {
    api.load_error = dlerror() ? dlerror() : "dlopen(libnccl.so.2) failed";
    return nullptr;
  }
#define SYM(f, n) api.f = reinterpret_cast<decltype(api.f)>(dlsym(api.lib, n))
  SYM(getUniqueId, "ncclGetUniqueId");
  SYM(commInitRank, "ncclCommInitRank");
  SYM(commDestroy, "ncclCommDestroy");
  SYM(send, "ncclSend");
  SYM(recv, "ncclRecv");
  SYM(groupStart, "ncclGroupStart");
  SYM(groupEnd, "ncclGroupEnd");
  SYM(allReduce, "ncclAllReduce");
  SYM(allGather, "ncclAllGather");
  SYM(errStr, "ncclGetErrorString");
#undef SYM
  if (!api.getUniqueId || !api.commInitRank || !api.commDestroy || !api.send || !api.recv || !api.groupStart ||
      !api.groupEnd || !api.allReduce || !api.allGather || !api.errStr) {
    api.load_error = "libnccl.so.2 lacks a required symbol";
    dlclose(api.lib);
    api.lib = nullptr;
    return nullptr;
  }
  return &api;
}

#define NC(h, call)                                                                                     \
  do {                                                                                                  \
    ncclResult_t r_ = (call);                                                                           \
    if (r_ != ncclSuccess)                                                                              \
      return fail((h), BDM_ENCCL, "%s: %s (%s:%d)", #call, nccl_api()->errStr(r_), __FILE__, __LINE__); \
  } while (0)

// ------------------------------------------------------------------------------------ device side
// Device counts of one slab (DistSlab::dc), read by the kernels of a step.
enum : int {
  DC_LIVE = 0,   // owned agents of the stepped buffer [0, LIVE) (after a step: A_END - A_BEGIN)
  DC_DEAD,       // emigrants marked dead in the owned region (dropped by the sort)
  DC_TOT,        // entries of ag[cur] after ingest: owned (incl. dead) + immigrants + ghosts
  DC_GLO,        // ghosts of box-x = x_begin - 1 (sort first)
  DC_GHI,        // ghosts of box-x = x_end (sort last)
  DC_SORTED,     // TOT - DEAD
  DC_ABEGIN,     // owned range of the sorted array [A_BEGIN, A_END)  (adjacent: read as a pair)
  DC_AEND,
  DC_CE0,        // column pass range [CE0, CE1): the appended records (the stepped ones were fused)
  DC_CE1,
  DC_OVF,        // sticky: a message or the buffer overflowed in this chunk (re-run it)
  DC_NEED,       // largest message need (emigrants + boundary stayers of one side) seen in this chunk
  DC_MIG,        // emigrants sent in this chunk
  DC_GHOSTS,     // ghosts of the last step
  DC_N
};
constexpr int HDR = 4;  // message header (fp64 slots): emigrants, boundary stayers, overflow, spare

__device__ __forceinline__ uint32_t hdr_u32(const double* m, int k) { return (uint32_t)m[k]; }

// Owned count after a step and the ranges the split scans: after a step only the first two and
// last two box-x layers of the step's sorted order can hold emigrants or boundary stayers
// (k_layer_bounds); mode 0 (first step of a chunk after setup or a restore): the whole array.
// (cnt4: the split's four counters, zeroed here so that no memset interrupts the launch chain)
__global__ void k_dist_prep(GridDev g, int mode, int32_t x_begin, int32_t x_end, uint32_t* __restrict__ dc,
                            uint32_t* __restrict__ r2, uint32_t* __restrict__ cnt4 = nullptr) {
  pdl_wait();
  if (cnt4 && threadIdx.x < 4) cnt4[threadIdx.x] = 0u;
  if (threadIdx.x != 0) return;
  uint32_t live = dc[DC_LIVE];
  if (mode == 1) {
    live = dc[DC_AEND] - dc[DC_ABEGIN];
    dc[DC_LIVE] = live;
  }
  if (mode == 0) {
    r2[0] = live;
    r2[1] = live;
    return;
  }
  const uint32_t n_lo = dc[DC_GLO];
  for (int t = 0; t < 2; ++t) {
    const int64_t X = t == 0 ? (int64_t)x_begin + 2 : (int64_t)x_end - 2;
    uint32_t r;
    if (t == 0 && x_begin == INT32_MIN) {
      r = 0u;
    } else if (t == 1 && x_end == INT32_MAX) {
      r = live;
    } else if (X <= g.lo[0]) {
      r = 0u;
    } else if (X > g.hi[0]) {
      r = live;
    } else {
      const uint32_t c = (uint32_t)(X - g.lo[0]) * (uint32_t)g.ny;
      const uint32_t k = g.table[g.coff[c]];
      r = k > n_lo ? k - n_lo : 0u;
      r = r < live ? r : live;
    }
    r2[t] = r;
  }
}

// Message headers from the split counters (cnt[0] emigrants lo, [1] stayers lo, [2] emigrants hi,
// [3] stayers hi); a side whose records exceed the capacity is flagged (the chunk is re-run).
__global__ void k_dist_header(const uint32_t* __restrict__ cnt, uint64_t cap, double* __restrict__ msg_lo,
                              double* __restrict__ msg_hi, uint32_t* __restrict__ dc) {
  pdl_wait();
  if (threadIdx.x != 0) return;
  const uint64_t nlo = (uint64_t)cnt[0] + cnt[1], nhi = (uint64_t)cnt[2] + cnt[3];
  const bool olo = nlo > cap, ohi = nhi > cap;
  msg_lo[0] = (double)cnt[0];
  msg_lo[1] = (double)cnt[1];
  msg_lo[2] = olo ? 1.0 : 0.0;
  msg_lo[3] = 0.0;
  msg_hi[0] = (double)cnt[2];
  msg_hi[1] = (double)cnt[3];
  msg_hi[2] = ohi ? 1.0 : 0.0;
  msg_hi[3] = 0.0;
  const uint32_t need = (uint32_t)(nlo > nhi ? nlo : nhi);
  if (need > dc[DC_NEED]) dc[DC_NEED] = need;
  if (olo || ohi) dc[DC_OVF] = 1u;
  dc[DC_MIG] += cnt[0] + cnt[2];
}

// Appends, after the owned region [0, LIVE): immigrants from below and above (owned from now on),
// then the ghosts of box-x = x_begin - 1 (the lower neighbour's boundary stayers + this rank's own
// emigrants to it: they moved less than a box, so they sit in the neighbour's last layer), then those
// of box-x = x_end.  The new counts are computed identically by every thread (inputs are read-only
// here) and written once.  Counts are clamped to the message capacity and to the buffer capacity
// `room`; a clamp flags the chunk for a re-run.
__global__ void k_dist_ingest(double4* __restrict__ ag, uint32_t* __restrict__ ids, uint32_t* __restrict__ dc,
                              const uint32_t* __restrict__ cnt, const double* __restrict__ send_lo,
                              const double* __restrict__ send_hi, const double* __restrict__ recv_lo,
                              const double* __restrict__ recv_hi, uint32_t cap, int has_lo, int has_hi, uint32_t room,
                              int fused) {
  pdl_wait();
  const uint32_t live = dc[DC_LIVE];
  bool ovf = false;
  // own split (the emigrants are at the front of the send records, the stayers at the back).  A message
  // whose records exceeded the capacity is not used at all (its front and back may overlap): the chunk
  // is void and re-run, and dropping it keeps the state consistent (no torn or duplicated agents)
  const bool own_lo_bad = (uint64_t)cnt[0] + cnt[1] > cap, own_hi_bad = (uint64_t)cnt[2] + cnt[3] > cap;
  ovf |= own_lo_bad || own_hi_bad;
  const uint32_t mig_lo = own_lo_bad ? 0u : cnt[0], mig_hi = own_hi_bad ? 0u : cnt[2];
  uint32_t imm_lo = 0, imm_hi = 0, gin_lo = 0, gin_hi = 0;
  if (has_lo) {
    if (recv_lo[2] != 0.0 || (uint64_t)hdr_u32(recv_lo, 0) + hdr_u32(recv_lo, 1) > cap) {
      ovf = true;
    } else {
      imm_lo = hdr_u32(recv_lo, 0);
      gin_lo = hdr_u32(recv_lo, 1);
    }
  }
  if (has_hi) {
    if (recv_hi[2] != 0.0 || (uint64_t)hdr_u32(recv_hi, 0) + hdr_u32(recv_hi, 1) > cap) {
      ovf = true;
    } else {
      imm_hi = hdr_u32(recv_hi, 0);
      gin_hi = hdr_u32(recv_hi, 1);
    }
  }
  // segments appended at `live`: [imm_lo][imm_hi][gin_lo][mig_lo][gin_hi][mig_hi]
  uint32_t seg[6] = {imm_lo, imm_hi, gin_lo, mig_lo, gin_hi, mig_hi};
  uint64_t total = 0;
  for (int k = 0; k < 6; ++k) {
    if ((uint64_t)live + total + seg[k] > room) {
      ovf = true;
      seg[k] = (uint32_t)(room - live - total);
    }
    total += seg[k];
  }
  const double* src[6] = {recv_lo + HDR, recv_hi + HDR, recv_lo + HDR, send_lo + HDR, recv_hi + HDR, send_hi + HDR};
  const bool back[6] = {false, false, true, false, true, false};  // stayers were written from the back
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t r = t;
    int k = 0;
    while (r >= seg[k]) {
      r -= seg[k];
      ++k;
    }
    const uint64_t rec = back[k] ? (uint64_t)cap - 1 - r : r;
    BDM_ASSERT(k < 6 && rec < cap && live + t < room);
    const double* q = src[k] + (size_t)REC * rec;
    ag[live + t] = make_double4(q[0], q[1], q[2], q[3]);
    ids[live + t] = (uint32_t)q[4];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const uint32_t tot = live + (uint32_t)total;
    const uint32_t dead = cnt[0] + cnt[2];  // every emigrant was marked dead (k_slab_mark_dead)
    const uint32_t glo = seg[2] + seg[3], ghi = seg[4] + seg[5];
    dc[DC_DEAD] = dead;
    dc[DC_TOT] = tot;
    dc[DC_GLO] = glo;
    dc[DC_GHI] = ghi;
    dc[DC_SORTED] = tot - dead;
    dc[DC_ABEGIN] = glo;
    dc[DC_AEND] = tot - dead - ghi;
    dc[DC_CE0] = fused ? live : 0u;
    dc[DC_CE1] = tot;
    dc[DC_GHOSTS] = glo + ghi;
    if (ovf) dc[DC_OVF] = 1u;
  }
}

// Chunk summary of one slab for the end-of-chunk all-reduce (max): overflow, largest message need,
// frame / range flags, -lo[3] and hi[3] of the owned agents' new boxes, owned count.
constexpr int SUMN = 10;
__global__ void k_dist_summary(const uint32_t* __restrict__ dc, const Extents* __restrict__ ext, double* __restrict__ out) {
  if (threadIdx.x != 0) return;
  const uint32_t live = dc[DC_AEND] - dc[DC_ABEGIN];
  out[0] = (double)dc[DC_OVF];
  out[1] = (double)dc[DC_NEED];
  out[2] = (double)((ext->range_err != 0) | (ext->col_bad != 0u) | (ext->sticky != 0u));
  for (int a = 0; a < 3; ++a) {
    out[3 + a] = live ? -(double)ext->lo[a] : -(double)INT32_MAX;
    out[6 + a] = live ? (double)ext->hi[a] : (double)INT32_MIN;
  }
  out[9] = (double)live;
}

// Destination rank of every input record (box-x against the cuts) and the count per destination.
__global__ void k_dist_dest(const double* __restrict__ rec, uint32_t n, double inv, const int32_t* __restrict__ cuts,
                            int world, uint32_t* __restrict__ dest, unsigned long long* __restrict__ count) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int bx = (int)floor(rec[(size_t)REC * i] * inv);
  int d = 0;  // cuts[1..world-1] are the inner cuts (cuts[0] = INT32_MIN, cuts[world] = INT32_MAX)
  while (d + 1 < world && bx >= cuts[d + 1]) ++d;
  dest[i] = (uint32_t)d;
  atomicAdd(&count[d], 1ull);
}

__global__ void k_dist_scatter(const double* __restrict__ rec, uint32_t n, const uint32_t* __restrict__ dest,
                               unsigned long long* __restrict__ slot, double* __restrict__ out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const unsigned long long k = atomicAdd(&slot[dest[i]], 1ull);
  for (int a = 0; a < REC; ++a) out[(size_t)REC * k + a] = rec[(size_t)REC * i + a];
}

// Input validation + records (x, y, z, D, id) + the local max D (O1) and box extents (O2).
__global__ void k_dist_pack_in(const double* __restrict__ pos, const double* __restrict__ diam,
                               const int64_t* __restrict__ ids, uint32_t n, double* __restrict__ rec,
                               unsigned long long* maxd_bits, ErrDev* err) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long b = 0ull;
  if (i < n) {
    const double x = pos[3 * (size_t)i], y = pos[3 * (size_t)i + 1], z = pos[3 * (size_t)i + 2], d = diam[i];
    const int64_t id = ids[i];
    if (!(d > 0.0) || !isfinite(d) || !isfinite(x) || !isfinite(y) || !isfinite(z) || id < 0 || id >= 0xffffffffll)
      report(err, 1u, i, i);
    double* r = rec + (size_t)REC * i;
    r[0] = x;
    r[1] = y;
    r[2] = z;
    r[3] = d;
    r[4] = (double)id;
    b = d > 0.0 ? (unsigned long long)__double_as_longlong(d) : 0ull;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long v = __shfl_xor_sync(FULL, b, o);
    b = v > b ? v : b;
  }
  if ((threadIdx.x & 31) == 0 && b) atomicMax(maxd_bits, b);
}

__global__ void k_rec_extents(const double* __restrict__ rec, uint32_t n, double inv, Extents* ext) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = i < n;
  bool bad = false;
  int b[3] = {0, 0, 0};
  if (valid)
    for (int a = 0; a < 3; ++a) b[a] = box_coord(rec[(size_t)REC * i + a], inv, bad);
  if (__any_sync(FULL, bad) && (threadIdx.x & 31) == 0) ext->range_err = 1;
  block_minmax_atomic(ext, b, valid);
}

__global__ void k_rec_layer_hist(const double* __restrict__ rec, uint32_t n, double inv, int32_t x0, uint32_t nx,
                                 unsigned long long* __restrict__ hist) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t k = 0xffffffffu;
  if (i < n) {
    const int bx = (int)floor(rec[(size_t)REC * i] * inv);
    const int64_t u = (int64_t)bx - x0;
    if (u >= 0 && u < nx) k = (uint32_t)u;
  }
  const unsigned peers = __match_any_sync(FULL, k);
  if (k != 0xffffffffu && (int)(threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&hist[k], (unsigned long long)__popc(peers));
}

// Per box-x layer of a built grid: sum of box occupancies n_b and of n_b^2 (the work model).
__global__ void k_layer_work(GridDev g, int32_t x0, uint32_t nx, unsigned long long* __restrict__ sq) {
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < g.n_cols; c += gridDim.x * blockDim.x) {
    const int4 ci = g.col[c];
    if (ci.y < ci.x) continue;
    const int64_t u = (int64_t)g.lo[0] + (int64_t)(c / (uint32_t)g.ny) - x0;
    if (u < 0 || u >= nx) continue;
    unsigned long long s = 0;
    for (int z = 0; z <= ci.y - ci.x; ++z) {
      const unsigned long long m = g.table[ci.z + z + 1] - g.table[ci.z + z];
      s += m * m;
    }
    if (s) atomicAdd(&sq[u], s);
  }
}

__global__ void k_ag_maxd_rec(const double* __restrict__ rec, uint32_t n, unsigned long long* maxd_bits) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long b = i < n ? (unsigned long long)__double_as_longlong(rec[(size_t)REC * i + 3]) : 0ull;
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long v = __shfl_xor_sync(FULL, b, o);
    b = v > b ? v : b;
  }
  if ((threadIdx.x & 31) == 0 && b) atomicMax(maxd_bits, b);
}

// Owned agents back to records (a redistribution of the work pass).
__global__ void k_ag_to_rec(const double4* __restrict__ ag, const uint32_t* __restrict__ ids, uint32_t n,
                            double* __restrict__ rec) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double4 p = ag[i];
  double* r = rec + (size_t)REC * i;
  r[0] = p.x;
  r[1] = p.y;
  r[2] = p.z;
  r[3] = p.w;
  r[4] = (double)ids[i];
}

// Order-free pair digest of the current positions (bdm_get_pair_digest): per agent, the number of
// neighbour (kind 0, d2 <= L2) or contact (kind 1, delta > 0) partners and sum mix64(id_j) mod 2^64
// over them (O3 / O4 as written, the 27 boxes of O3), written by id.
__global__ void k_pair_digest(const double4* __restrict__ ag, const uint32_t* __restrict__ ids, uint32_t n, GridDev g,
                              int kind, uint32_t* __restrict__ count, unsigned long long* __restrict__ hash) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double4 me = ag[i];
  const double ri = 0.5 * me.w;
  const int bx = (int)floor(me.x * g.inv), by = (int)floor(me.y * g.inv), bz = (int)floor(me.z * g.inv);
  uint32_t c = 0;
  unsigned long long hsum = 0;
  for (int col = 0; col < 9; ++col) {
    uint32_t b = 0, e = 0;
    if (!zrun(g, bx + col / 3 - 1, by + col % 3 - 1, bz - 1, bz + 1, b, e)) continue;
    for (uint32_t j = b; j < e; ++j) {
      if (j == i) continue;
      const double4 o = ag[j];
      const double dx = me.x - o.x, dy = me.y - o.y, dz = me.z - o.z;
      const double d2 = (dx * dx + dy * dy) + dz * dz;
      bool hit;
      if (kind == 0) {
        hit = d2 <= g.L2;
      } else {
        const double s = ri + 0.5 * o.w;
        hit = s - sqrt(d2) > 0.0;
      }
      if (hit) {
        ++c;
        hsum += mix64((uint64_t)ids[j]);
      }
    }
  }
  const uint32_t id = ids[i];
  count[id] = c;
  hash[id] = hsum;
}

// ------------------------------------------------------------------------------------ host side
constexpr int DIST_CHUNK = 16;  // steps between host round trips (frame margin = chunk + 1 boxes)

struct DistSlab {
  bdm_ctx* h = nullptr;     // the slab handle (owned agents + ghosts)
  int rank = 0;             // global (virtual) rank
  int32_t xb = 0, xe = 0;   // owned box-x range
  uint32_t* dc = nullptr;   // device counts (DC_*)
  uint32_t* dc_host = nullptr;  // pinned mirror
  double* msg[4] = {nullptr, nullptr, nullptr, nullptr};  // send lo, send hi, recv lo, recv hi (HDR + cap REC)
  int64_t msg_cap = 0;        // records per message of the current buffers
  double* sum = nullptr;      // device chunk summary (SUMN doubles)
  double* sum_host = nullptr;
  double4* ck_ag = nullptr;   // chunk checkpoint of the owned agents
  uint32_t* ck_id = nullptr;
  int64_t ck_cap = 0;
  int64_t live = 0;           // owned agents (host view at the last synchronisation)
  bool stepped = false;       // a step ran since the last setup / restore (layer-range split possible)
  int64_t room = 0;           // capacity of the slab buffers
  int32_t flo[3] = {0, 0, 0}, fhi[3] = {0, 0, 0};  // grid frame of the current chunk
  double fm32 = 0.0;                                 // its fp32 prefilter margin
  bool fvalid = false;        // the frame above is in use (kept across chunks while it holds the agents)
  int32_t zbits = 0;          // packed new boxes (column << zbits | z - flo[2]) of the sum pass, 0 = off
};

struct DistGroup {
  NcclApi* api = nullptr;
  ncclComm_t comm = nullptr;
  bool virt = false;
  int world = 1;
  int device = 0;
  cudaStream_t stream = nullptr;
  std::vector<DistSlab> sl;
  std::vector<int32_t> cuts;  // world + 1
  double L = 0.0, inv = 0.0;
  int32_t glo[3] = {0, 0, 0}, ghi[3] = {0, 0, 0};  // global box extents at the last synchronisation
  int64_t cap = 0;                                 // message capacity (records), agreed by all ranks
  int64_t n_global = 0;
  // statistics
  int64_t steps = 0, chunks = 0, redo = 0, syncs = 0, bytes = 0, migrated = 0, ghosts = 0;
  double* red = nullptr;  // device scratch for reductions (64 doubles)
  // CUDA graph of two steady steps (fused columns, no displacements kept), replayed inside chunks;
  // valid while the signature of what its launches baked in is unchanged
  cudaGraphExec_t gexec = nullptr;
  std::vector<uintptr_t> gsig;
  int64_t graph_launches = 0, graph_bytes = 0;  // per replay: kernels and exchange bytes of the pair
  int64_t replays = 0;
};

// Host reductions across ranks.  Virtual mode: the local slabs are all the ranks (reduced here);
// otherwise one NCCL allreduce on the device scratch.
int dist_allreduce(bdm_ctx* H, DistGroup* G, std::vector<std::vector<double>>& per_local, ncclRedOp_t op,
                   std::vector<double>& out) {
  const size_t m = per_local[0].size();
  out.assign(m, 0.0);
  for (size_t k = 0; k < m; ++k) {
    double v = per_local[0][k];
    for (size_t s = 1; s < per_local.size(); ++s) {
      const double w = per_local[s][k];
      v = op == ncclMax ? std::max(v, w) : (op == ncclMin ? std::min(v, w) : v + w);
    }
    out[k] = v;
  }
  if (G->virt || G->world == 1) return BDM_OK;
  std::vector<double> tmp(out);
  double* d = nullptr;
  CU(H, cudaMalloc(&d, m * sizeof(double)));
  Scratch sc;
  sc.p = d;
  CU(H, cudaMemcpyAsync(d, tmp.data(), m * sizeof(double), cudaMemcpyHostToDevice, G->stream));
  NC(H, G->api->allReduce(d, d, m, ncclDouble, op, G->comm, G->stream));
  CU(H, cudaMemcpyAsync(out.data(), d, m * sizeof(double), cudaMemcpyDeviceToHost, G->stream));
  CU(H, cudaStreamSynchronize(G->stream));
  ++G->syncs;
  return BDM_OK;
}

// Balanced cuts on integer box-x from per-layer values w over [x0, x0 + nx) (counts, or the work
// model): cut g is the first layer after the g/world quantile of w.  Every inner slab is at least 2
// boxes wide -- the protocol relies on it: an emigrant moves less than one box, so it always lands in
// the neighbour's boundary layer, which no third rank holds as a ghost layer.  When the population
// spans fewer than 2 * world layers, the last ranks get empty 2-box slabs beyond it.
std::vector<int32_t> choose_cuts(const std::vector<double>& w, int32_t x0, int world) {
  const int64_t nx = (int64_t)w.size();
  std::vector<int32_t> b{INT32_MIN};
  if (world > 1) {
    std::vector<double> cum(nx);
    double t = 0.0;
    for (int64_t k = 0; k < nx; ++k) cum[k] = (t += w[k]);
    const double total = nx ? cum[nx - 1] : 0.0;
    int64_t prev = x0;
    for (int g = 1; g < world; ++g) {
      const double target = total * g / world;
      const int64_t k = (int64_t)(std::lower_bound(cum.begin(), cum.end(), target) - cum.begin()) + 1;
      const int64_t lo = prev + (g == 1 ? 1 : 2);
      int64_t cut = std::max<int64_t>(x0 + k, lo);
      const int64_t hi = x0 + nx - 1 - (int64_t)(world - 1 - g) * 2;  // room for the later slabs
      if (hi >= lo) cut = std::min<int64_t>(cut, hi);
      b.push_back((int32_t)cut);
      prev = cut;
    }
  }
  b.push_back(INT32_MAX);
  return b;
}

// One grouped NCCL exchange: each message (send buffer of local slot a -> recv buffer of rank b).
struct Msg {
  int from_rank, to_rank;
  const void* sbuf;  // valid when from_rank is local
  void* rbuf;        // valid when to_rank is local
  size_t count;      // doubles
};

bool is_local(DistGroup* G, int rank) {
  for (auto& s : G->sl)
    if (s.rank == rank) return true;
  return false;
}

int dist_p2p(bdm_ctx* H, DistGroup* G, const std::vector<Msg>& msgs) {
  if (msgs.empty()) return BDM_OK;
  // virtual mode: every rank is local, every message is a self send + recv of the 1-rank
  // communicator, matched in issue order; otherwise peers are the global ranks
  NC(H, G->api->groupStart());
  for (const Msg& m : msgs) {
    const bool loc_from = is_local(G, m.from_rank), loc_to = is_local(G, m.to_rank);
    const int peer_of_send = G->virt ? 0 : m.to_rank, peer_of_recv = G->virt ? 0 : m.from_rank;
    if (loc_from && m.count) NC(H, G->api->send(m.sbuf, m.count, ncclDouble, peer_of_send, G->comm, G->stream));
    if (loc_to && m.count) NC(H, G->api->recv(m.rbuf, m.count, ncclDouble, peer_of_recv, G->comm, G->stream));
    if (loc_from) G->bytes += (int64_t)(m.count * sizeof(double));
  }
  NC(H, G->api->groupEnd());
  return BDM_OK;
}

// All-to-all redistribution of records by box-x against G->cuts (setup only, host round trips).
// recs[s] / n[s]: records of local slot s (device, freed here); on return the records each slot owns.
int dist_redistribute(bdm_ctx* H, DistGroup* G, std::vector<double*>& recs, std::vector<int64_t>& n) {
  const int W = G->world, S = (int)G->sl.size();
  int32_t* dcuts = nullptr;
  CU(H, cudaMalloc(&dcuts, (W + 1) * sizeof(int32_t)));
  Scratch sc_cuts;
  sc_cuts.p = dcuts;
  CU(H, cudaMemcpyAsync(dcuts, G->cuts.data(), (W + 1) * sizeof(int32_t), cudaMemcpyHostToDevice, G->stream));
  std::vector<std::vector<double>> cnt_local(S, std::vector<double>((size_t)W * W, 0.0));
  std::vector<uint32_t*> dest(S, nullptr);
  std::vector<double*> sorted(S, nullptr);
  std::vector<std::vector<int64_t>> mine(S, std::vector<int64_t>(W, 0));
  for (int s = 0; s < S; ++s) {
    unsigned long long* c = nullptr;
    CU(H, cudaMalloc(&c, W * sizeof(unsigned long long)));
    Scratch scc;
    scc.p = c;
    CU(H, cudaMalloc(&dest[s], std::max<int64_t>(n[s], 1) * sizeof(uint32_t)));
    CU(H, cudaMemsetAsync(c, 0, W * sizeof(unsigned long long), G->stream));
    if (n[s]) k_dist_dest<<<blocks(n[s], 256), 256, 0, G->stream>>>(recs[s], (uint32_t)n[s], G->inv, dcuts, W, dest[s], c);
    CU(H, cudaGetLastError());
    std::vector<unsigned long long> hc(W);
    CU(H, cudaMemcpyAsync(hc.data(), c, W * sizeof(unsigned long long), cudaMemcpyDeviceToHost, G->stream));
    CU(H, cudaStreamSynchronize(G->stream));
    ++G->syncs;
    // exclusive offsets -> scatter into destination order
    std::vector<unsigned long long> off(W, 0);
    for (int d = 1; d < W; ++d) off[d] = off[d - 1] + hc[d - 1];
    CU(H, cudaMemcpyAsync(c, off.data(), W * sizeof(unsigned long long), cudaMemcpyHostToDevice, G->stream));
    CU(H, cudaMalloc(&sorted[s], std::max<int64_t>(n[s], 1) * REC * sizeof(double)));
    if (n[s]) k_dist_scatter<<<blocks(n[s], 256), 256, 0, G->stream>>>(recs[s], (uint32_t)n[s], dest[s], c, sorted[s]);
    CU(H, cudaGetLastError());
    CU(H, cudaStreamSynchronize(G->stream));
    ++G->syncs;
    for (int d = 0; d < W; ++d) {
      mine[s][d] = (int64_t)hc[d];
      cnt_local[s][(size_t)G->sl[s].rank * W + d] = (double)hc[d];
    }
    cudaFree(recs[s]);
    cudaFree(dest[s]);
    recs[s] = nullptr;
  }
  // the count matrix [from][to] of all ranks (each rank fills its own row; summed)
  std::vector<double> mat;
  int rc = dist_allreduce(H, G, cnt_local, ncclSum, mat);
  if (rc) return rc;
  std::vector<double*> out(S, nullptr);
  std::vector<int64_t> nout(S, 0);
  std::vector<std::vector<int64_t>> roff(S, std::vector<int64_t>(W, 0));
  for (int s = 0; s < S; ++s) {
    const int r = G->sl[s].rank;
    int64_t tot = 0;
    for (int f = 0; f < W; ++f) {
      roff[s][f] = tot;
      tot += (int64_t)mat[(size_t)f * W + r];
    }
    nout[s] = tot;
    CU(H, cudaMalloc(&out[s], std::max<int64_t>(tot, 1) * REC * sizeof(double)));
  }
  std::vector<Msg> msgs;
  auto slot_of = [&](int rank) {
    for (int s = 0; s < S; ++s)
      if (G->sl[s].rank == rank) return s;
    return -1;
  };
  for (int f = 0; f < W; ++f)
    for (int t = 0; t < W; ++t) {
      const size_t cntm = (size_t)mat[(size_t)f * W + t];
      if (!cntm) continue;
      const int sf = slot_of(f), st = slot_of(t);
      if (sf < 0 && st < 0) continue;
      const double* sb = nullptr;
      if (sf >= 0) {
        int64_t o = 0;
        for (int d = 0; d < t; ++d) o += mine[sf][d];
        sb = sorted[sf] + (size_t)REC * o;
      }
      double* rb = st >= 0 ? out[st] + (size_t)REC * roff[st][f] : nullptr;
      if (sf >= 0 && st >= 0 && !G->virt) {  // (a rank's records to itself: a device copy)
        CU(H, cudaMemcpyAsync(rb, sb, cntm * REC * sizeof(double), cudaMemcpyDeviceToDevice, G->stream));
        continue;
      }
      msgs.push_back(Msg{f, t, sb, rb, cntm * REC});
    }
  rc = dist_p2p(H, G, msgs);
  if (rc) return rc;
  CU(H, cudaStreamSynchronize(G->stream));
  ++G->syncs;
  for (int s = 0; s < S; ++s) {
    cudaFree(sorted[s]);
    recs[s] = out[s];
    n[s] = nout[s];
  }
  return BDM_OK;
}

// Builds (or rebuilds) slab handle s with `cnt` owned records and enough room.
int dist_load_slab(bdm_ctx* H, DistGroup* G, int s, const double* rec, int64_t cnt) {
  DistSlab& D = G->sl[s];
  const int64_t room = std::max<int64_t>(cnt + cnt / 4 + 4 * G->cap + 4096, 1);
  if (!D.h || D.room < room) {
    if (D.h) bdm_destroy(D.h);
    D.h = nullptr;
    bdm_params p = H->prm;
    p.flags = BDM_DEVICE_PTRS;
    p.device = G->device;
    bdm_ctx* h = nullptr;
    // an empty slab handle of the given capacity (records are unpacked below)
    int rc = bdm_slab_init(&h, 0, room, nullptr, nullptr, nullptr, &p);
    if (rc) return fail(H, rc, "slab %d: %s", D.rank, bdm_last_error(nullptr));
    h->stream = G->stream;
    D.h = h;
    D.room = room;
  }
  bdm_ctx* h = D.h;
  h->cur = 0;
  h->n = cnt;
  h->n_dead = 0;
  h->split_pending = false;
  h->cols_next = false;
  h->have_dp = false;
  h->n_dp = 0;
  h->state = State::NoGrid;
  set_box_edge(h->grid, G->L);
  h->have_grid = true;
  k_ext_reset<<<1, 32, 0, G->stream>>>(h->ext, 0);  // (clears the sticky flags of a fresh allocation)
  {
    ErrDev e0{0u, 0xffffffffu, ERR_NONE};
    CU(H, cudaMemcpyAsync(h->err, &e0, sizeof e0, cudaMemcpyHostToDevice, G->stream));
  }
  if (cnt) k_unpack<<<blocks(cnt, 256), 256, 0, G->stream>>>(rec, (uint32_t)cnt, h->ag[0], h->id[0], 0u);
  CU(H, cudaGetLastError());
  if (!D.dc) {
    CU(H, cudaMalloc(&D.dc, DC_N * sizeof(uint32_t)));
    CU(H, cudaMallocHost(&D.dc_host, DC_N * sizeof(uint32_t)));
  }
  std::vector<uint32_t> z(DC_N, 0u);
  z[DC_LIVE] = (uint32_t)cnt;
  CU(H, cudaMemcpyAsync(D.dc, z.data(), DC_N * sizeof(uint32_t), cudaMemcpyHostToDevice, G->stream));
  CU(H, cudaStreamSynchronize(G->stream));
  ++G->syncs;
  D.live = cnt;
  D.stepped = false;
  D.fvalid = false;
  D.xb = G->cuts[D.rank];
  D.xe = G->cuts[D.rank + 1];
  return BDM_OK;
}

// Per-layer work of the slab's own agents (its grid over its own layers): sum n_b^2 per layer.
int dist_layer_sq(bdm_ctx* H, DistGroup* G, int s, int32_t x0, uint32_t nx, std::vector<double>& sq_out) {
  DistSlab& D = G->sl[s];
  bdm_ctx* h = D.h;
  sq_out.assign(nx, 0.0);
  if (D.live == 0) return BDM_OK;
  GridDev& g = h->grid;
  g.lo[0] = std::max<int32_t>(D.xb, G->glo[0]);
  g.hi[0] = std::min<int32_t>(D.xe - 1, G->ghi[0]);
  for (int a = 1; a < 3; ++a) {
    g.lo[a] = G->glo[a];
    g.hi[a] = G->ghi[a];
  }
  if (g.lo[0] > g.hi[0]) return BDM_OK;
  g.ny = g.hi[1] - g.lo[1] + 1;
  g.nz = g.hi[2] - g.lo[2] + 1;
  const int64_t nb = ((int64_t)g.hi[0] - g.lo[0] + 1) * g.ny * (int64_t)g.nz;
  if (nb >= (int64_t)0xffffffffll) return fail(H, BDM_ERANGE, "setup grid of rank %d: %lld boxes", D.rank, (long long)nb);
  g.n_boxes = (uint32_t)nb;
  h->cols_next = false;
  int rc = sort_into(h, (uint32_t)D.live, 0u);
  if (rc) return fail(H, rc, "setup grid of rank %d: %s", D.rank, h->error.c_str());
  unsigned long long* sq = nullptr;
  CU(H, cudaMalloc(&sq, nx * sizeof(unsigned long long)));
  Scratch scs;
  scs.p = sq;
  CU(H, cudaMemsetAsync(sq, 0, nx * sizeof(unsigned long long), G->stream));
  k_layer_work<<<h->sm_count * 4, 256, 0, G->stream>>>(h->grid, x0, nx, sq);
  CU(H, cudaGetLastError());
  std::vector<unsigned long long> hs(nx);
  CU(H, cudaMemcpyAsync(hs.data(), sq, nx * sizeof(unsigned long long), cudaMemcpyDeviceToHost, G->stream));
  CU(H, cudaStreamSynchronize(G->stream));
  ++G->syncs;
  for (uint32_t k = 0; k < nx; ++k) sq_out[k] = (double)hs[k];
  // back to unsorted owned records order is irrelevant: the sorted buffer is the owned state now
  return BDM_OK;
}

// ---- one step of every local slab (no host synchronisation)
int dist_split_all(bdm_ctx* H, DistGroup* G) {
  cudaStream_t st = G->stream;
  for (auto& D : G->sl) {
    bdm_ctx* h = D.h;
    CU(H, lx(k_dist_prep, 1, 32, 0, st, h->grid, D.stepped ? 1 : 0, D.xb, D.xe, D.dc, h->cnt + 4, h->cnt));
    DBG(h, "k_dist_prep");
    CU(H, lx(k_slab_split, h->sm_count * 4, 256, 0, st, h->ag[h->cur], h->id[h->cur], (uint32_t)D.room, h->cnt + 4,
             h->grid.inv, D.xb, D.xe, D.msg[0] + HDR, D.msg[1] + HDR, (uint64_t)G->cap, h->cnt, D.dc + DC_LIVE));
    DBG(h, "k_slab_split");
    CU(H, lx(k_dist_header, 1, 32, 0, st, h->cnt, (uint64_t)G->cap, D.msg[0], D.msg[1], D.dc));
    DBG(h, "k_dist_header");
    CU(H, cudaGetLastError());
    h->launches += 3;
  }
  // the exchange: every rank sends its lower message to r-1 and its upper one to r+1
  std::vector<Msg> msgs;
  const size_t cnt = (size_t)HDR + (size_t)REC * (size_t)G->cap;
  auto slot = [&](int rank) -> DistSlab* {
    for (auto& D : G->sl)
      if (D.rank == rank) return &D;
    return nullptr;
  };
  for (int r = 0; r < G->world; ++r) {
    for (int side = 0; side < 2; ++side) {  // side 0: r -> r-1 (arrives as the receiver's upper message)
      const int to = side == 0 ? r - 1 : r + 1;
      if (to < 0 || to >= G->world) continue;
      DistSlab* a = slot(r);
      DistSlab* b = slot(to);
      if (!a && !b) continue;
      msgs.push_back(Msg{r, to, a ? a->msg[side] : nullptr, b ? b->msg[side == 0 ? 3 : 2] : nullptr, cnt});
    }
  }
  return dist_p2p(H, G, msgs);
}

int dist_ingest_build_force(bdm_ctx* H, DistGroup* G, DistSlab& D, bool want_dp) {
  bdm_ctx* h = D.h;
  cudaStream_t st = G->stream;
  const uint32_t room = (uint32_t)D.room;
  // emigrants of the split are marked dead in place (the sort drops them)
  const bool packed = h->cols_next && D.zbits > 0;  // the last sum pass wrote packed new boxes of [0, LIVE)
  CU(H, lx(k_slab_mark_dead, h->sm_count * 4, 256, 0, st, h->ag[h->cur], room, h->cnt + 4, h->grid.inv, D.xb, D.xe,
           D.dc + DC_LIVE, packed ? h->pbox : nullptr));
  DBG(h, "k_slab_mark_dead");
  const bool fused = h->cols_next;
  CU(H, lx(k_dist_ingest, h->sm_count * 2, 256, 0, st, h->ag[h->cur], h->id[h->cur], D.dc, h->cnt, D.msg[0], D.msg[1],
           D.msg[2], D.msg[3], (uint32_t)G->cap, D.rank > 0 ? 1 : 0, D.rank + 1 < G->world ? 1 : 0, room,
           fused ? 1 : 0));
  DBG(h, "k_dist_ingest");
  CU(H, cudaGetLastError());
  h->launches += 2;
  TimedStep ts{};
  if (h->timing) {
    CU(H, cudaEventCreate(&ts.e0));
    CU(H, cudaEventCreate(&ts.e1));
    CU(H, cudaEventCreate(&ts.e2));
    h->timed.push_back(ts);
    CU(H, cudaEventRecord(ts.e0, st));
  }
  // slab-local grid over the chunk's fixed frame (G->glo/ghi +- margin, x clipped to the slab)
  GridDev& g = h->grid;
  for (int a = 0; a < 3; ++a) {
    g.lo[a] = D.flo[a];
    g.hi[a] = D.fhi[a];
  }
  g.ny = g.hi[1] - g.lo[1] + 1;
  g.nz = g.hi[2] - g.lo[2] + 1;
  g.n_boxes = (uint32_t)(((int64_t)g.hi[0] - g.lo[0] + 1) * g.ny * (int64_t)g.nz);
  g.m32 = D.fm32;
  const int src0 = h->cur;
  {
    const uint64_t nc = (uint64_t)(g.hi[0] - g.lo[0] + 1) * (uint64_t)g.ny;
    g.n_cols = (uint32_t)nc;
    int rc = ensure_columns(h, nc + 1);
    if (rc) return fail(H, rc, "%s", h->error.c_str());
    rc = ensure_table(h, (size_t)g.n_boxes + 1, nc + 1);
    if (rc) return fail(H, rc, "%s", h->error.c_str());
    if (fused) {  // z-ranges of the stepped agents were accumulated by the last sum pass
      std::swap(h->czlo, h->czlo2);
      std::swap(h->czhi, h->czhi2);
      std::swap(h->col_cap, h->col2_cap);
      h->cols_next = false;
      rc = ensure_columns(h, nc + 1);
      if (rc) return fail(H, rc, "%s", h->error.c_str());
    } else {
      const unsigned gs = (unsigned)std::min<uint64_t>((nc + 256) / 256, 148u * 16u);
      CU(H, lx(k_col_reset, gs, 256, 0, st, h->czlo, h->czhi, g.n_cols));
      h->launches += 1;
    }
    g.czlo = h->czlo;
    g.czhi = h->czhi;
    g.coff = h->coff;
    g.table = h->table;
    g.col = h->colrec;
    CU(H, lx(k_col_ext, fused ? h->sm_count * 2 : blocks(room, 512), 256, 0, st, h->ag[src0], room, g, h->czlo,
             h->czhi, D.dc + DC_CE0));
    DBG(h, "k_col_ext(dist)");
    const unsigned gs = (unsigned)std::min<uint64_t>((nc + 256) / 256, 148u * 16u);
    rc = scan_reserve(h, nc + 1);  // (k_col_len zeroes the offset scan's tile states, k_table_zero the table scan's)
    if (rc) return fail(H, rc, "%s", h->error.c_str());
    CU(H, lx(k_col_len, gs, 256, 0, st, h->czlo, h->czhi, g.n_cols, h->coff, h->scan_state,
             (uint32_t)((nc + 1 + SCAN_TILE - 1) / SCAN_TILE), h->scan_ticket));
    DBG(h, "k_col_len(dist)");
    rc = scan(h, h->coff, nc + 1, nullptr, true);
    if (rc) return fail(H, rc, "%s", h->error.c_str());
    CU(H, lx(k_table_zero, h->sm_count * 8, 256, 0, st, h->table, h->coff, g.n_cols, h->czlo, h->czhi, h->colrec,
             h->scan_state, (uint32_t)h->scan_tiles_cap, h->scan_ticket, nullptr));
    DBG(h, "k_table_zero(dist)");
    if (packed) {  // the stepped agents' boxes from the sum pass (4 B), the appended records from their state
      CU(H, lx(k_key_hist_packed<true>, blocks(room, 256 * KHP), 256, 0, st, h->pbox, room, g, D.flo[2], D.zbits,
               h->key, h->slot, h->table, h->err, D.dc + DC_LIVE));
      CU(H, lx(k_key_hist<true>, h->sm_count * 4, 256, 0, st, h->ag[src0], room, g, h->key, h->slot, h->table, h->err,
               D.dc + DC_TOT, D.dc + DC_LIVE));
      h->launches += 1;
    } else {
      CU(H, lx(k_key_hist<true>, blocks(room, 512), 256, 0, st, h->ag[src0], room, g, h->key, h->slot, h->table,
               h->err, D.dc + DC_TOT, nullptr));
    }
    DBG(h, "k_key_hist(dist)");
    rc = scan(h, h->table, 0, h->coff + nc, true);
    if (rc) return fail(H, rc, "%s", h->error.c_str());
    CU(H, lx(k_scatter, blocks(room, 256 * KSC), 256, 0, st, h->key, h->slot, h->id[src0], h->table, room, h->tsrc,
             h->tid, h->tkey, D.dc + DC_TOT));
    DBG(h, "k_scatter(dist)");
    CU(H, lx(k_place, blocks(room, PLACE_T), PLACE_T, 0, st, h->tsrc, h->tid, h->tkey, h->table, h->ag[src0], room,
             h->ag[1 - src0], h->id[1 - src0], h->agf, nullptr, nullptr, D.dc + DC_SORTED, h->id[src0],
             D.dc + DC_ABEGIN));
    DBG(h, "k_place(dist)");
    CU(H, cudaGetLastError());
    h->launches += 7;
    h->cur = 1 - src0;
  }
  if (h->timing) CU(H, cudaEventRecord(ts.e1, st));
  // half-shell force phase on the owned range [A_BEGIN, A_END) of the sorted array
  const int src = h->cur, dst = 1 - h->cur;
  ParamsDev pd = params_dev(h->prm);
  ColNext cn{0, 0, 0, 0, nullptr, nullptr, nullptr, 0, 0};
  {
    cn.lo0 = g.lo[0];
    cn.lo1 = g.lo[1];
    cn.nx = g.hi[0] - g.lo[0] + 1;
    cn.ny = g.ny;
    const size_t nc2 = (size_t)cn.nx * (size_t)cn.ny;
    int rc = ensure_columns(h, nc2 + 1, true);
    if (rc) return fail(H, rc, "%s", h->error.c_str());
    cn.czlo = h->czlo2;
    cn.czhi = h->czhi2;
    if (D.zbits > 0) {  // packed new boxes for the next build's key pass (the frame is fixed for the chunk)
      cn.pbox = h->pbox;
      cn.z0 = D.flo[2];
      cn.zbits = D.zbits;
    }
    // one launch: extents reset, the next build's column ranges, the pair counters
    const uint64_t w = std::max<uint64_t>(nc2, (uint64_t)room / 4 + 1);
    const unsigned gr = (unsigned)std::min<uint64_t>((w + 255) / 256, 148u * 16u);
    CU(H, lx(k_force_reset, gr, 256, 0, st, h->ext, 1, h->czlo2, h->czhi2, (uint32_t)nc2, h->h_bcnt,
             std::max<uint32_t>(room, 1u)));
  }
  if (g_htile) {
    const unsigned gt = (unsigned)h->sm_count * h->tile_blocks_per_sm;
    k_half_search_tile<<<gt, TILE_THREADS, TILE_SMEM_BYTES, st>>>(h->ag[src], h->agf, 0u, room, g, h->h_fwd, h->h_fcnt,
                                                              h->h_bwd, h->h_bcnt, h->ext, false, D.dc + DC_AEND);
  } else {
    const unsigned ga = (unsigned)h->sm_count * h->half_a_blocks_per_sm;
    CU(H, lx(k_half_search, ga, HA_THREADS, HA_SMEM_BYTES, st, h->ag[src], h->agf, 0u, room, g, h->h_fwd, h->h_fcnt,
             h->h_bwd, h->h_bcnt, h->ext, false, D.dc + DC_AEND, nullptr));
  }
  DBG(h, "k_half_search(dist)");
  if (h->timing && !h->timed.empty() && !h->timed.back().e3) {
    CU(H, cudaEventCreate(&h->timed.back().e3));
    CU(H, cudaEventRecord(h->timed.back().e3, st));
  }
  const unsigned gb = (unsigned)h->sm_count * h->half_b_blocks_per_sm;
  double* dp = want_dp ? h->dp : nullptr;
  uint32_t* dpi = want_dp ? h->dp_ids : nullptr;
  CU(H, lx(k_half_sum<false>, gb, FORCE_THREADS, HB_SMEM_BYTES, st, h->ag[src], h->id[src], 0u, room, g, pd,
           h->ag[dst], nullptr /* (ids: k_place wrote the owned range) */, dp, dpi, h->ext, h->err, h->h_fwd, h->h_fcnt,
           h->h_bwd, h->h_bcnt, cn, nullptr,
           h->h_slow, D.dc + DC_ABEGIN, nullptr, (int64_t)-1));
  DBG(h, "k_half_sum(dist)");
  CU(H, lx(k_half_slow<false>, (unsigned)h->sm_count * 4, 128, 0, st, h->ag[src], h->id[src], 0u, g, pd, h->ag[dst],
           h->id[dst], dp, dpi, h->ext, h->err, cn, nullptr, h->h_slow, D.dc + DC_ABEGIN));
  DBG(h, "k_half_slow(dist)");
  CU(H, lx(k_locate_nonfinite, 1, 32, 0, st, h->ag[src], h->id[src], g, pd, h->err));
  CU(H, cudaGetLastError());
  h->launches += 5;  // k_force_reset, search, sum, slow, locate
  if (h->timing) CU(H, cudaEventRecord(ts.e2, st));
  h->cur = dst;
  h->cols_next = true;
  h->nlo[0] = cn.lo0;
  h->nlo[1] = cn.lo1;
  h->nnx = cn.nx;
  h->nny = cn.ny;
  h->last_half = true;
  h->state = State::Stepped;
  if (want_dp) h->have_dp = true;
  D.stepped = true;
  return BDM_OK;
}

// Chunk set-up: frame, capacities, checkpoint.
int dist_chunk_begin(bdm_ctx* H, DistGroup* G, int K) {
  const int32_t M = K + 1;
  for (auto& D : G->sl) {
    bdm_ctx* h = D.h;
    // buffers: room for the owned agents + 4 messages; message buffers of the agreed capacity
    const int64_t room_need = D.live + D.live / 8 + 4 * G->cap + 4096;
    if (room_need > D.room) {  // grow the slab (keeps the owned agents)
      bdm_params p = H->prm;
      p.flags = BDM_DEVICE_PTRS;
      p.device = G->device;
      bdm_ctx* nh = nullptr;
      const int64_t nroom = room_need + room_need / 4;
      int rc = bdm_slab_init(&nh, 0, nroom, nullptr, nullptr, nullptr, &p);
      if (rc) return fail(H, rc, "slab %d regrow: %s", D.rank, bdm_last_error(nullptr));
      nh->stream = G->stream;
      k_ext_reset<<<1, 32, 0, G->stream>>>(nh->ext, 0);
      CU(H, cudaMemcpyAsync(nh->ag[0], h->ag[h->cur], D.live * sizeof(double4), cudaMemcpyDeviceToDevice, G->stream));
      CU(H, cudaMemcpyAsync(nh->id[0], h->id[h->cur], D.live * sizeof(uint32_t), cudaMemcpyDeviceToDevice, G->stream));
      CU(H, cudaStreamSynchronize(G->stream));
      ++G->syncs;
      nh->timing = h->timing;
      nh->launches = h->launches;
      nh->grid = h->grid;
      nh->grid.pad = (uint32_t)nroom;  // (its own padding agent)
      bdm_destroy(h);
      D.h = h = nh;
      D.room = nroom;
      D.stepped = false;
      D.fvalid = false;
      h->cur = 0;
      h->cols_next = false;
      h->state = State::NoGrid;
    }
    h->n = D.live;
    init_device_info(h);
    h->cap = D.room;
    if (!ensure_half(h)) return fail(H, BDM_ENOMEM, "rank %d: pair rows for %lld agents", D.rank, (long long)D.room);
    if (D.msg_cap != G->cap) {  // (re)allocated only when the agreed capacity changes
      const size_t mcount = (size_t)HDR + (size_t)REC * (size_t)G->cap;
      for (int k = 0; k < 4; ++k) {
        if (D.msg[k]) cudaFree(D.msg[k]);
        D.msg[k] = nullptr;
        CU(H, cudaMalloc(&D.msg[k], mcount * sizeof(double)));
        CU(H, cudaMemsetAsync(D.msg[k], 0, HDR * sizeof(double), G->stream));
      }
      D.msg_cap = G->cap;
    }
    if (!D.sum) {
      CU(H, cudaMalloc(&D.sum, SUMN * sizeof(double)));
      CU(H, cudaMallocHost(&D.sum_host, SUMN * sizeof(double)));
    }
    if (D.ck_cap < D.live || !D.ck_ag) {
      if (D.ck_ag) cudaFree(D.ck_ag);
      if (D.ck_id) cudaFree(D.ck_id);
      D.ck_cap = std::max<int64_t>(D.live + D.live / 4 + 1024, 1);
      CU(H, cudaMalloc(&D.ck_ag, D.ck_cap * sizeof(double4)));
      CU(H, cudaMalloc(&D.ck_id, D.ck_cap * sizeof(uint32_t)));
    }
    if (D.live) {
      CU(H, cudaMemcpyAsync(D.ck_ag, h->ag[h->cur], D.live * sizeof(double4), cudaMemcpyDeviceToDevice, G->stream));
      CU(H, cudaMemcpyAsync(D.ck_id, h->id[h->cur], D.live * sizeof(uint32_t), cudaMemcpyDeviceToDevice, G->stream));
    }
    // the frame of this chunk: x = [xb - 1, xe] clipped to the global extents +- M; y, z global +- M
    // (applied by the chunk's first build: the first split still reads the last step's grid).  The
    // previous chunk's frame is kept while it holds every agent of this chunk (the global extents
    // +- (K + 1) boxes): then the last sum pass's fused columns and packed boxes stay valid.
    int32_t nlo[3], nhi[3];
    nlo[0] = (int32_t)std::max<int64_t>((int64_t)D.xb - 1, (int64_t)G->glo[0] - M);
    nhi[0] = (int32_t)std::min<int64_t>((int64_t)D.xe, (int64_t)G->ghi[0] + M);
    if (nlo[0] > nhi[0]) nhi[0] = nlo[0];  // (a rank without agents near its slab)
    for (int a = 1; a < 3; ++a) {
      nlo[a] = G->glo[a] - M;
      nhi[a] = G->ghi[a] + M;
    }
    bool keep = D.fvalid;
    for (int a = 0; a < 3; ++a) keep = keep && nlo[a] >= D.flo[a] && nhi[a] <= D.fhi[a];
    const bool keep_cols = keep && h->cols_next;
    if (!keep) {  // a new frame, with the full margin of a longest chunk (kept for longer)
      const int32_t MM = DIST_CHUNK + 1;
      D.flo[0] = (int32_t)std::max<int64_t>((int64_t)D.xb - 1, (int64_t)G->glo[0] - MM);
      D.fhi[0] = (int32_t)std::min<int64_t>((int64_t)D.xe, (int64_t)G->ghi[0] + MM);
      if (D.flo[0] > D.fhi[0]) D.fhi[0] = D.flo[0];
      for (int a = 1; a < 3; ++a) {
        D.flo[a] = G->glo[a] - MM;
        D.fhi[a] = G->ghi[a] + MM;
      }
      D.fvalid = true;
    }
    for (int a = 0; a < 3; ++a)
      if (D.flo[a] < -(1 << 20) + 2 || D.fhi[a] > (1 << 20) - 2)
        return fail(H, BDM_ERANGE, "an agent lies >= 2^20 boxes from the origin (DESIGN.md R9)");
    const int64_t nb = ((int64_t)D.fhi[0] - D.flo[0] + 1) * ((int64_t)D.fhi[1] - D.flo[1] + 1) *
                       ((int64_t)D.fhi[2] - D.flo[2] + 1);
    if (nb >= (int64_t)0xffffffffll) return fail(H, BDM_ERANGE, "rank %d frame: %lld boxes >= 2^32", D.rank, (long long)nb);
    // the fp32 prefilter margin of this frame (as sort_into)
    double P = 0.0;
    for (int a = 0; a < 3; ++a)
      P = std::max(P, std::max(std::fabs((double)D.flo[a]), std::fabs((double)D.fhi[a] + 1.0)) * G->L * (1.0 + 0x1p-20));
    const double ulp32 = P > 0.0 ? std::ldexp(1.0, std::ilogb(P) - 23) : 0x1p-149;
    D.fm32 = 2.0 * ulp32 + 0x1p-18 + G->L * 0x1p-20;
    h->cols_next = keep_cols;  // else the first build of the chunk runs its own column pass
    {  // packed new boxes: (column << zbits | z - flo[2]) when that fits 32 bits
      const uint64_t ncols = (uint64_t)(D.fhi[0] - D.flo[0] + 1) * (uint64_t)(D.fhi[1] - D.flo[1] + 1);
      int zb = 1;
      while ((1 << zb) < D.fhi[2] - D.flo[2] + 1) ++zb;
      D.zbits = zb < 31 && ncols <= (0xffffffffull >> zb) ? zb : 0;
      if (D.zbits && (int64_t)h->pbox_cap < D.room) {
        if (h->pbox) cudaFree(h->pbox);
        h->pbox = nullptr;
        CU(H, cudaMalloc(&h->pbox, D.room * sizeof(uint32_t)));
        h->pbox_cap = (size_t)D.room;
      }
    }
    CU(H, cudaMemsetAsync(D.dc + DC_OVF, 0, 4 * sizeof(uint32_t), G->stream));  // OVF, NEED, MIG, GHOSTS
  }
  return BDM_OK;  // (no host synchronisation: everything above is ordered on the stream)
}

// Chunk end: the one host round trip.  Every slab's summary is all-reduced on the device (NCCL;
// virtual ranks: reduced here), then read back with the counts and errors; returns 1 in *redo if some
// message or buffer overflowed (the chunk is re-run).
int dist_chunk_end(bdm_ctx* H, DistGroup* G, int* redo) {
  for (auto& D : G->sl) {
    bdm_ctx* h = D.h;
    k_dist_summary<<<1, 32, 0, G->stream>>>(D.dc, h->ext, D.sum);
    CU(H, cudaGetLastError());
    h->launches += 1;
  }
  if (!G->virt && G->world > 1) NC(H, G->api->allReduce(G->sl[0].sum, G->sl[0].sum, SUMN, ncclDouble, ncclMax,
                                                        G->comm, G->stream));
  for (auto& D : G->sl) {
    bdm_ctx* h = D.h;
    CU(H, cudaMemcpyAsync(D.sum_host, D.sum, SUMN * sizeof(double), cudaMemcpyDeviceToHost, G->stream));
    CU(H, cudaMemcpyAsync(D.dc_host, D.dc, DC_N * sizeof(uint32_t), cudaMemcpyDeviceToHost, G->stream));
    CU(H, cudaMemcpyAsync(h->err_host, h->err, sizeof(ErrDev), cudaMemcpyDeviceToHost, G->stream));
  }
  CU(H, cudaStreamSynchronize(G->stream));
  ++G->syncs;
  double mx[SUMN];
  for (int k = 0; k < SUMN; ++k) {
    mx[k] = G->sl[0].sum_host[k];
    for (size_t s = 1; s < G->sl.size(); ++s) mx[k] = std::max(mx[k], G->sl[s].sum_host[k]);
  }
  *redo = mx[0] != 0.0;
  const double need = mx[1];
  if (*redo) {  // results of this chunk are void: clear its error state, grow the messages, re-run it
    ErrDev e0{0u, 0xffffffffu, ERR_NONE};
    for (auto& D : G->sl) {
      CU(H, cudaMemcpyAsync(D.h->err, &e0, sizeof e0, cudaMemcpyHostToDevice, G->stream));
      k_ext_reset<<<1, 32, 0, G->stream>>>(D.h->ext, 0);
    }
    G->cap = std::max<int64_t>(G->cap * 2, (int64_t)(need * 1.5) + 4096);
    ++G->redo;
    return BDM_OK;
  }
  for (auto& D : G->sl) {
    bdm_ctx* h = D.h;
    if (h->err_host->code) {  // asynchronous data errors (non-finite force, agent outside the frame)
      const int rc = check_async(h);
      H->poisoned = true;
      return fail(H, rc ? rc : BDM_ECUDA, "rank %d: %s", D.rank, h->error.c_str());
    }
  }
  if (mx[2] != 0.0) {
    H->poisoned = true;
    return fail(H, BDM_ERANGE, "an agent left the grid frame of a chunk (|p*inv| >= 2^20 or a non-finite position)");
  }
  for (int a = 0; a < 3; ++a) {
    G->glo[a] = (int32_t)(-mx[3 + a]);
    G->ghi[a] = (int32_t)mx[6 + a];
  }
  int64_t mig = 0, gh = 0;
  for (auto& D : G->sl) {
    D.live = D.dc_host[DC_AEND] - D.dc_host[DC_ABEGIN];
    D.h->n = D.live;
    D.h->n_dp = D.live;
    mig += D.dc_host[DC_MIG];
    gh += D.dc_host[DC_GHOSTS];
  }
  G->migrated += mig;
  G->ghosts = gh;
  // keep the capacity ahead of the largest need (every rank computes the same value)
  if (need * 1.25 > (double)G->cap) G->cap = (int64_t)(need * 1.5) + 4096;
  return BDM_OK;
}

int dist_restore(bdm_ctx* H, DistGroup* G) {
  for (auto& D : G->sl) {
    bdm_ctx* h = D.h;
    h->cur = 0;
    if (D.live) {
      CU(H, cudaMemcpyAsync(h->ag[0], D.ck_ag, D.live * sizeof(double4), cudaMemcpyDeviceToDevice, G->stream));
      CU(H, cudaMemcpyAsync(h->id[0], D.ck_id, D.live * sizeof(uint32_t), cudaMemcpyDeviceToDevice, G->stream));
    }
    std::vector<uint32_t> z(DC_N, 0u);
    z[DC_LIVE] = (uint32_t)D.live;
    CU(H, cudaMemcpyAsync(D.dc, z.data(), DC_N * sizeof(uint32_t), cudaMemcpyHostToDevice, G->stream));
    D.stepped = false;
    h->cols_next = false;
  }
  CU(H, cudaStreamSynchronize(G->stream));
  ++G->syncs;
  return BDM_OK;
}

int dist_mech_step_(bdm_ctx* H, int32_t n_steps);
int dist_mech_step(bdm_ctx* H, int32_t n_steps) {
  const int rc = dist_mech_step_(H, n_steps);
  if (rc && H->error.empty()) H->error = g_tls_error;  // (a slab's failure message)
  return rc;
}

int dist_step(bdm_ctx* H, DistGroup* G, bool want_dp) {
  int rc = dist_split_all(H, G);
  if (rc) return rc;
  for (auto& D : G->sl)
    if ((rc = dist_ingest_build_force(H, G, D, want_dp))) return rc;
  return BDM_OK;
}

// What the steady pair's launches bake in: buffers, frame, capacity, parity, column arrays.
std::vector<uintptr_t> dist_signature(DistGroup* G) {
  std::vector<uintptr_t> v{(uintptr_t)G->cap, (uintptr_t)G->stream};
  for (auto& D : G->sl) {
    bdm_ctx* h = D.h;
    for (uintptr_t x : {(uintptr_t)h, (uintptr_t)h->cur, (uintptr_t)h->czlo, (uintptr_t)h->czlo2, (uintptr_t)h->table,
                        (uintptr_t)h->coff, (uintptr_t)h->colrec, (uintptr_t)h->pbox, (uintptr_t)h->h_fwd,
                        (uintptr_t)h->scan_state, (uintptr_t)D.room, (uintptr_t)D.zbits, (uintptr_t)D.msg[0],
                        (uintptr_t)D.msg[2], (uintptr_t)(uint32_t)D.flo[0], (uintptr_t)(uint32_t)D.flo[1],
                        (uintptr_t)(uint32_t)D.flo[2], (uintptr_t)(uint32_t)D.fhi[0], (uintptr_t)(uint32_t)D.fhi[1],
                        (uintptr_t)(uint32_t)D.fhi[2], (uintptr_t)h->cols_next, (uintptr_t)D.stepped})
      v.push_back(x);
  }
  return v;
}

// npairs x two steady steps through one CUDA graph (captured once per signature): the ~30 launches and
// the NCCL group of a step cost a few microseconds each when issued one by one.  The host-side state a
// step mutates (buffer parity, column array swaps) has period two, so it is back where it started.
int dist_steady_pairs(bdm_ctx* H, DistGroup* G, int npairs) {
  const std::vector<uintptr_t> sig = dist_signature(G);
  if (!G->gexec || sig != G->gsig) {
    if (G->gexec) cudaGraphExecDestroy(G->gexec);
    G->gexec = nullptr;
    int64_t l0 = 0, b0 = G->bytes;
    for (auto& D : G->sl) l0 += D.h->launches;
    CU(H, cudaStreamBeginCapture(G->stream, cudaStreamCaptureModeThreadLocal));
    int rc = dist_step(H, G, false);
    if (!rc) rc = dist_step(H, G, false);
    cudaGraph_t graph = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(G->stream, &graph);
    if (rc || ce != cudaSuccess || !graph) {
      (void)cudaGetLastError();
      if (graph) cudaGraphDestroy(graph);
      return rc ? rc : fail(H, BDM_ECUDA, "graph capture of the steady steps: %s", cudaGetErrorString(ce));
    }
    const cudaError_t ie = cudaGraphInstantiate(&G->gexec, graph, 0);
    cudaGraphDestroy(graph);
    if (ie != cudaSuccess) {
      (void)cudaGetLastError();
      G->gexec = nullptr;
      return fail(H, BDM_ECUDA, "graph instantiation: %s", cudaGetErrorString(ie));
    }
    int64_t l1 = 0;
    for (auto& D : G->sl) l1 += D.h->launches;
    G->graph_launches = l1 - l0;
    G->graph_bytes = G->bytes - b0;  // (the capture counted one pair: that of the launch just below)
    G->gsig = dist_signature(G);
    if (G->gsig != sig) return fail(H, BDM_ECUDA, "steady steps are not of period two");
    // the capture recorded one pair without running it: run it now
    --npairs;
    CU(H, cudaGraphLaunch(G->gexec, G->stream));
    ++G->replays;
  }
  for (int p = 0; p < npairs; ++p) {
    CU(H, cudaGraphLaunch(G->gexec, G->stream));
    ++G->replays;
    G->sl[0].h->launches += G->graph_launches;
    G->bytes += G->graph_bytes;
  }
  return BDM_OK;
}

int dist_mech_step_(bdm_ctx* H, int32_t n_steps) {
  DistGroup* G = H->dist;
  int done = 0;
  // graphs need a capturable stream (not the legacy default stream) and no per-step host work
  bool use_graph = G->stream != nullptr && !g_debug && !std::getenv("BDM_DIST_NOGRAPH");
  for (auto& D : G->sl) use_graph = use_graph && !D.h->timing;
  while (done < n_steps) {
    const int K = std::min(DIST_CHUNK, n_steps - done);
    int rc = dist_chunk_begin(H, G, K);
    if (rc) return rc;
    int k = 0;
    while (k < K) {
      const bool last = done + k == n_steps - 1;
      // steady pairs: after the chunk's first step (fused columns from then on), before the last step
      // of the call (which keeps the displacements)
      const int steady = (K - 1) - k - (done + K == n_steps ? 1 : 0);
      if (use_graph && k >= 1 && steady >= 2) {
        const int np = steady / 2;
        if ((rc = dist_steady_pairs(H, G, np))) return rc;
        k += 2 * np;
        continue;
      }
      if ((rc = dist_step(H, G, last))) return rc;
      ++k;
    }
    int redo = 0;
    if ((rc = dist_chunk_end(H, G, &redo))) return rc;
    if (redo) {  // a message or buffer overflowed: re-run the chunk from its checkpoint
      if ((rc = dist_restore(H, G))) return rc;
      continue;
    }
    done += K;
    G->steps += K;
    ++G->chunks;
  }
  H->n = 0;
  for (auto& D : G->sl) H->n += D.live;
  return BDM_OK;
}

int dist_sync(bdm_ctx* H) {
  DistGroup* G = H->dist;
  CU(H, cudaStreamSynchronize(G->stream));
  ++G->syncs;
  for (auto& D : G->sl) {
    int rc = check_async(D.h);
    if (rc) return fail(H, rc, "rank %d: %s", D.rank, D.h->error.c_str());
  }
  return BDM_OK;
}

void dist_set_timing(DistGroup* G, bool on) {
  for (auto& D : G->sl)
    if (D.h) D.h->timing = on;
}

// Timing of a distributed handle: the first local rank's events (bdm_get_timing_ex layout), launches
// of all local ranks.
int dist_get_timing(bdm_ctx* H, double* out6) {
  DistGroup* G = H->dist;
  int64_t launches = 0;
  for (size_t s = 1; s < G->sl.size(); ++s) {
    launches += G->sl[s].h->launches;
    G->sl[s].h->launches_total += G->sl[s].h->launches;
    G->sl[s].h->launches = 0;
    for (auto& t : G->sl[s].h->timed) {
      cudaEventDestroy(t.e0);
      cudaEventDestroy(t.e1);
      cudaEventDestroy(t.e2);
      if (t.e3) cudaEventDestroy(t.e3);
    }
    G->sl[s].h->timed.clear();
  }
  int rc = bdm_get_timing_ex(G->sl[0].h, out6);
  if (rc) return fail(H, rc, "%s", G->sl[0].h->error.c_str());
  out6[3] += (double)launches;
  return BDM_OK;
}

void dist_destroy(DistGroup* G) {
  if (!G) return;
  if (G->gexec) cudaGraphExecDestroy(G->gexec);
  for (auto& D : G->sl) {
    for (int k = 0; k < 4; ++k)
      if (D.msg[k]) cudaFree(D.msg[k]);
    if (D.ck_ag) cudaFree(D.ck_ag);
    if (D.ck_id) cudaFree(D.ck_id);
    if (D.sum) cudaFree(D.sum);
    if (D.sum_host) cudaFreeHost(D.sum_host);
    if (D.dc) cudaFree(D.dc);
    if (D.dc_host) cudaFreeHost(D.dc_host);
    if (D.h) bdm_destroy(D.h);
  }
  if (G->comm && G->api) G->api->commDestroy(G->comm);
  delete G;
}

// Shared set-up of bdm_init_dist (one local rank) and bdm_init_dist_local (all ranks local).
int dist_setup(bdm_ctx* H, DistGroup* G, std::vector<double*>& recs, std::vector<int64_t>& n) {
  const int S = (int)G->sl.size();
  // O1: the global box edge
  std::vector<std::vector<double>> loc(S), loc2(S);
  unsigned long long* mb = nullptr;
  CU(H, cudaMalloc(&mb, sizeof(unsigned long long)));
  Scratch scm;
  scm.p = mb;
  Extents* ext = nullptr;
  CU(H, cudaMalloc(&ext, sizeof(Extents)));
  Scratch sce;
  sce.p = ext;
  for (int s = 0; s < S; ++s) loc[s] = {0.0};
  // (records were validated and max D measured by the caller: H->ext_host holds nothing yet)
  for (int s = 0; s < S; ++s) {
    CU(H, cudaMemsetAsync(mb, 0, sizeof(unsigned long long), G->stream));
    // max D of the records
    k_ag_maxd_rec<<<blocks(std::max<int64_t>(n[s], 1), 256), 256, 0, G->stream>>>(recs[s], (uint32_t)n[s], mb);
    unsigned long long hb = 0;
    CU(H, cudaMemcpyAsync(&hb, mb, sizeof hb, cudaMemcpyDeviceToHost, G->stream));
    CU(H, cudaStreamSynchronize(G->stream));
    ++G->syncs;
    double d;
    std::memcpy(&d, &hb, sizeof d);
    loc[s][0] = d;
  }
  std::vector<double> r;
  int rc = dist_allreduce(H, G, loc, ncclMax, r);
  if (rc) return rc;
  G->L = std::max(r[0], H->prm.box_edge_min);
  if (!(G->L > 0.0)) G->L = 1.0;  // (no agents anywhere)
  G->inv = 1.0 / (G->L * (1.0 + 0x1p-30));
  if (!(H->prm.max_disp < G->L * (1.0 - 0x1p-20)))  // |dp| <= max_disp (1 + 4u) < L: boundary-layer exchange
    return fail(H, BDM_EINVAL, "distributed steps need max_disp (%g) < the box edge L (%g): a step must move an agent "
                "by less than one box (DESIGN.md §7)", H->prm.max_disp, G->L);
  // O2 extents
  for (int s = 0; s < S; ++s) {
    k_ext_reset<<<1, 32, 0, G->stream>>>(ext, 0);
    if (n[s]) k_rec_extents<<<blocks(n[s], 256), 256, 0, G->stream>>>(recs[s], (uint32_t)n[s], G->inv, ext);
    Extents he;
    CU(H, cudaMemcpyAsync(&he, ext, sizeof he, cudaMemcpyDeviceToHost, G->stream));
    CU(H, cudaStreamSynchronize(G->stream));
    ++G->syncs;
    if (he.range_err) return fail(H, BDM_ERANGE, "an agent lies >= 2^20 boxes from the origin (DESIGN.md R9)");
    loc2[s].clear();
    for (int a = 0; a < 3; ++a) loc2[s].push_back(n[s] ? -(double)he.lo[a] : -(double)INT32_MAX);
    for (int a = 0; a < 3; ++a) loc2[s].push_back(n[s] ? (double)he.hi[a] : (double)INT32_MIN);
    loc2[s].push_back((double)n[s]);
  }
  rc = dist_allreduce(H, G, loc2, ncclMax, r);
  if (rc) return rc;
  std::vector<double> tot;
  {
    std::vector<std::vector<double>> cn(S);
    for (int s = 0; s < S; ++s) cn[s] = {(double)n[s]};
    rc = dist_allreduce(H, G, cn, ncclSum, tot);
    if (rc) return rc;
  }
  G->n_global = (int64_t)tot[0];
  for (int a = 0; a < 3; ++a) {
    G->glo[a] = (int32_t)(-r[a]);
    G->ghi[a] = (int32_t)r[3 + a];
  }
  if (G->n_global == 0)
    for (int a = 0; a < 3; ++a) G->glo[a] = G->ghi[a] = 0;
  const int32_t x0 = G->glo[0];
  const uint32_t nx = (uint32_t)(G->ghi[0] - G->glo[0] + 1);
  // per-layer histogram -> count-balanced cuts
  std::vector<std::vector<double>> hl(S, std::vector<double>(nx, 0.0));
  unsigned long long* dh = nullptr;
  CU(H, cudaMalloc(&dh, nx * sizeof(unsigned long long)));
  Scratch sch;
  sch.p = dh;
  for (int s = 0; s < S; ++s) {
    CU(H, cudaMemsetAsync(dh, 0, nx * sizeof(unsigned long long), G->stream));
    if (n[s]) k_rec_layer_hist<<<blocks(n[s], 256), 256, 0, G->stream>>>(recs[s], (uint32_t)n[s], G->inv, x0, nx, dh);
    std::vector<unsigned long long> hh(nx);
    CU(H, cudaMemcpyAsync(hh.data(), dh, nx * sizeof(unsigned long long), cudaMemcpyDeviceToHost, G->stream));
    CU(H, cudaStreamSynchronize(G->stream));
    ++G->syncs;
    for (uint32_t k = 0; k < nx; ++k) hl[s][k] = (double)hh[k];
  }
  std::vector<double> hist;
  rc = dist_allreduce(H, G, hl, ncclSum, hist);
  if (rc) return rc;
  G->cuts = choose_cuts(hist, x0, G->world);
  // the message capacity: every rank computes the same value from the global histogram
  double mxl = 0.0;
  for (double v : hist) mxl = std::max(mxl, v);
  G->cap = (int64_t)(1.5 * mxl) + 4096;
  if (const char* e = std::getenv("BDM_DIST_CAP0")) G->cap = std::max<int64_t>(1, std::atoll(e));  // tests: force re-runs
  if ((rc = dist_redistribute(H, G, recs, n))) return rc;
  for (int s = 0; s < S; ++s)
    if ((rc = dist_load_slab(H, G, s, recs[s], n[s]))) return rc;
  // work-balanced cuts from each rank's own grid (its layers are complete now)
  if (G->world > 1 && G->n_global > 0) {
    std::vector<std::vector<double>> sq(S);
    for (int s = 0; s < S; ++s)
      if ((rc = dist_layer_sq(H, G, s, x0, nx, sq[s]))) return rc;
    std::vector<double> sqs;
    rc = dist_allreduce(H, G, sq, ncclSum, sqs);
    if (rc) return rc;
    double sum_sq = 0.0;
    for (double v : sqs) sum_sq += v;
    const double mean_sq = sum_sq / (double)G->n_global;
    std::vector<double> w(nx);
    for (uint32_t k = 0; k < nx; ++k) w[k] = hist[k] + (mean_sq > 0.0 ? sqs[k] / mean_sq : 0.0);
    const std::vector<int32_t> cuts2 = choose_cuts(w, x0, G->world);
    if (cuts2 != G->cuts) {  // owned agents back to records, redistributed by the work cuts
      G->cuts = cuts2;
      for (int s = 0; s < S; ++s) {
        DistSlab& D = G->sl[s];
        bdm_ctx* h = D.h;
        CU(H, cudaMalloc(&recs[s], std::max<int64_t>(D.live, 1) * REC * sizeof(double)));
        if (D.live)
          k_ag_to_rec<<<blocks(D.live, 256), 256, 0, G->stream>>>(h->ag[h->cur], h->id[h->cur], (uint32_t)D.live,
                                                                   recs[s]);
        CU(H, cudaGetLastError());
        n[s] = D.live;
      }
      if ((rc = dist_redistribute(H, G, recs, n))) return rc;
      for (int s = 0; s < S; ++s)
        if ((rc = dist_load_slab(H, G, s, recs[s], n[s]))) return rc;
    }
  }
  return BDM_OK;
}

}  // namespace

// ---------------------------------------------------------------------------------------- C ABI
namespace {

__global__ void k_local_out(const double4* __restrict__ ag, const double* __restrict__ dp,
                            const uint32_t* __restrict__ ids, uint32_t n, int64_t* __restrict__ out_ids,
                            double* __restrict__ out_vals) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (out_ids) out_ids[i] = (int64_t)ids[i];
  if (out_vals) {
    if (ag) {
      const double4 p = ag[i];
      out_vals[3 * (size_t)i] = p.x;
      out_vals[3 * (size_t)i + 1] = p.y;
      out_vals[3 * (size_t)i + 2] = p.z;
    } else {
      for (int a = 0; a < 3; ++a) out_vals[3 * (size_t)i + a] = dp[3 * (size_t)i + a];
    }
  }
}

// Validates and stages a batch of agents (counts[s] for local slot s, concatenated), then runs the
// set-up (box edge, extents, cuts, redistribution) over the group's communicator.
int dist_load(bdm_ctx* H, const std::vector<int64_t>& counts, const int64_t* ids, const double* pos,
              const double* diam) {
  DistGroup* G = H->dist;
  const bool dev = H->prm.flags & BDM_DEVICE_PTRS;
  const size_t S = G->sl.size();
  std::vector<double*> recs(S, nullptr);
  std::vector<int64_t> n(counts);
  struct Free {
    std::vector<double*>& r;
    ~Free() {
      for (double* q : r)
        if (q) cudaFree(q);
    }
  } free_recs{recs};
  ErrDev* err = nullptr;
  unsigned long long* mb = nullptr;
  if (cudaMalloc(&err, sizeof(ErrDev)) != cudaSuccess || cudaMalloc(&mb, sizeof(unsigned long long)) != cudaSuccess)
    return fail(H, BDM_ENOMEM, "distributed load: device allocation");
  Scratch sce, scm;
  sce.p = err;
  scm.p = mb;
  ErrDev e0{0u, 0xffffffffu, ERR_NONE};
  int64_t off = 0;
  for (size_t s = 0; s < S; ++s) {
    const int64_t m = n[s];
    CU(H, cudaMalloc(&recs[s], std::max<int64_t>(m, 1) * REC * sizeof(double)));
    if (m) {
      const double *dpos = pos + 3 * off, *ddiam = diam + off;
      const int64_t* dids = ids + off;
      Scratch stage;
      if (!dev) {  // host inputs: staged
        const size_t bytes = (size_t)m * (4 * sizeof(double) + sizeof(int64_t));
        CU(H, cudaMalloc(&stage.p, bytes));
        double* sp = static_cast<double*>(stage.p);
        CU(H, cudaMemcpyAsync(sp, dpos, 3 * m * sizeof(double), cudaMemcpyHostToDevice, G->stream));
        CU(H, cudaMemcpyAsync(sp + 3 * m, ddiam, m * sizeof(double), cudaMemcpyHostToDevice, G->stream));
        CU(H, cudaMemcpyAsync(sp + 4 * m, dids, m * sizeof(int64_t), cudaMemcpyHostToDevice, G->stream));
        dpos = sp;
        ddiam = sp + 3 * m;
        dids = reinterpret_cast<const int64_t*>(sp + 4 * m);
      }
      CU(H, cudaMemcpyAsync(err, &e0, sizeof e0, cudaMemcpyHostToDevice, G->stream));
      k_dist_pack_in<<<blocks(m, 256), 256, 0, G->stream>>>(dpos, ddiam, dids, (uint32_t)m, recs[s], mb, err);
      CU(H, cudaGetLastError());
      ErrDev he;
      CU(H, cudaMemcpyAsync(&he, err, sizeof he, cudaMemcpyDeviceToHost, G->stream));
      CU(H, cudaStreamSynchronize(G->stream));
      ++G->syncs;
      if (he.code)
        return fail(H, BDM_EINVAL, "distributed load: invalid agent %llu of rank %d (D > 0 and finite, finite "
                    "positions, 0 <= id < 2^32 - 1)", (unsigned long long)(he.bad >> 32), G->sl[s].rank);
    }
    off += m;
  }
  int rc = dist_setup(H, G, recs, n);
  if (rc) return rc;
  H->n = 0;
  for (auto& D : G->sl) H->n += D.live;
  H->have_grid = true;
  H->poisoned = false;
  return BDM_OK;
}

// Group handle shared by bdm_init_dist and bdm_init_dist_local: creates the communicator, then loads
// the first batch.
int dist_create(bdm_handle* out, int world, const std::vector<int>& ranks, const std::vector<int64_t>& counts,
                const int64_t* ids, const double* pos, const double* diam, const bdm_params* p, const void* uid,
                bool virt, int device, void* stream) {
  *out = nullptr;
  NcclApi* api = nccl_api();
  if (!api) return fail(nullptr, BDM_ENCCL, "NCCL unavailable: %s", "libnccl.so.2 could not be loaded");
  bdm_ctx* H = new (std::nothrow) bdm_ctx();
  if (!H) return fail(nullptr, BDM_ENOMEM, "bdm_init_dist: host allocation");
  H->prm = *p;
  H->device = device;
  H->stream = static_cast<cudaStream_t>(stream);
  DistGroup* G = new DistGroup();
  H->dist = G;
  G->api = api;
  G->virt = virt;
  G->world = world;
  G->device = device;
  G->stream = H->stream;
  auto bail = [&](int rc) {
    g_tls_error = H->error;
    bdm_destroy(H);
    return rc;
  };
  if (cudaSetDevice(device) != cudaSuccess) {
    (void)cudaGetLastError();
    return bail(fail(H, BDM_ECUDA, "bdm_init_dist: cudaSetDevice(%d) failed", device));
  }
  {
    ncclUniqueId id;
    if (virt) {
      ncclResult_t r = api->getUniqueId(&id);
      if (r != ncclSuccess) return bail(fail(H, BDM_ENCCL, "ncclGetUniqueId: %s", api->errStr(r)));
    } else {
      std::memcpy(&id, uid, sizeof id);
    }
    ncclResult_t r = api->commInitRank(&G->comm, virt ? 1 : world, id, virt ? 0 : ranks[0]);
    if (r != ncclSuccess) return bail(fail(H, BDM_ENCCL, "ncclCommInitRank(world %d): %s", world, api->errStr(r)));
  }
  for (int r : ranks) {
    DistSlab D;
    D.rank = r;
    G->sl.push_back(D);
  }
  int rc = dist_load(H, counts, ids, pos, diam);
  if (rc) return bail(rc);
  *out = H;
  return BDM_OK;
}

}  // namespace

extern "C" {

int bdm_nccl_unique_id(void* out128) {
  if (!out128) return fail(nullptr, BDM_EINVAL, "bdm_nccl_unique_id: NULL output");
  NcclApi* api = nccl_api();
  if (!api) return fail(nullptr, BDM_ENCCL, "NCCL unavailable: libnccl.so.2 could not be loaded");
  ncclUniqueId id;
  ncclResult_t r = api->getUniqueId(&id);
  if (r != ncclSuccess) return fail(nullptr, BDM_ENCCL, "ncclGetUniqueId: %s", api->errStr(r));
  std::memcpy(out128, &id, sizeof id);
  return BDM_OK;
}

int bdm_init_dist(bdm_handle* h, int64_t n_local, const int64_t* ids, const double* pos, const double* diam,
                  const bdm_params* p, int rank, int world, const void* nccl_uid, int device, void* cuda_stream) {
  if (!h) return fail(nullptr, BDM_EINVAL, "bdm_init_dist: handle pointer is NULL");
  *h = nullptr;
  if (!params_ok(p)) return fail(nullptr, BDM_EINVAL, "bdm_init_dist: invalid params");
  if (world < 1 || rank < 0 || rank >= world || !nccl_uid || device < 0)
    return fail(nullptr, BDM_EINVAL, "bdm_init_dist: need 0 <= rank < world, a unique id and a device");
  if (n_local < 0 || n_local >= (int64_t)0xffffffffll || (n_local > 0 && (!ids || !pos || !diam)))
    return fail(nullptr, BDM_EINVAL, "bdm_init_dist: need 0 <= n_local < 2^32 - 1 and non-NULL arrays");
  return dist_create(h, world, {rank}, {n_local}, ids, pos, diam, p, nccl_uid, false, device, cuda_stream);
}

int bdm_init_dist_local(bdm_handle* h, int world, const int64_t* counts, const int64_t* ids, const double* pos,
                        const double* diam, const bdm_params* p, void* cuda_stream) {
  if (!h) return fail(nullptr, BDM_EINVAL, "bdm_init_dist_local: handle pointer is NULL");
  *h = nullptr;
  if (!params_ok(p)) return fail(nullptr, BDM_EINVAL, "bdm_init_dist_local: invalid params");
  if (world < 1 || world > 1024 || !counts) return fail(nullptr, BDM_EINVAL, "bdm_init_dist_local: 1 <= world <= 1024");
  std::vector<int> ranks;
  std::vector<int64_t> cnt;
  int64_t tot = 0;
  for (int r = 0; r < world; ++r) {
    if (counts[r] < 0) return fail(nullptr, BDM_EINVAL, "bdm_init_dist_local: negative count");
    ranks.push_back(r);
    cnt.push_back(counts[r]);
    tot += counts[r];
  }
  if (tot >= (int64_t)0xffffffffll || (tot > 0 && (!ids || !pos || !diam)))
    return fail(nullptr, BDM_EINVAL, "bdm_init_dist_local: need < 2^32 - 1 agents and non-NULL arrays");
  int dev = p->device;
  if (dev < 0 && cudaGetDevice(&dev) != cudaSuccess) {
    (void)cudaGetLastError();
    return fail(nullptr, BDM_ECUDA, "bdm_init_dist_local: no CUDA device");
  }
  return dist_create(h, world, ranks, cnt, ids, pos, diam, p, nullptr, true, dev, cuda_stream);
}

int bdm_set_agents_dist(bdm_handle h, int64_t n_local, const int64_t* ids, const double* pos, const double* diam) {
  if (!h || !h->dist) return fail(h, BDM_EINVAL, "bdm_set_agents_dist: needs a distributed handle");
  if (h->dist->sl.size() != 1) return fail(h, BDM_EINVAL, "bdm_set_agents_dist: one local rank per handle");
  if (n_local < 0 || n_local >= (int64_t)0xffffffffll || (n_local > 0 && (!ids || !pos || !diam)))
    return fail(h, BDM_EINVAL, "bdm_set_agents_dist: need 0 <= n_local < 2^32 - 1 and non-NULL arrays");
  CU(h, cudaSetDevice(h->dist->device));
  return dist_load(h, {n_local}, ids, pos, diam);
}

int bdm_get_local(bdm_handle h, int what, int64_t* n, int64_t* ids, double* vals) {
  if (!h || !n || (what != BDM_OWNED_POSITIONS && what != BDM_LAST_DISPLACEMENTS))
    return fail(h, BDM_EINVAL, "bdm_get_local: bad arguments");
  if (!h->dist) return fail(h, BDM_ESTATE, "bdm_get_local: not a distributed handle (bdm_init_dist)");
  DistGroup* G = h->dist;
  CU(h, cudaSetDevice(G->device));
  int64_t tot = 0;
  for (auto& D : G->sl) tot += D.live;
  *n = tot;
  if (what == BDM_LAST_DISPLACEMENTS)
    for (auto& D : G->sl)
      if (!D.h->have_dp) return fail(h, BDM_ESTATE, "bdm_get_local: no step has been run");
  if (tot == 0 || (!ids && !vals)) return BDM_OK;
  const bool dev = h->prm.flags & BDM_DEVICE_PTRS;
  Scratch sc;
  int64_t* oi = ids;
  double* ov = vals;
  if (!dev) {
    CU(h, cudaMalloc(&sc.p, tot * (sizeof(int64_t) + 3 * sizeof(double))));
    oi = ids ? static_cast<int64_t*>(sc.p) : nullptr;
    ov = vals ? reinterpret_cast<double*>(static_cast<int64_t*>(sc.p) + tot) : nullptr;
  }
  int64_t o = 0;
  for (auto& D : G->sl) {
    bdm_ctx* s = D.h;
    if (D.live)
      k_local_out<<<blocks(D.live, 256), 256, 0, G->stream>>>(
          what == BDM_OWNED_POSITIONS ? s->ag[s->cur] : nullptr, s->dp,
          what == BDM_OWNED_POSITIONS ? s->id[s->cur] : s->dp_ids, (uint32_t)D.live, oi ? oi + o : nullptr,
          ov ? ov + 3 * o : nullptr);
    o += D.live;
  }
  CU(h, cudaGetLastError());
  if (!dev) {
    if (ids) CU(h, cudaMemcpyAsync(ids, oi, tot * sizeof(int64_t), cudaMemcpyDeviceToHost, G->stream));
    if (vals) CU(h, cudaMemcpyAsync(vals, ov, 3 * tot * sizeof(double), cudaMemcpyDeviceToHost, G->stream));
  }
  CU(h, cudaStreamSynchronize(G->stream));
  ++G->syncs;
  return BDM_OK;
}

int bdm_get_cuts(bdm_handle h, int32_t* out, int32_t cap) {
  if (!h || !out || !h->dist) return fail(h, BDM_EINVAL, "bdm_get_cuts: needs a distributed handle and an output");
  const DistGroup* G = h->dist;
  if (cap < (int32_t)G->cuts.size()) return fail(h, BDM_ETRUNC, "bdm_get_cuts: need %d entries", (int)G->cuts.size());
  for (size_t k = 0; k < G->cuts.size(); ++k) out[k] = G->cuts[k];
  return BDM_OK;
}

int bdm_get_pair_digest(bdm_handle h, int kind, uint32_t* count, uint64_t* hash) {
  if (!h || (kind != BDM_NEIGHBOR && kind != BDM_CONTACT) || (h->n > 0 && (!count || !hash)))
    return fail(h, BDM_EINVAL, "bdm_get_pair_digest: bad arguments");
  if (h->dist || h->slab) return fail(h, BDM_ESTATE, "bdm_get_pair_digest: single handles only");
  if (h->n == 0) return BDM_OK;
  CU(h, cudaSetDevice(h->device));
  if (h->state != State::Fresh) {
    int rc = grid_build(h);
    if (rc) return rc;
  }
  const uint32_t n = (uint32_t)h->n;
  const bool dev = h->prm.flags & BDM_DEVICE_PTRS;
  Scratch sc;
  uint32_t* c = count;
  unsigned long long* hs = reinterpret_cast<unsigned long long*>(hash);
  if (!dev) {
    CU(h, cudaMalloc(&sc.p, (size_t)n * (sizeof(uint32_t) + sizeof(unsigned long long))));
    hs = static_cast<unsigned long long*>(sc.p);
    c = reinterpret_cast<uint32_t*>(hs + n);
  }
  k_pair_digest<<<blocks(n, 128), 128, 0, h->stream>>>(h->ag[h->cur], h->id[h->cur], n, h->grid, kind, c, hs);
  CU(h, cudaGetLastError());
  h->launches += 1;
  if (!dev) {
    CU(h, cudaMemcpyAsync(count, c, (size_t)n * sizeof(uint32_t), cudaMemcpyDeviceToHost, h->stream));
    CU(h, cudaMemcpyAsync(hash, hs, (size_t)n * sizeof(uint64_t), cudaMemcpyDeviceToHost, h->stream));
  }
  return check_async(h);
}

int bdm_get_stats(bdm_handle h, bdm_stats* out) {
  if (!h || !out) return fail(h, BDM_EINVAL, "bdm_get_stats: NULL argument");
  std::memset(out, 0, sizeof *out);
  if (h->dist) {
    const DistGroup* G = h->dist;
    out->n_agents = 0;
    for (auto& D : G->sl) {
      out->n_agents += D.live;
      out->launches += D.h ? D.h->launches_total + D.h->launches : 0;
    }
    out->steps = G->steps;
    out->host_syncs = G->syncs;
    out->half_path = G->steps ? 1 : -1;
    out->migrated = G->migrated;
    out->ghosts = G->ghosts;
    out->exchange_bytes = G->bytes;
    out->chunks = G->chunks;
    out->redo_chunks = G->redo;
    out->world = G->world;
    out->local_ranks = (int64_t)G->sl.size();
    return BDM_OK;
  }
  out->n_agents = h->n;
  out->steps = (int64_t)h->steps_total;
  out->launches = h->launches_total + h->launches;
  out->host_syncs = h->host_syncs;
  out->half_path = h->steps_total ? (h->last_half ? (h->ring_band ? 2 : 1) : 0) : -1;
  out->world = 1;
  out->local_ranks = 1;
  return BDM_OK;
}

}  // extern "C"
