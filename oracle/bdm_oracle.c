/*
 * bdm_oracle.c -- plain, slow CPU oracle for one BioDynaMo mechanical-interaction step.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or constant generator with the CUDA path in paper_2006_06775_b200/.
 *
 * It follows, step by step, the reading recorded in DESIGN.md §3:
 *
 *   O1  box edge   L = max(max_i D_i, box_edge_min); L2 = L*L; inv = 1/(L*(1+2^-30))
 *                  PAPER.md:321-322 (§2.1 "box size is chosen based on the largest agent")
 *   O2  boxes      b_i = (floor(x_i*inv), floor(y_i*inv), floor(z_i*inv))
 *                  PAPER.md:315-317 (§2.1 "assigns agents to boxes based on the center of mass")
 *   O3  neighbours j != i in the 27 boxes b_i + {-1,0,1}^3 with d2 <= L2,
 *                  d2 = (dx*dx + dy*dy) + dz*dz, dx = x_i - x_j
 *                  PAPER.md:318-320 (§2.1 "iterating over the assigned box and all its
 *                  surrounding boxes (27 boxes in total)")
 *   O4  pair force d = sqrt(d2); r_i = 0.5*D_i; s = r_i + r_j; delta = s - d; contact iff delta > 0;
 *                  r = (r_i*r_j)/s; f = k*delta - gamma*sqrt(r*delta); m = f/d; F_ij = m*(dx,dy,dz)
 *                  (BASELINE.json north_star: "overlap delta=r1+r2-d gives a repulsion term minus
 *                  a sqrt(r*delta) attraction term"; PAPER.md:109, 724-725 defer to Zubler-Douglas)
 *                  d2 == 0 exactly: delta = s, force +f*x_hat on the higher id (R8)
 *   O5  sum        F_i = sum of F_ij over contacts, boxes in (dx,dy,dz) lexicographic order from
 *                  (-1,-1,-1), within a box by ascending id (R13/R14)
 *   O6  displacement |F| = sqrt((Fx*Fx + Fy*Fy) + Fz*Fz); |F| <= adherence -> 0;
 *                  c = dt/eta; |F|*c > max_disp -> F*(max_disp/|F|); else F*c
 *                  (north_star "displacement rule with its adherence threshold and
 *                  max-displacement clamp"; "Delta p = F/eta*Delta t, clamps")
 *   O7  update     p_i' = p_i + Delta p_i after all forces (Jacobi)
 *
 * Every +, -, * is a separately rounded IEEE binary64 operation: build with
 * -ffp-contract=off (no FMA).  sqrt and / are correctly rounded (libm sqrt).
 *
 * Implementation is deliberately plain: agents are sorted by (box key, id) with qsort and each
 * of the 27 boxes is found by binary search.  No blocking, no fusion.  Optional OpenMP over
 * agents (each agent's sum is independent and computed in the same order).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_OK 0
#define ORC_EINVAL (-1)
#define ORC_ENOMEM (-3)
#define ORC_ENONFINITE (-6)
#define ORC_ERANGE (-7)
#define ORC_ETRUNC (-8)

typedef struct {
  double k_rep, gamma_att, adherence, dt, eta, max_disp, box_edge_min;
} orc_params;

typedef struct {
  double L, L2, inv;
  int64_t lo[3], hi[3];
} orc_grid;

/* per-agent record; any pointer may be NULL */
typedef struct {
  int32_t* n_cand;   /* candidates visited in the 27 boxes (self excluded) */
  int32_t* n_nb;     /* |{j : d2 <= L2}| */
  int32_t* n_ct;     /* |{j : delta > 0}| */
  double* s_abs;     /* sum |f_ij| over contacts */
  int8_t* branch;    /* 0 = below adherence, 1 = clamped, 2 = free */
  uint64_t* nb_hash; /* sum mix64(j) over neighbours (mod 2^64) */
  uint64_t* ct_hash; /* sum mix64(j) over contacts   (mod 2^64) */
  double* force;     /* 3n summed force F_i */
} orc_record;

int orc_version(void) { return 1; }

void orc_params_default(orc_params* p) {
  p->k_rep = 10.0;       /* SPEC.md:248 k=10 */
  p->gamma_att = 4.0;    /* SPEC.md:248 k_adh = 0.4 k, re-read as gamma (R3) */
  p->adherence = 0.1;    /* DESIGN.md R4 */
  p->dt = 1.0;
  p->eta = 1.0;
  p->max_disp = 3.0;
  p->box_edge_min = 0.0;
}

uint64_t orc_mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

/* O1 + the box extents used by O2's key. */
int orc_grid_params(int64_t n, const double* pos, const double* diam, double box_edge_min, orc_grid* g) {
  double maxd = 0.0;
  for (int64_t i = 0; i < n; ++i)
    if (diam[i] > maxd) maxd = diam[i];
  double L = maxd > box_edge_min ? maxd : box_edge_min;
  g->L = L;
  g->L2 = L * L;
  g->inv = 1.0 / (L * (1.0 + 0x1p-30));
  for (int a = 0; a < 3; ++a) {
    g->lo[a] = 0;
    g->hi[a] = 0;
  }
  for (int64_t i = 0; i < n; ++i) {
    for (int a = 0; a < 3; ++a) {
      double q = pos[3 * i + a] * g->inv;
      if (!(fabs(q) < 1048576.0)) return ORC_ERANGE; /* |p*inv| < 2^20 keeps the 2^-30 margin valid */
      int64_t b = (int64_t)floor(q);
      if (i == 0 || b < g->lo[a]) g->lo[a] = b;
      if (i == 0 || b > g->hi[a]) g->hi[a] = b;
    }
  }
  return ORC_OK;
}

void orc_box_coords(int64_t n, const double* pos, const orc_grid* g, int64_t* b) {
  for (int64_t i = 0; i < 3 * n; ++i) b[i] = (int64_t)floor(pos[i] * g->inv);
}

/* ---- the grid: agents sorted by (key, id) ---- */
typedef struct {
  uint64_t key;
  int64_t id;
} orc_entry;

static int cmp_entry(const void* a, const void* b) {
  const orc_entry* x = (const orc_entry*)a;
  const orc_entry* y = (const orc_entry*)b;
  if (x->key != y->key) return x->key < y->key ? -1 : 1;
  if (x->id != y->id) return x->id < y->id ? -1 : 1;
  return 0;
}

typedef struct {
  orc_grid g;
  int64_t n;
  int64_t ny, nz;
  int64_t* b;        /* 3n box coordinates */
  orc_entry* sorted; /* n entries sorted by (key, id) */
} orc_index;

static uint64_t key_of(const orc_index* ix, int64_t bx, int64_t by, int64_t bz) {
  return (uint64_t)(((bx - ix->g.lo[0]) * ix->ny + (by - ix->g.lo[1])) * ix->nz + (bz - ix->g.lo[2]));
}

static void free_index(orc_index* ix) {
  free(ix->b);
  free(ix->sorted);
}

static int build_index(orc_index* ix, int64_t n, const double* pos, const double* diam, double box_edge_min) {
  memset(ix, 0, sizeof(*ix));
  ix->n = n;
  int rc = orc_grid_params(n, pos, diam, box_edge_min, &ix->g);
  if (rc) return rc;
  ix->ny = ix->g.hi[1] - ix->g.lo[1] + 1;
  ix->nz = ix->g.hi[2] - ix->g.lo[2] + 1;
  ix->b = (int64_t*)malloc(sizeof(int64_t) * 3 * (n > 0 ? n : 1));
  ix->sorted = (orc_entry*)malloc(sizeof(orc_entry) * (n > 0 ? n : 1));
  if (!ix->b || !ix->sorted) {
    free_index(ix);
    return ORC_ENOMEM;
  }
  orc_box_coords(n, pos, &ix->g, ix->b);
  for (int64_t i = 0; i < n; ++i) {
    ix->sorted[i].key = key_of(ix, ix->b[3 * i], ix->b[3 * i + 1], ix->b[3 * i + 2]);
    ix->sorted[i].id = i;
  }
  qsort(ix->sorted, (size_t)n, sizeof(orc_entry), cmp_entry);
  return ORC_OK;
}

/* first position in sorted[] whose key >= k */
static int64_t lower_bound(const orc_index* ix, uint64_t k) {
  int64_t lo = 0, hi = ix->n;
  while (lo < hi) {
    int64_t mid = lo + (hi - lo) / 2;
    if (ix->sorted[mid].key < k)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

/* O4 for one pair (i, j) with d2 already known to be a neighbour.  Returns 1 on contact and
 * writes the force on i into t[3] and f into *fout. */
static int pair_force(const double* pi, const double* pj, double Di, double Dj, int64_t idi, int64_t idj,
                      double dx, double dy, double dz, double d2, const orc_params* p, double* t, double* fout) {
  double d = sqrt(d2);
  double ri = 0.5 * Di;
  double rj = 0.5 * Dj;
  double s = ri + rj;
  double delta = s - d;
  (void)pi;
  (void)pj;
  if (!(delta > 0.0)) return 0;
  double r = (ri * rj) / s;
  double f = p->k_rep * delta - p->gamma_att * sqrt(r * delta);
  *fout = f;
  if (d2 == 0.0) { /* coincident centres, R8 */
    double sign = idi > idj ? 1.0 : -1.0;
    t[0] = sign * f;
    t[1] = 0.0;
    t[2] = 0.0;
    return 1;
  }
  double m = f / d;
  t[0] = m * dx;
  t[1] = m * dy;
  t[2] = m * dz;
  return 1;
}

/* O6 */
static int displacement(const double F[3], const orc_params* p, double dp[3]) {
  double fn = sqrt((F[0] * F[0] + F[1] * F[1]) + F[2] * F[2]);
  if (fn <= p->adherence) {
    dp[0] = 0.0;
    dp[1] = 0.0;
    dp[2] = 0.0;
    return 0;
  }
  double c = p->dt / p->eta;
  if (fn * c > p->max_disp) {
    double scale = p->max_disp / fn;
    dp[0] = F[0] * scale;
    dp[1] = F[1] * scale;
    dp[2] = F[2] * scale;
    return 1;
  }
  dp[0] = F[0] * c;
  dp[1] = F[1] * c;
  dp[2] = F[2] * c;
  return 2;
}

/* O3-O6 for agent i using the index. */
static int agent_update(const orc_index* ix, int64_t i, const double* pos, const double* diam, const orc_params* p,
                        double* dp_out, const orc_record* rec) {
  const double* pi = pos + 3 * i;
  double F[3] = {0.0, 0.0, 0.0};
  int32_t n_cand = 0, n_nb = 0, n_ct = 0;
  double s_abs = 0.0;
  uint64_t nb_hash = 0, ct_hash = 0;
  for (int ddx = -1; ddx <= 1; ++ddx)
    for (int ddy = -1; ddy <= 1; ++ddy)
      for (int ddz = -1; ddz <= 1; ++ddz) {
        int64_t cx = ix->b[3 * i] + ddx, cy = ix->b[3 * i + 1] + ddy, cz = ix->b[3 * i + 2] + ddz;
        if (cx < ix->g.lo[0] || cx > ix->g.hi[0] || cy < ix->g.lo[1] || cy > ix->g.hi[1] || cz < ix->g.lo[2] ||
            cz > ix->g.hi[2])
          continue;
        uint64_t k = key_of(ix, cx, cy, cz);
        for (int64_t q = lower_bound(ix, k); q < ix->n && ix->sorted[q].key == k; ++q) {
          int64_t j = ix->sorted[q].id;
          if (j == i) continue;
          ++n_cand;
          const double* pj = pos + 3 * j;
          double dx = pi[0] - pj[0];
          double dy = pi[1] - pj[1];
          double dz = pi[2] - pj[2];
          double d2 = (dx * dx + dy * dy) + dz * dz;
          if (!(d2 <= ix->g.L2)) continue;
          ++n_nb;
          nb_hash += orc_mix64((uint64_t)j);
          double t[3], f;
          if (pair_force(pi, pj, diam[i], diam[j], i, j, dx, dy, dz, d2, p, t, &f)) {
            ++n_ct;
            ct_hash += orc_mix64((uint64_t)j);
            s_abs += fabs(f);
            F[0] = F[0] + t[0];
            F[1] = F[1] + t[1];
            F[2] = F[2] + t[2];
          }
        }
      }
  int br = displacement(F, p, dp_out);
  if (rec) {
    if (rec->n_cand) rec->n_cand[i] = n_cand;
    if (rec->n_nb) rec->n_nb[i] = n_nb;
    if (rec->n_ct) rec->n_ct[i] = n_ct;
    if (rec->s_abs) rec->s_abs[i] = s_abs;
    if (rec->branch) rec->branch[i] = (int8_t)br;
    if (rec->nb_hash) rec->nb_hash[i] = nb_hash;
    if (rec->ct_hash) rec->ct_hash[i] = ct_hash;
    if (rec->force) {
      rec->force[3 * i] = F[0];
      rec->force[3 * i + 1] = F[1];
      rec->force[3 * i + 2] = F[2];
    }
  }
  if (!isfinite(F[0]) || !isfinite(F[1]) || !isfinite(F[2])) return ORC_ENONFINITE;
  return ORC_OK;
}

static int check_inputs(int64_t n, const double* pos, const double* diam, const orc_params* p) {
  if (n < 0 || (n > 0 && (!pos || !diam)) || !p) return ORC_EINVAL;
  if (!(p->eta > 0.0) || !(p->max_disp > 0.0) || !isfinite(p->eta) || !isfinite(p->max_disp)) return ORC_EINVAL;
  if (!(p->k_rep >= 0.0) || !(p->gamma_att >= 0.0) || !(p->adherence >= 0.0) || !(p->dt >= 0.0) ||
      !(p->box_edge_min >= 0.0) || !isfinite(p->k_rep) || !isfinite(p->gamma_att) || !isfinite(p->adherence) ||
      !isfinite(p->dt) || !isfinite(p->box_edge_min))
    return ORC_EINVAL;
  for (int64_t i = 0; i < n; ++i) {
    if (!(diam[i] > 0.0) || !isfinite(diam[i])) return ORC_EINVAL;
    for (int a = 0; a < 3; ++a)
      if (!isfinite(pos[3 * i + a])) return ORC_EINVAL;
  }
  return ORC_OK;
}

/*
 * One step (O1-O7) for the agents listed in sample[0..n_sample) (all agents if sample == NULL).
 * dp: 3*n_out displacements (n_out = n_sample or n); pos_new: 3*n_out or NULL;
 * rec arrays are indexed by agent id (length n).  nthreads <= 0: OpenMP default.
 */
int orc_step_sample(int64_t n, const double* pos, const double* diam, const orc_params* p, int64_t n_sample,
                    const int64_t* sample, double* dp, double* pos_new, const orc_record* rec, int nthreads) {
  int rc = check_inputs(n, pos, diam, p);
  if (rc) return rc;
  if (n == 0) return ORC_OK;
  orc_index ix;
  rc = build_index(&ix, n, pos, diam, p->box_edge_min);
  if (rc) return rc;
  int64_t m = sample ? n_sample : n;
  int bad = 0;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1024) reduction(| : bad)
#endif
  for (int64_t q = 0; q < m; ++q) {
    int64_t i = sample ? sample[q] : q;
    if (i < 0 || i >= n) {
      bad |= 1;
      continue;
    }
    if (agent_update(&ix, i, pos, diam, p, dp + 3 * q, rec)) bad |= 2;
    if (pos_new)
      for (int a = 0; a < 3; ++a) pos_new[3 * q + a] = pos[3 * i + a] + dp[3 * q + a];
  }
  (void)nthreads;
  free_index(&ix);
  if (bad & 1) return ORC_EINVAL;
  if (bad & 2) return ORC_ENONFINITE;
  return ORC_OK;
}

int orc_step(int64_t n, const double* pos, const double* diam, const orc_params* p, double* dp, double* pos_new,
             const orc_record* rec, int nthreads) {
  return orc_step_sample(n, pos, diam, p, n, NULL, dp, pos_new, rec, nthreads);
}

/* O8: n_steps repetitions of O1-O7 in place on pos; dp receives the last step's displacement. */
int orc_run(int64_t n, double* pos, const double* diam, const orc_params* p, int32_t n_steps, double* dp,
            int nthreads) {
  if (n_steps < 0) return ORC_EINVAL;
  double* tmp = (double*)malloc(sizeof(double) * 3 * (n > 0 ? n : 1));
  if (!tmp) return ORC_ENOMEM;
  for (int32_t s = 0; s < n_steps; ++s) {
    int rc = orc_step(n, pos, diam, p, dp, tmp, NULL, nthreads);
    if (rc) {
      free(tmp);
      return rc;
    }
    memcpy(pos, tmp, sizeof(double) * 3 * n);
  }
  free(tmp);
  return ORC_OK;
}

/*
 * Unordered pair sets.  kind 0 = neighbour set N (d2 <= L2), kind 1 = contact set C (delta > 0).
 * Writes (min id, max id) pairs, sorted lexicographically, into out[2*cap]; returns the number of
 * pairs (>= 0) or an error code.  If the count exceeds cap, nothing beyond cap is written and the
 * caller learns the size from the return value.
 */
static int cmp_pair(const void* a, const void* b) {
  const int64_t* x = (const int64_t*)a;
  const int64_t* y = (const int64_t*)b;
  if (x[0] != y[0]) return x[0] < y[0] ? -1 : 1;
  if (x[1] != y[1]) return x[1] < y[1] ? -1 : 1;
  return 0;
}

int64_t orc_pairs(int64_t n, const double* pos, const double* diam, const orc_params* p, int kind, int64_t* out,
                  int64_t cap) {
  int rc = check_inputs(n, pos, diam, p);
  if (rc) return rc;
  if (n == 0) return 0;
  orc_index ix;
  rc = build_index(&ix, n, pos, diam, p->box_edge_min);
  if (rc) return rc;
  int64_t cnt = 0;
  for (int64_t i = 0; i < n; ++i) {
    const double* pi = pos + 3 * i;
    for (int ddx = -1; ddx <= 1; ++ddx)
      for (int ddy = -1; ddy <= 1; ++ddy)
        for (int ddz = -1; ddz <= 1; ++ddz) {
          int64_t cx = ix.b[3 * i] + ddx, cy = ix.b[3 * i + 1] + ddy, cz = ix.b[3 * i + 2] + ddz;
          if (cx < ix.g.lo[0] || cx > ix.g.hi[0] || cy < ix.g.lo[1] || cy > ix.g.hi[1] || cz < ix.g.lo[2] ||
              cz > ix.g.hi[2])
            continue;
          uint64_t k = key_of(&ix, cx, cy, cz);
          for (int64_t q = lower_bound(&ix, k); q < n && ix.sorted[q].key == k; ++q) {
            int64_t j = ix.sorted[q].id;
            if (j <= i) continue; /* each unordered pair once */
            const double* pj = pos + 3 * j;
            double dx = pi[0] - pj[0];
            double dy = pi[1] - pj[1];
            double dz = pi[2] - pj[2];
            double d2 = (dx * dx + dy * dy) + dz * dz;
            if (!(d2 <= ix.g.L2)) continue;
            if (kind == 1) {
              double t[3], f;
              if (!pair_force(pi, pj, diam[i], diam[j], i, j, dx, dy, dz, d2, p, t, &f)) continue;
            }
            if (cnt < cap) {
              out[2 * cnt] = i;
              out[2 * cnt + 1] = j;
            }
            ++cnt;
          }
        }
  }
  free_index(&ix);
  if (cnt <= cap) qsort(out, (size_t)cnt, 2 * sizeof(int64_t), cmp_pair);
  return cnt;
}

/* Force on agent i from agent j alone (O4), for closed-form pins.  Returns 1 on contact. */
int orc_pair_force(const double* pi, const double* pj, double Di, double Dj, int64_t idi, int64_t idj,
                   const orc_params* p, double* t) {
  double dx = pi[0] - pj[0];
  double dy = pi[1] - pj[1];
  double dz = pi[2] - pj[2];
  double d2 = (dx * dx + dy * dy) + dz * dz;
  double f;
  t[0] = t[1] = t[2] = 0.0;
  return pair_force(pi, pj, Di, Dj, idi, idj, dx, dy, dz, d2, p, t, &f);
}

/* O6 alone, for pins.  Returns the branch (0 adherence, 1 clamp, 2 free). */
int orc_displacement(const double* F, const orc_params* p, double* dp) { return displacement(F, p, dp); }

int orc_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ------------------------------------------------------------------------------------------------
 * NEXT-2: cell growth and division (readings G1-G3).  PAPER.md:711-712, 772 (the
 * "cell growth and division" GPU benchmark); SPEC.md:82-91 (CellDivision: volume-conserving split,
 * daughter displaced so the two spheres touch), SPEC.md:101 (2^n doubling oracle).
 *   G1 growth   D <- D + growth                                   (diameter rate, um per step)
 *   G2 division if D >= div_diam: D' = D * c, c = 2^(-1/3) (binary64 nearest), h = 0.5 * D',
 *               u = v/|v|, v_a = 2 * U(seed, step, id, a) - 1 (counter hash, a = 0..2; v = 0 -> x_hat),
 *               mother p - h*u (same id), daughter p + h*u with id N + (rank of the mother among this
 *               step's dividers in ascending id order)
 *   G3 order    a growth step runs after the mechanics of the same step (new agents are visible from
 *               the next step on)
 * ---------------------------------------------------------------------------------------------- */
typedef struct {
  double growth;   /* diameter increase per step, um */
  double div_diam; /* division threshold on the grown diameter, um */
  uint64_t seed;
} orc_growth;

static const double ORC_CBRT_HALF = 0.79370052598409973737585281963615; /* 2^(-1/3) */

static double orc_u01(uint64_t seed, uint64_t step, uint64_t id, uint64_t a) {
  uint64_t h = orc_mix64(seed * 0x9E3779B97F4A7C15ULL + ((step << 32) + id) * 4ULL + a);
  return (double)(h >> 11) * 0x1p-53;
}

/* One growth + division pass in id order.  pos (3*cap), diam (cap) are updated in place; returns the
 * new agent count, or ORC_ERANGE when cap is too small. */
int64_t orc_grow_divide(int64_t n, double* pos, double* diam, const orc_growth* gp, int64_t step, int64_t cap) {
  int64_t nd = 0;
  for (int64_t i = 0; i < n; ++i) {
    diam[i] = diam[i] + gp->growth;
    if (diam[i] >= gp->div_diam) ++nd;
  }
  if (n + nd > cap) return ORC_ERANGE;
  int64_t k = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (!(diam[i] >= gp->div_diam)) continue;
    double v[3], u[3];
    for (int a = 0; a < 3; ++a) v[a] = 2.0 * orc_u01(gp->seed, (uint64_t)step, (uint64_t)i, (uint64_t)a) - 1.0;
    double norm = sqrt((v[0] * v[0] + v[1] * v[1]) + v[2] * v[2]);
    if (norm == 0.0) {
      u[0] = 1.0;
      u[1] = 0.0;
      u[2] = 0.0;
    } else {
      for (int a = 0; a < 3; ++a) u[a] = v[a] / norm;
    }
    double Dd = diam[i] * ORC_CBRT_HALF;
    double h = 0.5 * Dd;
    int64_t d = n + k;
    for (int a = 0; a < 3; ++a) {
      double p = pos[3 * i + a];
      double off = h * u[a];
      pos[3 * i + a] = p - off;
      pos[3 * d + a] = p + off;
    }
    diam[i] = Dd;
    diam[d] = Dd;
    ++k;
  }
  return n + nd;
}

/* n_steps of (mechanics O1-O7, then growth + division); returns the final count (<0: error).
 * dp (3*cap) receives the mechanics displacement of the last step for the agents of that step. */
int64_t orc_run_growth(int64_t n, double* pos, double* diam, const orc_params* p, const orc_growth* gp,
                       int32_t n_steps, int64_t step0, int64_t cap, double* dp, int nthreads) {
  double* tmp = (double*)malloc(sizeof(double) * 3 * (cap > 0 ? cap : 1));
  if (!tmp) return ORC_ENOMEM;
  for (int32_t s = 0; s < n_steps; ++s) {
    int rc = orc_step(n, pos, diam, p, dp, tmp, NULL, nthreads);
    if (rc) {
      free(tmp);
      return rc;
    }
    memcpy(pos, tmp, sizeof(double) * 3 * n);
    n = orc_grow_divide(n, pos, diam, gp, step0 + s, cap);
    if (n < 0) break;
  }
  free(tmp);
  return n;
}

/* ------------------------------------------------------------------------------------------------
 * NEXT-3: soma clustering (readings S1-S5).  PAPER.md:711-712, 773 (the "soma
 * clustering" GPU benchmark: two cell types, each secreting its own substance and moving up its
 * gradient); SPEC.md:260-329 (diffusion-field: explicit Euler, 7-point stencil, closed boundary,
 * trilinear sampling, central-difference gradients), SPEC.md:477 (soma_clustering benchmark).
 *   S1 secretion  every agent of type t adds `secretion` to the node nearest to it in field t:
 *                 node_a = clamp(floor((p_a - origin_a) * (1/h) + 0.5), 0, dims_a - 1);
 *                 c[node] += count(node) * secretion  (one multiply per node)
 *   S2 diffusion  c' = c + dt * (D * lap - mu * c), lap = (((xm + xp) + (ym + yp)) + (zm + zp) - 6c) * (1/h^2),
 *                 closed boundary: a missing neighbour is the node itself; both fields; a negative c' is
 *                 clamped to 0 ("Concentrations remain >= 0 (clamped)")
 *   S3 chemotaxis g = grad c_t(p): central differences (g_a = (c[+1] - c[-1]) * (0.5/h), one-sided
 *                 (c[+1]-c[0])/h or (c[0]-c[-1])/h on the boundary layers) at the 8 nodes of the cell
 *                 containing p, trilinearly interpolated (weights clamped to the lattice);
 *                 p <- p + speed * g / |g| (no move if |g| == 0)
 *   S4 mechanics  O1-O7 on the moved agents
 * ---------------------------------------------------------------------------------------------- */
typedef struct {
  double h, origin[3];
  int32_t dims[3];
  double diff, decay, dt, secretion, speed;
} orc_fields;

static int64_t fidx(const orc_fields* f, int64_t x, int64_t y, int64_t z) {
  return (x * f->dims[1] + y) * f->dims[2] + z;
}

static int64_t clampi(int64_t v, int64_t lo, int64_t hi) { return v < lo ? lo : (v > hi ? hi : v); }

void orc_secrete(int64_t n, const double* pos, const int8_t* type, const orc_fields* f, double* c0, double* c1) {
  int64_t nn = (int64_t)f->dims[0] * f->dims[1] * f->dims[2];
  uint32_t* cnt = (uint32_t*)calloc((size_t)(2 * nn), sizeof(uint32_t));
  double invh = 1.0 / f->h;
  for (int64_t i = 0; i < n; ++i) {
    int64_t b[3];
    for (int a = 0; a < 3; ++a)
      b[a] = clampi((int64_t)floor((pos[3 * i + a] - f->origin[a]) * invh + 0.5), 0, f->dims[a] - 1);
    cnt[(type[i] ? nn : 0) + fidx(f, b[0], b[1], b[2])] += 1;
  }
  for (int64_t k = 0; k < nn; ++k) {
    if (cnt[k]) c0[k] = c0[k] + (double)cnt[k] * f->secretion;
    if (cnt[nn + k]) c1[k] = c1[k] + (double)cnt[nn + k] * f->secretion;
  }
  free(cnt);
}

void orc_diffuse(const orc_fields* f, const double* c, double* out) {
  double ih2 = 1.0 / (f->h * f->h);
  for (int64_t x = 0; x < f->dims[0]; ++x)
    for (int64_t y = 0; y < f->dims[1]; ++y)
      for (int64_t z = 0; z < f->dims[2]; ++z) {
        double c0 = c[fidx(f, x, y, z)];
        double xm = c[fidx(f, x > 0 ? x - 1 : x, y, z)], xp = c[fidx(f, x + 1 < f->dims[0] ? x + 1 : x, y, z)];
        double ym = c[fidx(f, x, y > 0 ? y - 1 : y, z)], yp = c[fidx(f, x, y + 1 < f->dims[1] ? y + 1 : y, z)];
        double zm = c[fidx(f, x, y, z > 0 ? z - 1 : z)], zp = c[fidx(f, x, y, z + 1 < f->dims[2] ? z + 1 : z)];
        double lap = ((((xm + xp) + (ym + yp)) + (zm + zp)) - 6.0 * c0) * ih2;
        double v = c0 + f->dt * (f->diff * lap - f->decay * c0);
        out[fidx(f, x, y, z)] = v < 0.0 ? 0.0 : v; /* negative results clamped to 0 */
      }
}

/* central-difference gradient component a at node (x,y,z), one-sided on the boundary layers */
static double node_grad(const orc_fields* f, const double* c, int64_t x, int64_t y, int64_t z, int a) {
  int64_t v[3] = {x, y, z};
  int64_t lo[3] = {x, y, z}, hi[3] = {x, y, z};
  if (v[a] > 0) lo[a] = v[a] - 1;
  if (v[a] + 1 < f->dims[a]) hi[a] = v[a] + 1;
  double cl = c[fidx(f, lo[0], lo[1], lo[2])], ch = c[fidx(f, hi[0], hi[1], hi[2])];
  if (lo[a] == v[a] && hi[a] == v[a]) return 0.0;
  if (lo[a] == v[a] || hi[a] == v[a]) return (ch - cl) * (1.0 / f->h);
  return (ch - cl) * (0.5 / f->h);
}

void orc_gradient_at(const orc_fields* f, const double* c, const double* p, double* g) {
  double invh = 1.0 / f->h;
  int64_t b[3];
  double w[3];
  for (int a = 0; a < 3; ++a) {
    double q = (p[a] - f->origin[a]) * invh;
    double fl = floor(q);
    int64_t i0 = (int64_t)fl;
    double t = q - fl;
    if (i0 < 0) {
      i0 = 0;
      t = 0.0;
    }
    if (i0 > f->dims[a] - 2) {
      i0 = f->dims[a] - 2 >= 0 ? f->dims[a] - 2 : 0;
      t = f->dims[a] >= 2 ? 1.0 : 0.0;
    }
    b[a] = i0;
    w[a] = t;
  }
  for (int a = 0; a < 3; ++a) {
    double acc = 0.0;
    for (int k = 0; k < 8; ++k) {
      int dx = (k >> 2) & 1, dy = (k >> 1) & 1, dz = k & 1;
      int64_t x = b[0] + dx, y = b[1] + dy, z = b[2] + dz;
      if (x >= f->dims[0]) x = f->dims[0] - 1;
      if (y >= f->dims[1]) y = f->dims[1] - 1;
      if (z >= f->dims[2]) z = f->dims[2] - 1;
      double wk = (dx ? w[0] : 1.0 - w[0]) * (dy ? w[1] : 1.0 - w[1]);
      wk = wk * (dz ? w[2] : 1.0 - w[2]);
      acc = acc + wk * node_grad(f, c, x, y, z, a);
    }
    g[a] = acc;
  }
}

void orc_chemotaxis(int64_t n, double* pos, const int8_t* type, const orc_fields* f, const double* c0,
                    const double* c1) {
  for (int64_t i = 0; i < n; ++i) {
    double g[3];
    orc_gradient_at(f, type[i] ? c1 : c0, pos + 3 * i, g);
    double gn = sqrt((g[0] * g[0] + g[1] * g[1]) + g[2] * g[2]);
    if (!(gn > 0.0)) continue;
    double sc = f->speed / gn;
    for (int a = 0; a < 3; ++a) pos[3 * i + a] = pos[3 * i + a] + g[a] * sc;
  }
}

/* n_steps of S1-S4; c0/c1 are updated in place (scratch allocated here). */
int orc_run_soma(int64_t n, double* pos, const double* diam, const int8_t* type, const orc_params* p,
                 const orc_fields* f, double* c0, double* c1, int32_t n_steps, double* dp, int nthreads) {
  int64_t nn = (int64_t)f->dims[0] * f->dims[1] * f->dims[2];
  double* tmp = (double*)malloc(sizeof(double) * (size_t)(nn > 3 * n ? nn : 3 * n + 1));
  if (!tmp) return ORC_ENOMEM;
  for (int32_t s = 0; s < n_steps; ++s) {
    orc_secrete(n, pos, type, f, c0, c1);
    orc_diffuse(f, c0, tmp);
    memcpy(c0, tmp, sizeof(double) * nn);
    orc_diffuse(f, c1, tmp);
    memcpy(c1, tmp, sizeof(double) * nn);
    orc_chemotaxis(n, pos, type, f, c0, c1);
    int rc = orc_step(n, pos, diam, p, dp, tmp, NULL, nthreads);
    if (rc) {
      free(tmp);
      return rc;
    }
    memcpy(pos, tmp, sizeof(double) * 3 * n);
  }
  free(tmp);
  return ORC_OK;
}

/* ------------------------------------------------------------------------------------------------
 * NEXT-4: neurite elements (cylinders) -- sphere-cylinder contacts and spring chains (DESIGN.md §13,
 * readings N1-N6).  PAPER.md:402-415 (§2.2 "approximated as a spring with a point mass on its distal
 * end ... springs are connected to each other to transmit forces along the chain")
 * (the paper's GPU kernel lacks cylinders); SPEC.md:230-238 (sphere_cylinder_force: closest point on
 * the axis segment, then the sphere law; reaction on the distal point mass)
 * (neurite_mechanics_op: axial spring force k_s (actual - resting)/resting).
 *   N1 element e: distal point Q_e, diameter d_e, resting length l0_e, mother m_e (-1: root with
 *      fixed proximal anchor A_e), daughters c1_e, c2_e; P_e = Q_{m_e} or A_e; v = Q - P;
 *      len = sqrt((vx*vx + vy*vy) + vz*vz); centre C_e = P + 0.5*v
 *   N2 box edge L = max(max_s D_s, max_e (len_e + d_e), box_edge_min), one frame for both grids
 *   N3 spring: T_e = k_s * ((len - l0)/l0); u = v * (1/len); on Q_e: -T_e*u; on Q_{m_e}: +T_e*u
 *   N4 sphere-cylinder: t = clamp(((c-P).v)/(v.v), 0, 1) (v.v = 0: t = 0); X = P + t*v; w = c - X;
 *      d2 = (wx*wx + wy*wy) + wz*wz; d = sqrt(d2); delta = (r_s + r_e) - d; contact iff delta > 0 and
 *      d2 > 0; r = (r_s*r_e)/(r_s + r_e); f = k*delta - gamma*sqrt(r*delta); on the sphere (f/d)*w,
 *      on Q_e the reaction -(f/d)*w
 *   N5 sums: sphere: sphere-sphere sum (O5), then element terms over the 27 element boxes around its
 *      box in (dx,dy,dz) order, ascending element id.  Distal point Q_e: -T_e*u_e, then +T_c*u_c for
 *      daughters c in ascending id, then sphere reactions over the 27 sphere boxes around box(C_e),
 *      ascending sphere id
 *   N6 displacement O6 for spheres and distal points alike; p' = p + dp, Q' = Q + dQ (Jacobi)
 * ---------------------------------------------------------------------------------------------- */
typedef struct {
  double k_spring;
} orc_neurite;

static void el_geom(int64_t e, const double* Q, const double* A, const int64_t* mother, double* P, double* v,
                    double* len, double* C) {
  const double* pp = mother[e] >= 0 ? Q + 3 * mother[e] : A + 3 * e;
  for (int a = 0; a < 3; ++a) {
    P[a] = pp[a];
    v[a] = Q[3 * e + a] - pp[a];
  }
  *len = sqrt((v[0] * v[0] + v[1] * v[1]) + v[2] * v[2]);
  for (int a = 0; a < 3; ++a) C[a] = P[a] + 0.5 * v[a];
}

/* N4: force on the sphere at c (radius rs) from element (P, v, re); returns 1 on contact */
static int sc_term(const double* c, double rs, const double* P, const double* v, double re, const orc_params* p,
                   double* t3) {
  double cp[3] = {c[0] - P[0], c[1] - P[1], c[2] - P[2]};
  double vv = (v[0] * v[0] + v[1] * v[1]) + v[2] * v[2];
  double t = 0.0;
  if (vv > 0.0) {
    t = ((cp[0] * v[0] + cp[1] * v[1]) + cp[2] * v[2]) / vv;
    t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
  }
  double w[3];
  for (int a = 0; a < 3; ++a) w[a] = c[a] - (P[a] + t * v[a]);
  double d2 = (w[0] * w[0] + w[1] * w[1]) + w[2] * w[2];
  if (!(d2 > 0.0)) return 0;
  double d = sqrt(d2);
  double s = rs + re;
  double delta = s - d;
  if (!(delta > 0.0)) return 0;
  double r = (rs * re) / s;
  double f = p->k_rep * delta - p->gamma_att * sqrt(r * delta);
  double m = f / d;
  for (int a = 0; a < 3; ++a) t3[a] = m * w[a];
  return 1;
}

/* One step of spheres + neurite elements.  Sphere arrays as orc_step; elements: Q (3E), d (E),
 * l0 (E), anchor A (3E), mother/c1/c2 (E).  Outputs dp_s (3n), dQ (3E); positions updated in place. */
int orc_neurite_step(int64_t n, double* pos, const double* diam, int64_t E, double* Q, const double* de,
                     const double* l0, const double* A, const int64_t* mother, const int64_t* c1, const int64_t* c2,
                     const orc_params* p, const orc_neurite* np, double* dp_s, double* dQ) {
  double* P = (double*)malloc(sizeof(double) * 3 * (E > 0 ? E : 1));
  double* V = (double*)malloc(sizeof(double) * 3 * (E > 0 ? E : 1));
  double* LEN = (double*)malloc(sizeof(double) * (E > 0 ? E : 1));
  double* C = (double*)malloc(sizeof(double) * 3 * (E > 0 ? E : 1));
  double* Ce_d = (double*)malloc(sizeof(double) * (E > 0 ? E : 1));
  double* F = (double*)malloc(sizeof(double) * 3 * (n > 0 ? n : 1));
  if (!P || !V || !LEN || !C || !Ce_d || !F) return ORC_ENOMEM;
  double L = p->box_edge_min;
  for (int64_t i = 0; i < n; ++i)
    if (diam[i] > L) L = diam[i];
  for (int64_t e = 0; e < E; ++e) {
    el_geom(e, Q, A, mother, P + 3 * e, V + 3 * e, LEN + e, C + 3 * e);
    Ce_d[e] = LEN[e] + de[e];
    if (Ce_d[e] > L) L = Ce_d[e];
  }
  /* sphere-sphere sums with the common box edge (N2) */
  orc_params ps = *p;
  ps.box_edge_min = L;
  orc_record rec;
  memset(&rec, 0, sizeof rec);
  rec.force = F;
  double* scratch = (double*)malloc(sizeof(double) * 3 * (n > 0 ? n : 1));
  int rc = n > 0 ? orc_step_sample(n, pos, diam, &ps, n, NULL, scratch, NULL, &rec, 0) : ORC_OK;
  free(scratch);
  if (rc) return rc;
  orc_index sx, ex;
  memset(&sx, 0, sizeof sx);
  memset(&ex, 0, sizeof ex);
  if (n > 0 && (rc = build_index(&sx, n, pos, diam, L))) return rc;
  if (E > 0 && (rc = build_index(&ex, E, C, Ce_d, L))) return rc;
  /* spheres: + element terms (N5), O6 */
  for (int64_t i = 0; i < n; ++i) {
    double Fi[3] = {F[3 * i], F[3 * i + 1], F[3 * i + 2]};
    if (E > 0) {
      int64_t b[3];
      for (int a = 0; a < 3; ++a) b[a] = (int64_t)floor(pos[3 * i + a] * ex.g.inv);
      for (int ddx = -1; ddx <= 1; ++ddx)
        for (int ddy = -1; ddy <= 1; ++ddy)
          for (int ddz = -1; ddz <= 1; ++ddz) {
            int64_t cx = b[0] + ddx, cy = b[1] + ddy, cz = b[2] + ddz;
            if (cx < ex.g.lo[0] || cx > ex.g.hi[0] || cy < ex.g.lo[1] || cy > ex.g.hi[1] || cz < ex.g.lo[2] ||
                cz > ex.g.hi[2])
              continue;
            uint64_t k = key_of(&ex, cx, cy, cz);
            for (int64_t q = lower_bound(&ex, k); q < E && ex.sorted[q].key == k; ++q) {
              int64_t e = ex.sorted[q].id;
              double t3[3];
              if (sc_term(pos + 3 * i, 0.5 * diam[i], P + 3 * e, V + 3 * e, 0.5 * de[e], p, t3)) {
                Fi[0] = Fi[0] + t3[0];
                Fi[1] = Fi[1] + t3[1];
                Fi[2] = Fi[2] + t3[2];
              }
            }
          }
    }
    displacement(Fi, p, dp_s + 3 * i);
  }
  /* distal points (N3, N5), O6 */
  for (int64_t e = 0; e < E; ++e) {
    double Fe[3] = {0.0, 0.0, 0.0};
    double T = np->k_spring * ((LEN[e] - l0[e]) / l0[e]);
    double inv = 1.0 / LEN[e];
    for (int a = 0; a < 3; ++a) Fe[a] = Fe[a] + (-T) * (V[3 * e + a] * inv);
    int64_t ch[2] = {c1[e], c2[e]};
    if (ch[0] > ch[1] && ch[1] >= 0) {
      int64_t t = ch[0];
      ch[0] = ch[1];
      ch[1] = t;
    }
    for (int k = 0; k < 2; ++k) {
      int64_t c = ch[k];
      if (c < 0) continue;
      double Tc = np->k_spring * ((LEN[c] - l0[c]) / l0[c]);
      double invc = 1.0 / LEN[c];
      for (int a = 0; a < 3; ++a) Fe[a] = Fe[a] + Tc * (V[3 * c + a] * invc);
    }
    if (n > 0) {
      int64_t b[3];
      for (int a = 0; a < 3; ++a) b[a] = (int64_t)floor(C[3 * e + a] * sx.g.inv);
      for (int ddx = -1; ddx <= 1; ++ddx)
        for (int ddy = -1; ddy <= 1; ++ddy)
          for (int ddz = -1; ddz <= 1; ++ddz) {
            int64_t cx = b[0] + ddx, cy = b[1] + ddy, cz = b[2] + ddz;
            if (cx < sx.g.lo[0] || cx > sx.g.hi[0] || cy < sx.g.lo[1] || cy > sx.g.hi[1] || cz < sx.g.lo[2] ||
                cz > sx.g.hi[2])
              continue;
            uint64_t k = key_of(&sx, cx, cy, cz);
            for (int64_t q = lower_bound(&sx, k); q < n && sx.sorted[q].key == k; ++q) {
              int64_t s = sx.sorted[q].id;
              double t3[3];
              if (sc_term(pos + 3 * s, 0.5 * diam[s], P + 3 * e, V + 3 * e, 0.5 * de[e], p, t3)) {
                Fe[0] = Fe[0] - t3[0];
                Fe[1] = Fe[1] - t3[1];
                Fe[2] = Fe[2] - t3[2];
              }
            }
          }
    }
    displacement(Fe, p, dQ + 3 * e);
  }
  for (int64_t i = 0; i < 3 * n; ++i) pos[i] = pos[i] + dp_s[i];
  for (int64_t i = 0; i < 3 * E; ++i) Q[i] = Q[i] + dQ[i];
  if (n > 0) free_index(&sx);
  if (E > 0) free_index(&ex);
  free(P);
  free(V);
  free(LEN);
  free(C);
  free(Ce_d);
  free(F);
  return ORC_OK;
}
