/*
 * lj_oracle.c -- CPU restatement of the reference LJ force path (TEST INFRASTRUCTURE).
 *
 * This file is the *checker*: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  The product path never calls it.
 *
 * It restates, in plain C with strict IEEE double arithmetic (compile with
 * -O2 -ffp-contract=off, no -ffast-math), the algorithm of the reference package
 * `lanemd` (/root/reference/pkg/src/lanemd, read-only; paths below are relative
 * to it).  Every function cites the reference file:line it follows.  The goal is
 * bit-identical forces and identical integer statistics to the reference's
 * driver.force_phase on the same inputs; tests/golden pins that claim with
 * fixtures generated from the unmodified reference (tests/golden/make_golden.py).
 *
 * Extensions the reference does not have (north star; parity for them is pinned
 * only by internal consistency):
 *   - potential energy and virial accumulated in the sweep,
 *   - plain Verlet lists with a skin (orc_force_phase_vl),
 *   - the velocity-Verlet step and boundary wrap (integrator.py / domain.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OWNED 0
#define HALO 1
#define DUMMY 2

#define ORC_OK 0
#define ORC_OVERLAP 1      /* ParticleOverlapError */
#define ORC_DEGENERATE 2   /* DegenerateDomainError */
#define ORC_CONFIG 3       /* ConfigurationError */
#define ORC_NOMEM 4

/* traversal codes (traversals.py:40-48 + extension) */
#define TRAV_C01 0
#define TRAV_C08 1
#define TRAV_C18 2
#define TRAV_VCL 3
#define TRAV_VL 4

typedef struct {
  int64_t kernel_invocations;
  int64_t lane_slots;
  int64_t useful_interactions;
  int64_t pair_interactions;
  double epot;   /* extension */
  double virial; /* extension */
  int32_t overlap;
  int32_t pad;
} orc_stats;

/* Neumaier-compensated accumulator for the energy/virial extension. */
typedef struct { double s, c; } kahan;
static inline void kadd(kahan* k, double v) {
  double t = k->s + v;
  if (fabs(k->s) >= fabs(v)) k->c += (k->s - t) + v; else k->c += (v - t) + k->s;
  k->s = t;
}

/* SoA particle buffer (particles.py:54-164). */
typedef struct {
  int64_t n;
  double *x, *y, *z, *fx, *fy, *fz;
  int8_t* own;
  int64_t* id;
} pbuf;

static int pbuf_alloc(pbuf* b, int64_t n) {
  b->n = n;
  int64_t m = n > 0 ? n : 1;
  b->x = calloc(m, 8); b->y = calloc(m, 8); b->z = calloc(m, 8);
  b->fx = calloc(m, 8); b->fy = calloc(m, 8); b->fz = calloc(m, 8);
  b->own = calloc(m, 1); b->id = calloc(m, 8);
  return (b->x && b->y && b->z && b->fx && b->fy && b->fz && b->own && b->id) ? 0 : -1;
}
static void pbuf_free(pbuf* b) {
  free(b->x); free(b->y); free(b->z); free(b->fx); free(b->fy); free(b->fz);
  free(b->own); free(b->id); memset(b, 0, sizeof(*b));
}

/* ------------------------------------------------------------------ sweep */
typedef struct { double eps24, sigma2, rc2, eps4; } ljk;

/* executor.py:72-115 (_sweep_span) == kernels.py:197-239 (_pair_sweep):
 * identical expression order, no contraction.  Energy/virial (extension):
 * weight 1 for a dual-write (newton3) pair, 1/2 for a one-sided evaluation. */
static int64_t sweep_span(const pbuf* I, const pbuf* J, int64_t i0, int64_t ni,
                          int64_t j0, int64_t nj, int newton3, int same,
                          const ljk* k, kahan* epot, kahan* vir) {
  int64_t pairs = 0;
  const double w = newton3 ? 1.0 : 0.5;
  for (int64_t p = i0; p < i0 + ni; ++p) {
    if (I->own[p] != OWNED) continue;
    double px = I->x[p], py = I->y[p], pz = I->z[p];
    double ax = 0.0, ay = 0.0, az = 0.0;
    int64_t start = (same && newton3) ? p + 1 : j0;
    for (int64_t q = start; q < j0 + nj; ++q) {
      if (same && q == p) continue;
      if (J->own[q] == DUMMY) continue;
      double dx = px - J->x[q];
      double dy = py - J->y[q];
      double dz = pz - J->z[q];
      double r2 = dx * dx + dy * dy + dz * dz;
      if (r2 >= k->rc2) continue;
      if (r2 == 0.0) return -1;
      double s2 = k->sigma2 / r2;
      double s6 = s2 * s2 * s2;
      double f = k->eps24 * (2.0 * s6 * s6 - s6) / r2;
      ax += f * dx;
      ay += f * dy;
      az += f * dz;
      if (newton3) {
        J->fx[q] -= f * dx;
        J->fy[q] -= f * dy;
        J->fz[q] -= f * dz;
      }
      if (epot) {
        kadd(epot, w * (k->eps4 * (s6 * s6 - s6)));
        kadd(vir, w * (f * r2));
      }
      pairs += 1;
    }
    I->fx[p] += ax;
    I->fy[p] += ay;
    I->fz[p] += az;
  }
  return pairs;
}

/* ------------------------------------------------------------ stats helpers */
/* particles.py:166-198 (ownership_counts, self_pair_slots) on a span. */
static void span_counts(const pbuf* b, int64_t o, int64_t n, int64_t* owned, int64_t* nondummy) {
  int64_t a = 0, c = 0;
  for (int64_t k = o; k < o + n; ++k) { a += b->own[k] == OWNED; c += b->own[k] != DUMMY; }
  *owned = a; *nondummy = c;
}
static int64_t self_pair_slots(const pbuf* b, int64_t o, int64_t n, int newton3) {
  int64_t owned, total;
  span_counts(b, o, n, &owned, &total);
  if (!newton3) return owned * (total - 1 > 0 ? total - 1 : 0);
  int64_t acc = 0, seen = 0;
  for (int64_t k = o; k < o + n; ++k) {
    seen += b->own[k] != DUMMY;                 /* cumsum(nondummy)[k] */
    if (b->own[k] == OWNED) acc += total - seen;
  }
  return acc;
}
static inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

/* ----------------------------------------------------------- work units */
typedef struct {
  int64_t i_off, i_len, j_off, j_len;
  int8_t j_halo, newton3, same;
  int32_t color;
  int64_t base;
  int64_t seq; /* emission order, for the stable color sort */
} unit;

typedef struct { unit* u; int64_t n, cap; } unitvec;
static int uv_push(unitvec* v, unit x) {
  if (v->n == v->cap) {
    int64_t nc = v->cap ? 2 * v->cap : 1024;
    unit* nu = realloc(v->u, nc * sizeof(unit));
    if (!nu) return -1;
    v->u = nu; v->cap = nc;
  }
  x.seq = v->n;
  v->u[v->n++] = x;
  return 0;
}
static int unit_cmp(const void* a, const void* b) {
  const unit* x = a; const unit* y = b;
  if (x->color != y->color) return x->color < y->color ? -1 : 1;
  return x->seq < y->seq ? -1 : (x->seq > y->seq);
}
/* traversals.py:168-170 (_finish): stable sort by color. */
static void finish_units(unitvec* v) { qsort(v->u, v->n, sizeof(unit), unit_cmp); }

/* executor.py:118-171 (_batch_sweep / execute_packed) + pack_schedule's
 * useful-lane count (executor.py:38-69). */
static int execute_units(const unitvec* v, pbuf* own_b, pbuf* halo_b, const ljk* k,
                         int a, int b, int V, orc_stats* st, int want_ev) {
  kahan ep = {0, 0}, vr = {0, 0};
  int64_t total = 0, inv = 0, useful = 0;
  for (int64_t u = 0; u < v->n; ++u) {
    const unit* w = &v->u[u];
    const pbuf* J = w->j_halo ? halo_b : own_b;
    inv += cdiv(w->i_len, a) * cdiv(w->j_len, b);
    if (w->same) useful += self_pair_slots(own_b, w->i_off, w->i_len, w->newton3);
    else {
      int64_t io, in_, jo, jn;
      span_counts(own_b, w->i_off, w->i_len, &io, &in_);
      span_counts(J, w->j_off, w->j_len, &jo, &jn);
      useful += io * jn;
    }
    int64_t p = sweep_span(own_b, J, w->i_off, w->i_len, w->j_off, w->j_len, w->newton3,
                           w->same, k, want_ev ? &ep : NULL, want_ev ? &vr : NULL);
    if (p < 0) { st->overlap = 1; return ORC_OVERLAP; }
    total += p;
  }
  st->kernel_invocations = inv;
  st->lane_slots = inv * V;
  st->useful_interactions = useful;
  st->pair_interactions = total;
  st->epot = ep.s + ep.c;
  st->virial = vr.s + vr.c;
  return ORC_OK;
}

/* -------------------------------------------------------------------- box */
typedef struct {
  double lo[3], hi[3], len[3];
  int periodic[3];
} obox;

/* domain.py:97-144 (build_halo): images in itertools.product order of the
 * per-axis shift options [0, hi-lo, lo-hi], each piece in ascending index. */
static int build_halo(const pbuf* b, const obox* bx, double margin, pbuf* out) {
  int64_t n = b->n;
  double opts[3][3]; int nopt[3];
  for (int ax = 0; ax < 3; ++ax) {
    opts[ax][0] = 0.0;
    if (bx->periodic[ax]) { opts[ax][1] = bx->hi[ax] - bx->lo[ax]; opts[ax][2] = bx->lo[ax] - bx->hi[ax]; nopt[ax] = 3; }
    else nopt[ax] = 1;
  }
  int any = bx->periodic[0] || bx->periodic[1] || bx->periodic[2];
  if (!any) return pbuf_alloc(out, 0);
  const double* pos[3] = {b->x, b->y, b->z};
  /* count first */
  int64_t cnt = 0;
  for (int s0 = 0; s0 < nopt[0]; ++s0) for (int s1 = 0; s1 < nopt[1]; ++s1) for (int s2 = 0; s2 < nopt[2]; ++s2) {
    if (s0 == 0 && s1 == 0 && s2 == 0) continue;
    int s[3] = {s0, s1, s2};
    for (int64_t p = 0; p < n; ++p) {
      if (b->own[p] != OWNED) continue;
      int ok = 1;
      for (int ax = 0; ax < 3 && ok; ++ax) {
        if (s[ax] == 1) ok = (pos[ax][p] - bx->lo[ax]) < margin;
        else if (s[ax] == 2) ok = (bx->hi[ax] - pos[ax][p]) < margin;
      }
      cnt += ok;
    }
  }
  if (pbuf_alloc(out, cnt)) return ORC_NOMEM;
  int64_t w = 0;
  for (int s0 = 0; s0 < nopt[0]; ++s0) for (int s1 = 0; s1 < nopt[1]; ++s1) for (int s2 = 0; s2 < nopt[2]; ++s2) {
    if (s0 == 0 && s1 == 0 && s2 == 0) continue;
    int s[3] = {s0, s1, s2};
    for (int64_t p = 0; p < n; ++p) {
      if (b->own[p] != OWNED) continue;
      int ok = 1;
      for (int ax = 0; ax < 3 && ok; ++ax) {
        if (s[ax] == 1) ok = (pos[ax][p] - bx->lo[ax]) < margin;
        else if (s[ax] == 2) ok = (bx->hi[ax] - pos[ax][p]) < margin;
      }
      if (!ok) continue;
      out->x[w] = b->x[p] + opts[0][s0];
      out->y[w] = b->y[p] + opts[1][s1];
      out->z[w] = b->z[p] + opts[2][s2];
      out->own[w] = HALO;
      out->id[w] = b->id[p];
      ++w;
    }
  }
  return ORC_OK;
}

/* -------------------------------------------------------- linked cells */
typedef struct {
  int64_t dims[3], tdims[3];
  double cell_len[3], lo[3];
  int64_t ncell;
  /* owned backing */
  pbuf ob; int64_t* perm; int64_t* o_start; int64_t* o_count;
  /* halo backing */
  pbuf hb; int64_t* h_start; int64_t* h_count;
  uint8_t* occ;          /* 0 empty, 1 owned, 2 halo-only (containers.py:93-94) */
  int64_t* owned_occ; int64_t n_owned_occ;
  int64_t* halo_occ; int64_t n_halo_occ;
} lc_t;

/* containers.py:71-98 */
static int lc_init(lc_t* c, const obox* bx, double length) {
  memset(c, 0, sizeof(*c));
  for (int ax = 0; ax < 3; ++ax) {
    double d = floor(bx->len[ax] / length);
    if (!(d >= 1.0)) return ORC_DEGENERATE;
    c->dims[ax] = (int64_t)d;
    c->cell_len[ax] = bx->len[ax] / (double)c->dims[ax];
    c->tdims[ax] = c->dims[ax] + 2;
    c->lo[ax] = bx->lo[ax];
  }
  c->ncell = c->tdims[0] * c->tdims[1] * c->tdims[2];
  return ORC_OK;
}

/* containers.py:104-115 (cell_coords + linear_index) */
static int64_t lc_cell_of(const lc_t* c, double x, double y, double z, int ring) {
  double p[3] = {x, y, z};
  int64_t q[3];
  for (int ax = 0; ax < 3; ++ax) {
    double s = floor((p[ax] - c->lo[ax]) / c->cell_len[ax]);
    int64_t v = (int64_t)s + 1;
    int64_t lo = ring ? 0 : 1, hi = ring ? c->dims[ax] + 1 : c->dims[ax];
    if (v < lo) v = lo;
    if (v > hi) v = hi;
    q[ax] = v;
  }
  return q[0] + c->tdims[0] * (q[1] + c->tdims[1] * q[2]);
}

/* stable counting sort of keys in [0, ncell): perm[k] = index of k-th sorted */
static int stable_bin(const int64_t* key, int64_t n, int64_t ncell, int64_t* perm,
                      int64_t* start, int64_t* count) {
  memset(count, 0, ncell * sizeof(int64_t));
  for (int64_t k = 0; k < n; ++k) count[key[k]]++;
  int64_t acc = 0;
  for (int64_t c = 0; c < ncell; ++c) { start[c] = acc; acc += count[c]; }
  int64_t* cur = malloc((ncell > 0 ? ncell : 1) * sizeof(int64_t));
  if (!cur) return ORC_NOMEM;
  memcpy(cur, start, ncell * sizeof(int64_t));
  for (int64_t k = 0; k < n; ++k) perm[cur[key[k]]++] = k;
  free(cur);
  return ORC_OK;
}

static void take(const pbuf* src, const int64_t* perm, pbuf* dst) {
  for (int64_t k = 0; k < dst->n; ++k) {
    int64_t s = perm[k];
    dst->x[k] = src->x[s]; dst->y[k] = src->y[s]; dst->z[k] = src->z[s];
    dst->own[k] = src->own[s]; dst->id[k] = src->id[s];
    dst->fx[k] = 0.0; dst->fy[k] = 0.0; dst->fz[k] = 0.0;
  }
}

/* containers.py:122-139 (rebuild) + 141-172 (refresh). */
static int lc_build(lc_t* c, const pbuf* owned, const pbuf* halo) {
  int64_t n = owned->n, nh = halo->n, nc = c->ncell;
  int rc = ORC_NOMEM;
  int64_t* key = malloc((n > nh ? n : nh) * sizeof(int64_t) + 8);
  c->perm = malloc((n + 1) * sizeof(int64_t));
  int64_t* hperm = malloc((nh + 1) * sizeof(int64_t));
  c->o_start = malloc(nc * sizeof(int64_t)); c->o_count = malloc(nc * sizeof(int64_t));
  c->h_start = malloc(nc * sizeof(int64_t)); c->h_count = malloc(nc * sizeof(int64_t));
  c->occ = calloc(nc, 1);
  c->owned_occ = malloc(nc * sizeof(int64_t)); c->halo_occ = malloc(nc * sizeof(int64_t));
  if (!key || !c->perm || !hperm || !c->o_start || !c->o_count || !c->h_start || !c->h_count ||
      !c->occ || !c->owned_occ || !c->halo_occ) goto out;
  for (int64_t k = 0; k < n; ++k) key[k] = lc_cell_of(c, owned->x[k], owned->y[k], owned->z[k], 0);
  if ((rc = stable_bin(key, n, nc, c->perm, c->o_start, c->o_count))) goto out;
  if ((rc = pbuf_alloc(&c->ob, n))) goto out;
  take(owned, c->perm, &c->ob);
  for (int64_t k = 0; k < nh; ++k) key[k] = lc_cell_of(c, halo->x[k], halo->y[k], halo->z[k], 1);
  if ((rc = stable_bin(key, nh, nc, hperm, c->h_start, c->h_count))) goto out;
  if ((rc = pbuf_alloc(&c->hb, nh))) goto out;
  take(halo, hperm, &c->hb);
  c->n_owned_occ = 0; c->n_halo_occ = 0;
  for (int64_t q = 0; q < nc; ++q) {
    if (c->o_count[q]) { c->owned_occ[c->n_owned_occ++] = q; c->occ[q] = 1; }
  }
  for (int64_t q = 0; q < nc; ++q) {
    if (c->h_count[q]) {
      c->halo_occ[c->n_halo_occ++] = q;
      if (c->occ[q] == 0) c->occ[q] = 2;  /* owned cells shadow halo marks */
    }
  }
  rc = ORC_OK;
out:
  free(key); free(hperm);
  return rc;
}

static void lc_free(lc_t* c) {
  pbuf_free(&c->ob); pbuf_free(&c->hb);
  free(c->perm); free(c->o_start); free(c->o_count); free(c->h_start); free(c->h_count);
  free(c->occ); free(c->owned_occ); free(c->halo_occ);
}

/* containers.py:178-184 (buffer_at): owned cell view, else halo cell view. */
static void lc_buffer_at(const lc_t* c, int64_t lin, int* is_halo, int64_t* off, int64_t* len) {
  if (c->o_count[lin]) { *is_halo = 0; *off = c->o_start[lin]; *len = c->o_count[lin]; }
  else { *is_halo = 1; *off = c->h_start[lin]; *len = c->h_count[lin]; }
}

static void coords_of(const lc_t* c, int64_t lin, int64_t* x, int64_t* y, int64_t* z) {
  *x = lin % c->tdims[0];
  int64_t r = lin / c->tdims[0];
  *y = r % c->tdims[1];
  *z = r / c->tdims[1];
}
static inline int64_t pymod(int64_t a, int64_t m) { int64_t r = a % m; return r < 0 ? r + m : r; }

/* traversals.py:79-84: 13 forward directions, itertools.product order. */
static int FWD[13][3]; static int ALL[27][3]; static int dirs_ready = 0;
static void init_dirs(void) {
  if (dirs_ready) return;
  int nf = 0, na = 0;
  for (int a = -1; a <= 1; ++a) for (int b = -1; b <= 1; ++b) for (int c = -1; c <= 1; ++c) {
    ALL[na][0] = a; ALL[na][1] = b; ALL[na][2] = c; ++na;
    int fwd = (c > 0) || (c == 0 && b > 0) || (c == 0 && b == 0 && a > 0);
    if (fwd) { FWD[nf][0] = a; FWD[nf][1] = b; FWD[nf][2] = c; ++nf; }
  }
  dirs_ready = 1;
}

/* traversals.py:152-165 (_emit_pair) */
static int emit_pair(unitvec* v, const lc_t* c, int64_t a, int64_t b, int ah, int bh,
                     int newton3, int color, int64_t base) {
  int ha, hb; int64_t oa, la, ob, lb;
  if (ah || bh) {
    if (ah) { int64_t t = a; a = b; b = t; }
    lc_buffer_at(c, a, &ha, &oa, &la);
    lc_buffer_at(c, b, &hb, &ob, &lb);
    unit u = {oa, la, ob, lb, (int8_t)hb, 0, 0, color, base, 0};
    return uv_push(v, u);
  }
  lc_buffer_at(c, a, &ha, &oa, &la);
  lc_buffer_at(c, b, &hb, &ob, &lb);
  if (newton3) {
    unit u = {oa, la, ob, lb, (int8_t)hb, 1, 0, color, base, 0};
    return uv_push(v, u);
  }
  unit u1 = {oa, la, ob, lb, (int8_t)hb, 0, 0, color, base, 0};
  unit u2 = {ob, lb, oa, la, (int8_t)ha, 0, 0, color, base, 0};
  if (uv_push(v, u1)) return -1;
  return uv_push(v, u2);
}

/* traversals.py:94-105 */
static void block_offset_rank(const int* d, int* r1, int* r2) {
  int o1[3], o2[3];
  for (int k = 0; k < 3; ++k) { o1[k] = -d[k] > 0 ? -d[k] : 0; o2[k] = d[k] > 0 ? d[k] : 0; }
  *r1 = 4 * o1[0] + 2 * o1[1] + o1[2];
  *r2 = 4 * o2[0] + 2 * o2[1] + o2[2];
}

/* traversals.py:125-149 (_occupied_pairs) driving c18 (190-211) / c08 (214-241). */
static int schedule_lc(const lc_t* c, int trav, int newton3, unitvec* v) {
  init_dirs();
  const int64_t* T = c->tdims;
  if (trav == TRAV_C01) {  /* traversals.py:173-187 */
    if (newton3) return ORC_CONFIG;
    for (int d = 0; d < 27; ++d) {
      for (int64_t k = 0; k < c->n_owned_occ; ++k) {
        int64_t a = c->owned_occ[k], x, y, z;
        coords_of(c, a, &x, &y, &z);
        int64_t nl = (x + ALL[d][0]) + T[0] * ((y + ALL[d][1]) + T[1] * (z + ALL[d][2]));
        if (c->occ[nl] == 0) continue;
        int ha, hb; int64_t oa, la, ob, lb;
        lc_buffer_at(c, a, &ha, &oa, &la);
        lc_buffer_at(c, nl, &hb, &ob, &lb);
        unit u = {oa, la, ob, lb, (int8_t)hb, 0, (int8_t)(a == nl), 0, a, 0};
        if (uv_push(v, u)) return ORC_NOMEM;
      }
    }
    finish_units(v);
    return ORC_OK;
  }
  /* self units */
  for (int64_t k = 0; k < c->n_owned_occ; ++k) {
    int64_t a = c->owned_occ[k], x, y, z;
    coords_of(c, a, &x, &y, &z);
    int col = trav == TRAV_C18 ? (int)((x % 3) + 3 * (y % 3) + 9 * (z % 2))
                               : (int)((x % 2) + 2 * (y % 2) + 4 * (z % 2));
    unit u = {c->o_start[a], c->o_count[a], c->o_start[a], c->o_count[a], 0, (int8_t)newton3, 1, col, a, 0};
    if (uv_push(v, u)) return ORC_NOMEM;
  }
  /* occ = concat(owned_occupied, halo_occupied) (may repeat a cell, as the reference does) */
  int64_t nocc = c->n_owned_occ + c->n_halo_occ;
  for (int d = 0; d < 13; ++d) {
    const int* D = FWD[d];
    int r1 = 0, r2 = 0;
    if (trav == TRAV_C08) block_offset_rank(D, &r1, &r2);
    for (int64_t k = 0; k < nocc; ++k) {
      int64_t a = k < c->n_owned_occ ? c->owned_occ[k] : c->halo_occ[k - c->n_owned_occ];
      int64_t x, y, z;
      coords_of(c, a, &x, &y, &z);
      int ah = c->occ[a] == 2;
      int64_t nx = x + D[0], ny = y + D[1], nz = z + D[2];
      if (nx < 0 || nx >= T[0] || ny < 0 || ny >= T[1] || nz < 0 || nz >= T[2]) continue;
      int64_t nl = nx + T[0] * (ny + T[1] * nz);
      int st = c->occ[nl];
      if (st == 0 || (ah && st == 2)) continue;
      int bh = st == 2;
      if (trav == TRAV_C18) {
        int col = (int)((x % 3) + 3 * (y % 3) + 9 * (z % 2));
        if (emit_pair(v, c, a, nl, ah, bh, newton3, col, a)) return ORC_NOMEM;
      } else {
        int64_t bx = x + (D[0] < 0 ? D[0] : 0), by = y + (D[1] < 0 ? D[1] : 0), bz = z + (D[2] < 0 ? D[2] : 0);
        int64_t base = bx + T[0] * (by + T[1] * bz);
        int col = (int)(pymod(bx, 2) + 2 * pymod(by, 2) + 4 * pymod(bz, 2));
        int64_t aa = a, bb = nl; int aah = ah, bbh = bh;
        if (r2 < r1) { aa = nl; bb = a; aah = bh; bbh = ah; }
        if (emit_pair(v, c, aa, bb, aah, bbh, newton3, col, base)) return ORC_NOMEM;
      }
    }
  }
  finish_units(v);
  return ORC_OK;
}

static int check_pattern(int a, int b, int V) {
  if (V < 4 || (V & (V - 1)) != 0) return ORC_CONFIG;  /* kernels.py:92-95 */
  if (a * b != V || a < 1 || b < 1) return ORC_CONFIG;
  return ORC_OK;
}

static void make_box(obox* bx, const double* lo, const double* hi, const int32_t* periodic) {
  for (int ax = 0; ax < 3; ++ax) {
    bx->lo[ax] = lo[ax]; bx->hi[ax] = hi[ax]; bx->len[ax] = hi[ax] - lo[ax];
    bx->periodic[ax] = periodic[ax] != 0;
  }
}

static void wrap_input(pbuf* b, int64_t n, const double* x, const double* y, const double* z,
                       const int8_t* own) {
  memset(b, 0, sizeof(*b));
  b->n = n; b->x = (double*)x; b->y = (double*)y; b->z = (double*)z; b->own = (int8_t*)own;
}

static ljk make_ljk(double eps, double sigma, double cutoff) {
  ljk k; k.eps24 = 24.0 * eps; k.sigma2 = sigma * sigma; k.rc2 = cutoff * cutoff; k.eps4 = 4.0 * eps;
  return k;
}

/* driver.py:107-129 (force_phase) for the linked-cells container.
 * Forces are OVERWRITTEN in the caller's (original) order. */
int orc_force_phase_lc(int64_t n, const double* x, const double* y, const double* z,
                       const int8_t* own, const double* lo, const double* hi, const int32_t* periodic,
                       double eps, double sigma, double cutoff, double skin,
                       int trav, int newton3, int a, int b, int V,
                       double* fx, double* fy, double* fz, orc_stats* st) {
  memset(st, 0, sizeof(*st));
  int rc = check_pattern(a, b, V);
  if (rc) return rc;
  if (trav == TRAV_C01 && newton3) return ORC_CONFIG;
  if (trav != TRAV_C01 && trav != TRAV_C08 && trav != TRAV_C18) return ORC_CONFIG;
  obox bx; make_box(&bx, lo, hi, periodic);
  pbuf in; wrap_input(&in, n, x, y, z, own);
  int64_t* ids = malloc((n + 1) * 8);
  if (!ids) return ORC_NOMEM;
  for (int64_t k = 0; k < n; ++k) ids[k] = k;
  in.id = ids;
  lc_t c;
  if ((rc = lc_init(&c, &bx, cutoff + skin))) { free(ids); return rc; }
  pbuf halo;
  if ((rc = build_halo(&in, &bx, cutoff + skin, &halo))) { free(ids); return rc; }
  if ((rc = lc_build(&c, &in, &halo))) goto out;
  unitvec v = {0};
  if ((rc = schedule_lc(&c, trav, newton3, &v))) { free(v.u); goto out; }
  ljk k = make_ljk(eps, sigma, cutoff);
  rc = execute_units(&v, &c.ob, &c.hb, &k, a, b, V, st, 1);
  free(v.u);
  /* containers.py:186-189 (collect_forces) */
  for (int64_t q = 0; q < n; ++q) {
    int64_t s = c.perm[q];
    fx[s] = c.ob.fx[q]; fy[s] = c.ob.fy[q]; fz[s] = c.ob.fz[q];
  }
out:
  lc_free(&c); pbuf_free(&halo); free(ids);
  return rc;
}

/* Cell assignment and stable permutation of the owned particles
 * (containers.py:104-139): cell[k] = linear ring-padded index, perm = argsort(stable). */
int orc_lc_bin(int64_t n, const double* x, const double* y, const double* z,
               const double* lo, const double* hi, double length, int ring,
               int64_t* cell, int64_t* perm, int64_t* dims_out) {
  obox bx; int32_t per[3] = {0, 0, 0}; make_box(&bx, lo, hi, per);
  lc_t c;
  int rc = lc_init(&c, &bx, length);
  if (rc) return rc;
  for (int ax = 0; ax < 3; ++ax) dims_out[ax] = c.dims[ax];
  for (int64_t k = 0; k < n; ++k) cell[k] = lc_cell_of(&c, x[k], y[k], z[k], ring);
  int64_t* st = malloc(c.ncell * 8); int64_t* ct = malloc(c.ncell * 8);
  if (!st || !ct) { free(st); free(ct); return ORC_NOMEM; }
  rc = stable_bin(cell, n, c.ncell, perm, st, ct);
  free(st); free(ct);
  return rc;
}

/* build_halo restated; returns count, fills the caller's arrays (size >= 7n). */
int64_t orc_build_halo(int64_t n, const double* x, const double* y, const double* z,
                       const int8_t* own, const double* lo, const double* hi,
                       const int32_t* periodic, double margin,
                       double* hx, double* hy, double* hz, int64_t* hid) {
  obox bx; make_box(&bx, lo, hi, periodic);
  pbuf in; wrap_input(&in, n, x, y, z, own);
  int64_t* ids = malloc((n + 1) * 8);
  for (int64_t k = 0; k < n; ++k) ids[k] = k;
  in.id = ids;
  pbuf h;
  if (build_halo(&in, &bx, margin, &h)) { free(ids); return -1; }
  for (int64_t k = 0; k < h.n; ++k) { hx[k] = h.x[k]; hy[k] = h.y[k]; hz[k] = h.z[k]; hid[k] = h.id[k]; }
  int64_t cnt = h.n;
  pbuf_free(&h); free(ids);
  return cnt;
}

/* kernels.py:377-424 (compute_pair_vectorized, fast path) on two caller buffers;
 * forces accumulate (+=).  same_buffer: pass the same arrays for i and j. */
int orc_pair_sweep(int64_t ni, const double* xi, const double* yi, const double* zi, const int8_t* owni,
                   double* fxi, double* fyi, double* fzi,
                   int64_t nj, const double* xj, const double* yj, const double* zj, const int8_t* ownj,
                   double* fxj, double* fyj, double* fzj,
                   double eps, double sigma, double cutoff, int newton3, int same,
                   int a, int b, int V, orc_stats* st) {
  memset(st, 0, sizeof(*st));
  int rc = check_pattern(a, b, V);
  if (rc) return rc;
  pbuf I = {ni, (double*)xi, (double*)yi, (double*)zi, fxi, fyi, fzi, (int8_t*)owni, NULL};
  pbuf J = {nj, (double*)xj, (double*)yj, (double*)zj, fxj, fyj, fzj, (int8_t*)ownj, NULL};
  if (same) J = I;
  ljk k = make_ljk(eps, sigma, cutoff);
  kahan ep = {0, 0}, vr = {0, 0};
  int64_t p = sweep_span(&I, &J, 0, ni, 0, nj, newton3, same, &k, &ep, &vr);
  if (p < 0) { st->overlap = 1; return ORC_OVERLAP; }
  int64_t inv = cdiv(ni, a) * cdiv(nj, b);
  st->kernel_invocations = inv;
  st->lane_slots = inv * V;
  if (same) st->useful_interactions = self_pair_slots(&I, 0, ni, newton3);
  else {
    int64_t io, in_, jo, jn;
    span_counts(&I, 0, ni, &io, &in_); span_counts(&J, 0, nj, &jo, &jn);
    st->useful_interactions = io * jn;
  }
  st->pair_interactions = p;
  st->epot = ep.s + ep.c; st->virial = vr.s + vr.c;
  return ORC_OK;
}

/* ------------------------------------------------------- cluster lists */
typedef struct {
  int M;
  double col;
  int64_t n_cl;          /* owned clusters */
  pbuf ob;               /* padded owned backing, n_cl*M */
  int64_t* perm; int64_t* slots;
  double *amin, *amax;   /* n_cl x 3 */
  int64_t n_hcl;
  pbuf hb;               /* padded halo backing */
  double *hmin, *hmax;
} vcl_t;

typedef struct { int64_t col; double z; int64_t idx; } ckey;
static int ckey_cmp(const void* a, const void* b) {
  const ckey* x = a; const ckey* y = b;
  if (x->col != y->col) return x->col < y->col ? -1 : 1;
  if (x->z < y->z) return -1;
  if (y->z < x->z) return 1;
  return x->idx < y->idx ? -1 : (x->idx > y->idx);
}

/* containers.py:335-367 (_column_key, _chunk_columns): lexsort((z, col)). */
static int chunk_columns(const pbuf* b, const obox* bx, double col, int M,
                         int64_t** order_o, int64_t** slots_o, int64_t** counts_o, int64_t* ncl_o) {
  int64_t n = b->n;
  ckey* keys = malloc((n + 1) * sizeof(ckey));
  int64_t* order = malloc((n + 1) * 8); int64_t* slots = malloc((n + 1) * 8);
  int64_t* counts = malloc((n + 1) * 8);
  if (!keys || !order || !slots || !counts) { free(keys); free(order); free(slots); free(counts); return ORC_NOMEM; }
  int64_t width = (int64_t)(bx->len[0] / col) + 4;
  for (int64_t k = 0; k < n; ++k) {
    int64_t cx = (int64_t)floor((b->x[k] - bx->lo[0]) / col) + 1;
    int64_t cy = (int64_t)floor((b->y[k] - bx->lo[1]) / col) + 1;
    keys[k].col = cx + width * cy; keys[k].z = b->z[k]; keys[k].idx = k;
  }
  qsort(keys, n, sizeof(ckey), ckey_cmp);
  for (int64_t k = 0; k < n; ++k) order[k] = keys[k].idx;
  int64_t ncl = 0, pad = 0, lo = 0;
  while (lo < n) {
    int64_t hi = lo;
    while (hi < n && keys[hi].col == keys[lo].col) ++hi;
    for (int64_t s = lo; s < hi; s += M) {
      int64_t chunk = (s + M < hi ? s + M : hi) - s;
      for (int64_t t = 0; t < chunk; ++t) slots[s + t] = pad + t;
      counts[ncl++] = chunk;
      pad += M;
    }
    lo = hi;
  }
  free(keys);
  *order_o = order; *slots_o = slots; *counts_o = counts; *ncl_o = ncl;
  return ORC_OK;
}

/* containers.py:369-376 (_padded_backing) */
static int padded_backing(const pbuf* b, const int64_t* order, const int64_t* slots, int64_t ncl, int M, pbuf* out) {
  if (pbuf_alloc(out, ncl * M)) return ORC_NOMEM;
  for (int64_t k = 0; k < out->n; ++k) { out->id[k] = -1; out->own[k] = DUMMY; }
  for (int64_t k = 0; k < b->n; ++k) {
    int64_t s = slots[k], o = order[k];
    out->x[s] = b->x[o]; out->y[s] = b->y[o]; out->z[s] = b->z[o];
    out->own[s] = b->own[o]; out->id[s] = b->id[o];
  }
  return ORC_OK;
}

/* containers.py:393-406 (_compute_aabbs): dummies parked at the AABB min. */
static void compute_aabbs(pbuf* b, int64_t ncl, int M, double* mn, double* mx) {
  double* pos[3] = {b->x, b->y, b->z};
  for (int64_t c = 0; c < ncl; ++c) {
    for (int ax = 0; ax < 3; ++ax) {
      double lo = INFINITY, hi = -INFINITY;
      for (int t = 0; t < M; ++t) {
        int64_t s = c * M + t;
        if (b->own[s] == DUMMY) continue;
        double v = pos[ax][s];
        if (v < lo) lo = v;   /* np.min / np.max over real entries */
        if (v > hi) hi = v;
      }
      for (int t = 0; t < M; ++t) {
        int64_t s = c * M + t;
        if (b->own[s] == DUMMY) pos[ax][s] = lo;
      }
      mn[c * 3 + ax] = lo; mx[c * 3 + ax] = hi;
    }
  }
}

/* containers.py:271-273 (_box_distance_sq), summed x, y, z in order. */
static inline double box_d2(const double* amin, const double* amax, const double* bmin, const double* bmax) {
  double s = 0.0;
  for (int ax = 0; ax < 3; ++ax) {
    double u = amin[ax] - bmax[ax], v = bmin[ax] - amax[ax];
    double m = u > v ? u : v;
    double g = m > 0.0 ? m : 0.0;
    s = ax == 0 ? g * g : s + g * g;
  }
  return s;
}

/* traversals.py:269-287 (_greedy_base_colors) */
static int greedy_colors(int64_t n, int64_t** lists, const int64_t* nl, int32_t* colors, int32_t* ncol) {
  /* writers[z] = bases k (ascending) whose write set {k} U lists[k] contains z */
  int64_t* wcount = calloc(n + 1, 8);
  if (!wcount) return ORC_NOMEM;
  for (int64_t k = 0; k < n; ++k) { wcount[k]++; for (int64_t t = 0; t < nl[k]; ++t) wcount[lists[k][t]]++; }
  int64_t* wstart = malloc((n + 1) * 8);
  int64_t acc = 0;
  for (int64_t k = 0; k < n; ++k) { wstart[k] = acc; acc += wcount[k]; }
  wstart[n] = acc;
  int64_t* writers = malloc((acc + 1) * 8); int64_t* cur = malloc((n + 1) * 8);
  memcpy(cur, wstart, n * 8);
  for (int64_t k = 0; k < n; ++k) {
    writers[cur[k]++] = k;
    for (int64_t t = 0; t < nl[k]; ++t) { int64_t z = lists[k][t]; writers[cur[z]++] = k; }
  }
  /* writers[z] must be ascending in k: k is pushed in ascending order per z */
  int32_t maxc = -1;
  int32_t cap = 64; uint8_t* used = calloc(cap, 1);
  for (int64_t k = 0; k < n; ++k) colors[k] = -1;
  for (int64_t k = 0; k < n; ++k) {
    memset(used, 0, cap);
    for (int64_t t = -1; t < nl[k]; ++t) {
      int64_t z = t < 0 ? k : lists[k][t];
      for (int64_t w = wstart[z]; w < wstart[z + 1]; ++w) {
        int64_t o = writers[w];
        if (o != k && colors[o] >= 0) {
          if (colors[o] >= cap) { int32_t nc = cap * 2; while (nc <= colors[o]) nc *= 2; used = realloc(used, nc); memset(used + cap, 0, nc - cap); cap = nc; }
          used[colors[o]] = 1;
        }
      }
    }
    int32_t c = 0;
    while (c < cap && used[c]) ++c;
    colors[k] = c;
    if (c > maxc) maxc = c;
  }
  *ncol = maxc + 1 > 0 ? maxc + 1 : 1;
  free(wcount); free(wstart); free(writers); free(cur); free(used);
  return ORC_OK;
}

/* driver.py:107-129 with VerletClusterContainer (containers.py:302-479) and
 * the vcl schedule (traversals.py:244-266).  Dense O(C^2) cluster lists as in
 * the reference (containers.py:276-299): use at small sizes only. */
int orc_force_phase_vcl(int64_t n, const double* x, const double* y, const double* z,
                        const int8_t* own, const double* lo, const double* hi, const int32_t* periodic,
                        double eps, double sigma, double cutoff, double skin, int M,
                        int newton3, int a, int b, int V,
                        double* fx, double* fy, double* fz, orc_stats* st,
                        int64_t* n_clusters_out, int32_t* n_colors_out) {
  memset(st, 0, sizeof(*st));
  int rc = check_pattern(a, b, V);
  if (rc) return rc;
  if (M < 2) return ORC_CONFIG;
  obox bx; make_box(&bx, lo, hi, periodic);
  pbuf in; wrap_input(&in, n, x, y, z, own);
  int64_t* ids = malloc((n + 1) * 8);
  for (int64_t k = 0; k < n; ++k) ids[k] = k;
  in.id = ids;
  double length = cutoff + skin;
  double limit = length * length;
  vcl_t c; memset(&c, 0, sizeof(c)); c.M = M; c.col = length;
  int64_t *order = NULL, *counts = NULL, *horder = NULL, *hslots = NULL, *hcounts = NULL;
  int64_t** lists = NULL; int64_t* nl = NULL; int64_t** hl = NULL; int64_t* nhl = NULL;
  int32_t* colors = NULL;
  pbuf halo; memset(&halo, 0, sizeof(halo));
  unitvec v = {0};
  if ((rc = chunk_columns(&in, &bx, length, M, &order, &c.slots, &counts, &c.n_cl))) goto out;
  c.perm = order;
  if ((rc = padded_backing(&in, order, c.slots, c.n_cl, M, &c.ob))) goto out;
  c.amin = malloc((c.n_cl * 3 + 1) * 8); c.amax = malloc((c.n_cl * 3 + 1) * 8);
  compute_aabbs(&c.ob, c.n_cl, M, c.amin, c.amax);
  /* neighbor lists (containers.py:276-299) */
  lists = calloc(c.n_cl + 1, sizeof(int64_t*)); nl = calloc(c.n_cl + 1, 8);
  for (int64_t k = 0; k < c.n_cl; ++k) {
    int64_t cap = 16; lists[k] = malloc(cap * 8);
    for (int64_t zz = 0; zz < c.n_cl; ++zz) {
      if (newton3 ? (zz <= k) : (zz == k)) continue;
      if (box_d2(c.amin + 3 * k, c.amax + 3 * k, c.amin + 3 * zz, c.amax + 3 * zz) <= limit) {
        if (nl[k] == cap) { cap *= 2; lists[k] = realloc(lists[k], cap * 8); }
        lists[k][nl[k]++] = zz;
      }
    }
  }
  /* refresh: halo clusters + halo links (containers.py:431-469) */
  if ((rc = build_halo(&in, &bx, length, &halo))) goto out;
  hl = calloc(c.n_cl + 1, sizeof(int64_t*)); nhl = calloc(c.n_cl + 1, 8);
  if (halo.n) {
    if ((rc = chunk_columns(&halo, &bx, length, M, &horder, &hslots, &hcounts, &c.n_hcl))) goto out;
    if ((rc = padded_backing(&halo, horder, hslots, c.n_hcl, M, &c.hb))) goto out;
    c.hmin = malloc((c.n_hcl * 3 + 1) * 8); c.hmax = malloc((c.n_hcl * 3 + 1) * 8);
    compute_aabbs(&c.hb, c.n_hcl, M, c.hmin, c.hmax);
    for (int64_t k = 0; k < c.n_cl; ++k) {
      int64_t cap = 16; hl[k] = malloc(cap * 8);
      for (int64_t h = 0; h < c.n_hcl; ++h) {
        if (box_d2(c.amin + 3 * k, c.amax + 3 * k, c.hmin + 3 * h, c.hmax + 3 * h) <= limit) {
          if (nhl[k] == cap) { cap *= 2; hl[k] = realloc(hl[k], cap * 8); }
          hl[k][nhl[k]++] = h;
        }
      }
    }
  } else {
    if ((rc = pbuf_alloc(&c.hb, 0))) goto out;
  }
  /* schedule (traversals.py:244-266) */
  colors = malloc((c.n_cl + 1) * 4);
  int32_t ncol = 1;
  if (newton3) { if ((rc = greedy_colors(c.n_cl, lists, nl, colors, &ncol))) goto out; }
  else for (int64_t k = 0; k < c.n_cl; ++k) colors[k] = 0;
  for (int64_t k = 0; k < c.n_cl; ++k) {
    unit u = {k * M, M, k * M, M, 0, (int8_t)newton3, 1, colors[k], k, 0};
    if (uv_push(&v, u)) { rc = ORC_NOMEM; goto out; }
    for (int64_t t = 0; t < nl[k]; ++t) {
      unit w = {k * M, M, lists[k][t] * M, M, 0, (int8_t)newton3, 0, colors[k], k, 0};
      if (uv_push(&v, w)) { rc = ORC_NOMEM; goto out; }
    }
    for (int64_t t = 0; t < nhl[k]; ++t) {
      unit w = {k * M, M, hl[k][t] * M, M, 1, 0, 0, colors[k], k, 0};
      if (uv_push(&v, w)) { rc = ORC_NOMEM; goto out; }
    }
  }
  finish_units(&v);
  ljk kk = make_ljk(eps, sigma, cutoff);
  rc = execute_units(&v, &c.ob, &c.hb, &kk, a, b, V, st, 1);
  /* containers.py:475-479 (collect_forces) */
  for (int64_t q = 0; q < n; ++q) {
    int64_t o = c.perm[q], s = c.slots[q];
    fx[o] = c.ob.fx[s]; fy[o] = c.ob.fy[s]; fz[o] = c.ob.fz[s];
  }
  if (n_clusters_out) *n_clusters_out = c.n_cl;
  if (n_colors_out) *n_colors_out = ncol;
out:
  if (lists) for (int64_t k = 0; k < c.n_cl; ++k) free(lists[k]);
  if (hl) for (int64_t k = 0; k < c.n_cl; ++k) free(hl[k]);
  free(lists); free(nl); free(hl); free(nhl); free(colors); free(v.u);
  free(order); free(counts); free(horder); free(hslots); free(hcounts);
  free(c.slots); free(c.amin); free(c.amax); free(c.hmin); free(c.hmax);
  pbuf_free(&c.ob); pbuf_free(&c.hb); pbuf_free(&halo); free(ids);
  return rc;
}

/* Cluster structure of the owned particles (containers.py:343-406) for
 * bit-exact checks of the GPU cluster build: order (perm), slots, counts,
 * AABBs and padded positions. */
int orc_vcl_structure(int64_t n, const double* x, const double* y, const double* z,
                      const double* lo, const double* hi, double length, int M,
                      int64_t* order, int64_t* slots, int64_t* counts, int64_t* ncl_out,
                      double* amin, double* amax, double* px, double* py, double* pz) {
  obox bx; int32_t per[3] = {0, 0, 0}; make_box(&bx, lo, hi, per);
  int8_t* own = calloc(n + 1, 1);
  pbuf in; wrap_input(&in, n, x, y, z, own);
  int64_t* ids = malloc((n + 1) * 8);
  for (int64_t k = 0; k < n; ++k) ids[k] = k;
  in.id = ids;
  int64_t *o, *s, *cnt, ncl;
  int rc = chunk_columns(&in, &bx, length, M, &o, &s, &cnt, &ncl);
  if (rc) { free(own); free(ids); return rc; }
  memcpy(order, o, n * 8); memcpy(slots, s, n * 8); memcpy(counts, cnt, ncl * 8);
  pbuf pb;
  rc = padded_backing(&in, o, s, ncl, M, &pb);
  if (!rc) {
    compute_aabbs(&pb, ncl, M, amin, amax);
    memcpy(px, pb.x, ncl * M * 8); memcpy(py, pb.y, ncl * M * 8); memcpy(pz, pb.z, ncl * M * 8);
    pbuf_free(&pb);
  }
  *ncl_out = ncl;
  free(o); free(s); free(cnt); free(own); free(ids);
  return rc;
}

/* ------------------------------------------------------ Verlet lists (ext) */
/* Extension (no reference implementation; SPEC.md:8 excludes it).  Candidates
 * come from the linked-cells grid built with interaction_length = rc + skin
 * (containers.py:71-139); a pair (i, j) is listed iff r2 < (rc+skin)^2 with r2
 * evaluated exactly as executor.py:93-94.  Lists are per owned particle in the
 * cell-sorted order; candidates are the owned particles of the 27 cells
 * (itertools.product order, cell order) followed by the images binned to
 * those cells.  Unlike buffer_at (containers.py:178-184) no image is shadowed
 * by owned particles of the same cell, so images of particles that sit
 * outside [lo, hi) still interact (the physically exact pair set).  Half
 * lists (newton3): owned j only if j's sorted index > i; images always (the
 * owned side is i, traversals.py:157-160). */
static int vl_build(const lc_t* c, double rl2, int newton3, int64_t** off_o, int64_t** nbr_o, int8_t** halo_o) {
  init_dirs();
  int64_t n = c->ob.n;
  int64_t* off = malloc((n + 1) * 8);
  int64_t cap = 1024, cnt = 0;
  int64_t* nbr = malloc(cap * 8); int8_t* hal = malloc(cap);
  if (!off || !nbr || !hal) return ORC_NOMEM;
  for (int64_t p = 0; p < n; ++p) {
    off[p] = cnt;
    if (c->ob.own[p] != OWNED) continue;
    int64_t cell = lc_cell_of(c, c->ob.x[p], c->ob.y[p], c->ob.z[p], 0);
    int64_t x, y, z; coords_of(c, cell, &x, &y, &z);
    for (int ih = 0; ih < 2; ++ih) {
      for (int d = 0; d < 27; ++d) {
        int64_t nlin = (x + ALL[d][0]) + c->tdims[0] * ((y + ALL[d][1]) + c->tdims[1] * (z + ALL[d][2]));
        int64_t o = ih ? c->h_start[nlin] : c->o_start[nlin];
        int64_t l = ih ? c->h_count[nlin] : c->o_count[nlin];
        const pbuf* J = ih ? &c->hb : &c->ob;
        for (int64_t q = o; q < o + l; ++q) {
          if (!ih && q == p) continue;
          if (J->own[q] == DUMMY) continue;
          if (newton3 && !ih && q < p) continue;
          double dx = c->ob.x[p] - J->x[q];
          double dy = c->ob.y[p] - J->y[q];
          double dz = c->ob.z[p] - J->z[q];
          double r2 = dx * dx + dy * dy + dz * dz;
          if (!(r2 < rl2)) continue;
          if (cnt == cap) { cap *= 2; nbr = realloc(nbr, cap * 8); hal = realloc(hal, cap); }
          nbr[cnt] = q; hal[cnt] = (int8_t)ih; ++cnt;
        }
      }
    }
  }
  off[n] = cnt;
  *off_o = off; *nbr_o = nbr; *halo_o = hal;
  return ORC_OK;
}

/* VL force phase (extension) at the build positions.  Stats per DESIGN.md:
 * i-tiles of `a` consecutive owned-backing particles; each tile's j-stream is
 * padded to the longest list in the tile and chunked by b. */
int orc_force_phase_vl(int64_t n, const double* x, const double* y, const double* z,
                       const int8_t* own, const double* lo, const double* hi, const int32_t* periodic,
                       double eps, double sigma, double cutoff, double skin,
                       int newton3, int a, int b, int V,
                       double* fx, double* fy, double* fz, orc_stats* st, int64_t* n_entries) {
  memset(st, 0, sizeof(*st));
  int rc = check_pattern(a, b, V);
  if (rc) return rc;
  obox bx; make_box(&bx, lo, hi, periodic);
  pbuf in; wrap_input(&in, n, x, y, z, own);
  int64_t* ids = malloc((n + 1) * 8);
  for (int64_t k = 0; k < n; ++k) ids[k] = k;
  in.id = ids;
  double length = cutoff + skin;
  lc_t c;
  if ((rc = lc_init(&c, &bx, length))) { free(ids); return rc; }
  pbuf halo;
  if ((rc = build_halo(&in, &bx, length, &halo))) { free(ids); return rc; }
  int64_t *off = NULL, *nbr = NULL; int8_t* hal = NULL;
  if ((rc = lc_build(&c, &in, &halo))) goto out;
  if ((rc = vl_build(&c, length * length, newton3, &off, &nbr, &hal))) goto out;
  ljk k = make_ljk(eps, sigma, cutoff);
  kahan ep = {0, 0}, vr = {0, 0};
  int64_t pairs = 0, useful = 0, inv = 0;
  int64_t N = c.ob.n;
  for (int64_t p = 0; p < N; ++p) {
    if (c.ob.own[p] != OWNED) continue;
    double px = c.ob.x[p], py = c.ob.y[p], pz = c.ob.z[p];
    double ax = 0.0, ay = 0.0, az = 0.0;
    for (int64_t e = off[p]; e < off[p + 1]; ++e) {
      pbuf* J = hal[e] ? &c.hb : &c.ob;
      int64_t q = nbr[e];
      int n3 = newton3 && !hal[e];
      double dx = px - J->x[q];
      double dy = py - J->y[q];
      double dz = pz - J->z[q];
      double r2 = dx * dx + dy * dy + dz * dz;
      if (r2 >= k.rc2) continue;
      if (r2 == 0.0) { rc = ORC_OVERLAP; st->overlap = 1; goto out; }
      double s2 = k.sigma2 / r2;
      double s6 = s2 * s2 * s2;
      double f = k.eps24 * (2.0 * s6 * s6 - s6) / r2;
      ax += f * dx; ay += f * dy; az += f * dz;
      if (n3) { J->fx[q] -= f * dx; J->fy[q] -= f * dy; J->fz[q] -= f * dz; }
      double w = n3 ? 1.0 : 0.5;
      kadd(&ep, w * (k.eps4 * (s6 * s6 - s6)));
      kadd(&vr, w * (f * r2));
      pairs += 1;
    }
    c.ob.fx[p] += ax; c.ob.fy[p] += ay; c.ob.fz[p] += az;
  }
  /* stats over i-tiles of a consecutive backing slots */
  for (int64_t t0 = 0; t0 < N; t0 += a) {
    int64_t mx = 0;
    for (int64_t p = t0; p < t0 + a && p < N; ++p) {
      int64_t L = off[p + 1] - off[p];
      useful += L;
      if (L > mx) mx = L;
    }
    inv += cdiv(mx, b);
  }
  st->kernel_invocations = inv;
  st->lane_slots = inv * V;
  st->useful_interactions = useful;
  st->pair_interactions = pairs;
  st->epot = ep.s + ep.c; st->virial = vr.s + vr.c;
  if (n_entries) *n_entries = off[N];
  for (int64_t q = 0; q < n; ++q) {
    int64_t s = c.perm[q];
    fx[s] = c.ob.fx[q]; fy[s] = c.ob.fy[q]; fz[s] = c.ob.fz[q];
  }
out:
  free(off); free(nbr); free(hal);
  lc_free(&c); pbuf_free(&halo); free(ids);
  return rc;
}

/* VL pair set for bit-exact comparison: (id_i, id_j, j_is_halo) triples in
 * list order.  Returns the count; arrays must hold max_out entries. */
int64_t orc_vl_pairs(int64_t n, const double* x, const double* y, const double* z,
                     const double* lo, const double* hi, const int32_t* periodic,
                     double length, int newton3, int64_t max_out,
                     int64_t* pi, int64_t* pj, int8_t* ph) {
  obox bx; make_box(&bx, lo, hi, periodic);
  int8_t* own = calloc(n + 1, 1);
  pbuf in; wrap_input(&in, n, x, y, z, own);
  int64_t* ids = malloc((n + 1) * 8);
  for (int64_t k = 0; k < n; ++k) ids[k] = k;
  in.id = ids;
  lc_t c;
  int64_t ret = -1;
  if (lc_init(&c, &bx, length)) { free(own); free(ids); return -2; }
  pbuf halo;
  build_halo(&in, &bx, length, &halo);
  int64_t *off = NULL, *nbr = NULL; int8_t* hal = NULL;
  if (lc_build(&c, &in, &halo)) goto out;
  if (vl_build(&c, length * length, newton3, &off, &nbr, &hal)) goto out;
  ret = off[c.ob.n];
  if (ret > max_out) { ret = -3; goto out; }
  for (int64_t p = 0; p < c.ob.n; ++p)
    for (int64_t e = off[p]; e < off[p + 1]; ++e) {
      pi[e] = c.ob.id[p];
      pj[e] = hal[e] ? c.hb.id[nbr[e]] : c.ob.id[nbr[e]];
      ph[e] = hal[e];
    }
out:
  free(off); free(nbr); free(hal);
  lc_free(&c); pbuf_free(&halo); free(own); free(ids);
  return ret;
}

/* ------------------------------------------------ integrator + boundaries */
/* integrator.py:21-48: phase 0 = pre-force, 1 = post-force. */
void orc_verlet(int64_t n, int phase, double dt, double mass,
                double* x, double* y, double* z, double* vx, double* vy, double* vz,
                double* fx, double* fy, double* fz, double* ox, double* oy, double* oz) {
  double h = 0.5 / mass;
  double* X[3] = {x, y, z}; double* Vv[3] = {vx, vy, vz}; double* F[3] = {fx, fy, fz}; double* O[3] = {ox, oy, oz};
  for (int ax = 0; ax < 3; ++ax) {
    if (phase == 0) {
      double c = h * dt * dt;
      for (int64_t k = 0; k < n; ++k) {
        X[ax][k] = X[ax][k] + (Vv[ax][k] * dt + F[ax][k] * c);
        O[ax][k] = F[ax][k];
        F[ax][k] = 0.0;
      }
    } else {
      double c = h * dt;
      for (int64_t k = 0; k < n; ++k) Vv[ax][k] = Vv[ax][k] + (F[ax][k] + O[ax][k]) * c;
    }
  }
}

/* numpy's np.mod for doubles (npy_divmod's remainder). */
static double py_mod(double a, double b) {
  double m = fmod(a, b);
  if (m != 0.0) { if ((b < 0) != (m < 0)) m += b; }
  else m = copysign(0.0, b);
  return m;
}

/* domain.py:69-94 (apply_boundaries); returns 1 on divergence. */
int orc_apply_boundaries(int64_t n, const double* lo, const double* hi, const int32_t* periodic,
                         double* x, double* y, double* z, double* vx, double* vy, double* vz) {
  double* X[3] = {x, y, z}; double* Vv[3] = {vx, vy, vz};
  for (int ax = 0; ax < 3; ++ax) {
    double l = lo[ax], h = hi[ax], L = h - l;
    for (int64_t k = 0; k < n; ++k)
      if (X[ax][k] > h + L || X[ax][k] < l - L) return 1;
    if (periodic[ax]) {
      for (int64_t k = 0; k < n; ++k) X[ax][k] = py_mod(X[ax][k] - l, L) + l;
    } else {
      for (int64_t k = 0; k < n; ++k) {
        if (X[ax][k] > h) { X[ax][k] = 2.0 * h - X[ax][k]; Vv[ax][k] = -Vv[ax][k]; }
      }
      for (int64_t k = 0; k < n; ++k) {
        if (X[ax][k] < l) { X[ax][k] = 2.0 * l - X[ax][k]; Vv[ax][k] = -Vv[ax][k]; }
      }
    }
  }
  return 0;
}

/* ------------------------------------------- prepared execution (baseline) */
/* The reference's metric region covers execute_packed only (driver.py:203-207);
 * rebuild / halo / schedule / pack happen before it.  orc_lc_prepare does the
 * latter once; orc_lc_execute times like execute_packed.  With Newton3 off the
 * units of one i-cell write only that cell, so they are grouped per i-cell and
 * the groups run in parallel (OpenMP) -- in unit order within a group, which
 * keeps every particle's summation order, i.e. bitwise the sequential result. */
typedef struct {
  lc_t c; pbuf halo; unitvec v; ljk k;
  int a, b, V, newton3;
  int64_t n; int64_t* ids;
  int64_t ngroups; int64_t* gstart; int64_t* gunits;
  int64_t inv, useful;
} orc_lc_handle;

static int unit_by_i(const void* x, const void* y) {
  const unit* const* a = x; const unit* const* b = y;
  if ((*a)->i_off != (*b)->i_off) return (*a)->i_off < (*b)->i_off ? -1 : 1;
  return (*a)->seq < (*b)->seq ? -1 : ((*a)->seq > (*b)->seq);
}

void* orc_lc_prepare(int64_t n, const double* x, const double* y, const double* z,
                     const int8_t* own, const double* lo, const double* hi, const int32_t* periodic,
                     double eps, double sigma, double cutoff, double skin,
                     int trav, int newton3, int a, int b, int V, int* status) {
  orc_lc_handle* h = calloc(1, sizeof(orc_lc_handle));
  *status = check_pattern(a, b, V);
  if (*status) { free(h); return NULL; }
  obox bx; make_box(&bx, lo, hi, periodic);
  pbuf in; wrap_input(&in, n, x, y, z, own);
  h->ids = malloc((n + 1) * 8);
  for (int64_t k = 0; k < n; ++k) h->ids[k] = k;
  in.id = h->ids;
  h->n = n; h->a = a; h->b = b; h->V = V; h->newton3 = newton3;
  if ((*status = lc_init(&h->c, &bx, cutoff + skin))) { free(h->ids); free(h); return NULL; }
  if ((*status = build_halo(&in, &bx, cutoff + skin, &h->halo))) { free(h->ids); free(h); return NULL; }
  if ((*status = lc_build(&h->c, &in, &h->halo))) return h;
  if ((*status = schedule_lc(&h->c, trav, newton3, &h->v))) return h;
  h->k = make_ljk(eps, sigma, cutoff);
  /* geometric stats once (they do not change between executions) */
  for (int64_t u = 0; u < h->v.n; ++u) {
    const unit* w = &h->v.u[u];
    const pbuf* J = w->j_halo ? &h->c.hb : &h->c.ob;
    h->inv += cdiv(w->i_len, a) * cdiv(w->j_len, b);
    if (w->same) h->useful += self_pair_slots(&h->c.ob, w->i_off, w->i_len, w->newton3);
    else {
      int64_t io, in_, jo, jn;
      span_counts(&h->c.ob, w->i_off, w->i_len, &io, &in_);
      span_counts(J, w->j_off, w->j_len, &jo, &jn);
      h->useful += io * jn;
    }
  }
  if (!newton3) {
    unit** ptrs = malloc((h->v.n + 1) * sizeof(unit*));
    for (int64_t u = 0; u < h->v.n; ++u) ptrs[u] = &h->v.u[u];
    qsort(ptrs, h->v.n, sizeof(unit*), unit_by_i);
    h->gunits = malloc((h->v.n + 1) * 8);
    h->gstart = malloc((h->v.n + 2) * 8);
    int64_t g = 0;
    for (int64_t u = 0; u < h->v.n; ++u) {
      h->gunits[u] = ptrs[u] - h->v.u;
      if (u == 0 || ptrs[u]->i_off != ptrs[u - 1]->i_off) h->gstart[g++] = u;
    }
    h->gstart[g] = h->v.n;
    h->ngroups = g;
    free(ptrs);
  }
  *status = ORC_OK;
  return h;
}

int orc_lc_execute(void* hv, int threads, orc_stats* st, double* fx, double* fy, double* fz) {
  orc_lc_handle* h = hv;
  memset(st, 0, sizeof(*st));
  pbuf* ob = &h->c.ob;
  memset(ob->fx, 0, ob->n * 8); memset(ob->fy, 0, ob->n * 8); memset(ob->fz, 0, ob->n * 8);
  int64_t total = 0; int bad = 0;
  if (h->newton3 || threads <= 1) {
    for (int64_t u = 0; u < h->v.n && !bad; ++u) {
      const unit* w = &h->v.u[u];
      const pbuf* J = w->j_halo ? &h->c.hb : ob;
      int64_t p = sweep_span(ob, J, w->i_off, w->i_len, w->j_off, w->j_len, w->newton3, w->same,
                             &h->k, NULL, NULL);
      if (p < 0) bad = 1; else total += p;
    }
  } else {
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic, 64) num_threads(threads) reduction(+:total) reduction(|:bad)
#endif
    for (int64_t g = 0; g < h->ngroups; ++g) {
      for (int64_t t = h->gstart[g]; t < h->gstart[g + 1]; ++t) {
        const unit* w = &h->v.u[h->gunits[t]];
        const pbuf* J = w->j_halo ? &h->c.hb : ob;
        int64_t p = sweep_span(ob, J, w->i_off, w->i_len, w->j_off, w->j_len, 0, w->same,
                               &h->k, NULL, NULL);
        if (p < 0) bad = 1; else total += p;
      }
    }
  }
  if (bad) { st->overlap = 1; return ORC_OVERLAP; }
  st->kernel_invocations = h->inv;
  st->lane_slots = h->inv * h->V;
  st->useful_interactions = h->useful;
  st->pair_interactions = total;
  if (fx) {
    for (int64_t q = 0; q < h->n; ++q) {
      int64_t s = h->c.perm[q];
      fx[s] = ob->fx[q]; fy[s] = ob->fy[q]; fz[s] = ob->fz[q];
    }
  }
  return ORC_OK;
}

void orc_lc_free(void* hv) {
  orc_lc_handle* h = hv;
  if (!h) return;
  lc_free(&h->c); pbuf_free(&h->halo); free(h->v.u); free(h->ids);
  free(h->gstart); free(h->gunits); free(h);
}

int orc_omp_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
