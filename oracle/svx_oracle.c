/*
 * svx_oracle.c -- CPU restatement of the reference's integration path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker and the CPU
 * baseline ("port") for the B200 engine; only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  The
 * product (paper_2512_12945_b200/libsvx.so) never links or calls it.
 *
 * It restates, operation for operation, the reference semvox package
 * (/root/reference/pkg/src/semvox):
 *   prep      integrate_frame masks and ray setup     fusion.py:228-263
 *   K1        _dda_ray band walk                      _core.pyx:478-579 (_pycore.py:326-372)
 *   rows      row_distances_weights                   _pycore.py:384-396, _core.pyx:553-566
 *   drop      w <= 0 rows                              _core.pyx:688-702
 *   K2        (voxel key, row) sort, 21-bit pack      _core.pyx:707-738 (_pycore.py:375-381,484-491)
 *   K3        grouping                                _core.pyx:742-753
 *   K4        first-occurrence leaf allocation        _core.pyx:377-420, 248-280
 *   K5        sequential per-voxel reduce             _core.pyx:759-843
 *   K6        apply_tsdf / apply_closed / apply_open  _pycore.py:399-446
 *   queries   active_slots order, probe, cosine,      _core.pyx:424-463, 324-375,
 *             classify_means, label readouts          gaussian.py:132-170, dirichlet.py:81-88,
 *                                                     evalbench.py:30-55
 * Compiled with -ffp-contract=off (as pkg/setup.py:14) so double expressions
 * round exactly like the reference's C++ and numpy.  Parity against the real
 * reference is pinned by tests/golden (fixtures generated from semvox itself,
 * tests/golden/make_golden.py) and the reference's own known-answer cases.
 *
 * Layout note: payloads are stored per active voxel (dense ids) rather than
 * per leaf; the observable semantics (active set, active order = leaf
 * allocation order then slot order, values, backgrounds) are the reference's.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_COORD_LIMIT (1LL << 30)
#define ORC_PACK_BITS 21
#define ORC_STEP_BUDGET (1LL << 20)

enum { ORC_OK = 0, ORC_E_CONFIG = 1, ORC_E_PAYLOAD = 2, ORC_E_INPUT = 3, ORC_E_RANGE = 4,
       ORC_E_INTERNAL = 6, ORC_E_NOMEM = 8 };

typedef struct {
    double voxel_size, truncation, max_range;
    int32_t weight_fn, space_carving, sem_kind, num_classes, last_wins, feature_dim;
    double prior_beta, lambda_floor;
    int32_t tsdf_f32;   /* store d, w rounded through float (compact mode) */
    int32_t sem_f32;    /* store counts / m / beta rounded through float (f32 dtypes) */
    int32_t threads;
} orc_config;

typedef struct {
    int64_t points_in, points_used, skipped_nonfinite, skipped_range, skipped_degenerate,
        skipped_bad_label, band_hits, touched_voxels, new_blocks, new_voxels;
    double t_emit_ms, t_sort_ms, t_group_ms, t_ensure_ms, t_update_ms;
} orc_report;

typedef struct {
    orc_config cfg;
    int P;  /* payload width: C or D */
    /* leaves */
    int64_t nleaves, lcap;
    int32_t* lcoord;  /* 3 per leaf */
    uint64_t* lmask;  /* 8 per leaf */
    int32_t* lslot;   /* 512 per leaf: voxel id or -1 */
    /* leaf hash */
    int64_t hcap, hcount;
    int32_t* hkey;    /* 3 per slot */
    int32_t* hval;    /* -1 empty */
    /* voxels */
    int64_t nvox, vcap;
    double *d, *w, *s0, *s1;
    int64_t frames;
} orc_map;

static const char* g_msg = "";
const char* orc_last_error(void) { return g_msg; }
static int orc_fail(int code, const char* msg) { g_msg = msg; return code; }

static double now_ms(void) {
#ifdef _OPENMP
    return omp_get_wtime() * 1e3;
#else
    return 0.0;
#endif
}

static uint64_t leaf_hash(int32_t a, int32_t b, int32_t c) {
    uint64_t h = (uint64_t)(uint32_t)a * 0x9E3779B97F4A7C15ULL;
    h ^= ((uint64_t)(uint32_t)b + 0x632BE59BD9B4E019ULL) * 0xBF58476D1CE4E5B9ULL;
    h ^= ((uint64_t)(uint32_t)c + 0x85EBCA77C2B2AE63ULL) * 0x94D049BB133111EBULL;
    h ^= h >> 31;
    return h;
}

static int grow_hash(orc_map* m) {
    int64_t ncap = m->hcap ? 2 * m->hcap : 1024;
    int32_t* nk = (int32_t*)malloc(sizeof(int32_t) * 3 * ncap);
    int32_t* nv = (int32_t*)malloc(sizeof(int32_t) * ncap);
    if (!nk || !nv) { free(nk); free(nv); return ORC_E_NOMEM; }
    for (int64_t i = 0; i < ncap; ++i) nv[i] = -1;
    for (int64_t i = 0; i < m->hcap; ++i) {
        if (m->hval[i] < 0) continue;
        int32_t* k = m->hkey + 3 * i;
        int64_t pos = (int64_t)(leaf_hash(k[0], k[1], k[2]) & (uint64_t)(ncap - 1));
        while (nv[pos] >= 0) pos = (pos + 1) & (ncap - 1);
        memcpy(nk + 3 * pos, k, 12);
        nv[pos] = m->hval[i];
    }
    free(m->hkey); free(m->hval);
    m->hkey = nk; m->hval = nv; m->hcap = ncap;
    return ORC_OK;
}

static int64_t hash_find(const orc_map* m, int32_t a, int32_t b, int32_t c) {
    if (!m->hcap) return -1;
    int64_t pos = (int64_t)(leaf_hash(a, b, c) & (uint64_t)(m->hcap - 1));
    while (m->hval[pos] >= 0) {
        const int32_t* k = m->hkey + 3 * pos;
        if (k[0] == a && k[1] == b && k[2] == c) return m->hval[pos];
        pos = (pos + 1) & (m->hcap - 1);
    }
    return -1;
}

static void* grow(void* p, size_t elem, int64_t old, int64_t cap, int fill) {
    void* np = realloc(p, elem * (size_t)cap);
    if (np && fill >= 0) memset((char*)np + elem * (size_t)old, fill, elem * (size_t)(cap - old));
    return np;
}

/* _resolve_leaf_alloc (_core.pyx:248-280): find or append a leaf. */
static int64_t leaf_alloc(orc_map* m, int32_t a, int32_t b, int32_t c, int64_t* new_leaves) {
    int64_t id = hash_find(m, a, b, c);
    if (id >= 0) return id;
    if ((m->hcount + 1) * 2 > m->hcap && grow_hash(m)) return -1;
    if (m->nleaves == m->lcap) {
        int64_t cap = m->lcap ? 2 * m->lcap : 256;
        m->lcoord = (int32_t*)grow(m->lcoord, 12, m->lcap, cap, 0);
        m->lmask = (uint64_t*)grow(m->lmask, 64, m->lcap, cap, 0);
        m->lslot = (int32_t*)grow(m->lslot, 2048, m->lcap, cap, 0xFF);
        if (!m->lcoord || !m->lmask || !m->lslot) return -1;
        m->lcap = cap;
    }
    id = m->nleaves++;
    m->lcoord[3 * id] = a; m->lcoord[3 * id + 1] = b; m->lcoord[3 * id + 2] = c;
    int64_t pos = (int64_t)(leaf_hash(a, b, c) & (uint64_t)(m->hcap - 1));
    while (m->hval[pos] >= 0) pos = (pos + 1) & (m->hcap - 1);
    m->hkey[3 * pos] = a; m->hkey[3 * pos + 1] = b; m->hkey[3 * pos + 2] = c;
    m->hval[pos] = (int32_t)id;
    m->hcount++;
    (*new_leaves)++;
    return id;
}

static int reserve_voxels(orc_map* m, int64_t need) {
    if (need <= m->vcap) return ORC_OK;
    int64_t cap = m->vcap ? 2 * m->vcap : 4096;
    while (cap < need) cap *= 2;
    m->d = (double*)grow(m->d, 8, m->vcap, cap, -1);
    m->w = (double*)grow(m->w, 8, m->vcap, cap, -1);
    if (!m->d || !m->w) return ORC_E_NOMEM;
    if (m->cfg.sem_kind) {
        m->s0 = (double*)grow(m->s0, 8 * (size_t)m->P, m->vcap, cap, -1);
        if (!m->s0) return ORC_E_NOMEM;
    }
    if (m->cfg.sem_kind == 2) {
        m->s1 = (double*)grow(m->s1, 8 * (size_t)m->P, m->vcap, cap, -1);
        if (!m->s1) return ORC_E_NOMEM;
    }
    m->vcap = cap;
    return ORC_OK;
}

orc_map* orc_create(const orc_config* cfg) {
    orc_map* m = (orc_map*)calloc(1, sizeof(orc_map));
    if (!m) return NULL;
    m->cfg = *cfg;
    m->P = cfg->sem_kind == 1 ? cfg->num_classes : (cfg->sem_kind == 2 ? cfg->feature_dim : 0);
    if (grow_hash(m) || reserve_voxels(m, 4096)) { free(m); return NULL; }
    return m;
}

void orc_destroy(orc_map* m) {
    if (!m) return;
    free(m->lcoord); free(m->lmask); free(m->lslot); free(m->hkey); free(m->hval);
    free(m->d); free(m->w); free(m->s0); free(m->s1);
    free(m);
}

/* ---- K1: the fp64 band walk (_core.pyx:478-579) ---------------------------- */
typedef struct { int64_t i, j, k; double d, w; } orc_row;

static double store_f(double v, int f32) { return f32 ? (double)(float)v : v; }

/* Walk a ray; writes rows when out != NULL.  Returns emitted count or -1. */
static int64_t dda_ray(double ox, double oy, double oz, double ux, double uy, double uz,
                       double ts, double h, double trunc, int carving, int wfn, orc_row* out) {
    double t_lo = carving ? 0.0 : fmax(ts - trunc, 0.0);
    double t_hi = ts + trunc;
    double px = ox + ux * t_lo, py = oy + uy * t_lo, pz = oz + uz * t_lo;
    int64_t ci = (int64_t)floor(px / h), cj = (int64_t)floor(py / h), ck = (int64_t)floor(pz / h);
    int sx = ux == 0 ? 0 : (ux > 0 ? 1 : -1);
    int sy = uy == 0 ? 0 : (uy > 0 ? 1 : -1);
    int sz = uz == 0 ? 0 : (uz > 0 ? 1 : -1);
    double tmx, tmy, tmz, tdx, tdy, tdz;
    if (sx > 0) { tmx = t_lo + ((ci + 1) * h - px) / ux; tdx = h / fabs(ux); }
    else if (sx < 0) { tmx = t_lo + (ci * h - px) / ux; tdx = h / fabs(ux); }
    else { tmx = INFINITY; tdx = INFINITY; }
    if (sy > 0) { tmy = t_lo + ((cj + 1) * h - py) / uy; tdy = h / fabs(uy); }
    else if (sy < 0) { tmy = t_lo + (cj * h - py) / uy; tdy = h / fabs(uy); }
    else { tmy = INFINITY; tdy = INFINITY; }
    if (sz > 0) { tmz = t_lo + ((ck + 1) * h - pz) / uz; tdz = h / fabs(uz); }
    else if (sz < 0) { tmz = t_lo + (ck * h - pz) / uz; tdz = h / fabs(uz); }
    else { tmz = INFINITY; tdz = INFINITY; }
    double t_enter = t_lo;
    int64_t cnt = 0, k = 0;
    while (t_enter < t_hi) {
        if (k >= ORC_STEP_BUDGET) return -1;
        int axis = 0;
        double tmin = tmx;
        if (tmy < tmin) { axis = 1; tmin = tmy; }
        if (tmz < tmin) { axis = 2; tmin = tmz; }
        if (tmin > t_lo) {
            if (out) {
                /* row_distances_weights (_pycore.py:384-396) */
                double cx = (ci + 0.5) * h - ox, cy = (cj + 0.5) * h - oy, cz = (ck + 0.5) * h - oz;
                double proj = cx * ux + cy * uy + cz * uz;
                double dd = ts - proj;
                if (dd < -trunc) dd = -trunc;
                if (dd > trunc) dd = trunc;
                out[cnt].i = ci; out[cnt].j = cj; out[cnt].k = ck;
                out[cnt].d = dd;
                out[cnt].w = wfn == 1 ? (dd >= 0.0 ? 1.0 : (trunc + dd) / trunc) : 1.0;
            }
            ++cnt;
        }
        if (axis == 0) { ci += sx; tmx += tdx; }
        else if (axis == 1) { cj += sy; tmy += tdy; }
        else { ck += sz; tmz += tdz; }
        t_enter = tmin;
        ++k;
    }
    return cnt;
}

/* Single-ray band (raycast_band, _pycore.py:275-323): coords (cap x 3). */
int64_t orc_raycast_band(const double origin[3], const double endpoint[3], double h, double trunc,
                         int carving, int64_t* coords, int64_t cap) {
    double dx = endpoint[0] - origin[0], dy = endpoint[1] - origin[1], dz = endpoint[2] - origin[2];
    double ts = sqrt((dx * dx + dy * dy) + dz * dz);
    if (ts == 0.0) return 0;
    double ux = dx / ts, uy = dy / ts, uz = dz / ts;
    int64_t n = dda_ray(origin[0], origin[1], origin[2], ux, uy, uz, ts, h, trunc, carving, 0, NULL);
    if (n < 0) return -1;
    orc_row* rows = (orc_row*)malloc(sizeof(orc_row) * (size_t)(n ? n : 1));
    dda_ray(origin[0], origin[1], origin[2], ux, uy, uz, ts, h, trunc, carving, 0, rows);
    for (int64_t r = 0; r < n && r < cap; ++r) {
        coords[3 * r] = rows[r].i; coords[3 * r + 1] = rows[r].j; coords[3 * r + 2] = rows[r].k;
    }
    free(rows);
    return n;
}

/* ---- K2: stable LSD radix sort of (key, row) by key ------------------------- */
static void radix_sort(uint64_t* key, int64_t* row, uint64_t* k2, int64_t* r2, int64_t n, int bits) {
    for (int shift = 0; shift < bits; shift += 11) {
        int64_t cnt[2048];
        memset(cnt, 0, sizeof(cnt));
        for (int64_t i = 0; i < n; ++i) cnt[(key[i] >> shift) & 2047]++;
        int64_t s = 0;
        for (int b = 0; b < 2048; ++b) { int64_t c = cnt[b]; cnt[b] = s; s += c; }
        for (int64_t i = 0; i < n; ++i) {
            int64_t p = cnt[(key[i] >> shift) & 2047]++;
            k2[p] = key[i]; r2[p] = row[i];
        }
        memcpy(key, k2, 8 * (size_t)n);
        memcpy(row, r2, 8 * (size_t)n);
    }
}

/*
 * Integrate one frame.  points: (n,3) f64.  sensor != 0: points are in the
 * sensor frame and pose (4x4 row-major) maps them to the world as
 * ((R0 x + R1 y) + R2 z) + t (the engine's defined order; identical to the
 * reference's BLAS product for identity rotations).  sensor == 0: points are
 * world-frame and pose[3], pose[7], pose[11] hold the origin.
 */
/* Frame.points_world (fusion.py:98-100): `points @ R.T + t`.  numpy hands
 * an (n, 3) @ (3, 3) product with n >= 2 to OpenBLAS dgemm, whose microkernel
 * accumulates k = 0, 1, 2 with fused multiply-adds starting from the k = 0
 * product; a single row goes through the vector-matrix path, which starts
 * from the k = 1 product and fuses k = 0, then k = 2.  Both orders were
 * measured against numpy in the build container (make_golden.py rotated). */
static double world_pt(const double* pose, int r, double x, double y, double z, int single) {
    const double* R = pose + 4 * r;
    const double acc = single ? fma(R[0], x, R[1] * y) : fma(R[1], y, R[0] * x);
    return fma(R[2], z, acc) + R[3];
}

int orc_integrate(orc_map* m, const double* pts, int64_t n, const double pose[16], int sensor,
                  const int32_t* labels, const double* feats, orc_report* rep) {
    const orc_config* c = &m->cfg;
    memset(rep, 0, sizeof(*rep));
    rep->points_in = n;
    if (c->sem_kind == 1 && !labels) return orc_fail(ORC_E_PAYLOAD, "closed-set grid requires per-point labels");
    if (c->sem_kind == 2 && !feats) return orc_fail(ORC_E_PAYLOAD, "open-set grid requires per-point features");
    m->frames++;
    if (n == 0) return ORC_OK;
#ifdef _OPENMP
    if (c->threads > 0) omp_set_num_threads(c->threads);
#endif
    const double ox = pose[3], oy = pose[7], oz = pose[11];
    const double h = c->voxel_size, trunc = c->truncation;
    const int D = c->feature_dim;
    double t0 = now_ms();
    /* prep (fusion.py:228-263) */
    double* ray = (double*)malloc(sizeof(double) * 4 * (size_t)n);
    int64_t* cnt = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
    if (!ray || !cnt) { free(ray); free(cnt); return orc_fail(ORC_E_NOMEM, "out of memory"); }
    int64_t nf = 0, nr = 0, ndg = 0, nbl = 0, nused = 0, hits = 0;
    int budget = 0;
#pragma omp parallel for schedule(static) reduction(+ : nf, nr, ndg, nbl, nused, hits) reduction(| : budget)
    for (int64_t i = 0; i < n; ++i) {
        double x = pts[3 * i], y = pts[3 * i + 1], z = pts[3 * i + 2];
        double wx = x, wy = y, wz = z;
        if (sensor) {   /* points @ R.T + t in numpy/OpenBLAS order (world_pt) */
            wx = world_pt(pose, 0, x, y, z, n == 1);
            wy = world_pt(pose, 1, x, y, z, n == 1);
            wz = world_pt(pose, 2, x, y, z, n == 1);
        }
        int finite = isfinite(wx) && isfinite(wy) && isfinite(wz);
        double dx = wx - ox, dy = wy - oy, dz = wz - oz;
        double ts = sqrt((dx * dx + dy * dy) + dz * dz);
        if (!isfinite(ts)) ts = INFINITY;
        int degenerate = finite && ts == 0.0;
        int in_range = ts <= c->max_range;
        int keep = finite && !degenerate && in_range;
        nf += !finite;
        ndg += degenerate;
        nr += finite && !degenerate && !in_range;
        if (c->sem_kind == 1) {
            int good = labels[i] >= 1 && labels[i] <= c->num_classes;
            nbl += keep && !good;
            keep = keep && good;
        } else if (c->sem_kind == 2) {
            int good = 1;
            for (int q = 0; q < D; ++q) good = good && isfinite(feats[(int64_t)i * D + q]);
            nbl += keep && !good;
            keep = keep && good;
        }
        cnt[i] = 0;
        if (keep) {
            nused++;
            double ux = dx / ts, uy = dy / ts, uz = dz / ts;
            ray[4 * i] = ux; ray[4 * i + 1] = uy; ray[4 * i + 2] = uz; ray[4 * i + 3] = ts;
            int64_t e = dda_ray(ox, oy, oz, ux, uy, uz, ts, h, trunc, c->space_carving,
                                c->weight_fn, NULL);
            if (e < 0) budget = 1;
            else { cnt[i] = e; hits += e; }
        }
    }
    rep->skipped_nonfinite = nf; rep->skipped_range = nr; rep->skipped_degenerate = ndg;
    rep->skipped_bad_label = nbl; rep->points_used = nused; rep->band_hits = hits;
    if (budget) {
        free(ray); free(cnt);
        return orc_fail(ORC_E_INTERNAL, "ray band exceeds step budget; shrink max_range or grow voxels");
    }
    /* offsets + fill */
    int64_t total = 0;
    for (int64_t i = 0; i < n; ++i) { int64_t v = cnt[i]; cnt[i] = total; total += v; }
    cnt[n] = total;
    orc_row* rows = (orc_row*)malloc(sizeof(orc_row) * (size_t)(total ? total : 1));
    int64_t* rid = (int64_t*)malloc(sizeof(int64_t) * (size_t)(total ? total : 1));
    if (!rows || !rid) { free(ray); free(cnt); free(rows); free(rid); return orc_fail(ORC_E_NOMEM, "out of memory"); }
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        if (cnt[i + 1] == cnt[i]) continue;
        dda_ray(ox, oy, oz, ray[4 * i], ray[4 * i + 1], ray[4 * i + 2], ray[4 * i + 3], h, trunc,
                c->space_carving, c->weight_fn, rows + cnt[i]);
        for (int64_t r = cnt[i]; r < cnt[i + 1]; ++r) rid[r] = i;
    }
    /* drop zero-weight rows (_core.pyx:688-702) */
    int64_t R = 0;
    for (int64_t r = 0; r < total; ++r) {
        if (rows[r].w > 0.0) { rows[R] = rows[r]; rid[R] = rid[r]; ++R; }
    }
    double t1 = now_ms();
    rep->t_emit_ms = t1 - t0;
    if (R == 0) { free(ray); free(cnt); free(rows); free(rid); return ORC_OK; }
    int64_t mn[3] = {rows[0].i, rows[0].j, rows[0].k}, mx[3] = {rows[0].i, rows[0].j, rows[0].k};
    for (int64_t r = 1; r < R; ++r) {
        int64_t v[3] = {rows[r].i, rows[r].j, rows[r].k};
        for (int a = 0; a < 3; ++a) { if (v[a] < mn[a]) mn[a] = v[a]; if (v[a] > mx[a]) mx[a] = v[a]; }
    }
    for (int a = 0; a < 3; ++a) {
        if (mx[a] - mn[a] >= (1LL << ORC_PACK_BITS)) {
            free(ray); free(cnt); free(rows); free(rid);
            return orc_fail(ORC_E_INTERNAL, "frame voxel extent exceeds 2^21 per axis; shrink max_range or grow voxels");
        }
    }
    for (int a = 0; a < 3; ++a) {
        if (llabs(mn[a]) >= ORC_COORD_LIMIT || llabs(mx[a]) >= ORC_COORD_LIMIT) {
            free(ray); free(cnt); free(rows); free(rid);
            return orc_fail(ORC_E_RANGE, "voxel coordinate beyond +/-2^30 addressable range");
        }
    }
    /* K2: (key, row) order; rows are already in (point, step) order */
    uint64_t* key = (uint64_t*)malloc(8 * (size_t)R);
    uint64_t* k2 = (uint64_t*)malloc(8 * (size_t)R);
    int64_t* order = (int64_t*)malloc(8 * (size_t)R);
    int64_t* o2 = (int64_t*)malloc(8 * (size_t)R);
    for (int64_t r = 0; r < R; ++r) {
        key[r] = ((uint64_t)(rows[r].i - mn[0]) << (2 * ORC_PACK_BITS)) |
                 ((uint64_t)(rows[r].j - mn[1]) << ORC_PACK_BITS) | (uint64_t)(rows[r].k - mn[2]);
        order[r] = r;
    }
    radix_sort(key, order, k2, o2, R, 3 * ORC_PACK_BITS);
    free(k2); free(o2);
    double t2 = now_ms();
    rep->t_sort_ms = t2 - t1;
    /* K3: groups */
    int64_t* start = (int64_t*)malloc(8 * (size_t)(R + 1));
    int64_t U = 0;
    for (int64_t r = 0; r < R; ++r)
        if (r == 0 || key[r] != key[r - 1]) start[U++] = r;
    start[U] = R;
    rep->touched_voxels = U;
    double t3 = now_ms();
    rep->t_group_ms = t3 - t2;
    /* K4: ensure in first-occurrence order */
    int64_t* gvid = (int64_t*)malloc(8 * (size_t)U);
    char* gnew = (char*)malloc((size_t)U);
    int err = reserve_voxels(m, m->nvox + U);
    int64_t new_leaves = 0, new_vox = 0;
    for (int64_t g = 0; g < U && !err; ++g) {
        const orc_row* rw = &rows[order[start[g]]];
        int64_t leaf = leaf_alloc(m, (int32_t)(rw->i >> 3), (int32_t)(rw->j >> 3),
                                  (int32_t)(rw->k >> 3), &new_leaves);
        if (leaf < 0) { err = ORC_E_NOMEM; break; }
        int slot = (int)(((rw->i & 7) << 6) | ((rw->j & 7) << 3) | (rw->k & 7));
        int32_t* sl = &m->lslot[leaf * 512 + slot];
        gnew[g] = *sl < 0;
        if (*sl < 0) {
            *sl = (int32_t)(m->nvox + new_vox++);
            m->lmask[leaf * 8 + (slot >> 6)] |= 1ULL << (slot & 63);
        }
        gvid[g] = *sl;
    }
    double t4 = now_ms();
    rep->t_ensure_ms = t4 - t3;
    if (err) {
        free(ray); free(cnt); free(rows); free(rid); free(key); free(order); free(start);
        free(gvid); free(gnew);
        return orc_fail(err, "out of memory");
    }
    m->nvox += new_vox;
    rep->new_blocks = new_leaves;
    rep->new_voxels = new_vox;
    /* K5 + K6: sequential per-voxel reduce, then the apply arithmetic */
    const int P = m->P;
    const int kind = c->sem_kind;
#pragma omp parallel
    {
        double* sz = kind == 2 ? (double*)malloc(sizeof(double) * 2 * (size_t)D) : NULL;
        double* cntv = kind == 1 ? (double*)malloc(sizeof(double) * (size_t)P) : NULL;
#pragma omp for schedule(static)
        for (int64_t g = 0; g < U; ++g) {
            const int64_t v = gvid[g];
            const int isnew = gnew[g];
            double sw = 0.0, swd = 0.0, mind = INFINITY, maxd = -INFINITY;
            int last = 0;
            if (cntv) memset(cntv, 0, sizeof(double) * (size_t)P);
            if (sz) memset(sz, 0, sizeof(double) * 2 * (size_t)D);
            for (int64_t s = start[g]; s < start[g + 1]; ++s) {
                const int64_t r = order[s];
                const double dd = rows[r].d, ww = rows[r].w;
                sw += ww;
                swd += ww * dd;
                if (dd < mind) mind = dd;
                if (dd > maxd) maxd = dd;
                const int64_t pi = rid[r];
                if (kind == 1) {
                    if (c->last_wins) last = labels[pi] - 1;
                    else cntv[labels[pi] - 1] += 1.0;
                } else if (kind == 2) {
                    const double* z = feats + pi * D;
                    for (int q = 0; q < D; ++q) {
                        sz[q] += z[q];
                        sz[D + q] += z[q] * z[q];
                    }
                }
            }
            /* apply_tsdf (_pycore.py:399-417) */
            double w_old = isnew ? 0.0 : m->w[v];
            double d_old = isnew ? store_f(trunc, c->tsdf_f32) : m->d[v];
            double w_new = w_old + sw;
            double d_new = w_new > 0.0 ? (w_old * d_old + swd) / w_new : d_old;
            int same = c->tsdf_f32 ? ((float)d_old == (float)mind) : (d_old == mind);
            if (mind == maxd && (w_old == 0.0 || same)) d_new = mind;
            m->d[v] = store_f(d_new, c->tsdf_f32);
            m->w[v] = store_f(w_new, c->tsdf_f32);
            if (kind == 1) {
                /* apply_closed (_pycore.py:420-429) */
                double* row = m->s0 + v * P;
                for (int q = 0; q < P; ++q) {
                    double old = isnew ? 0.0 : row[q];
                    row[q] = c->last_wins ? (q == last ? 1.0 : 0.0)
                                          : store_f(old + store_f(cntv[q], c->sem_f32), c->sem_f32);
                }
            } else if (kind == 2) {
                /* apply_open (_pycore.py:432-446) */
                const double nobs = (double)(start[g + 1] - start[g]);
                const double lam = fmax(w_old, c->lambda_floor);
                const double lam_post = lam + nobs;
                const double coef = lam * nobs / lam_post;
                const double bbg = store_f(c->prior_beta, c->sem_f32);
                double* mrow = m->s0 + v * D;
                double* brow = m->s1 + v * D;
                for (int q = 0; q < D; ++q) {
                    double m_old = isnew ? 0.0 : mrow[q];
                    double b_old = isnew ? bbg : brow[q];
                    double m_new = (lam * m_old + sz[q]) / lam_post;
                    double zbar = sz[q] / nobs;
                    double ss = sz[D + q] - sz[q] * zbar;
                    if (ss < 0.0) ss = 0.0;
                    double diff = zbar - m_old;
                    double gap = coef * (diff * diff) * 0.5;
                    double b_new = b_old + 0.5 * ss + gap;
                    mrow[q] = store_f(m_new, c->sem_f32);
                    brow[q] = store_f(b_new, c->sem_f32);
                }
            }
        }
        free(sz);
        free(cntv);
    }
    rep->t_update_ms = now_ms() - t4;
    free(ray); free(cnt); free(rows); free(rid); free(key); free(order); free(start);
    free(gvid); free(gnew);
    return ORC_OK;
}

/* ---- queries ---------------------------------------------------------------- */
int64_t orc_active_count(const orc_map* m) { return m->nvox; }
int64_t orc_leaf_count(const orc_map* m) { return m->nleaves; }

static int64_t active_list(const orc_map* m, int64_t* vid, int64_t* coords) {
    int64_t p = 0;
    for (int64_t l = 0; l < m->nleaves; ++l) {
        for (int wd = 0; wd < 8; ++wd) {
            uint64_t bits = m->lmask[l * 8 + wd];
            while (bits) {
                int slot = wd * 64 + __builtin_ctzll(bits);
                bits &= bits - 1;
                if (vid) vid[p] = m->lslot[l * 512 + slot];
                if (coords) {
                    coords[3 * p] = ((int64_t)m->lcoord[3 * l] << 3) + ((slot >> 6) & 7);
                    coords[3 * p + 1] = ((int64_t)m->lcoord[3 * l + 1] << 3) + ((slot >> 3) & 7);
                    coords[3 * p + 2] = ((int64_t)m->lcoord[3 * l + 2] << 3) + (slot & 7);
                }
                ++p;
            }
        }
    }
    return p;
}

/* active_values (grid.py:163-168): all outputs f64; any may be NULL. */
int64_t orc_export(const orc_map* m, int64_t* coords, double* d, double* w, double* s0, double* s1) {
    int64_t n = m->nvox;
    int64_t* vid = (int64_t*)malloc(8 * (size_t)(n ? n : 1));
    active_list(m, vid, coords);
    const int P = m->P;
    for (int64_t i = 0; i < n; ++i) {
        int64_t v = vid[i];
        if (d) d[i] = m->d[v];
        if (w) w[i] = m->w[v];
        if (s0 && P) memcpy(s0 + i * P, m->s0 + v * P, 8 * (size_t)P);
        if (s1 && m->cfg.sem_kind == 2) memcpy(s1 + i * P, m->s1 + v * P, 8 * (size_t)P);
    }
    free(vid);
    return n;
}

/* probe_coords (_core.pyx:324-375) + backgrounds (grid.py:176-190). */
void orc_probe(const orc_map* m, const int64_t* coords, int64_t cnt, double* d, double* w,
               double* s0, double* s1, uint8_t* active) {
    const int P = m->P;
    for (int64_t i = 0; i < cnt; ++i) {
        int64_t x = coords[3 * i], y = coords[3 * i + 1], z = coords[3 * i + 2];
        int64_t leaf = hash_find(m, (int32_t)(x >> 3), (int32_t)(y >> 3), (int32_t)(z >> 3));
        int32_t v = -1;
        if (leaf >= 0) v = m->lslot[leaf * 512 + (((x & 7) << 6) | ((y & 7) << 3) | (z & 7))];
        active[i] = v >= 0;
        d[i] = v >= 0 ? m->d[v] : store_f(m->cfg.truncation, m->cfg.tsdf_f32);
        w[i] = v >= 0 ? m->w[v] : 0.0;
        for (int q = 0; q < P; ++q) {
            if (s0) s0[i * P + q] = v >= 0 ? m->s0[(int64_t)v * P + q] : 0.0;
            if (s1 && m->cfg.sem_kind == 2)
                s1[i * P + q] = v >= 0 ? m->s1[(int64_t)v * P + q]
                                       : store_f(m->cfg.prior_beta, m->cfg.sem_f32);
        }
    }
}

/* cosine_to_embeddings (gaussian.py:158-170) against q (D,), active order. */
void orc_cosine(const orc_map* m, const double* q, double* sims) {
    const int D = m->P;
    int64_t n = m->nvox;
    int64_t* vid = (int64_t*)malloc(8 * (size_t)(n ? n : 1));
    active_list(m, vid, NULL);
    double qn = 0.0;
    for (int c = 0; c < D; ++c) qn += q[c] * q[c];
    qn = sqrt(qn);
    for (int64_t i = 0; i < n; ++i) {
        const double* row = m->s0 + vid[i] * D;
        double dot = 0.0, nn = 0.0;
        for (int c = 0; c < D; ++c) { dot += row[c] * q[c]; nn += row[c] * row[c]; }
        double mn = sqrt(nn);
        sims[i] = mn == 0.0 ? NAN : dot / (mn * qn);
    }
    free(vid);
}

/* classify_means (gaussian.py:132-155) with weights = TSDF weight. */
void orc_classify(const orc_map* m, const double* emb, int k, double tau, double tp,
                  int32_t* labels, double* best) {
    const int D = m->P;
    int64_t n = m->nvox;
    int64_t* vid = (int64_t*)malloc(8 * (size_t)(n ? n : 1));
    active_list(m, vid, NULL);
    double* en = (double*)malloc(8 * (size_t)k);
    double* e = (double*)malloc(8 * (size_t)k);
    for (int j = 0; j < k; ++j) {
        double s = 0.0;
        for (int c = 0; c < D; ++c) s += emb[j * D + c] * emb[j * D + c];
        en[j] = sqrt(s);
    }
    for (int64_t i = 0; i < n; ++i) {
        const double* row = m->s0 + vid[i] * D;
        double nn = 0.0;
        for (int c = 0; c < D; ++c) nn += row[c] * row[c];
        double mn = sqrt(nn);
        labels[i] = 0;
        best[i] = 0.0;
        if (mn == 0.0 || !(m->w[vid[i]] > 0.0)) continue;
        double lmax = -INFINITY;
        for (int j = 0; j < k; ++j) {
            double dot = 0.0;
            for (int c = 0; c < D; ++c) dot += row[c] * emb[j * D + c];
            e[j] = (dot / (mn * en[j])) / tau;
            if (e[j] > lmax) lmax = e[j];
        }
        double den = 0.0, emax = -1.0;
        int arg = 0;
        for (int j = 0; j < k; ++j) {
            e[j] = exp(e[j] - lmax);
            den += e[j];
            if (e[j] > emax) { emax = e[j]; arg = j; }
        }
        double top = emax / den;
        labels[i] = top < tp ? 0 : arg + 1;
        best[i] = top;
    }
    free(vid); free(en); free(e);
}

/* Closed-set readouts: mode 0 label_map (dirichlet.py:81-88), 1 grid_labels (evalbench.py:30-55). */
void orc_label_map(const orc_map* m, int mode, int32_t* labels) {
    const int C = m->P;
    int64_t n = m->nvox;
    int64_t* vid = (int64_t*)malloc(8 * (size_t)(n ? n : 1));
    active_list(m, vid, NULL);
    for (int64_t i = 0; i < n; ++i) {
        const double* row = m->s0 + vid[i] * C;
        int arg = 0;
        double total = row[0];
        for (int q = 1; q < C; ++q) { total += row[q]; if (row[q] > row[arg]) arg = q; }
        labels[i] = (mode == 1 && !(total > 0.0)) ? 0 : arg + 1;
    }
    free(vid);
}
