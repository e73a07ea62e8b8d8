/*
 * nbb_oracle.c -- CPU restatement of the reference's compact-fractal stencil path.
 *
 * TEST INFRASTRUCTURE ONLY (see nbb_oracle.h).  Plain C, scalar, one function per
 * reference routine, each citing the reference file:line it restates.  Pinned
 * against the reference build (oracle/_ref) via tests/golden/ and
 * tests/test_oracle.py.
 */
#include "nbb_oracle.h"

#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ipow with overflow guard, proj/src/geometry.cpp:10-21 */
static int ipow_ok(int64_t base, int e, int64_t* out) {
    int64_t r = 1;
    for (int i = 0; i < e; ++i) {
        if (base != 0 && r > INT64_MAX / base) return 0;
        r *= base;
    }
    *out = r;
    return 1;
}

/* CoordMapper ctor, proj/src/maps.cpp:45-78; validate(), proj/src/descriptor.cpp:12-44;
 * unfold_stride, proj/src/maps.cpp:28-34; compact_dims, proj/src/maps.cpp:36-43. */
int nbbo_mapper_init(nbbo_mapper* m, const int32_t* rep, int k, int s, int r) {
    memset(m, 0, sizeof(*m));
    if (k < 1 || s < 2 || s > NBBO_MAX_S || (int64_t)k > (int64_t)s * s) return -1;
    if (r < 0 || r > NBBO_MAX_LEVEL) return -1;
    m->k = k; m->s = s; m->r = r;
    if (!ipow_ok(s, r, &m->side)) return -1;
    if (!ipow_ok(k, (r + 1) / 2, &m->w)) return -1;
    if (!ipow_ok(k, r / 2, &m->h)) return -1;
    for (int i = 0; i < s * s; ++i) m->id_of_subbox[i] = -1;
    for (int i = 0; i < k; ++i) {
        int gx = rep[2 * i], gy = rep[2 * i + 1];
        if (gx < 0 || gy < 0 || gx >= s || gy >= s) return -1;
        if (m->id_of_subbox[gy * s + gx] >= 0) return -1; /* duplicate */
        m->id_of_subbox[gy * s + gx] = (int16_t)i;
        m->rep_gx[i] = gx;
        m->rep_gy[i] = gy;
    }
    m->spow[0] = 1;
    for (int mu = 0; mu < r; ++mu) m->spow[mu + 1] = m->spow[mu] * s;
    int64_t p = 1;
    for (int mu = 0; mu < r; ++mu) {
        if (mu > 0 && mu % 2 == 0) p *= k;          /* p = k^(mu/2) */
        m->stride_x[mu] = (mu % 2 == 0) ? p : 0;
        m->stride_y[mu] = (mu % 2 == 0) ? 0 : p;
    }
    return 0;
}

/* CoordMapper::try_to_compact, proj/src/maps.cpp:80-107 (generic-s branch; the
 * s == 2 shift branch at :83-93 computes the same digits for x, y >= 0). */
int nbbo_try_to_compact(const nbbo_mapper* m, int64_t x, int64_t y, int64_t* cx, int64_t* cy) {
    int64_t ax = 0, ay = 0;
    const int s = m->s;
    for (int mu = 0; mu < m->r; ++mu) {
        const int id = m->id_of_subbox[(y % s) * s + (x % s)];
        if (id < 0) return 0;
        ax += m->stride_x[mu] * id;
        ay += m->stride_y[mu] * id;
        x /= s;
        y /= s;
    }
    *cx = ax;
    *cy = ay;
    return 1;
}

/* CoordMapper::to_embedded, proj/src/maps.cpp:123-146 (range check omitted). */
void nbbo_to_embedded(const nbbo_mapper* m, int64_t cx, int64_t cy, int64_t* x, int64_t* y) {
    int64_t ex = 0, ey = 0;
    for (int mu = 0; mu < m->r; ++mu) {
        int digit;
        if (mu % 2 == 0) { digit = (int)(cx % m->k); cx /= m->k; }
        else             { digit = (int)(cy % m->k); cy /= m->k; }
        ex += m->rep_gx[digit] * m->spow[mu];
        ey += m->rep_gy[digit] * m->spow[mu];
    }
    *x = ex;
    *y = ey;
}

/* build_map_matrices + mma_multiply_accumulate + to_compact_via_mma,
 * proj/src/maps.cpp:163-199: A row0 = x strides, row1 = y strides,
 * B column 0 = replica IDs H(e, mu) (replica_id, proj/src/maps.cpp:9-21). */
int nbbo_to_compact_via_mma(const nbbo_mapper* m, int64_t x, int64_t y, int64_t* cx, int64_t* cy) {
    const int side = m->r > 16 ? m->r : 16;
    int64_t* a = (int64_t*)calloc((size_t)side * side, sizeof(int64_t));
    int64_t* b = (int64_t*)calloc((size_t)side * side, sizeof(int64_t));
    int64_t* c = (int64_t*)calloc((size_t)side * side, sizeof(int64_t));
    int ok = 1;
    for (int mu = 0; mu < m->r; ++mu) {
        const int64_t sc = m->spow[mu];
        const int gx = (int)((x / sc) % m->s), gy = (int)((y / sc) % m->s);
        const int id = m->id_of_subbox[gy * m->s + gx];
        if (id < 0) { ok = 0; break; }
        a[0 * side + mu] = m->stride_x[mu];
        a[1 * side + mu] = m->stride_y[mu];
        b[mu * side + 0] = id;
    }
    if (ok) {
        for (int i = 0; i < side; ++i)
            for (int l = 0; l < side; ++l) {
                const int64_t av = a[i * side + l];
                if (av == 0) continue;
                for (int j = 0; j < side; ++j) c[i * side + j] += av * b[l * side + j];
            }
        *cx = c[0];
        *cy = c[side];
    }
    free(a); free(b); free(c);
    return ok;
}

/* splitmix64, proj/include/nbb/rng.hpp:9-14 */
uint64_t nbbo_splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

/* cell_key + cell_alive, proj/include/nbb/rng.hpp:18-33 */
int nbbo_cell_alive(uint64_t seed, int64_t x, int64_t y, double density) {
    const uint64_t key = nbbo_splitmix64(nbbo_splitmix64(seed) ^ ((uint64_t)x << 32) ^
                                         (uint64_t)(uint32_t)y);
    const double u = (double)(key >> 11) * (1.0 / 9007199254740992.0);
    return u < density;
}

/* coord_mix, proj/include/nbb/rng.hpp:36-39 */
uint64_t nbbo_coord_mix(int64_t x, int64_t y) {
    return nbbo_splitmix64(((uint64_t)x << 32) ^ (uint64_t)(uint32_t)y);
}

/* Simulation::seed_random, proj/src/stencil.cpp:138-180 (linear + embedded). */
void nbbo_seed(const nbbo_mapper* m, int mode, uint64_t seed, double density, uint8_t* f) {
    if (mode == 1 || mode == 2) { /* embedded storage (bb, lambda) */
        for (int64_t y = 0; y < m->side; ++y)
            for (int64_t x = 0; x < m->side; ++x) {
                int64_t cx, cy;
                if (nbbo_try_to_compact(m, x, y, &cx, &cy))
                    f[y * m->side + x] = nbbo_cell_alive(seed, x, y, density) ? 1 : 0;
            }
    } else {
        const int64_t total = m->w * m->h;
        for (int64_t i = 0; i < total; ++i) {
            int64_t x, y;
            nbbo_to_embedded(m, i % m->w, i / m->w, &x, &y);
            f[i] = nbbo_cell_alive(seed, x, y, density) ? 1 : 0;
        }
    }
}

/* Simulation::state_hash, proj/src/stencil.cpp:196-234 (embedded + linear). */
uint64_t nbbo_state_hash(const nbbo_mapper* m, int mode, const uint8_t* f) {
    uint64_t hash = 0;
    if (mode == 1 || mode == 2) { /* embedded storage (bb, lambda) */
        const int64_t total = m->side * m->side;
        for (int64_t i = 0; i < total; ++i)
            if (f[i]) hash += nbbo_coord_mix(i % m->side, i / m->side);
    } else {
        const int64_t total = m->w * m->h;
        for (int64_t i = 0; i < total; ++i)
            if (f[i]) {
                int64_t x, y;
                nbbo_to_embedded(m, i % m->w, i / m->w, &x, &y);
                hash += nbbo_coord_mix(x, y);
            }
    }
    return hash;
}

/* state_hash restricted to linear-compact indices [i0, i1) (the partial sums of
 * stencil.cpp:207-216 add up to the full hash: the sum is order independent). */
uint64_t nbbo_state_hash_range(const nbbo_mapper* m, const uint8_t* f, int64_t i0, int64_t i1) {
    uint64_t hash = 0;
    for (int64_t i = i0; i < i1; ++i)
        if (f[i]) {
            int64_t x, y;
            nbbo_to_embedded(m, i % m->w, i / m->w, &x, &y);
            hash += nbbo_coord_mix(x, y);
        }
    return hash;
}

/* neighbor_offsets, proj/src/stencil.cpp:55-61 */
static const int kOff[8][2] = {{1, 0}, {-1, 0}, {0, 1}, {0, -1},
                               {1, 1}, {1, -1}, {-1, 1}, {-1, -1}};

/* StencilRule::born_with / survives_with, proj/include/nbb/stencil.hpp:23-24 */
static inline uint8_t apply_rule(uint16_t birth, uint16_t survive, uint8_t alive, int count) {
    return alive ? (uint8_t)((survive >> count) & 1) : (uint8_t)((birth >> count) & 1);
}

/* Simulation::step_compact_linear (no neighbour table), proj/src/stencil.cpp:353-367 */
void nbbo_step_compact(const nbbo_mapper* m, uint16_t birth, uint16_t survive, int moore,
                       const uint8_t* f, uint8_t* b, int64_t i0, int64_t i1) {
    const int deg = moore ? 8 : 4;
    const int64_t n = m->side, w = m->w;
    for (int64_t i = i0; i < i1; ++i) {
        int64_t ex, ey;
        nbbo_to_embedded(m, i % w, i / w, &ex, &ey);
        int count = 0;
        for (int j = 0; j < deg; ++j) {
            const int64_t nx = ex + kOff[j][0], ny = ey + kOff[j][1];
            if (nx < 0 || ny < 0 || nx >= n || ny >= n) continue;
            int64_t cx, cy;
            if (nbbo_try_to_compact(m, nx, ny, &cx, &cy)) count += f[cy * w + cx];
        }
        b[i] = apply_rule(birth, survive, f[i], count);
    }
}

/* Simulation::step_bounding_box, proj/src/stencil.cpp:291-311 */
void nbbo_step_bb(const nbbo_mapper* m, uint16_t birth, uint16_t survive, int moore,
                  const uint8_t* f, uint8_t* b, int64_t y0, int64_t y1) {
    const int deg = moore ? 8 : 4;
    const int64_t n = m->side;
    for (int64_t y = y0; y < y1; ++y)
        for (int64_t x = 0; x < n; ++x) {
            int64_t cx, cy;
            if (!nbbo_try_to_compact(m, x, y, &cx, &cy)) continue; /* holes never change */
            int count = 0;
            for (int j = 0; j < deg; ++j) {
                const int64_t nx = x + kOff[j][0], ny = y + kOff[j][1];
                if (nx >= 0 && ny >= 0 && nx < n && ny < n) count += f[ny * n + nx];
            }
            b[y * n + x] = apply_rule(birth, survive, f[y * n + x], count);
        }
}

/* Simulation::step_compact_grid (the "lambda" backend), proj/src/stencil.cpp:313-332:
 * embedded storage, the loop visits exactly the k^r compact indices [i0, i1),
 * neighbours are read in embedded coordinates (no nu). */
void nbbo_step_lambda(const nbbo_mapper* m, uint16_t birth, uint16_t survive, int moore,
                      const uint8_t* f, uint8_t* b, int64_t i0, int64_t i1) {
    const int deg = moore ? 8 : 4;
    const int64_t n = m->side, w = m->w;
    for (int64_t i = i0; i < i1; ++i) {
        int64_t ex, ey;
        nbbo_to_embedded(m, i % w, i / w, &ex, &ey);
        int count = 0;
        for (int j = 0; j < deg; ++j) {
            const int64_t nx = ex + kOff[j][0], ny = ey + kOff[j][1];
            if (nx >= 0 && ny >= 0 && nx < n && ny < n) count += f[ny * n + nx];
        }
        b[ey * n + ex] = apply_rule(birth, survive, f[ey * n + ex], count);
    }
}

/* ---- blocked compact layout (Layout::BlockedCompact) ----------------------------
 * block b of the coarse mapper mc (level r - m, rho = s^m) holds the rho x rho
 * embedded mini box with corner lambda_c(b) * rho, row-major: slot
 * b*rho^2 + ly*rho + lx (grid.cpp:54-63).  mf is the full-level mapper. */

/* Grid::storage_index, BlockedCompact branch (grid.cpp:54-63); -1 if the coarse
 * cell is not in the coarse fractal. */
int64_t nbbo_blocked_index(const nbbo_mapper* mf, const nbbo_mapper* mc, int64_t rho, int64_t x, int64_t y) {
    (void)mf;
    int64_t cx, cy;
    if (!nbbo_try_to_compact(mc, x / rho, y / rho, &cx, &cy)) return -1;
    return (cy * mc->w + cx) * rho * rho + (y % rho) * rho + (x % rho);
}

/* Simulation::seed_random, BlockedCompact branch (stencil.cpp:161-177) */
void nbbo_blocked_seed(const nbbo_mapper* mf, const nbbo_mapper* mc, int64_t rho, uint64_t seed,
                       double density, uint8_t* f) {
    const int64_t blocks = mc->w * mc->h;
    for (int64_t bk = 0; bk < blocks; ++bk) {
        int64_t cxe, cye;
        nbbo_to_embedded(mc, bk % mc->w, bk / mc->w, &cxe, &cye);
        for (int64_t ly = 0; ly < rho; ++ly)
            for (int64_t lx = 0; lx < rho; ++lx) {
                const int64_t x = cxe * rho + lx, y = cye * rho + ly;
                int64_t a, c;
                if (nbbo_try_to_compact(mf, x, y, &a, &c))
                    f[bk * rho * rho + ly * rho + lx] = nbbo_cell_alive(seed, x, y, density) ? 1 : 0;
            }
    }
}

/* Simulation::state_hash, BlockedCompact branch (stencil.cpp:217-231) */
uint64_t nbbo_blocked_hash(const nbbo_mapper* mf, const nbbo_mapper* mc, int64_t rho, const uint8_t* f) {
    (void)mf;
    uint64_t hash = 0;
    const int64_t blocks = mc->w * mc->h;
    for (int64_t bk = 0; bk < blocks; ++bk) {
        int64_t cxe, cye;
        nbbo_to_embedded(mc, bk % mc->w, bk / mc->w, &cxe, &cye);
        for (int64_t ly = 0; ly < rho; ++ly)
            for (int64_t lx = 0; lx < rho; ++lx)
                if (f[bk * rho * rho + ly * rho + lx]) hash += nbbo_coord_mix(cxe * rho + lx, cye * rho + ly);
    }
    return hash;
}

/* Simulation::step_compact_blocked, proj/src/stencil.cpp:370-399, blocks [b0, b1) */
void nbbo_blocked_step(const nbbo_mapper* mf, const nbbo_mapper* mc, int64_t rho, uint16_t birth,
                       uint16_t survive, int moore, const uint8_t* f, uint8_t* b, int64_t b0, int64_t b1) {
    const int deg = moore ? 8 : 4;
    const int64_t n = mf->side;
    for (int64_t bk = b0; bk < b1; ++bk) {
        int64_t cxe, cye;
        nbbo_to_embedded(mc, bk % mc->w, bk / mc->w, &cxe, &cye);
        for (int64_t ly = 0; ly < rho; ++ly)
            for (int64_t lx = 0; lx < rho; ++lx) {
                const int64_t x = cxe * rho + lx, y = cye * rho + ly;
                int64_t a, c;
                if (!nbbo_try_to_compact(mf, x, y, &a, &c)) continue; /* filler slot, stays dead */
                int count = 0;
                for (int j = 0; j < deg; ++j) {
                    const int64_t nx = x + kOff[j][0], ny = y + kOff[j][1];
                    if (nx < 0 || ny < 0 || nx >= n || ny >= n) continue;
                    if (nbbo_try_to_compact(mf, nx, ny, &a, &c))
                        count += f[nbbo_blocked_index(mf, mc, rho, nx, ny)];
                }
                const int64_t slot = bk * rho * rho + ly * rho + lx;
                b[slot] = apply_rule(birth, survive, f[slot], count);
            }
    }
}

typedef struct {
    const nbbo_mapper* m;
    int mode, moore;
    uint16_t birth, survive;
    const uint8_t* f;
    uint8_t* b;
    int64_t lo, hi;
} step_job;

static void* step_worker(void* arg) {
    step_job* j = (step_job*)arg;
    if (j->mode == 1) nbbo_step_bb(j->m, j->birth, j->survive, j->moore, j->f, j->b, j->lo, j->hi);
    else if (j->mode == 2) nbbo_step_lambda(j->m, j->birth, j->survive, j->moore, j->f, j->b, j->lo, j->hi);
    else nbbo_step_compact(j->m, j->birth, j->survive, j->moore, j->f, j->b, j->lo, j->hi);
    return NULL;
}

/* Simulation::step + parallel_for, proj/src/stencil.cpp:236-289: BB splits rows,
 * compact splits compact indices into ceil(D/W) chunks. */
void nbbo_step(const nbbo_mapper* m, int mode, uint16_t birth, uint16_t survive, int moore,
               const uint8_t* f, uint8_t* b, int nthreads) {
    const int64_t domain = mode == 1 ? m->side : m->w * m->h;  /* mode 2: compact indices */
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    if (nthreads == 1 || domain < 2) {
        step_job j = {m, mode, moore, birth, survive, f, b, 0, domain};
        step_worker(&j);
        return;
    }
    pthread_t th[256];
    step_job jobs[256];
    const int64_t chunk = (domain + nthreads - 1) / nthreads;
    int spawned = 0;
    for (int t = 0; t < nthreads; ++t) {
        const int64_t lo = t * chunk, hi = lo + chunk < domain ? lo + chunk : domain;
        if (lo >= hi) break;
        step_job j = {m, mode, moore, birth, survive, f, b, lo, hi};
        jobs[t] = j;
        pthread_create(&th[t], NULL, step_worker, &jobs[t]);
        ++spawned;
    }
    for (int t = 0; t < spawned; ++t) pthread_join(th[t], NULL);
}

uint64_t nbbo_fnv1a64(const uint8_t* p, int64_t n) {
    uint64_t h = 0xcbf29ce484222325ull;
    for (int64_t i = 0; i < n; ++i) {
        h ^= p[i];
        h *= 0x100000001b3ull;
    }
    return h;
}
