/*
 * nbb_oracle.h -- CPU restatement of the reference compact-fractal stencil path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the parity checker for the CUDA engine in
 * paper_2110_12952_b200/.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load it; the product path never links or calls it.
 *
 * Every function restates the algorithm of the reference implementation under
 * /root/reference/proj (cited file:line).  The restatement is pinned against the
 * reference itself (oracle/_ref, built from the reference sources by
 * oracle/Makefile) through the golden vectors in tests/golden/.
 */
#ifndef NBB_ORACLE_H
#define NBB_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NBBO_MAX_LEVEL 40
#define NBBO_MAX_S 16

/* Mirrors CoordMapper's precomputed tables (proj/include/nbb/maps.hpp:61-70). */
typedef struct {
    int k, s, r;
    int64_t side, w, h;
    int64_t spow[NBBO_MAX_LEVEL + 1];          /* s^mu                         */
    int16_t id_of_subbox[NBBO_MAX_S * NBBO_MAX_S]; /* gy*s+gx -> id, -1 = hole */
    int32_t rep_gx[NBBO_MAX_S * NBBO_MAX_S];
    int32_t rep_gy[NBBO_MAX_S * NBBO_MAX_S];
    int64_t stride_x[NBBO_MAX_LEVEL], stride_y[NBBO_MAX_LEVEL];
} nbbo_mapper;

/* 0 on success, -1 on an invalid descriptor / level (validate(),
 * proj/src/descriptor.cpp:12-44). replicas_xy = k (gx, gy) pairs. */
int nbbo_mapper_init(nbbo_mapper* m, const int32_t* replicas_xy, int k, int s, int r);

/* nu: embedded -> compact, proj/src/maps.cpp:80-107.  Returns 1 if fractal. */
int nbbo_try_to_compact(const nbbo_mapper* m, int64_t x, int64_t y, int64_t* cx, int64_t* cy);
/* lambda: compact -> embedded, proj/src/maps.cpp:123-146 (no range check). */
void nbbo_to_embedded(const nbbo_mapper* m, int64_t cx, int64_t cy, int64_t* x, int64_t* y);
/* proj/src/maps.cpp:163-199: nu through the Figure-8 matrix product (int64). */
int nbbo_to_compact_via_mma(const nbbo_mapper* m, int64_t x, int64_t y, int64_t* cx, int64_t* cy);

/* proj/include/nbb/rng.hpp:9-39 */
uint64_t nbbo_splitmix64(uint64_t x);
int nbbo_cell_alive(uint64_t seed, int64_t x, int64_t y, double density);
uint64_t nbbo_coord_mix(int64_t x, int64_t y);

/* Seeding, proj/src/stencil.cpp:138-180.  mode 0 = linear compact (k^r bytes),
 * mode 1 = embedded (n^2 bytes).  Buffer must be pre-zeroed by the caller. */
void nbbo_seed(const nbbo_mapper* m, int mode, uint64_t seed, double density, uint8_t* f);

/* state_hash, proj/src/stencil.cpp:196-234. */
uint64_t nbbo_state_hash(const nbbo_mapper* m, int mode, const uint8_t* f);

/* state_hash over linear-compact indices [i0, i1) (partial sums add up). */
uint64_t nbbo_state_hash_range(const nbbo_mapper* m, const uint8_t* f, int64_t i0, int64_t i1);

/* step_compact_linear over compact indices [i0, i1), proj/src/stencil.cpp:334-368.
 * moore != 0 -> 8 Moore offsets, else 4 von Neumann (proj/src/stencil.cpp:55-61). */
void nbbo_step_compact(const nbbo_mapper* m, uint16_t birth, uint16_t survive, int moore,
                       const uint8_t* f, uint8_t* b, int64_t i0, int64_t i1);
/* step_bounding_box over rows [y0, y1), proj/src/stencil.cpp:291-311. */
void nbbo_step_bb(const nbbo_mapper* m, uint16_t birth, uint16_t survive, int moore,
                  const uint8_t* f, uint8_t* b, int64_t y0, int64_t y1);

/* Whole-grid step split over nthreads pthreads (the reference's parallel_for,
 * proj/src/stencil.cpp:236-260).  mode as in nbbo_seed. */
void nbbo_step(const nbbo_mapper* m, int mode, uint16_t birth, uint16_t survive, int moore,
               const uint8_t* f, uint8_t* b, int nthreads);

/* FNV-1a 64 over a byte buffer (the golden-vector fingerprint). */
uint64_t nbbo_fnv1a64(const uint8_t* p, int64_t n);

/* "lambda" backend step (CompactGrid, stencil.cpp:313-332): embedded buffers,
 * compact indices [i0, i1).  nbbo_step / nbbo_seed / nbbo_state_hash accept
 * mode 2 = lambda (embedded storage, compact iteration). */
void nbbo_step_lambda(const nbbo_mapper* m, uint16_t birth, uint16_t survive, int moore,
                      const uint8_t* f, uint8_t* b, int64_t i0, int64_t i1);

/* Blocked compact layout (Layout::BlockedCompact, grid.cpp:54-63): mf = full-level
 * mapper, mc = mapper at level r - m with rho = s^m. */
int64_t nbbo_blocked_index(const nbbo_mapper* mf, const nbbo_mapper* mc, int64_t rho, int64_t x, int64_t y);
void nbbo_blocked_seed(const nbbo_mapper* mf, const nbbo_mapper* mc, int64_t rho, uint64_t seed,
                       double density, uint8_t* f);
uint64_t nbbo_blocked_hash(const nbbo_mapper* mf, const nbbo_mapper* mc, int64_t rho, const uint8_t* f);
void nbbo_blocked_step(const nbbo_mapper* mf, const nbbo_mapper* mc, int64_t rho, uint16_t birth,
                       uint16_t survive, int moore, const uint8_t* f, uint8_t* b, int64_t b0, int64_t b1);

#ifdef __cplusplus
}
#endif
#endif
