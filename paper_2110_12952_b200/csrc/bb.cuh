// bb.cuh -- the bounding-box GPU baseline (north-star item 3), any growth factor s.
//
// Simulation::step_bounding_box (stencil.cpp:291-311) over the reference's embedded
// layout (n x n bytes, row-major, holes 0) as a dense row-streaming stencil:
//
// * Chunks.  The buffer is cut into 16-byte aligned chunks.  "Aligned row" y is the
//   chunk range [floor16(y n), floor16((y+1) n)) (the last row runs to ceil16(n^2),
//   into the 64 B allocation pad), so rows of any width n tile the buffer and
//   every chunk holds at most one row boundary.  A linear byte i has the
//   neighbours i +- 1, i +- n, i +- n +- 1 whatever the row alignment; only the
//   column edges (x = 0 / x = n - 1) need masks, and out-of-buffer bytes read 0.
// * CTA = one strip of cps chunks of every aligned row of a band of R rows.  It
//   streams the band top to bottom through an NS-slot shared-memory ring of row
//   segments (cps + 4 chunks: 32 B margins either side) with cp.async (zero-fill
//   outside the buffer), so every byte crosses HBM -> SM once per step; one
//   __syncthreads per row.  Thread t computes chunk t of the row: the middle
//   16 bytes of each of the 3 rows by LDS.128 (the rows above / below are
//   shifted by the warp-uniform delta = floor16(y n) -+ n - floor16((y -+ 1) n)),
//   the edge bytes from the neighbouring lanes by shuffles, SWAR neighbour
//   counts (bytes <= 8), the rule by SWAR compares / PRMT tables, a 16-bit hole
//   mask, one 16-byte store.
// * Membership (cell_in_fractal, maps.cpp:80-107) = the low m levels (S = s^m >= 32
//   columns) from a doubled bit table in shared memory AND the top r - m levels
//   from a coarse bitmap ((n / S)^2 bits, L2-resident).
// * Holes are 0 in both buffers and never change, so a warp whose 512 bytes of a
//   row are all holes (one coarse-bitmap test) neither loads (its ring slots are
//   zeroed in shared memory) nor computes nor stores them: the baseline touches
//   the box only where the fractal is (the reference skips holes the same way,
//   stencil.cpp:300-301).
#pragma once

#include "common.cuh"

namespace nbbgpu {

struct BBRowParams {
    uint64_t n;         // side s^r (>= 32)
    uint64_t alloc;     // bytes readable at the buffer (n^2 + pad)
    uint32_t magic;     // floor(2^32 / S) + 1: x / S = umulhi(x, magic) for x < 2^32 / S
    uint32_t S;         // low-table side s^m
    uint32_t CW;        // coarse side n / S
    uint32_t lt_words;  // words per doubled low-table row
    uint32_t cps;       // chunks per strip (2 per thread, multiple of 64, <= 256)
    uint32_t rows;      // rows per CTA (band height)
    uint32_t birth, survive;
    int moore;
};

// 4 bits -> 4 bytes of 0/1
__device__ __forceinline__ uint32_t bb_spread4(uint32_t nib) { return ((nib & 0xFu) * 0x00204081u) & 0x01010101u; }

// SWAR rule: bytes of cnt in 0..8, alive bytes 0/1 -> next-state bytes 0/1
template <bool CONWAY>
__device__ __forceinline__ uint32_t bb_rule(uint32_t cnt, uint32_t alive, uint32_t tb_lo, uint32_t tb_hi,
                                            uint32_t ts_lo, uint32_t ts_hi, uint32_t b8, uint32_t s8) {
    if (CONWAY) {
        // next = ((cnt | alive) == 3) per byte
        const uint32_t v = (cnt | alive) ^ 0x03030303u;
        const uint32_t z = ~(((v & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | v | 0x7F7F7F7Fu);  // 0x80 where v == 0
        return z >> 7;
    } else {
        // PRMT lookup of cnt & 7 in the 8-entry birth / survive byte tables
        const uint32_t c = cnt & 0x07070707u;
        const uint32_t nib = c | (c >> 4);                  // bytes 0, 2: two 4-bit selectors each
        const uint32_t sel = __byte_perm(nib, 0, 0x0020);  // 4 nibbles = the 4 counts
        const uint32_t rb = __byte_perm(tb_lo, tb_hi, sel);
        const uint32_t rs = __byte_perm(ts_lo, ts_hi, sel);
        const uint32_t am = alive * 0xFFu;                  // 0x00 / 0xFF per byte
        uint32_t r = (rs & am) | (rb & ~am);
        const uint32_t m8 = ((cnt >> 3) & 0x01010101u) * 0xFFu;  // count == 8
        const uint32_t v8 = (s8 & am) | (b8 & ~am);
        return (r & ~m8) | (v8 & m8);
    }
}

// The coarse bitmap rows / columns a CTA touches, cached in shared memory: rows
// [cy0, cy0 + nrows), columns [cx0, cx1] (wpr words per row), and column CW - 1
// per row in `last` (strip 0's row-straddling chunks end the previous row).
struct BBCoarse {
    const uint32_t* bits;
    uint32_t cy0, cx0, cx1, wpr, last;
};

__device__ __forceinline__ uint32_t bb_div(const BBRowParams& p, uint32_t x) { return __umulhi(x, p.magic); }

__device__ __forceinline__ bool bb_coarse_bit(const BBCoarse& c, uint32_t cx, uint32_t cy) {
    const uint32_t ry = cy - c.cy0;
    if (cx >= c.cx0 && cx <= c.cx1) {
        const uint32_t b = cx - c.cx0;
        return (c.bits[ry * c.wpr + (b >> 5)] >> (b & 31)) & 1u;
    }
    return (c.last >> ry) & 1u;
}

// membership bits of cells (x .. x+NB-1, y), NB = 16 or 32, 0 <= x, y < n; bits at
// x' >= n are 0.  S >= 32 > NB: the run meets at most two coarse cells.
template <int NB>
__device__ __forceinline__ uint32_t bb_member(const BBRowParams& p, const uint32_t* lt, const BBCoarse& cc,
                                              uint32_t x, uint32_t y) {
    const uint32_t cx = bb_div(p, x), cy = bb_div(p, y);
    const uint32_t xl = x - cx * p.S, yl = y - cy * p.S;
    const uint32_t* row = lt + yl * p.lt_words;
    const uint32_t w = xl >> 5;
    constexpr uint32_t ALL = NB == 32 ? 0xFFFFFFFFu : (1u << NB) - 1u;
    uint32_t bits = __funnelshift_r(row[w], row[w + 1], xl & 31) & ALL;  // doubled row: no wrap
    const uint32_t split = p.S - xl;  // bits >= split lie in coarse cell cx + 1
    uint32_t keep = bb_coarse_bit(cc, cx, cy) ? ALL : 0u;
    if (split < (uint32_t)NB) {
        const uint32_t lo = (1u << split) - 1u;
        const bool c1 = cx + 1 < p.CW && bb_coarse_bit(cc, cx + 1, cy);
        keep = (keep & lo) | (c1 ? (~lo & ALL) : 0u);
    }
    bits &= keep;
    const uint64_t left = p.n - x;
    if (left < (uint64_t)NB) bits &= (1u << left) - 1u;
    return bits;
}

// does row y hold a fractal cell in [x0, x0 + 1024)?  (coarse test, x0 >= 0; a
// conservative "yes" when the range reaches past the row)
__device__ __forceinline__ bool bb_run_live(const BBRowParams& p, const BBCoarse& cc, int64_t x0, int64_t y) {
    if (x0 + 1024 > (int64_t)p.n) return true;
    const uint32_t cy = bb_div(p, (uint32_t)y);
    const uint32_t cx0 = bb_div(p, (uint32_t)x0), cx1 = bb_div(p, (uint32_t)x0 + 1023u);  // <= cx0 + 33
    const uint32_t b0 = cx0 - cc.cx0, nb = cx1 - cx0 + 1;
    const uint32_t* row = cc.bits + (cy - cc.cy0) * cc.wpr;
    const uint32_t w = b0 >> 5, sh = b0 & 31;
    const uint64_t lo = (uint64_t)row[w] | ((uint64_t)row[w + 1] << 32);
    const uint64_t v = sh ? (lo >> sh) | ((uint64_t)row[w + 2] << (64 - sh)) : lo;
    return (v & ((1ull << nb) - 1ull)) != 0ull;
}

__device__ __forceinline__ void bb_cp_async16(uint32_t saddr, const void* g, uint32_t src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(saddr), "l"(g), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void bb_cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bb_cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

__device__ __forceinline__ int64_t bb_floor16(int64_t v) { return v & ~(int64_t)15; }

// the 32 bytes [off, off + 32) of a ring slot; off & 15 is warp-uniform
__device__ __forceinline__ void bb_mid32(const uint8_t* slot, uint32_t off, uint32_t m[8]) {
    const uint32_t a = off & ~15u, o = off & 15u;
    const uint4 v0 = *reinterpret_cast<const uint4*>(slot + a);
    const uint4 v1 = *reinterpret_cast<const uint4*>(slot + a + 16);
    if (o == 0u) {
        m[0] = v0.x; m[1] = v0.y; m[2] = v0.z; m[3] = v0.w;
        m[4] = v1.x; m[5] = v1.y; m[6] = v1.z; m[7] = v1.w;
        return;
    }
    const uint4 v2 = *reinterpret_cast<const uint4*>(slot + a + 32);
    const uint32_t v[12] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w, v2.x, v2.y, v2.z, v2.w};
    const uint32_t sh = 8u * (o & 3u);
    switch (o >> 2) {  // uniform across the warp: no divergence, static register indices
    case 0:
#pragma unroll
        for (int j = 0; j < 8; ++j) m[j] = __funnelshift_r(v[j], v[j + 1], sh);
        break;
    case 1:
#pragma unroll
        for (int j = 0; j < 8; ++j) m[j] = __funnelshift_r(v[j + 1], v[j + 2], sh);
        break;
    case 2:
#pragma unroll
        for (int j = 0; j < 8; ++j) m[j] = __funnelshift_r(v[j + 2], v[j + 3], sh);
        break;
    default:
#pragma unroll
        for (int j = 0; j < 8; ++j) m[j] = __funnelshift_r(v[j + 3], v[j + 4], sh);
        break;
    }
}

// 0xFF in byte b (0..31) of a 32-byte pair, as word j
__device__ __forceinline__ uint32_t bb_byte_mask(int b, int j) {
    return ((unsigned)b < 32u && (b >> 2) == j) ? 0xFFu << (8 * (b & 3)) : 0u;
}

// shared-memory layout of step_bb_rows_kernel: NS ring slots, the low table, the
// coarse cache (kBBCacheWords), the live flags [NS][warps], two mask rows
constexpr uint32_t kBBCacheWords = 64;
constexpr int kBBStages = 6;
constexpr int kBBMaxThreads = 128;

// coarse rows / columns of tile (sx, band): rows y0 - 1 .. y1 + NS, x within
// [xs - 16, xs + 16 cps + 16], plus column CW - 1
__device__ __host__ __forceinline__ void bb_tile_cover(const BBRowParams& p, uint32_t sx, uint32_t band, int ns,
                                                       uint32_t& cy0, uint32_t& cy1, uint32_t& cx0, uint32_t& cx1) {
    const int64_t n = (int64_t)p.n;
    const int64_t y0 = (int64_t)band * p.rows, y1 = y0 + p.rows < n ? y0 + p.rows : n;
    const int64_t xs = (int64_t)sx * p.cps * 16;
    const int64_t ya = y0 - 1 > 0 ? y0 - 1 : 0, yb = y1 + ns < n - 1 ? y1 + ns : n - 1;
    const int64_t xa = xs - 16 > 0 ? xs - 16 : 0;
    const int64_t xb = xs + 16 * (int64_t)p.cps + 16 < n - 1 ? xs + 16 * (int64_t)p.cps + 16 : n - 1;
    cy0 = (uint32_t)(ya / p.S);
    cy1 = (uint32_t)(yb / p.S);
    cx0 = (uint32_t)(xa / p.S);
    cx1 = (uint32_t)(xb / p.S);
}

// One CTA per live tile (strip sx of the aligned rows of band b: tiles whose output
// bytes are all holes are left out of the list on the host); 2 chunks per thread.
template <bool CONWAY, int NS>
__global__ void __launch_bounds__(kBBMaxThreads, 8)
step_bb_rows_kernel(const BBRowParams p, const uint2* __restrict__ tiles, const uint32_t* __restrict__ lowtab,
                    const uint32_t* __restrict__ coarse, const uint8_t* __restrict__ src, uint8_t* __restrict__ dst) {
    static_assert(NS >= 4, "rows y-1, y, y+1 plus one in flight");
    extern __shared__ __align__(16) uint8_t sm[];
    const uint32_t W = (p.cps + 4) * 16;  // slot bytes
    const int TPB = blockDim.x, NW = TPB >> 5;
    uint32_t* lt = reinterpret_cast<uint32_t*>(sm + NS * W);
    uint32_t* ccw = lt + p.S * p.lt_words;
    uint32_t* mrow = ccw + kBBCacheWords;                         // [2][TPB + 2]
    uint8_t* flags = reinterpret_cast<uint8_t*>(mrow + 2 * (TPB + 2));  // [NS][NW]
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int64_t n = (int64_t)p.n;
    const uint2 tile = tiles[blockIdx.x];
    const int64_t y0 = (int64_t)tile.y * p.rows;
    const int64_t y1 = min(y0 + (int64_t)p.rows, n);
    const int64_t xs = (int64_t)tile.x * p.cps * 16;  // strip offset within an aligned row
    BBCoarse cc;
    uint32_t cy1;
    bb_tile_cover(p, tile.x, tile.y, NS, cc.cy0, cy1, cc.cx0, cc.cx1);
    cc.wpr = (cc.cx1 - cc.cx0 + 1 + 31) / 32 + 2;
    cc.bits = ccw;
    cc.last = 0;
    for (uint32_t ry = 0; ry <= cy1 - cc.cy0; ++ry) {
        const uint64_t b = (uint64_t)(cc.cy0 + ry) * p.CW + p.CW - 1;
        cc.last |= ((__ldg(coarse + (b >> 5)) >> (b & 31)) & 1u) << ry;
    }
    for (uint32_t i = t; i < (cy1 - cc.cy0 + 1) * cc.wpr; i += TPB) {
        const uint32_t ry = i / cc.wpr, k = i % cc.wpr;
        const uint64_t b0 = (uint64_t)(cc.cy0 + ry) * p.CW + cc.cx0 + 32ull * k;  // first bit of word k
        const uint32_t ncols = cc.cx1 - cc.cx0 + 1;
        uint32_t v = 0;
        if (32 * k < ncols) {
            v = __funnelshift_r(__ldg(coarse + (b0 >> 5)), __ldg(coarse + (b0 >> 5) + 1), (uint32_t)(b0 & 31));
            const uint32_t left = ncols - 32 * k;
            if (left < 32) v &= (1u << left) - 1u;
        }
        ccw[i] = v;
    }
    for (uint32_t i = t; i < p.S * p.lt_words; i += TPB) lt[i] = __ldg(lowtab + i);
    __syncthreads();

    // rule tables (bytes 0/1) for counts 0..7 and the count-8 entries
    uint32_t tb_lo = 0, tb_hi = 0, ts_lo = 0, ts_hi = 0;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        tb_lo |= ((p.birth >> c) & 1u) << (8 * c);
        tb_hi |= ((p.birth >> (c + 4)) & 1u) << (8 * c);
        ts_lo |= ((p.survive >> c) & 1u) << (8 * c);
        ts_hi |= ((p.survive >> (c + 4)) & 1u) << (8 * c);
    }
    const uint32_t b8 = ((p.birth >> 8) & 1u) * 0x01010101u, s8 = ((p.survive >> 8) & 1u) * 0x01010101u;

    // row rho (-1 .. n) -> the next ring slot; thread t loads chunks 2t+2, 2t+3 of
    // the segment, threads 0..3 also the margin chunks 0, 1, cps+2, cps+3.  A warp
    // whose own 64 chunks are holes zero-fills them instead and flags the slot.
    const int64_t wx = xs + (int64_t)warp * 1024;  // the warp's first byte past floor16(rho n)
    auto load_row = [&](int64_t rho, int64_t rn, int sl) {  // rn = rho * n
        uint8_t* slot = sm + sl * W;
        const int64_t base = bb_floor16(rn) + xs - 32;
        const int64_t x0 = bb_floor16(rn) + wx - rn;
        const bool live = rho < 0 || rho >= n || x0 < 0 || bb_run_live(p, cc, x0, rho);
        if (lane == 0) flags[sl * NW + warp] = live;
        auto one = [&](uint32_t ch, bool want) {
            const int64_t a = base + 16 * (int64_t)ch;
            const bool in = want && a >= 0 && a + 16 <= (int64_t)p.alloc;
            if (in) bb_cp_async16((uint32_t)__cvta_generic_to_shared(slot + 16 * ch), src + a, 16);
            else *reinterpret_cast<uint4*>(slot + 16 * ch) = make_uint4(0, 0, 0, 0);
        };
        one(2 * (uint32_t)t + 2, live);
        one(2 * (uint32_t)t + 3, live);
        if (t < 4) one(t < 2 ? (uint32_t)t : p.cps + (uint32_t)t, true);
    };
    // membership bits of row y for x in [xs - 16 + 32k, +32), k = 0 .. TPB
    auto mask_row = [&](int64_t y, uint32_t* m) {
        if (y >= y1) return;
        for (int k = t; k <= TPB; k += TPB) {
            const int64_t x0 = xs - 16 + 32 * (int64_t)k;
            uint32_t v = 0;
            if (x0 < 0) v = bb_member<32>(p, lt, cc, 0u, (uint32_t)y) << 16;  // strip 0: x0 = -16
            else if (x0 < n) v = bb_member<32>(p, lt, cc, (uint32_t)x0, (uint32_t)y);
            m[k] = v;
        }
    };

    int sl_load = 0;  // slot of row y0 - 1 (rows map to slots in order)
    {
        int64_t rn = (y0 - 1) * n;
        for (int i = 0; i < NS - 1; ++i, rn += n) {
            load_row(y0 - 1 + i, rn, sl_load);
            sl_load = sl_load + 1 == NS ? 0 : sl_load + 1;
            bb_cp_commit();
        }
    }
    mask_row(y0, mrow);
    int slU = 0;  // slot of row y - 1
    int64_t yn = y0 * n;
    int64_t rn_load = (y0 + NS - 2) * n;
    const uint32_t offM = 32 + 32 * t;
    for (int64_t y = y0; y < y1; ++y, yn += n, rn_load += n) {
        bb_cp_wait<NS - 4>();  // rows <= y + 1 landed (this thread's copies)
        __syncthreads();       // ... everyone's; slot of row y - 2 and mask row y - 1 are free
        load_row(y + NS - 2, rn_load, sl_load);
        sl_load = sl_load + 1 == NS ? 0 : sl_load + 1;
        bb_cp_commit();
        const int par = (int)((y - y0) & 1);
        mask_row(y + 1, mrow + (par ^ 1) * (TPB + 2));

        const int slM = slU + 1 == NS ? 0 : slU + 1, slD = slM + 1 == NS ? 0 : slM + 1;
        const uint8_t* sU = sm + slU * W;
        const uint8_t* sM = sm + slM * W;
        const uint8_t* sD = sm + slD * W;
        slU = slM;
        if (!flags[slM * NW + warp]) continue;  // warp-uniform: 1024 bytes of holes stay 0
        const int64_t sty = bb_floor16(yn);
        const int d = (int)(sty - yn);  // -15 .. 0
        const uint32_t offU = (uint32_t)(sty - n - bb_floor16(yn - n)) + offM;
        const uint32_t offD = (uint32_t)(sty + n - bb_floor16(yn + n)) + offM;
        const uint32_t* mr = mrow + par * (TPB + 2);
        uint32_t mem = __funnelshift_r(mr[t], mr[t + 1], (uint32_t)(16 + d));
        const int64_t c = sty + xs + 32 * (int64_t)t;
        const int64_t xc = c - yn;  // x of the pair's first byte in row y (< 0: straddles)
        if (xc < 0)  // strip 0, thread 0: the first -xc bytes end row y - 1
            mem |= bb_member<16>(p, lt, cc, (uint32_t)(n + xc), (uint32_t)(y - 1)) & ((1u << (-xc)) - 1u);
        const int64_t end = y == n - 1 ? (n * n + 15) & ~(int64_t)15 : bb_floor16(yn + n);
        if (c + 16 >= end) mem &= c >= end ? 0u : 0xFFFFu;
        uint32_t U[8], M[8], D[8];
        bb_mid32(sM, offM, M);
        uint32_t E[10];
        if (p.moore) {
            bb_mid32(sU, offU, U);
            bb_mid32(sD, offD, D);
#pragma unroll
            for (int j = 0; j < 8; ++j) E[j + 1] = U[j] + M[j] + D[j];  // bytes <= 3
        } else {
            bb_mid32(sU, offU, U);
            bb_mid32(sD, offD, D);
#pragma unroll
            for (int j = 0; j < 8; ++j) E[j + 1] = M[j];
        }
        // the columns west / east neighbours come from (Moore: vertical sums,
        // von Neumann: M); the pair's edge bytes from the neighbouring lanes
        E[0] = __shfl_up_sync(0xFFFFFFFFu, E[8], 1);
        E[9] = __shfl_down_sync(0xFFFFFFFFu, E[1], 1);
        if (lane == 0) {
            uint32_t v = sM[offM - 1];
            if (p.moore) v += sU[offU - 1] + sD[offD - 1];
            E[0] = v << 24;
        }
        if (lane == 31) {
            uint32_t v = sM[offM + 32];
            if (p.moore) v += sU[offU + 32] + sD[offD + 32];
            E[9] = v;
        }
        if (mem == 0u) continue;
        // column edges inside the pair: x = 0 at byte -xc (row y) and n - xc (row
        // y + 1); x = n - 1 one byte before each
        const int64_t b2 = n - xc;
        const bool edge = (uint64_t)(-xc) <= 32u || (uint64_t)b2 <= 32u;
        uint32_t wm[8], em[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) wm[j] = em[j] = 0u;
        if (edge) {
            const int ib1 = (int)(-xc), ib2 = (int)b2;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                wm[j] = bb_byte_mask(ib1, j) | bb_byte_mask(ib2, j);
                em[j] = bb_byte_mask(ib1 - 1, j) | bb_byte_mask(ib2 - 1, j);
            }
        }
        uint32_t out[8];
#pragma unroll
        for (int j = 1; j <= 8; ++j) {
            const uint32_t w = __funnelshift_l(E[j - 1], E[j], 8) & ~wm[j - 1];
            const uint32_t e = __funnelshift_r(E[j], E[j + 1], 8) & ~em[j - 1];
            const uint32_t cnt = p.moore ? w + E[j] + e - M[j - 1] : U[j - 1] + D[j - 1] + w + e;
            const uint32_t r = bb_rule<CONWAY>(cnt, M[j - 1], tb_lo, tb_hi, ts_lo, ts_hi, b8, s8);
            out[j - 1] = r & bb_spread4(mem >> (4 * (j - 1)));
        }
        if (mem & 0xFFFFu) *reinterpret_cast<uint4*>(dst + c) = make_uint4(out[0], out[1], out[2], out[3]);
        if (mem >> 16) *reinterpret_cast<uint4*>(dst + c + 16) = make_uint4(out[4], out[5], out[6], out[7]);
    }
    bb_cp_wait<0>();
}

// tile liveness: any fractal cell among the coarse cells covering a tile's output
// bytes (rows y0 - 1 .. y1 - 1, x in [xs - 16, xs + 16 cps + 16], column CW - 1 for
// strip 0's row-straddling chunks)
__global__ void bb_tile_live_kernel(const BBRowParams p, const uint32_t* __restrict__ coarse, uint32_t nsx,
                                    uint32_t nbands, uint8_t* __restrict__ live) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < (uint64_t)nsx * nbands;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t sx = (uint32_t)(i % nsx), band = (uint32_t)(i / nsx);
        uint32_t cy0, cy1, cx0, cx1;
        bb_tile_cover(p, sx, band, 0, cy0, cy1, cx0, cx1);
        bool any = false;
        for (uint32_t cy = cy0; cy <= cy1 && !any; ++cy) {
            for (uint32_t cx = cx0; cx <= cx1 && !any; ++cx) {
                const uint64_t b = (uint64_t)cy * p.CW + cx;
                any = (coarse[b >> 5] >> (b & 31)) & 1u;
            }
            if (sx == 0) {
                const uint64_t b = (uint64_t)cy * p.CW + p.CW - 1;
                any = any || ((coarse[b >> 5] >> (b & 31)) & 1u);
            }
        }
        live[i] = any ? 1 : 0;
    }
}

// coarse membership bitmap: bit cy * CW + cx = cells (cx, cy) of the level-L
// coarse box are in the fractal (the top L levels of maps.cpp:80-107)
__global__ void bb_coarse_kernel(Frac f, int L, uint32_t CW, uint32_t* __restrict__ out, uint64_t nwords) {
    for (uint64_t wi = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; wi < nwords;
         wi += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t v = 0;
        for (int b = 0; b < 32; ++b) {
            const uint64_t i = wi * 32 + b;
            if (i >= (uint64_t)CW * CW) break;
            uint32_t x = (uint32_t)(i % CW), y = (uint32_t)(i / CW);
            bool in = true;
            for (int mu = 0; mu < L && in; ++mu) {
                in = f.id_of_subbox[(y % f.s) * f.s + (x % f.s)] >= 0;
                x /= f.s;
                y /= f.s;
            }
            if (in) v |= 1u << b;
        }
        out[wi] = v;
    }
}

}  // namespace nbbgpu
