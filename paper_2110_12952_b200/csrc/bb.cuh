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
#include "tiled.cuh"  // count8, apply_rule_bits (bit-sliced counts and rules)

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
    uint32_t ntiles;    // live tiles (the tile list)
    uint32_t birth, survive;
    int moore;
};

// 4 bits -> 4 bytes of 0/1
__device__ __forceinline__ uint32_t bb_spread4(uint32_t nib) { return ((nib & 0xFu) * 0x00204081u) & 0x01010101u; }

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

// 32 bytes of 0/1 (8 words) -> 32 bits, bit i = byte i
__device__ __forceinline__ uint32_t bb_pack32(const uint4 a, const uint4 b) {
    const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    uint32_t bits = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) bits |= ((w[j] * 0x01020408u) >> 24) << (4 * j);  // b0 + 2 b1 + 4 b2 + 8 b3
    return bits;
}

// the 32 cells [off, off + 32) of a bit row, and the cells off - 1 (top bit of
// west) and off + 32 (bit 0 of east); off & 31 is warp-uniform, off >= 1
__device__ __forceinline__ void bb_bits_window(const uint32_t* row, uint32_t off, uint32_t& v, uint32_t& west,
                                               uint32_t& east) {
    const uint32_t w = off >> 5, sh = off & 31;
    const uint32_t a = row[w], b = row[w + 1];
    v = __funnelshift_r(a, b, sh);
    west = sh ? a << (32 - sh) : row[w - 1];
    east = __funnelshift_r(b, row[w + 2], sh);
}

// shared-memory layout of step_bb_rows_kernel: NS ring slots, the low table, the
// coarse cache (kBBCacheWords), the live flags [NS][warps], two mask rows
constexpr uint32_t kBBCacheWords = 64;
constexpr int kBBStages = 6;  // byte ring (rows y+2 .. y+4 in flight)
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
// bytes are all holes are left out of the list on the host); 32 cells per thread.
// Rows stream in as bytes (cp.async ring, NS slots), each thread packs its own 32
// bytes of row y + 2 to one bit word (bit ring of 4 rows), and row y is computed
// bit-sliced: 32 cells per word op (count8 adders + the rule), unpacked to bytes
// only for the two 16-byte stores.
template <bool CONWAY, int NS>
__global__ void __launch_bounds__(kBBMaxThreads, 8)
step_bb_rows_kernel(const BBRowParams p, const uint2* __restrict__ tiles, const uint32_t* __restrict__ memb,
                    const uint32_t* __restrict__ coarse, const uint8_t* __restrict__ src, uint8_t* __restrict__ dst) {
    static_assert(NS >= 5, "rows y+3.. in flight while row y+2 is packed");
    constexpr int NB = 4;  // bit ring: rows y-1 .. y+2
    extern __shared__ __align__(16) uint8_t sm[];
    const uint32_t W = (p.cps + 4) * 16;  // byte slot
    const int TPB = blockDim.x, NW = TPB >> 5;
    const uint32_t BWS = (uint32_t)TPB + 4;  // bit slot words (+ pad for the shifted windows)
    const uint32_t MWS = (uint32_t)TPB + 4;  // membership words per slot
    uint32_t* bits = reinterpret_cast<uint32_t*>(sm + NS * W);    // [NB][BWS]
    uint32_t* mslot = bits + NB * BWS;                            // [NS][MWS] membership bits of the slot
    uint32_t* ccw = mslot + NS * MWS;
    uint8_t* flags = reinterpret_cast<uint8_t*>(ccw + kBBCacheWords);  // [NS][NW]
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int64_t n = (int64_t)p.n;
    uint32_t KB[9], KS[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) {
        KB[i] = ((p.birth >> i) & 1u) ? 0xFFFFFFFFu : 0u;
        KS[i] = ((p.survive >> i) & 1u) ? 0xFFFFFFFFu : 0u;
    }
    const uint2 tile = tiles[blockIdx.x];  // one live tile per CTA
    const int64_t y0 = (int64_t)tile.y * p.rows;
    const int64_t y1 = min(y0 + (int64_t)p.rows, n);
    const int64_t xs = (int64_t)tile.x * p.cps * 16;  // strip offset within an aligned row
    BBCoarse cc;  // (the hole-skip test)
    uint32_t cy1;
    bb_tile_cover(p, tile.x, tile.y, NS, cc.cy0, cy1, cc.cx0, cc.cx1);
    cc.wpr = (cc.cx1 - cc.cx0 + 1 + 31) / 32 + 2;
    cc.bits = ccw;
    cc.last = 0;
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
    for (uint32_t i = t; i < NB * BWS; i += TPB) bits[i] = 0u;
    __syncthreads();

    // row rho (-1 .. n) -> the next byte slot; thread t loads chunks 2t+2, 2t+3 of
    // the segment, thread 0 also the margin chunks 0, 1 and thread 1 cps+2, cps+3,
    // and the segment's membership words (static bitmap, bit i = linear byte i).
    // A warp whose own 64 chunks are holes loads nothing and flags the slot.
    const int64_t wx = xs + (int64_t)warp * 1024;  // the warp's first byte past floor16(rho n)
    const int64_t mwords = ((int64_t)p.alloc + 31) / 32;
    auto load_row = [&](int64_t rho, int64_t rn, int sl) {  // rn = rho * n
        uint8_t* slot = sm + sl * W;
        const int64_t base = bb_floor16(rn) + xs - 32;
        const int64_t x0 = bb_floor16(rn) + wx - rn;
        const bool live = rho < 0 || rho >= n || x0 < 0 || bb_run_live(p, cc, x0, rho);
        if (lane == 0) flags[sl * NW + warp] = live;
        // (the whole segment inside the buffer: no per-chunk bounds)
        const bool inside = base >= 0 && base + (int64_t)W <= (int64_t)p.alloc;
        const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(slot);
        auto one = [&](uint32_t ch) {
            const int64_t a = base + 16 * (int64_t)ch;
            const bool in = inside || (a >= 0 && a + 16 <= (int64_t)p.alloc);
            bb_cp_async16(sbase + 16 * ch, in ? src + a : src, in ? 16u : 0u);
        };
        if (live) {
            one(2 * (uint32_t)t + 2);
            one(2 * (uint32_t)t + 3);
        }
        if (t < 2) {
            one(t == 0 ? 0u : p.cps + 2);
            one(t == 0 ? 1u : p.cps + 3);
        }
        // membership words floor32(base) / 32 + k, k = 0 .. TPB + 2 (thread t: k = t, and
        // threads 0..2 also k = TPB .. TPB + 2)
        const int64_t w0 = (base >= 0 ? base : base - 31) / 32;
        const uint32_t mbase = (uint32_t)__cvta_generic_to_shared(mslot + sl * MWS);
        for (int k = t; k < TPB + 3; k += TPB) {
            const int64_t w = w0 + k;
            const bool in = w >= 0 && w < mwords;
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(mbase + 4u * (uint32_t)k),
                         "l"(in ? memb + w : memb), "r"(in ? 4u : 0u)
                         : "memory");
        }
    };
    // the thread's own 32 bytes of byte slot sl -> bit word of bit slot bl
    auto pack_row = [&](int sl, int bl) {
        const uint8_t* slot = sm + sl * W;
        uint32_t* brow = bits + bl * BWS;
        if (flags[sl * NW + warp]) {
            const uint4* v = reinterpret_cast<const uint4*>(slot + 32 + 32 * t);
            brow[1 + t] = bb_pack32(v[0], v[1]);
        } else {
            brow[1 + t] = 0u;
        }
        if (t < 2) {
            const uint4* v = reinterpret_cast<const uint4*>(slot + (t == 0 ? 0u : 16 * (p.cps + 2)));
            brow[t == 0 ? 0 : TPB + 1] = bb_pack32(v[0], v[1]);
        }
    };

    // prologue: rows y0-1 .. y0+NS-3 in flight, rows y0-1 .. y0+1 packed
    {
        int64_t rn = (y0 - 1) * n;
        for (int i = 0; i < NS - 1; ++i, rn += n) {
            load_row(y0 - 1 + i, rn, i);
            bb_cp_commit();
        }
    }
    __syncwarp();  // lane 0's live flags
    bb_cp_wait<NS - 4>();  // rows y0-1 .. y0+1 (this thread's copies)
    for (int i = 0; i < 3; ++i) pack_row(i, i);
    int sl_load = NS - 1;  // byte slot of the next row to load (y0 + NS - 2)
    int sl_y = 1 % NS;     // byte slot of row y (row y0 - 1 is in slot 0)
    int bU = 0;            // bit slot of row y - 1 (rows map to bit slots in order)
    int64_t yn = y0 * n;
    int64_t rn_load = (y0 + NS - 2) * n;
    const uint32_t offM = 32 + 32 * t;  // the thread's cells in a segment (bit offset == byte offset)
    for (int64_t y = y0; y < y1; ++y, yn += n, rn_load += n) {
        bb_cp_wait<NS - 5>();  // row y + 2 landed (this thread's copies)
        __syncthreads();       // rows <= y + 1 packed (and their membership words landed); slots of rows y - 2 free
        load_row(y + NS - 2, rn_load, sl_load);
        sl_load = sl_load + 1 == NS ? 0 : sl_load + 1;
        bb_cp_commit();
        const int sl_c = sl_y;  // byte slot of row y (its live flags, its membership words)
        sl_y = sl_y + 1 == NS ? 0 : sl_y + 1;
        const int sl2 = sl_c + 2 >= NS ? sl_c + 2 - NS : sl_c + 2;  // byte slot of row y + 2
        const int bM = bU + 1 == NB ? 0 : bU + 1, bD = bM + 1 == NB ? 0 : bM + 1, b2 = bD + 1 == NB ? 0 : bD + 1;
        pack_row(sl2, b2);

        const uint32_t* Ub = bits + bU * BWS;
        const uint32_t* Mb = bits + bM * BWS;
        const uint32_t* Db = bits + bD * BWS;
        bU = bM;
        if (!flags[sl_c * NW + warp]) continue;  // warp-uniform: 1024 hole bytes stay 0
        const int64_t sty = bb_floor16(yn);
        // the pair's membership: bits (32 + 32 t + (base & 31)) of the slot's words,
        // base = the slot's first byte (floor16: its bit offset in word 0 is 0 or 16)
        const uint32_t* ms = mslot + sl_c * MWS;
        const uint32_t sh = (uint32_t)((sty + xs - 32) & 31);
        uint32_t mem = __funnelshift_r(ms[1 + t], ms[2 + t], sh);
        const int64_t c = sty + xs + 32 * (int64_t)t;
        const int64_t xc = c - yn;  // x of the pair's first byte in row y (< 0: straddles)
        const int64_t end = y == n - 1 ? (n * n + 15) & ~(int64_t)15 : bb_floor16(yn + n);
        if (c + 16 >= end) mem &= c >= end ? 0u : 0xFFFFu;
        if (mem == 0u) continue;
        // the three rows: own 32 cells + the cells west / east of them
        const uint32_t m = Mb[1 + t], mwb = Mb[t], meb = Mb[t + 2];
        uint32_t u, uwb, ueb, dd, dwb, deb;
        bb_bits_window(Ub, (uint32_t)(sty - n - bb_floor16(yn - n)) + offM, u, uwb, ueb);
        bb_bits_window(Db, (uint32_t)(sty + n - bb_floor16(yn + n)) + offM, dd, dwb, deb);
        // column edges inside the pair: x = 0 at bit -xc (row y) and n - xc (row y + 1);
        // x = n - 1 one bit before each: no west / east neighbours there
        const int64_t b1 = -xc, b2e = n - xc;
        uint32_t wm = 0u, em = 0u;
        if ((uint64_t)b1 <= 32u || (uint64_t)b2e <= 32u) {
            if (b1 >= 0 && b1 < 32) wm |= 1u << b1;
            if (b2e >= 0 && b2e < 32) wm |= 1u << b2e;
            if (b1 >= 1 && b1 <= 32) em |= 1u << (b1 - 1);
            if (b2e >= 1 && b2e <= 32) em |= 1u << (b2e - 1);
        }
        const uint32_t mw = ((m << 1) | (mwb >> 31)) & ~wm, me = ((m >> 1) | (meb << 31)) & ~em;
        uint32_t r;
        if (p.moore) {
            const uint32_t uw = ((u << 1) | (uwb >> 31)) & ~wm, ue = ((u >> 1) | (ueb << 31)) & ~em;
            const uint32_t dw = ((dd << 1) | (dwb >> 31)) & ~wm, de = ((dd >> 1) | (deb << 31)) & ~em;
            r = apply_rule_bits<CONWAY>(count8(uw, u, ue, mw, me, dw, dd, de), m, KB, KS);
        } else {
            r = apply_rule_bits<false>(count8(u, dd, mw, me, 0u, 0u, 0u, 0u), m, KB, KS);
        }
        r &= mem;
        if (mem & 0xFFFFu)
            *reinterpret_cast<uint4*>(dst + c) = make_uint4(bb_spread4(r), bb_spread4(r >> 4), bb_spread4(r >> 8),
                                                            bb_spread4(r >> 12));
        if (mem >> 16)
            *reinterpret_cast<uint4*>(dst + c + 16) = make_uint4(bb_spread4(r >> 16), bb_spread4(r >> 20),
                                                                 bb_spread4(r >> 24), bb_spread4(r >> 28));
    }
    bb_cp_wait<0>();
}

// membership bitmap of the box (static, built once per handle): bit i of word w =
// linear byte 32 w + i is a fractal cell (0 past n^2)
__global__ void bb_member_bitmap_kernel(const BBRowParams p, const uint32_t* __restrict__ lowtab,
                                        const uint32_t* __restrict__ coarse, uint32_t* __restrict__ out,
                                        uint64_t nwords) {
    const uint64_t cells = p.n * p.n;
    for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < nwords;
         w += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t v = 0;
        for (int b = 0; b < 32; ++b) {
            const uint64_t i = w * 32 + b;
            if (i >= cells) break;
            const uint32_t x = (uint32_t)(i % p.n), y = (uint32_t)(i / p.n);
            const uint32_t cx = bb_div(p, x), cy = bb_div(p, y);
            const uint32_t xl = x - cx * p.S, yl = y - cy * p.S;
            const bool lo = (__ldg(lowtab + yl * p.lt_words + (xl >> 5)) >> (xl & 31)) & 1u;
            const uint64_t cb = (uint64_t)cy * p.CW + cx;
            const bool hi = (__ldg(coarse + (cb >> 5)) >> (cb & 31)) & 1u;
            v |= (uint32_t)(lo && hi) << b;
        }
        out[w] = v;
    }
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
