// tiled.cuh -- the throughput path: tile-parallel bit-sliced compact stencil.
//
// Structure used: fixing the top r-q replica digits (q even)
// selects a level-q sub-fractal that is exactly a WQ x WQ (WQ = k^(q/2))
// sub-rectangle of the compact array, laid out like the level-q compact array.
// Every tile therefore shares ONE local neighbour structure; only the links that
// leave the tile need the coarse (level r-q) maps.
//
// Work unit = a "group": 32 horizontally consecutive tiles of one coarse row.
// Bit b of a 32-bit word is tile b of the group (SIMD over tiles), so the
// stencil of a local cell is a fixed bit-sliced adder over the words of its
// neighbours -- no per-cell maps at all.  Per group and per local row a, one lane
//   forward : loads the 32*WQ contiguous bytes of row a (32-B vector loads),
//             packs bytes to bits, cuts the 32 WQ-bit tile rows and transposes
//             the 32x32 bit matrix in registers -> WQ words W[a][c] (bit b);
//   program : all lanes run the table-driven bit-sliced Life step per word;
//   backward: transposes back, unpacks bits to bytes, stores 32-B vectors.
// The reference semantics (stencil.cpp:334-368) are preserved bit for bit:
// out-of-box and hole neighbours count 0, states are read from src and written
// to dst only (double buffer).
#pragma once

#include "common.cuh"

namespace nbbgpu {

constexpr int kTiledWarps = 1;       // warps per block (smem-limited occupancy: fine-grained)
constexpr int kStageChunks = 4;      // 32-B chunks per row per load stage (128 B)
constexpr int kStageBufs = 2;        // stage buffers per warp (double buffering)
constexpr int kStageRow = kStageChunks * 32 + 16;  // padded row stride: conflict-free LDS.128
constexpr int kHaloBatch = 8;        // halo slots gathered per batch
constexpr int kMaxHalo = 512;

struct TiledParams {
    Frac f;                  // full-level tables (k, s, replica tables)
    int L;                   // coarse level r - q
    int C;                   // cells per tile k^q
    int nH;                  // halo slots
    int nD;                  // directions with halo slots
    int8_t dlist[8];         // D (= (dy+1)*3 + dx+1) of each used direction slot
    uint32_t Wc, Hc;         // coarse compact dims (< 65535)
    uint32_t gpr;            // groups per coarse row = ceil(Wc / 32)
    uint32_t row0, row1;     // owned coarse rows [row0, row1)
    uint64_t w;              // compact row stride (bytes)
    uint32_t birth, survive;
    const uint32_t* nbr;     // C x 8 smem byte offsets into the group's word array
    const uint32_t* ntab;    // [nD][Hc][Wc] coarse neighbour tile, (Y2 << 16) | X2, ~0 = none
    const uint8_t* halo_D;   // per slot: direction slot (index into dlist)
    const uint16_t* halo_a;  // per slot: source local row in the neighbour tile
    const uint16_t* halo_c;  // per slot: source local column
    const uint64_t* halo_off;// per slot: halo_a * w + halo_c (byte offset inside the tile)
    uint32_t smem_per_warp;  // bytes
    uint32_t words_per_group;// C + nH + 1 (padded)
};

// ---------------------------------------------------------------------------
// coarse neighbour: nu(lambda(X, Y) + (dx, dy)) at level L as a carry walk over
// the replica digits (only the levels the +-1 carry touches change), exactly the
// composition CoordMapper::to_embedded -> offset -> try_to_compact
// (maps.cpp:80-146) restricted to the changed digits.
// ---------------------------------------------------------------------------
template <int K, int S>
__device__ __forceinline__ bool coarse_neighbor(const Frac& f, int L, uint32_t X, uint32_t Y,
                                                int dx, int dy, uint32_t& X2, uint32_t& Y2) {
    const int k = K ? K : f.k, s = S ? S : f.s;
    uint32_t cx = X, cy = Y;
    int pw = 1;
    int nx = (int)X, ny = (int)Y;
    for (int mu = 0; mu < L; ++mu) {
        if (dx == 0 && dy == 0) break;
        int d;
        if ((mu & 1) == 0) { d = (int)(cx % (uint32_t)k); cx /= (uint32_t)k; }
        else               { d = (int)(cy % (uint32_t)k); cy /= (uint32_t)k; }
        int gx = f.gx[d] + dx, gy = f.gy[d] + dy;
        dx = gx < 0 ? -1 : (gx >= s ? 1 : 0);
        gx -= dx * s;
        dy = gy < 0 ? -1 : (gy >= s ? 1 : 0);
        gy -= dy * s;
        const int id = f.id_of_subbox[gy * s + gx];
        if (id < 0) return false;
        if ((mu & 1) == 0) nx += (id - d) * pw;
        else { ny += (id - d) * pw; pw *= k; }
    }
    X2 = (uint32_t)nx;
    Y2 = (uint32_t)ny;
    return dx == 0 && dy == 0;
}

// Static coarse-neighbour table (setup, once per tile plan): for every coarse tile
// (X, Y) and every direction slot ds, the packed neighbour tile (Y2 << 16) | X2 or
// ~0 when the neighbour is a hole or outside the box.
template <int K, int S>
__global__ void build_ntab_kernel(Frac f, int L, uint32_t Wc, uint32_t Hc, int nD, int8_t d0,
                                  int8_t d1, int8_t d2, int8_t d3, int8_t d4, int8_t d5, int8_t d6,
                                  int8_t d7, uint32_t* __restrict__ out) {
    const int8_t dl[8] = {d0, d1, d2, d3, d4, d5, d6, d7};
    const uint64_t n = (uint64_t)Wc * Hc;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t X = (uint32_t)(i % Wc), Y = (uint32_t)(i / Wc);
        for (int ds = 0; ds < nD; ++ds) {
            const int D = dl[ds];
            uint32_t X2, Y2, v = 0xFFFFFFFFu;
            if (coarse_neighbor<K, S>(f, L, X, Y, D % 3 - 1, D / 3 - 1, X2, Y2)) v = (Y2 << 16) | X2;
            out[(uint64_t)ds * n + i] = v;
        }
    }
}

struct u32x8 { uint32_t v[8]; };

__device__ __forceinline__ u32x8 ldg256(const void* p) {
    u32x8 r;
    asm volatile("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r.v[0]), "=r"(r.v[1]), "=r"(r.v[2]), "=r"(r.v[3]),
                   "=r"(r.v[4]), "=r"(r.v[5]), "=r"(r.v[6]), "=r"(r.v[7])
                 : "l"(p));
    return r;
}

__device__ __forceinline__ void stg256(void* p, const u32x8& r) {
    asm volatile("st.global.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                 :: "l"(p), "r"(r.v[0]), "r"(r.v[1]), "r"(r.v[2]), "r"(r.v[3]),
                    "r"(r.v[4]), "r"(r.v[5]), "r"(r.v[6]), "r"(r.v[7])
                 : "memory");
}

__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(p), "r"(bytes) : "memory");
}

// cp.async (LDGSTS): global -> shared without holding registers; per-thread groups.
__device__ __forceinline__ void cp_async16(uint32_t saddr, const void* g) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(saddr), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" :: "n"(N) : "memory"); }

__device__ __forceinline__ u32x8 lds256(uint32_t saddr) {
    u32x8 r;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.v[0]), "=r"(r.v[1]), "=r"(r.v[2]), "=r"(r.v[3]) : "r"(saddr));
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.v[4]), "=r"(r.v[5]), "=r"(r.v[6]), "=r"(r.v[7]) : "r"(saddr + 16));
    return r;
}

// 8 bytes (each 0/1) in (lo, hi) -> bits 24..31 of the result, bit 24+j = byte j:
// the high word of the 64-bit product (hi:lo) * 0x0102040810204080 (byte j's bit 0
// lands on bit 56+j; no two partial products share a bit, so no carries).
__device__ __forceinline__ uint32_t pack8_top(uint32_t lo, uint32_t hi) {
    uint32_t r = __umulhi(lo, 0x10204080u);
    r += lo * 0x01020408u;
    r += hi * 0x10204080u;
    return r;
}

// 32 bytes (each 0/1) -> 32 bits, bit t = byte t: 12 IMAD (FMA pipe) + 3 PRMT.
__device__ __forceinline__ uint32_t pack32(const u32x8& r) {
    const uint32_t a = pack8_top(r.v[0], r.v[1]), b = pack8_top(r.v[2], r.v[3]);
    const uint32_t c = pack8_top(r.v[4], r.v[5]), d = pack8_top(r.v[6], r.v[7]);
    return __byte_perm(__byte_perm(a, b, 0x0073), __byte_perm(c, d, 0x0073), 0x5410);
}

// 32 bits -> 32 bytes of 0/1 (bit j of a nibble -> bit 8j via * 0x00204081)
__device__ __forceinline__ u32x8 unpack32(uint32_t w) {
    u32x8 r;
#pragma unroll
    for (int j = 0; j < 8; ++j) r.v[j] = (((w >> (4 * j)) & 0xFu) * 0x00204081u) & 0x01010101u;
    return r;
}

// In-register 32x32 bit transpose: A[i] bit j -> A[j] bit i (Hacker's Delight 7-3).
__device__ __forceinline__ void transpose32(uint32_t (&A)[32]) {
#pragma unroll
    for (int j = 16, m = 0x0000FFFF; j != 0; j >>= 1, m ^= (m << j)) {
#pragma unroll
        for (int k = 0; k < 32; k = (k + j + 1) & ~j) {
            const uint32_t t = ((A[k] >> j) ^ A[k + j]) & (uint32_t)m;
            A[k] ^= t << j;
            A[k + j] ^= t;
        }
    }
}

// Byte-exact store of bytes [lo, hi) (0 <= lo < hi <= 32) of the 32-B chunk whose
// 0/1 bytes are the bits of w: whole 4-B words inside the range as u32 stores,
// the (at most two) boundary words byte/half-word wise.  No dynamic indexing.
__device__ __forceinline__ uint32_t nibble_bytes(uint32_t w, int word) {
    return (((w >> (4 * word)) & 0xFu) * 0x00204081u) & 0x01010101u;
}

__device__ __forceinline__ void store_bits_range(uint8_t* p32, uint32_t w, int lo, int hi) {
    if (lo == 0 && hi == 32) { stg256(p32, unpack32(w)); return; }
    const int wlo = (lo + 3) >> 2, whi = hi >> 2;  // whole words [wlo, whi)
#pragma unroll
    for (int q = 0; q < 8; ++q)
        if (q >= wlo && q < whi) *reinterpret_cast<uint32_t*>(p32 + 4 * q) = nibble_bytes(w, q);
    if (lo & 3) {  // head boundary word: bytes [lo, min(hi, 4*wlo))
        const int q = lo >> 2;
        const uint32_t v = nibble_bytes(w, q);
        const int e = min(hi, 4 * q + 4);
        for (int i = lo; i < e; ++i) p32[i] = (uint8_t)(v >> (8 * (i & 3)));
    }
    if ((hi & 3) && (hi >> 2) >= wlo) {  // tail boundary word: bytes [4*(hi>>2), hi)
        const int q = hi >> 2;
        const uint32_t v = nibble_bytes(w, q);
        for (int i = 4 * q; i < hi; ++i) p32[i] = (uint8_t)(v >> (8 * (i & 3)));
    }
}

// Bit-sliced neighbour count of up to 8 words: count = b0 + 2 b1 + 4 b2 + 8 b3.
struct Count4 { uint32_t b0, b1, d1, d2; };  // b2 = d1 ^ d2, b3 = d1 & d2

__device__ __forceinline__ Count4 count8(uint32_t x0, uint32_t x1, uint32_t x2, uint32_t x3,
                                         uint32_t x4, uint32_t x5, uint32_t x6, uint32_t x7) {
    const uint32_t s1 = x0 ^ x1 ^ x2, c1 = (x0 & x1) | (x2 & (x0 ^ x1));
    const uint32_t s2 = x3 ^ x4 ^ x5, c2 = (x3 & x4) | (x5 & (x3 ^ x4));
    const uint32_t s3 = s1 ^ s2 ^ x6, c3 = (s1 & s2) | (x6 & (s1 ^ s2));
    Count4 r;
    r.b0 = s3 ^ x7;
    const uint32_t c4 = s3 & x7;
    const uint32_t t1 = c1 ^ c2 ^ c3;
    r.d1 = (c1 & c2) | (c3 & (c1 ^ c2));
    r.b1 = t1 ^ c4;
    r.d2 = t1 & c4;
    return r;
}

__device__ __forceinline__ uint32_t sel(uint32_t p, uint32_t a, uint32_t b) {
    return (p & a) | (~p & b);  // p ? a : b per bit (one LOP3)
}

// Outer-totalistic rule on bit-sliced counts.  CONWAY: B3/S23 specialisation.
template <bool CONWAY>
__device__ __forceinline__ uint32_t apply_rule_bits(const Count4& c, uint32_t alive,
                                                    const uint32_t (&KB)[9],
                                                    const uint32_t (&KS)[9]) {
    if (CONWAY) {
        // count in {2,3} and (count == 3 or alive)
        return c.b1 & ~(c.d1 | c.d2) & (c.b0 | alive);
    } else {
        const uint32_t b2 = c.d1 ^ c.d2, b3 = c.d1 & c.d2;
        uint32_t L[9];
#pragma unroll
        for (int i = 0; i < 9; ++i) L[i] = sel(alive, KS[i], KB[i]);
        const uint32_t m01 = sel(c.b0, L[1], L[0]), m23 = sel(c.b0, L[3], L[2]);
        const uint32_t m45 = sel(c.b0, L[5], L[4]), m67 = sel(c.b0, L[7], L[6]);
        const uint32_t m03 = sel(c.b1, m23, m01), m47 = sel(c.b1, m67, m45);
        const uint32_t m07 = sel(b2, m47, m03);
        return sel(b3, L[8], m07);
    }
}

template <int WQ>
struct TileGeom {
    static constexpr int HQ = WQ;
    static constexpr int C = WQ * WQ;
    static constexpr int G = (32 / HQ) > 0 ? (32 / HQ) : 1;    // groups per warp
    static constexpr int ROWS = G * HQ;                         // staged rows per warp
    static constexpr int NW = WQ;                               // 32-bit words of a 32-tile row
    static constexpr int NCH = NW + 1;                          // 32-B chunks of a row (aligned)
    static constexpr int NSTG = (NCH + kStageChunks - 1) / kStageChunks;
    static constexpr int SBUF = ROWS * kStageRow;               // bytes of one stage buffer
    static constexpr int NPL = (G * C + 31) / 32;               // program cells per lane
};

// bytes of dynamic smem per warp for a tile width (host and device agree)
__host__ __device__ constexpr uint32_t tiled_smem_per_warp(int wq, uint32_t wpg) {
    return (uint32_t)((32 / wq > 0 ? 32 / wq : 1) * wpg * 4                 // word arrays
                      + 2 * 32 * 8                                           // row table (2 x 32 u64)
                      + 2 * 8 * 32 * 4                                       // neighbour tiles NT[2][8][32]
                      + kStageBufs * (32 / wq > 0 ? 32 / wq : 1) * wq * kStageRow);  // stages
}

template <int WQ, int K, int S, bool CONWAY>
__global__ void __launch_bounds__(kTiledWarps * 32, 17)
step_tiled_kernel(const TiledParams p, const uint8_t* __restrict__ src, uint8_t* __restrict__ dst) {
    using TG = TileGeom<WQ>;
    constexpr int HQ = TG::HQ, C = TG::C, G = TG::G, ROWS = TG::ROWS, NW = TG::NW;
    constexpr int NSTG = TG::NSTG, SBUF = TG::SBUF, NPL = TG::NPL;
    extern __shared__ __align__(16) uint8_t smem_raw[];

    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    // per warp: G word arrays WD [wpg] | row table RT[2][32] (u64: aligned base | span<<48)
    //           | kStageBufs stage buffers [ROWS][kStageRow]
    uint8_t* wsm = smem_raw + warp * p.smem_per_warp;
    uint32_t* wbase = reinterpret_cast<uint32_t*>(wsm);
    const uint32_t wpg = p.words_per_group;
    uint64_t* RT = reinterpret_cast<uint64_t*>(wsm + G * wpg * 4);
    uint32_t* NT = reinterpret_cast<uint32_t*>(wsm + G * wpg * 4 + 2 * 32 * 8);
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(wsm + G * wpg * 4 + 2 * 32 * 8 + 2 * 8 * 32 * 4);

    uint32_t KB[9], KS[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) {
        KB[i] = ((p.birth >> i) & 1u) ? 0xFFFFFFFFu : 0u;
        KS[i] = ((p.survive >> i) & 1u) ? 0xFFFFFFFFu : 0u;
    }

    const uint32_t total_groups = (p.row1 - p.row0) * p.gpr;   // < 2^32 (Wc, Hc < 2^16)
    const uint32_t warp_global = blockIdx.x * kTiledWarps + warp;
    const uint32_t nwarps = gridDim.x * kTiledWarps;

    // group g -> coarse row Y and first coarse column X0 of its 32 tiles
    auto gpos = [&](uint32_t g, uint32_t& Y, uint32_t& X0) {
        const uint32_t yy = g / p.gpr;
        Y = p.row0 + yy;
        X0 = (g - yy * p.gpr) * 32;
    };
    // row table for the groups starting at gbase: lane r < ROWS records its row's
    // 32-B aligned start and the span [0, delta + segbytes) of the aligned frame
    auto fill_rows = [&](uint32_t gbase, int buf) {
        if (lane < ROWS) {
            const int gs = lane / HQ, a = lane - (lane / HQ) * HQ;
            const uint32_t g = gbase + gs;
            uint64_t e = 0;
            if (g < total_groups) {
                uint32_t Y, X0;
                gpos(g, Y, X0);
                const uint64_t seg = ((uint64_t)Y * HQ + a) * p.w + (uint64_t)X0 * WQ;
                const uint64_t span = (seg & 31) + min(32u, p.Wc - X0) * WQ;
                e = (seg & ~31ull) | (span << 48);
            }
            RT[buf * 32 + lane] = e;
        }
    };
    // stage st of the rows in RT[buf]: 16-B pieces, 8 consecutive lanes per 128-B row
    // piece -> coalesced full-line requests; one cp.async group per stage per thread
    auto issue_stage = [&](int buf, int st) {
        if (st < NSTG) {
#pragma unroll
            for (int i = 0; i < (ROWS * 8 + 31) / 32; ++i) {
                const int pc = 32 * i + lane;
                const int r = pc >> 3, off = (pc & 7) * 16;
                if (r < ROWS) {
                    const uint64_t e = RT[buf * 32 + r];
                    const int cb = st * (kStageChunks * 32) + off;
                    if (cb < (int)(e >> 48))
                        cp_async16(sbase + (st % kStageBufs) * SBUF + r * kStageRow + off,
                                   src + (e & 0xFFFFFFFFFFFFull) + cb);
                }
            }
        }
        cp_async_commit();
    };
    // neighbour tile of tile X in coarse row Y for halo slot j (~0: none)
    auto halo_tile = [&](uint32_t Y, uint32_t X, int j) -> uint32_t {
        if (X >= p.Wc) return 0xFFFFFFFFu;
        return __ldg(p.ntab + ((uint64_t)p.halo_D[j] * p.Hc + Y) * p.Wc + X);
    };
    auto halo_load = [&](uint32_t t, int j) -> uint8_t {
        if (t == 0xFFFFFFFFu) return 0;
        return __ldg(src + (uint64_t)(t >> 16) * (HQ * p.w) + (uint64_t)(t & 0xFFFFu) * WQ +
                     __ldg(p.halo_off + j));
    };
    // neighbour tiles of group slot 0 of group gbase -> NT[buf] via cp.async (no
    // registers held; lands one group ahead of its use)
    auto nt_request = [&](uint32_t gbase, int buf) {
        uint32_t Y = 0, X0 = 0;
        const bool gv = gbase < total_groups;
        if (gv) gpos(gbase, Y, X0);
        const uint32_t X = X0 + lane;
        const uint32_t ntb = (uint32_t)__cvta_generic_to_shared(NT + buf * 8 * 32 + lane);
#pragma unroll
        for (int ds = 0; ds < 8; ++ds) {
            if (ds < p.nD) {
                if (gv && X < p.Wc)
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(ntb + ds * 32 * 4),
                                 "l"(p.ntab + ((uint64_t)ds * p.Hc + Y) * p.Wc + X) : "memory");
                else
                    NT[buf * 8 * 32 + ds * 32 + lane] = 0xFFFFFFFFu;
            }
        }
    };

    // ---- prologue: first group's row table, stages 0..1, halo bytes ------------------
    int rbuf = 0;
    fill_rows(warp_global * G, rbuf);
    __syncwarp();
    issue_stage(rbuf, 0);
    nt_request(warp_global * G + nwarps * G, 1);  // completes with stage 1's group
    issue_stage(rbuf, 1);
    uint8_t hv0[kHaloBatch];
    {
        uint32_t Y = 0, X0 = 0;
        const bool gv = warp_global * G < total_groups;
        if (gv) gpos(warp_global * G, Y, X0);
#pragma unroll
        for (int jj = 0; jj < kHaloBatch; ++jj)
            hv0[jj] = (gv && jj < p.nH) ? halo_load(halo_tile(Y, X0 + lane, jj), jj) : 0;
    }

    for (uint32_t g0 = warp_global * G; g0 < total_groups; g0 += nwarps * G) {
        // ---- forward: bytes -> bit-sliced words ------------------------------------
        // Per lane (row a of group slot gs): a runtime loop over the 32-B chunks of
        // the aligned frame packs bytes to bits and stores the delta-shifted words
        // SW_t (bit i = byte seg + 32t + i) into the lane's scratch row of WD; the
        // 32 tile rows R_b are then cut from SW with static shifts and transposed.
        // Stage st + 2 is requested as soon as stage st is consumed.
        {
            const int gs = lane / HQ, a = lane - (lane / HQ) * HQ;
            const bool act = lane < ROWS && g0 + gs < total_groups;
            const uint64_t e = act ? RT[rbuf * 32 + lane] : 0;
            const int span = (int)(e >> 48);
            uint32_t Y = 0, X0 = 0;
            if (act) gpos(g0 + gs, Y, X0);
            const int dl = act ? (int)((((uint64_t)Y * HQ + a) * p.w + (uint64_t)X0 * WQ) & 31) : 0;
            const int segbytes = span - dl;
            const int nb = act ? segbytes / WQ : 0;
            const uint32_t rowsm = sbase + lane * kStageRow;
            uint32_t* SWs = wbase + gs * wpg + a * WQ;  // scratch: this lane's row of WD
            constexpr uint32_t mask = (WQ >= 32) ? 0xFFFFFFFFu : ((1u << WQ) - 1u);
            auto chunk = [&](int c) -> uint32_t {  // packed bits of aligned chunk c
                return (act && 32 * c < span)
                           ? pack32(lds256(rowsm + ((c / kStageChunks) % kStageBufs) * SBUF +
                                           (c % kStageChunks) * 32))
                           : 0u;
            };
            cp_async_wait<1>();  // stage 0 landed (stage 1 may be in flight)
            __syncwarp();
            uint32_t awprev = chunk(0);
#pragma unroll 1
            for (int c = 1; c <= NW; ++c) {
                if ((c % kStageChunks) == 0) {
                    // entering stage c/4: stage c/4 - 1 fully consumed -> refill its buffer
                    __syncwarp();
                    issue_stage(rbuf, c / kStageChunks + 1);
                    cp_async_wait<1>();
                    __syncwarp();
                }
                const uint32_t aw = chunk(c);
                if (act) SWs[c - 1] = __funnelshift_r(awprev, aw, dl);
                awprev = aw;
            }
            if (act) {
                // bits past the segment belong to the next group: only R_b with b >= nb
                // would see them, and those are zeroed below
                uint32_t SW[NW];
#pragma unroll
                for (int t = 0; t < NW; ++t) SW[t] = SWs[t];
                uint32_t R[32];
#pragma unroll
                for (int b = 0; b < 32; ++b) {
                    const int bit = WQ * b, t0 = bit >> 5, sh = bit & 31;
                    uint32_t v = SW[t0] >> sh;
                    if (sh + WQ > 32 && t0 + 1 < NW) v = __funnelshift_r(SW[t0], SW[t0 + 1], sh);
                    R[b] = (b < nb) ? (v & mask) : 0u;
                }
                transpose32(R);  // R[c] bit b = tile b, local (a, c)
#pragma unroll
                for (int c = 0; c < WQ; ++c) SWs[c] = R[c];
            }
        }
        // ---- next group: row table + stages 0, 1 in flight from here on -------------
        const uint32_t gn = g0 + nwarps * G;
        cp_async_wait<0>();  // also completes NT for group gn (requested one group ago)
        __syncwarp();
        rbuf ^= 1;
        fill_rows(gn, rbuf);
        __syncwarp();
        issue_stage(rbuf, 0);
        // ---- halo words: first batch (requested one group ago), then the rest ---------
#pragma unroll
        for (int jj = 0; jj < kHaloBatch; ++jj) {
            const uint32_t word = __ballot_sync(0xffffffffu, hv0[jj] != 0);
            if (lane == jj && jj < p.nH) wbase[C + jj] = word;
        }
#pragma unroll 1
        for (int gs = 0; gs < G; ++gs) {
            uint32_t* WD = wbase + gs * wpg;
            uint32_t Y = 0, X0 = 0;
            const bool gv = g0 + gs < total_groups;
            if (gv) gpos(g0 + gs, Y, X0);
#pragma unroll 1
            for (int j0 = gs == 0 ? kHaloBatch : 0; j0 < p.nH; j0 += kHaloBatch) {
                uint8_t hv[kHaloBatch];
#pragma unroll
                for (int jj = 0; jj < kHaloBatch; ++jj) {
                    const int j = j0 + jj;
                    hv[jj] = (gv && j < p.nH) ? halo_load(halo_tile(Y, X0 + lane, j), j) : 0;
                }
#pragma unroll
                for (int jj = 0; jj < kHaloBatch; ++jj) {
                    const uint32_t word = __ballot_sync(0xffffffffu, hv[jj] != 0);
                    if (lane == jj && j0 + jj < p.nH) WD[C + j0 + jj] = word;
                }
            }
            if (lane == 0) WD[C + p.nH] = 0u;  // the "absent" neighbour
        }
        // next group's first halo batch, in flight during program + backward; then
        // request the neighbour tiles of the group after it (with stage 1's group)
        {
            const int nb = rbuf;  // NT buffer of group gn (alternates like rbuf)
#pragma unroll
            for (int jj = 0; jj < kHaloBatch; ++jj)
                hv0[jj] = jj < p.nH ? halo_load(NT[nb * 8 * 32 + p.halo_D[jj] * 32 + lane], jj) : 0;
            __syncwarp();
            nt_request(gn + nwarps * G, nb ^ 1);
            issue_stage(rbuf, 1);
        }
        __syncwarp();
        // ---- program: bit-sliced step on every local cell ------------------------
        // results stay in registers until every lane has read WD, then overwrite it
        uint32_t res[NPL];
#pragma unroll
        for (int m = 0; m < NPL; ++m) {
            const int i = lane + 32 * m;
            if (i < G * C) {
                const int gs = i / C, li = i - gs * C;
                const uint32_t* WD = wbase + gs * wpg;
                const uint4 n0 = __ldg(reinterpret_cast<const uint4*>(p.nbr + li * 8));
                const uint4 n1 = __ldg(reinterpret_cast<const uint4*>(p.nbr + li * 8) + 1);
                const uint8_t* WB = reinterpret_cast<const uint8_t*>(WD);
                const uint32_t x0 = *reinterpret_cast<const uint32_t*>(WB + n0.x);
                const uint32_t x1 = *reinterpret_cast<const uint32_t*>(WB + n0.y);
                const uint32_t x2 = *reinterpret_cast<const uint32_t*>(WB + n0.z);
                const uint32_t x3 = *reinterpret_cast<const uint32_t*>(WB + n0.w);
                const uint32_t x4 = *reinterpret_cast<const uint32_t*>(WB + n1.x);
                const uint32_t x5 = *reinterpret_cast<const uint32_t*>(WB + n1.y);
                const uint32_t x6 = *reinterpret_cast<const uint32_t*>(WB + n1.z);
                const uint32_t x7 = *reinterpret_cast<const uint32_t*>(WB + n1.w);
                const Count4 cnt = count8(x0, x1, x2, x3, x4, x5, x6, x7);
                res[m] = apply_rule_bits<CONWAY>(cnt, WD[li], KB, KS);
            }
        }
        __syncwarp();
#pragma unroll
        for (int m = 0; m < NPL; ++m) {
            const int i = lane + 32 * m;
            if (i < G * C) {
                const int gs = i / C, li = i - gs * C;
                wbase[gs * wpg + li] = res[m];
            }
        }
        __syncwarp();
        // ---- backward: words -> bytes ----------------------------------------------
        // Per lane: transpose back, assemble the delta-shifted words SW_t in the
        // lane's scratch row, then a runtime loop stores aligned 32-B chunks.
        {
            const int gs = lane / HQ, a = lane - (lane / HQ) * HQ;
            const uint32_t g = g0 + gs;
            if (lane < ROWS && g < total_groups) {
                uint32_t Y, X0;
                gpos(g, Y, X0);
                const int segbytes = (int)min(32u, p.Wc - X0) * WQ;
                const uint64_t seg = ((uint64_t)Y * HQ + a) * p.w + (uint64_t)X0 * WQ;
                const int delta = (int)(seg & 31);
                uint32_t* SWs = wbase + gs * wpg + a * WQ;  // program output overwrote WD
                uint32_t R[32];
#pragma unroll
                for (int c = 0; c < 32; ++c) R[c] = c < WQ ? SWs[c] : 0u;
                transpose32(R);  // R[b] bit c
#pragma unroll
                for (int t = 0; t < NW; ++t) {
                    uint32_t sw = 0;
#pragma unroll
                    for (int b = 0; b < 32; ++b) {
                        const int bit = WQ * b, t0 = bit >> 5, sh = bit & 31;
                        const int tend = (bit + WQ - 1) >> 5;
                        if (t0 == t) sw |= R[b] << sh;
                        else if (tend == t) sw |= R[b] >> (32 - sh);
                    }
                    SWs[t] = sw;
                }
                uint8_t* ap = dst + (seg - delta);
                const int end = delta + segbytes;  // exclusive, in the aligned frame
                const int nchunks = (end + 31) >> 5;
                uint32_t swprev = 0;
#pragma unroll 1
                for (int t = 0; t < nchunks; ++t) {
                    const uint32_t sw = t < NW ? SWs[t] : 0u;
                    const uint32_t wv = __funnelshift_l(swprev, sw, delta);
                    swprev = sw;
                    const int lo = t == 0 ? delta : 0;
                    const int hi = min(32, end - 32 * t);
                    if (lo == 0 && hi == 32) stg256(ap + 32 * t, unpack32(wv));
                    else store_bits_range(ap + 32 * t, wv, lo, hi);  // shared with a neighbour group
                }
            }
        }
        __syncwarp();
    }
    cp_async_wait<0>();
}

}  // namespace nbbgpu
