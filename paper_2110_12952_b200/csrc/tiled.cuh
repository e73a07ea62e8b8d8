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

constexpr int kTiledWarps = 4;       // warps per block
constexpr int kRing = 6;             // cp.async ring slots (32 B) per lane
constexpr int kRingLaneBytes = kRing * 32 + 16;  // +16: conflict-free LDS.128 across lanes
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
    const uint8_t* halo_D;   // per slot: direction slot (index into dlist)
    const uint16_t* halo_a;  // per slot: source local row in the neighbour tile
    const uint16_t* halo_c;  // per slot: source local column
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

// 32 bytes (each 0/1) -> 32 bits, bit t = byte t.
// (v * 0x10204080) >> 28 moves byte j's bit 0 to bit j with no carries for 0/1 bytes.
__device__ __forceinline__ uint32_t pack32(const u32x8& r) {
    uint32_t w = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) w |= ((r.v[j] * 0x10204080u) >> 28) << (4 * j);
    return w;
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

// Byte-exact store of bytes [lo, hi) of a 32-B chunk (0 <= lo < hi <= 32):
// statically indexed 8/4/2/1-byte pieces (no dynamic register indexing).
__device__ __forceinline__ void store_range32(uint8_t* p32, const u32x8& r, int lo, int hi) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {  // 8-byte slots
        const int s0 = 8 * q;
        if (lo <= s0 && s0 + 8 <= hi) {
            *reinterpret_cast<uint2*>(p32 + s0) = make_uint2(r.v[2 * q], r.v[2 * q + 1]);
            continue;
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {  // words
            const int w0 = s0 + 4 * h;
            const uint32_t v = r.v[2 * q + h];
            if (lo <= w0 && w0 + 4 <= hi) {
                *reinterpret_cast<uint32_t*>(p32 + w0) = v;
                continue;
            }
#pragma unroll
            for (int e = 0; e < 2; ++e) {  // half-words
                const int h0 = w0 + 2 * e;
                if (lo <= h0 && h0 + 2 <= hi) {
                    *reinterpret_cast<uint16_t*>(p32 + h0) = (uint16_t)(v >> (16 * e));
                } else {
                    if (lo <= h0 && h0 < hi) p32[h0] = (uint8_t)(v >> (16 * e));
                    if (lo <= h0 + 1 && h0 + 1 < hi) p32[h0 + 1] = (uint8_t)(v >> (16 * e + 8));
                }
            }
        }
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

template <int WQ, int K, int S, bool CONWAY>
__global__ void __launch_bounds__(kTiledWarps * 32, 5)
step_tiled_kernel(const TiledParams p, const uint8_t* __restrict__ src, uint8_t* __restrict__ dst) {
    constexpr int HQ = WQ;
    constexpr int C = WQ * WQ;
    constexpr int G = (32 / HQ) > 0 ? (32 / HQ) : 1;    // groups per warp
    constexpr int NW = WQ;                              // 32-bit words of a 32-tile row
    constexpr int NPL = (G * C + 31) / 32;              // program cells per lane
    extern __shared__ __align__(16) uint8_t smem_raw[];

    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    uint32_t* wbase = reinterpret_cast<uint32_t*>(smem_raw + warp * p.smem_per_warp);
    // per group slot: WD [words_per_group]; then HB: G x 8 x 32 packed tiles; then the
    // per-lane cp.async rings (32 x kRingLaneBytes)
    const uint32_t wpg = p.words_per_group;
    uint32_t* HB = wbase + G * wpg;
    const uint32_t ring = (uint32_t)__cvta_generic_to_shared(HB + G * 8 * 32) + lane * kRingLaneBytes;

    uint32_t KB[9], KS[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) {
        KB[i] = ((p.birth >> i) & 1u) ? 0xFFFFFFFFu : 0u;
        KS[i] = ((p.survive >> i) & 1u) ? 0xFFFFFFFFu : 0u;
    }

    const uint64_t rows = p.row1 - p.row0;
    const uint64_t total_groups = rows * p.gpr;
    const uint64_t warp_global = (uint64_t)blockIdx.x * kTiledWarps + warp;
    const uint64_t nwarps = (uint64_t)gridDim.x * kTiledWarps;

    // row segment of (group g, local row a): first byte and length
    auto row_seg = [&](uint64_t g, int a, uint64_t& seg, int& segbytes) {
        const uint32_t Y = p.row0 + (uint32_t)(g / p.gpr);
        const uint32_t X0 = (uint32_t)(g % p.gpr) * 32;
        segbytes = (int)min(32u, p.Wc - X0) * WQ;
        seg = ((uint64_t)Y * HQ + a) * p.w + (uint64_t)X0 * WQ;
    };
    for (uint64_t g0 = warp_global * G; g0 < total_groups; g0 += nwarps * G) {
        // ---- halo: coarse neighbour tiles (lane = tile b) ------------------------
#pragma unroll 1
        for (int gs = 0; gs < G; ++gs) {
            const uint64_t g = g0 + gs;
            const bool gvalid = g < total_groups;
            const uint32_t Y = p.row0 + (uint32_t)(gvalid ? g / p.gpr : 0);
            const uint32_t X = (uint32_t)(gvalid ? (g % p.gpr) : 0) * 32 + lane;
            const bool tvalid = gvalid && X < p.Wc;
#pragma unroll 1
            for (int ds = 0; ds < p.nD; ++ds) {
                const int D = p.dlist[ds];
                uint32_t packed = 0xFFFFFFFFu, X2, Y2;
                if (tvalid && coarse_neighbor<K, S>(p.f, p.L, X, Y, D % 3 - 1, D / 3 - 1, X2, Y2))
                    packed = (Y2 << 16) | X2;
                HB[(gs * 8 + ds) * 32 + lane] = packed;
            }
        }
        __syncwarp();
        // first halo batch of group slot 0: loads in flight during the forward phase
        uint8_t hv0[kHaloBatch];
#pragma unroll
        for (int jj = 0; jj < kHaloBatch; ++jj) {
            hv0[jj] = 0;
            if (jj < p.nH) {
                const uint32_t t = HB[p.halo_D[jj] * 32 + lane];
                if (t != 0xFFFFFFFFu)
                    hv0[jj] = __ldg(src + ((uint64_t)(t >> 16) * HQ + p.halo_a[jj]) * p.w +
                                    (uint64_t)(t & 0xFFFFu) * WQ + p.halo_c[jj]);
            }
        }
        // ---- forward: bytes -> bit-sliced words ------------------------------------
        {
            const int gs = lane / HQ, a = lane % HQ;
            const uint64_t g = g0 + gs;
            if (gs < G && g < total_groups) {
                uint64_t seg; int segbytes;
                row_seg(g, a, seg, segbytes);
                const int delta = (int)(seg & 31);
                const uint8_t* ap = src + (seg - delta);
                const int nchunks = (delta + segbytes + 31) >> 5;
                const int nb = segbytes / WQ;
                // Streamed: aligned word t (bit i = byte abase+32t+i) -> delta-shifted
                // word SW_t -> every tile row R_b whose last bit lies in SW_t.
                // Loads run PF chunks ahead; only a 2-word window stays live.
                constexpr uint32_t mask = (WQ >= 32) ? 0xFFFFFFFFu : ((1u << WQ) - 1u);
                // chunk c -> ring slot c % kRing; kRing-1 chunks stay in flight
#pragma unroll
                for (int c = 0; c < kRing - 1; ++c) {
                    if (c <= NW && c < nchunks) {
                        cp_async16(ring + 32 * c, ap + 32 * c);
                        cp_async16(ring + 32 * c + 16, ap + 32 * c + 16);
                    }
                    cp_async_commit();
                }
                cp_async_wait<kRing - 2>();
                uint32_t awcur = pack32(lds256(ring)), swprev = 0;
                uint32_t R[32];
#pragma unroll
                for (int t = 0; t < NW; ++t) {
                    // refill: chunk t + kRing - 1 into the slot chunk t just vacated
                    {
                        const int c = t + kRing - 1;
                        if (c <= NW && c < nchunks) {
                            cp_async16(ring + 32 * (c % kRing), ap + 32 * c);
                            cp_async16(ring + 32 * (c % kRing) + 16, ap + 32 * c + 16);
                        }
                        cp_async_commit();
                    }
                    cp_async_wait<kRing - 2>();  // chunk t + 1 has landed
                    const uint32_t awnext = (t + 1 < nchunks) ? pack32(lds256(ring + 32 * ((t + 1) % kRing))) : 0u;
                    const uint32_t sw = __funnelshift_r(awcur, awnext, delta);
#pragma unroll
                    for (int b = 0; b < 32; ++b) {
                        const int bit = WQ * b, t0 = bit >> 5, sh = bit & 31;
                        const int tend = (bit + WQ - 1) >> 5;
                        if (tend == t) {
                            const uint32_t v = (t0 == t) ? (sw >> sh) : __funnelshift_r(swprev, sw, sh);
                            R[b] = v & mask;
                        }
                    }
                    swprev = sw;
                    awcur = awnext;
                }
                cp_async_wait<0>();
                if (nb < 32) {
#pragma unroll
                    for (int b = 0; b < 32; ++b)
                        if (b >= nb) R[b] = 0;
                }
                transpose32(R);  // R[c] bit b = tile b, local (a, c)
                uint32_t* WD = wbase + gs * wpg;
#pragma unroll
                for (int c = 0; c < WQ; ++c) WD[a * WQ + c] = R[c];
            }
        }
        // ---- halo words ---------------------------------------------------------------
#pragma unroll
        for (int jj = 0; jj < kHaloBatch; ++jj) {
            const uint32_t word = __ballot_sync(0xffffffffu, hv0[jj] != 0);
            if (lane == jj && jj < p.nH) wbase[C + jj] = word;
        }
#pragma unroll 1
        for (int gs = 0; gs < G; ++gs) {
            uint32_t* WD = wbase + gs * wpg;
#pragma unroll 1
            for (int j0 = gs == 0 ? kHaloBatch : 0; j0 < p.nH; j0 += kHaloBatch) {
                uint8_t hv[kHaloBatch];
#pragma unroll
                for (int jj = 0; jj < kHaloBatch; ++jj) {
                    const int j = j0 + jj;
                    hv[jj] = 0;
                    if (j < p.nH) {
                        const uint32_t t = HB[(gs * 8 + p.halo_D[j]) * 32 + lane];
                        if (t != 0xFFFFFFFFu)
                            hv[jj] = __ldg(src + ((uint64_t)(t >> 16) * HQ + p.halo_a[j]) * p.w +
                                           (uint64_t)(t & 0xFFFFu) * WQ + p.halo_c[j]);
                    }
                }
#pragma unroll
                for (int jj = 0; jj < kHaloBatch; ++jj) {
                    const uint32_t word = __ballot_sync(0xffffffffu, hv[jj] != 0);
                    if (lane == jj && j0 + jj < p.nH) WD[C + j0 + jj] = word;
                }
            }
            if (lane == 0) WD[C + p.nH] = 0u;  // the "absent" neighbour
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
        {
            const int gs = lane / HQ, a = lane % HQ;
            const uint64_t g = g0 + gs;
            if (gs < G && g < total_groups) {
                uint64_t seg; int segbytes;
                row_seg(g, a, seg, segbytes);
                const int delta = (int)(seg & 31);
                const uint32_t* WO = wbase + gs * wpg;  // program output overwrote WD
                uint32_t R[32];
#pragma unroll
                for (int c = 0; c < 32; ++c) R[c] = c < WQ ? WO[a * WQ + c] : 0u;
                transpose32(R);  // R[b] bit c
                uint8_t* ap = dst + (seg - delta);
                const int end = delta + segbytes;  // exclusive, in the aligned frame
                const int nchunks = (end + 31) >> 5;
                // Streamed: SW_t (bit i = byte seg+32t+i) is complete once every R_b
                // overlapping it is or-ed in; aligned word t = funnel(SW_{t-1}, SW_t).
                uint32_t swprev = 0;
#pragma unroll
                for (int t = 0; t <= NW; ++t) {
                    uint32_t sw = 0;
                    if (t < NW) {
#pragma unroll
                        for (int b = 0; b < 32; ++b) {
                            const int bit = WQ * b, t0 = bit >> 5, sh = bit & 31;
                            const int tend = (bit + WQ - 1) >> 5;
                            if (t0 == t) sw |= R[b] << sh;
                            else if (tend == t) sw |= R[b] >> (32 - sh);
                        }
                    }
                    if (t < nchunks) {
                        const uint32_t wv = __funnelshift_l(swprev, sw, delta);
                        const u32x8 v = unpack32(wv);
                        const int lo = t == 0 ? delta : 0;
                        const int hi = min(32, end - 32 * t);
                        if (lo == 0 && hi == 32) stg256(ap + 32 * t, v);
                        else store_range32(ap + 32 * t, v, lo, hi);
                    }
                    swprev = sw;
                }
            }
        }
        __syncwarp();
    }
}

}  // namespace nbbgpu
