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
//   forward : loads the 32*WQ contiguous bytes of row a (16-B vector loads),
//             packs bytes to bits, cuts the 32 WQ-bit tile rows and transposes
//             the 32x32 bit matrix in registers -> WQ words W[a][c] (bit b);
//   program : all lanes run the table-driven bit-sliced Life step per word;
//   backward: transposes back, unpacks bits to bytes, stores 16-B vectors.
// The reference semantics (stencil.cpp:334-368) are preserved bit for bit:
// out-of-box and hole neighbours count 0, states are read from src and written
// to dst only (double buffer).
#pragma once

#include "common.cuh"

namespace nbbgpu {

constexpr int kTiledWarps = 8;       // warps per block
constexpr int kHaloBatch = 8;        // halo slots gathered per batch
constexpr int kMaxHalo = 512;

struct TiledParams {
    Frac f;                  // full-level tables (k, s, replica tables)
    int L;                   // coarse level r - q
    int C;                   // cells per tile k^q
    int nH;                  // halo slots
    uint32_t dmask;          // bit D (= (dy+1)*3 + dx+1) set if direction D has slots
    uint16_t halo_first[10]; // slots sorted by D: [halo_first[D], halo_first[D+1])
    uint32_t Wc, Hc;         // coarse compact dims
    uint32_t gpr;            // groups per coarse row = ceil(Wc / 32)
    uint32_t row0, row1;     // owned coarse rows [row0, row1)
    uint64_t w;              // compact row stride (bytes)
    uint32_t birth, survive;
    const uint32_t* nbr;     // C x 8 smem byte offsets into the group's word array
    const uint8_t* halo_D;   // per slot: direction index
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
__device__ __forceinline__ bool coarse_neighbor(const Frac& f, int L, uint32_t X, uint32_t Y,
                                                int dx, int dy, uint32_t& X2, uint32_t& Y2) {
    const int k = f.k, s = f.s;
    uint32_t cx = X, cy = Y;
    int pw = 1;
    int nx = (int)X, ny = (int)Y;
    for (int mu = 0; mu < L; ++mu) {
        if (dx == 0 && dy == 0) break;
        int d;
        if ((mu & 1) == 0) { d = (int)(cx % k); cx /= k; }
        else               { d = (int)(cy % k); cy /= k; }
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

// bytes (each 0/1) of a 16-B vector -> 16 bits, bit t = byte t
__device__ __forceinline__ uint32_t pack16(const uint4 v) {
    const uint32_t m = 0x10204080u;  // byte j bit0 -> bit 28+j, no carries for 0/1 bytes
    const uint32_t a = (v.x * m) >> 28, b = (v.y * m) >> 28;
    const uint32_t c = (v.z * m) >> 28, d = (v.w * m) >> 28;
    return a | (b << 4) | (c << 8) | (d << 12);
}

// 16 bits -> 16 bytes of 0/1
__device__ __forceinline__ uint4 unpack16(uint32_t p) {
    const uint32_t m = 0x00204081u;  // bit j -> bit 8j
    uint4 v;
    v.x = ((p & 0xFu) * m) & 0x01010101u;
    v.y = (((p >> 4) & 0xFu) * m) & 0x01010101u;
    v.z = (((p >> 8) & 0xFu) * m) & 0x01010101u;
    v.w = (((p >> 12) & 0xFu) * m) & 0x01010101u;
    return v;
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

// Store bytes [lo, hi) of a 16-B vector (0 <= lo < hi <= 16) with aligned pieces.
__device__ __forceinline__ void store_partial16(uint8_t* p16, const uint4 v, int lo, int hi) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    int i = lo;
    while (i < hi) {
        if ((i & 7) == 0 && i + 8 <= hi) {
            *reinterpret_cast<uint2*>(p16 + i) = make_uint2(w[i >> 2], w[(i >> 2) + 1]);
            i += 8;
        } else if ((i & 3) == 0 && i + 4 <= hi) {
            *reinterpret_cast<uint32_t*>(p16 + i) = w[i >> 2];
            i += 4;
        } else if ((i & 1) == 0 && i + 2 <= hi) {
            *reinterpret_cast<uint16_t*>(p16 + i) = (uint16_t)(w[i >> 2] >> ((i & 3) * 8));
            i += 2;
        } else {
            p16[i] = (uint8_t)(w[i >> 2] >> ((i & 3) * 8));
            i += 1;
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

template <int WQ, bool CONWAY>
__global__ void __launch_bounds__(kTiledWarps * 32)
step_tiled_kernel(const TiledParams p, const uint8_t* __restrict__ src, uint8_t* __restrict__ dst) {
    constexpr int HQ = WQ;
    constexpr int C = WQ * WQ;
    constexpr int G = (32 / HQ) > 0 ? (32 / HQ) : 1;    // groups per warp
    constexpr int NW = (32 * WQ + 31) / 32;             // words of a 32-tile row
    constexpr int CP = (C + 3) & ~3;                    // WO words, padded to 16 B
    extern __shared__ __align__(16) uint8_t smem_raw[];

    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    uint32_t* wbase = reinterpret_cast<uint32_t*>(smem_raw + warp * p.smem_per_warp);
    // per group slot: WD [words_per_group] | WO [CP] ; then HB: G x 9 x 32 u64
    const uint32_t wpg = p.words_per_group;
    uint64_t* HB = reinterpret_cast<uint64_t*>(wbase + G * (wpg + CP));

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

    for (uint64_t g0 = warp_global * G; g0 < total_groups; g0 += nwarps * G) {
        // ---------------- halo: coarse neighbour tile bases -------------------
#pragma unroll 1
        for (int gs = 0; gs < G; ++gs) {
            const uint64_t g = g0 + gs;
            const bool gvalid = g < total_groups;
            const uint32_t Y = p.row0 + (uint32_t)(gvalid ? g / p.gpr : 0);
            const uint32_t X0 = (uint32_t)(gvalid ? (g % p.gpr) : 0) * 32;
            const uint32_t X = X0 + lane;
            const bool tvalid = gvalid && X < p.Wc;
#pragma unroll
            for (int D = 0; D < 9; ++D) {
                if (!((p.dmask >> D) & 1u)) continue;
                uint64_t base = ~0ull;
                uint32_t X2, Y2;
                if (tvalid && coarse_neighbor(p.f, p.L, X, Y, D % 3 - 1, D / 3 - 1, X2, Y2))
                    base = (uint64_t)Y2 * HQ * p.w + (uint64_t)X2 * WQ;
                HB[(gs * 9 + D) * 32 + lane] = base;
            }
        }
        __syncwarp();
        // ---------------- forward: bytes -> bit-sliced words -------------------
        {
            const int gs = lane / HQ, a = lane % HQ;
            const uint64_t g = g0 + gs;
            if (gs < G && g < total_groups) {
                const uint32_t Y = p.row0 + (uint32_t)(g / p.gpr);
                const uint32_t X0 = (uint32_t)(g % p.gpr) * 32;
                const int nb = (int)min(32u, p.Wc - X0);
                const uint64_t seg = ((uint64_t)Y * HQ + a) * p.w + (uint64_t)X0 * WQ;
                const int segbytes = nb * WQ;
                const int delta = (int)(seg & 15);
                const uint4* ap = reinterpret_cast<const uint4*>(src + (seg - delta));
                const int nchunks = (delta + segbytes + 15) >> 4;
                // aligned bit string AW (bit t = byte abase + t), NW+1 words
                uint32_t AW[NW + 1];
#pragma unroll
                for (int t = 0; t <= NW; ++t) {
                    uint32_t lo = 0, hi = 0;
                    if (2 * t < nchunks) lo = pack16(__ldg(ap + 2 * t));
                    if (2 * t + 1 < nchunks) hi = pack16(__ldg(ap + 2 * t + 1));
                    AW[t] = lo | (hi << 16);
                }
                // shift by delta -> SW (bit t = byte seg + t), clip to segbytes
                uint32_t SW[NW];
#pragma unroll
                for (int t = 0; t < NW; ++t) {
                    uint32_t v = __funnelshift_r(AW[t], AW[t + 1], delta);
                    const int rem = segbytes - 32 * t;
                    if (rem < 32) v = rem <= 0 ? 0u : (v & ((1u << rem) - 1u));
                    SW[t] = v;
                }
                uint32_t R[32];
#pragma unroll
                for (int b = 0; b < 32; ++b) {
                    constexpr uint32_t mask = (WQ >= 32) ? 0xFFFFFFFFu : ((1u << WQ) - 1u);
                    const int bit = WQ * b, t0 = bit >> 5, sh = bit & 31;
                    uint32_t v = SW[t0] >> sh;
                    if (sh + WQ > 32 && t0 + 1 < NW) v = __funnelshift_r(SW[t0], SW[t0 + 1], sh);
                    R[b] = v & mask;
                }
                transpose32(R);  // R[c] bit b = tile b, local (a, c)
                uint32_t* WD = wbase + gs * (wpg + CP);
#pragma unroll
                for (int c = 0; c < WQ; ++c) WD[a * WQ + c] = R[c];
            }
        }
        // ---------------- halo words -----------------------------------------
#pragma unroll 1
        for (int gs = 0; gs < G; ++gs) {
            uint32_t* WD = wbase + gs * (wpg + CP);
#pragma unroll 1
            for (int j0 = 0; j0 < p.nH; j0 += kHaloBatch) {
                uint8_t hv[kHaloBatch];
#pragma unroll
                for (int jj = 0; jj < kHaloBatch; ++jj) {
                    const int j = j0 + jj;
                    hv[jj] = 0;
                    if (j < p.nH) {
                        const uint64_t base = HB[(gs * 9 + p.halo_D[j]) * 32 + lane];
                        if (base != ~0ull)
                            hv[jj] = __ldg(src + base + (uint64_t)p.halo_a[j] * p.w + p.halo_c[j]);
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
        // ---------------- program: bit-sliced step on every local cell ---------
#pragma unroll 1
        for (int i = lane; i < G * C; i += 32) {
            const int gs = i / C, li = i - gs * C;
            const uint32_t* WD = wbase + gs * (wpg + CP);
            uint32_t* WO = wbase + gs * (wpg + CP) + wpg;
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
            WO[li] = apply_rule_bits<CONWAY>(cnt, WD[li], KB, KS);
        }
        __syncwarp();
        // ---------------- backward: words -> bytes -----------------------------
        {
            const int gs = lane / HQ, a = lane % HQ;
            const uint64_t g = g0 + gs;
            if (gs < G && g < total_groups) {
                const uint32_t Y = p.row0 + (uint32_t)(g / p.gpr);
                const uint32_t X0 = (uint32_t)(g % p.gpr) * 32;
                const int nb = (int)min(32u, p.Wc - X0);
                const uint64_t seg = ((uint64_t)Y * HQ + a) * p.w + (uint64_t)X0 * WQ;
                const int segbytes = nb * WQ;
                const int delta = (int)(seg & 15);
                const uint32_t* WO = wbase + gs * (wpg + CP) + wpg;
                uint32_t R[32];
#pragma unroll
                for (int c = 0; c < 32; ++c) R[c] = c < WQ ? WO[a * WQ + c] : 0u;
                transpose32(R);  // R[b] bit c
                uint32_t SW[NW];
#pragma unroll
                for (int t = 0; t < NW; ++t) SW[t] = 0;
#pragma unroll
                for (int b = 0; b < 32; ++b) {
                    const int bit = WQ * b, t0 = bit >> 5, sh = bit & 31;
                    SW[t0] |= R[b] << sh;
                    if (sh + WQ > 32 && t0 + 1 < NW) SW[t0 + 1] |= R[b] >> (32 - sh);
                }
                // shift left by delta into the aligned frame
                uint32_t AW[NW + 1];
                AW[0] = SW[0] << delta;
#pragma unroll
                for (int t = 1; t < NW; ++t) AW[t] = __funnelshift_l(SW[t - 1], SW[t], delta);
                AW[NW] = delta ? (SW[NW - 1] >> (32 - delta)) : 0u;
                uint8_t* ap = dst + (seg - delta);
                const int end = delta + segbytes;  // exclusive, in aligned frame
                const int nchunks = (end + 15) >> 4;
#pragma unroll
                for (int t = 0; t <= NW; ++t) {
#pragma unroll
                    for (int hh = 0; hh < 2; ++hh) {
                        const int ch = 2 * t + hh;
                        if (ch < nchunks) {
                            const uint4 v = unpack16(hh ? (AW[t] >> 16) : (AW[t] & 0xFFFFu));
                            const int lo = ch == 0 ? delta : 0;
                            const int hi = min(16, end - 16 * ch);
                            if (lo == 0 && hi == 16)
                                *reinterpret_cast<uint4*>(ap + 16 * ch) = v;
                            else
                                store_partial16(ap + 16 * ch, v, lo, hi);
                        }
                    }
                }
            }
        }
        __syncwarp();
    }
}

}  // namespace nbbgpu
