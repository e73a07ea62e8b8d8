// bb.cuh -- vectorised bounding-box baseline (north-star item 3).
//
// Simulation::step_bounding_box (stencil.cpp:291-311) as a competent dense GPU
// stencil: each thread owns 16 consecutive bytes of a row of the embedded n x n
// box (n % 16 == 0, i.e. s = 2 or 4), loads the three rows with 16-B vector
// loads, gets the edge bytes from the neighbouring lanes by shuffles, sums the 8
// (or 4) neighbour bytes with SWAR adds (counts <= 8 fit a byte), applies the rule
// with SWAR byte compares / PRMT table lookups, masks holes to 0 (holes are 0 in
// both buffers, so writing 0 equals "never updated") and stores 16 B.
// Membership: low 4 bits of x, y through a 16x16-bit table (per y mod 16), the
// high digits by a scalar digit check per 16-cell vector (x & y == 0 fast path
// for the triangle).
#pragma once

#include "common.cuh"

namespace nbbgpu {

struct BBParams {
    Frac f;
    uint32_t n;          // side
    int mlow;            // levels covered by the low 4 bits (s=2: 4, s=4: 2)
    int triangle;        // fast path: member <=> (x & y) == 0
    uint16_t low[16];    // low[y & 15] bit i: low-level membership of (x0 + i, y)
    uint32_t birth, survive;
    int moore;
};

// high-level membership of the 16-aligned vector starting at (x0, y)
__device__ __forceinline__ bool bb_high_member(const BBParams& p, uint32_t x0, uint32_t y) {
    if (p.triangle) return ((x0 & y) & ~15u) == 0;
    const uint32_t s = p.f.s;
    uint32_t x = x0 >> 4, yy = y >> 4;  // 16 = s^mlow
    for (int mu = p.mlow; mu < p.f.r; ++mu) {
        if (p.f.id_of_subbox[(yy % s) * s + (x % s)] < 0) return false;
        x /= s;
        yy /= s;
    }
    return true;
}

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

template <bool CONWAY>
__global__ void __launch_bounds__(256) step_bb_vec_kernel(const BBParams p, const uint8_t* __restrict__ src,
                                                          uint8_t* __restrict__ dst) {
    const uint32_t n = p.n, vpr = n >> 4;  // vectors per row
    const uint64_t total = (uint64_t)n * vpr;
    const int lane = threadIdx.x & 31;
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
    // grid-stride over whole warps so the shuffles always see 32 active lanes
    const uint64_t nthreads = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u); base < total;
         base += nthreads) {
        const uint64_t v = base + lane;
        const bool valid = v < total;
        const uint32_t y = valid ? (uint32_t)(v / vpr) : 0u;
        const uint32_t xv = valid ? (uint32_t)(v - (uint64_t)y * vpr) : 0u;
        const uint32_t x0 = xv * 16;
        const uint8_t* row = src + (uint64_t)y * n;
        uint4 up = make_uint4(0, 0, 0, 0), mid = up, dn = up;
        if (valid) {
            mid = __ldg(reinterpret_cast<const uint4*>(row + x0));
            if (y > 0) up = __ldg(reinterpret_cast<const uint4*>(row - n + x0));
            if (y + 1 < n) dn = __ldg(reinterpret_cast<const uint4*>(row + n + x0));
        }
        // edge bytes: left = byte x0-1 (lane-1's .w top byte), right = byte x0+16
        uint32_t lu = __shfl_up_sync(0xffffffffu, up.w, 1), lm = __shfl_up_sync(0xffffffffu, mid.w, 1),
                 ld = __shfl_up_sync(0xffffffffu, dn.w, 1);
        uint32_t ru = __shfl_down_sync(0xffffffffu, up.x, 1), rm = __shfl_down_sync(0xffffffffu, mid.x, 1),
                 rd = __shfl_down_sync(0xffffffffu, dn.x, 1);
        const bool same_row_left = lane > 0 && xv > 0;        // lane-1 holds the previous vector
        const bool same_row_right = lane < 31 && xv + 1 < vpr;  // lane+1 holds the next vector
        if (valid && !same_row_left) {
            lu = lm = ld = 0;
            if (x0 > 0) {
                lm = (uint32_t)row[x0 - 1] << 24;
                if (y > 0) lu = (uint32_t)row[(int64_t)x0 - 1 - (int64_t)n] << 24;
                if (y + 1 < n) ld = (uint32_t)row[(int64_t)x0 - 1 + (int64_t)n] << 24;
            }
        }
        if (valid && !same_row_right) {
            ru = rm = rd = 0;
            if (x0 + 16 < n) {
                rm = row[x0 + 16];
                if (y > 0) ru = row[(int64_t)x0 + 16 - (int64_t)n];
                if (y + 1 < n) rd = row[(int64_t)x0 + 16 + (int64_t)n];
            }
        }
        if (!valid) continue;
        const uint32_t U[6] = {lu, up.x, up.y, up.z, up.w, ru};
        const uint32_t M[6] = {lm, mid.x, mid.y, mid.z, mid.w, rm};
        const uint32_t D[6] = {ld, dn.x, dn.y, dn.z, dn.w, rd};
        // membership of the 16 cells
        const uint32_t lowmask = bb_high_member(p, x0, y) ? p.low[y & 15] : 0u;
        uint32_t out[4];
#pragma unroll
        for (int j = 1; j <= 4; ++j) {
            // byte-shifted neighbours: west = byte x-1, east = byte x+1
            const uint32_t uw = __funnelshift_l(U[j - 1], U[j], 8), ue = __funnelshift_r(U[j], U[j + 1], 8);
            const uint32_t mw = __funnelshift_l(M[j - 1], M[j], 8), me = __funnelshift_r(M[j], M[j + 1], 8);
            const uint32_t dw = __funnelshift_l(D[j - 1], D[j], 8), de = __funnelshift_r(D[j], D[j + 1], 8);
            uint32_t cnt = U[j] + D[j] + mw + me;  // von Neumann: N, S, W, E
            if (p.moore) cnt += uw + ue + dw + de;
            const uint32_t r = bb_rule<CONWAY>(cnt, M[j], tb_lo, tb_hi, ts_lo, ts_hi, b8, s8);
            out[j - 1] = r & bb_spread4(lowmask >> (4 * (j - 1)));
        }
        *reinterpret_cast<uint4*>(dst + (uint64_t)y * n + x0) = make_uint4(out[0], out[1], out[2], out[3]);
    }
}

}  // namespace nbbgpu
