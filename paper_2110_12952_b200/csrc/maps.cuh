// maps.cuh -- batched lambda / nu maps, two variants each (north-star item 1).
//
//  DIGIT: the CUDA-core digit loop (maps.cpp:80-146), one thread per coordinate.
//  MMA:   the paper's matrix form (Figure 8; the reference's
//         MapMatrices / to_compact_via_mma, maps.cpp:163-199) as exact-integer
//         tensor-core products, mma.sync.m16n8k32 u8 x u8 -> s32:
//           nu:     D[p][n] = sum_mu H(p, mu) * limb_n(tau(mu))
//                   A = replica IDs H (16 points x 32 levels, u8),
//                   B = base-256 limbs of the unfold strides (n 0-3: tau_x,
//                   n 4-7: tau_y); cx = sum_n D[p][n] << 8n (exact: every
//                   partial sum < 32*255*255 < 2^31).
//           lambda: x = sum_mu gx(d_mu) * s^mu, y likewise: two products with
//                   A = gx / gy of the digits and B = limbs of s^mu.
//         Exact for any level r <= 32 (K = 32), unlike the paper's f16 form
//         (exact only while every tau is f16-representable).
#pragma once

#include "common.cuh"

namespace nbbgpu {

template <int K, int S>
__global__ void lambda_digit_kernel(Frac f, const int2* __restrict__ in, int2* __restrict__ out,
                                    uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const int2 c = in[i];
        int2 o = make_int2(-1, -1);
        if (c.x >= 0 && c.y >= 0 && (uint32_t)c.x < f.w && (uint32_t)c.y < f.h) {
            uint32_t x, y;
            lambda_map<K, S>(f, (uint32_t)c.x, (uint32_t)c.y, x, y);
            o = make_int2((int)x, (int)y);
        }
        out[i] = o;
    }
}

template <int K, int S>
__global__ void nu_digit_kernel(Frac f, const int2* __restrict__ in, int2* __restrict__ out,
                                uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const int2 e = in[i];
        int2 o = make_int2(-1, -1);
        uint32_t cx, cy;
        if (e.x >= 0 && e.y >= 0 && (uint32_t)e.x < f.side && (uint32_t)e.y < f.side &&
            nu_map<K, S>(f, (uint32_t)e.x, (uint32_t)e.y, cx, cy))
            o = make_int2((int)cx, (int)cy);
        out[i] = o;
    }
}

__device__ __forceinline__ void mma_u8_16832(int (&d)[4], const uint32_t (&a)[4],
                                             const uint32_t (&b)[2]) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 "
        "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
        : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

// Powers table for the MMA B operands (kernel parameter).
struct MmaTables {
    uint32_t tau[32];   // k^floor(mu/2): the unfold stride magnitude of level mu
    uint32_t spow[32];  // s^mu
};

// limb n (0..3) of v
__device__ __forceinline__ uint32_t limb(uint32_t v, int n) { return (v >> (8 * n)) & 0xFFu; }

// nu via tensor cores: one warp handles 16 points per mma.
// Fragment layouts (PTX ISA, mma.m16n8k32 8-bit): groupID g = lane>>2, t = lane&3;
//  A: a0 (row g, k 4t..4t+3), a1 (row g+8, same k), a2 (row g, k 16+4t..), a3 (row g+8, k 16+4t..)
//  B: b0 (k 4t..4t+3, col n=g), b1 (k 16+4t.., col g)
//  D: d0,d1 (row g, cols 2t, 2t+1), d2,d3 (row g+8, cols 2t, 2t+1)
template <int S>
__global__ void nu_mma_kernel(Frac f, MmaTables T, const int2* __restrict__ in,
                              int2* __restrict__ out, uint64_t n) {
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const uint32_t s = S ? S : f.s;
    // B fragment: column n = g; n < 4 -> limb n of tau_x(k), n >= 4 -> limb n-4 of tau_y(k)
    uint32_t b[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        uint32_t v = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int kk = 16 * h + 4 * t + i;
            uint32_t e = 0;
            if (kk < f.r) {
                const bool xlevel = (kk & 1) == 0;
                if ((g < 4) == xlevel) e = limb(T.tau[kk], g & 3);
            }
            v |= e << (8 * i);
        }
        b[h] = v;
    }
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t base = warp * 16; base < n; base += nwarps * 16) {
        // rows g and g+8 of this tile
        uint32_t a[4];
        bool bad[2];
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
            const uint64_t pi = base + g + 8 * rr;
            int2 e = pi < n ? in[pi] : make_int2(0, 0);
            bool oob = e.x < 0 || e.y < 0 || (uint32_t)e.x >= f.side || (uint32_t)e.y >= f.side;
            bool hole = false;
            uint32_t lo = 0, hi = 0;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                uint32_t v = 0;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int mu = 16 * h + 4 * t + i;
                    uint32_t id = 0;
                    if (mu < f.r && !oob) {
                        const uint32_t sc = T.spow[mu];
                        const uint32_t gx = ((uint32_t)e.x / sc) % s, gy = ((uint32_t)e.y / sc) % s;
                        const int r = f.id_of_subbox[gy * s + gx];
                        if (r < 0) hole = true; else id = (uint32_t)r;
                    }
                    v |= id << (8 * i);
                }
                if (h == 0) lo = v; else hi = v;
            }
            // the 4 lanes of a group cover all 32 levels: OR their hole flags
            const uint32_t hb = __ballot_sync(0xffffffffu, hole || oob);
            bad[rr] = ((hb >> (lane & ~3)) & 0xFu) != 0;
            a[rr] = lo;       // a0 (rr=0, row g) / a1 (rr=1, row g+8)
            a[2 + rr] = hi;   // a2 / a3
        }
        int d[4] = {0, 0, 0, 0};
        mma_u8_16832(d, a, b);
        // lane holds cols 2t, 2t+1 for rows g (d0,d1) and g+8 (d2,d3)
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
            // part = limb(2t) << 16t... weight of col n within x or y: 8*(n & 3)
            const uint32_t c0 = (uint32_t)d[2 * rr], c1 = (uint32_t)d[2 * rr + 1];
            uint32_t part = (c0 << (8 * ((2 * t) & 3))) + (c1 << (8 * ((2 * t + 1) & 3)));
            part += __shfl_xor_sync(0xffffffffu, part, 1);  // t0+t1 -> x, t2+t3 -> y
            const uint32_t other = __shfl_xor_sync(0xffffffffu, part, 2);
            const uint64_t pi = base + g + 8 * rr;
            if (t == 0 && pi < n)
                out[pi] = bad[rr] ? make_int2(-1, -1) : make_int2((int)part, (int)other);
        }
    }
}

// lambda via tensor cores: x and y as two products over the digit-position values.
template <int K>
__global__ void lambda_mma_kernel(Frac f, MmaTables T, const int2* __restrict__ in,
                                  int2* __restrict__ out, uint64_t n) {
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const uint32_t k = K ? K : f.k;
    // B: column n = g; n < 4 -> limb n of s^mu; n >= 4 -> 0 (unused)
    uint32_t b[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        uint32_t v = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int kk = 16 * h + 4 * t + i;
            uint32_t e = (kk < f.r && g < 4) ? limb(T.spow[kk], g) : 0u;
            v |= e << (8 * i);
        }
        b[h] = v;
    }
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t base = warp * 16; base < n; base += nwarps * 16) {
        uint32_t ax[4], ay[4];
        bool bad[2];
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
            const uint64_t pi = base + g + 8 * rr;
            int2 c = pi < n ? in[pi] : make_int2(0, 0);
            const bool oob = c.x < 0 || c.y < 0 || (uint32_t)c.x >= f.w || (uint32_t)c.y >= f.h;
            bad[rr] = oob;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                uint32_t vx = 0, vy = 0;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int mu = 16 * h + 4 * t + i;
                    if (mu < f.r && !oob) {
                        // digit mu: even -> cx digit mu/2, odd -> cy digit (mu-1)/2
                        const uint32_t src = (mu & 1) ? (uint32_t)c.y : (uint32_t)c.x;
                        const uint32_t d = (src / T.tau[mu]) % k;
                        vx |= (uint32_t)f.gx[d] << (8 * i);
                        vy |= (uint32_t)f.gy[d] << (8 * i);
                    }
                }
                ax[2 * h + rr] = vx;
                ay[2 * h + rr] = vy;
            }
        }
        int dx[4] = {0, 0, 0, 0}, dy[4] = {0, 0, 0, 0};
        mma_u8_16832(dx, ax, b);
        mma_u8_16832(dy, ay, b);
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
            // cols 2t, 2t+1 valid for t < 2 (limbs 0..3)
            uint32_t px = 0, py = 0;
            if (t < 2) {
                px = ((uint32_t)dx[2 * rr] << (16 * t)) + ((uint32_t)dx[2 * rr + 1] << (16 * t + 8));
                py = ((uint32_t)dy[2 * rr] << (16 * t)) + ((uint32_t)dy[2 * rr + 1] << (16 * t + 8));
            }
            px += __shfl_xor_sync(0xffffffffu, px, 1);
            py += __shfl_xor_sync(0xffffffffu, py, 1);
            const uint64_t pi = base + g + 8 * rr;
            if (t == 0 && pi < n) out[pi] = bad[rr] ? make_int2(-1, -1) : make_int2((int)px, (int)py);
        }
    }
}

}  // namespace nbbgpu

namespace nbbgpu {

// The paper's per-cell compact step (lambda of the own cell, nu of its 8
// neighbours, stencil.cpp:354-367) with the 8 nu maps evaluated on
// the tensor cores: a warp stages its 32 cells x 8 neighbour coordinates in smem,
// 16 mma.sync.m16n8k32 (u8 x u8 -> s32, the nu_mma_kernel formulation) turn them
// into compact coordinates, and every lane gathers its own 8 results.
// Used for the "lambda/nu tensor-core vs CUDA-core maps" comparison (config 2).
template <int S>
__global__ void __launch_bounds__(128) step_compact_naive_mma_kernel(Frac f, MmaTables T,
                                                                    const uint8_t* __restrict__ src,
                                                                    uint8_t* __restrict__ dst,
                                                                    uint64_t i0, uint64_t i1,
                                                                    uint32_t birth, uint32_t survive,
                                                                    int deg) {
    __shared__ int2 q[4][256];    // per warp: (x, y) of neighbour queries, (-1,-1) = none
    __shared__ int2 res[4][256];  // per warp: (cx, cy) results, (-1, -1) = absent
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
    const uint32_t s = S ? S : f.s;
    uint32_t b[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        uint32_t v = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int kk = 16 * h + 4 * t + i;
            uint32_t e = 0;
            if (kk < f.r && ((g < 4) == ((kk & 1) == 0))) e = limb(T.tau[kk], g & 3);
            v |= e << (8 * i);
        }
        b[h] = v;
    }
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t base = i0 + ((blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5) * 32; base < i1;
         base += nwarps * 32) {
        const uint64_t i = base + lane;
        const bool valid = i < i1;
        uint32_t ex = 0, ey = 0;
        if (valid) lambda_map<0, S>(f, (uint32_t)(i % f.w), (uint32_t)(i / f.w), ex, ey);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int nx = (int)ex + kOffX[j], ny = (int)ey + kOffY[j];
            const bool in = valid && j < deg && nx >= 0 && ny >= 0 && nx < (int)f.side && ny < (int)f.side;
            q[wid][lane * 8 + j] = in ? make_int2(nx, ny) : make_int2(-1, -1);
        }
        __syncwarp();
#pragma unroll 1
        for (int tile = 0; tile < 16; ++tile) {
            uint32_t a[4];
            bool bad[2];
#pragma unroll
            for (int rr = 0; rr < 2; ++rr) {
                const int2 e = q[wid][tile * 16 + g + 8 * rr];
                const bool oob = e.x < 0;
                bool hole = false;
                uint32_t lo = 0, hi = 0;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    uint32_t v = 0;
#pragma unroll
                    for (int ii = 0; ii < 4; ++ii) {
                        const int mu = 16 * h + 4 * t + ii;
                        uint32_t id = 0;
                        if (mu < f.r && !oob) {
                            const uint32_t sc = T.spow[mu];
                            const uint32_t gx = ((uint32_t)e.x / sc) % s, gy = ((uint32_t)e.y / sc) % s;
                            const int r = f.id_of_subbox[gy * s + gx];
                            if (r < 0) hole = true; else id = (uint32_t)r;
                        }
                        v |= id << (8 * ii);
                    }
                    if (h == 0) lo = v; else hi = v;
                }
                const uint32_t hb = __ballot_sync(0xffffffffu, hole || oob);
                bad[rr] = ((hb >> (lane & ~3)) & 0xFu) != 0;
                a[rr] = lo;
                a[2 + rr] = hi;
            }
            int d[4] = {0, 0, 0, 0};
            mma_u8_16832(d, a, b);
#pragma unroll
            for (int rr = 0; rr < 2; ++rr) {
                const uint32_t c0 = (uint32_t)d[2 * rr], c1 = (uint32_t)d[2 * rr + 1];
                uint32_t part = (c0 << (8 * ((2 * t) & 3))) + (c1 << (8 * ((2 * t + 1) & 3)));
                part += __shfl_xor_sync(0xffffffffu, part, 1);
                const uint32_t other = __shfl_xor_sync(0xffffffffu, part, 2);
                if (t == 0)
                    res[wid][tile * 16 + g + 8 * rr] = bad[rr] ? make_int2(-1, -1)
                                                               : make_int2((int)part, (int)other);
            }
        }
        __syncwarp();
        if (valid) {
            uint32_t count = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int2 c = res[wid][lane * 8 + j];
                if (c.x >= 0) count += src[(uint64_t)c.y * f.w + c.x];
            }
            dst[i] = apply_rule(birth, survive, src[i], count);
        }
        __syncwarp();
    }
}

}  // namespace nbbgpu
