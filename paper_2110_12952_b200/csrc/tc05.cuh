// tc05.cuh -- the paper's tensor-core map formulation on Blackwell's 5th-generation
// tensor cores (tcgen05.mma kind::i8, accumulators in TMEM), north-star item 1.
//
// Same contraction as the mma.sync variant (maps.cuh, the
// reference's MapMatrices / to_compact_via_mma, maps.cpp:163-199), one CTA tile of
// M = 128 points per instruction:
//   nu:     D[p][n] = sum_mu H(p, mu) * limb_n(tau(mu))       (K = 32 levels, u8 x u8 -> s32)
//           A = replica ids H of point p (row p, K-major), B = base-256 limbs of the
//           unfold strides (columns 0-3: tau at x levels, 4-7: tau at y levels);
//   lambda: D[p][n] = sum_mu gx(d_mu) limb_n(s^mu) (+ gy for n = 4..7): two K = 32
//           instructions accumulating into the same TMEM columns.
// cx = sum_n D[p][n] << 8n: exact for every level r <= 32 (each D entry < 32 * 255^2).
// Roles: all 128 threads build their point's A row in shared memory (canonical
// K-major no-swizzle layout: 8-row x 16-byte core matrices, LBO = 128 B between the
// two K halves, SBO = 256 B between 8-row groups), thread 0 issues tcgen05.mma and
// tcgen05.commit to an mbarrier, warp w reads TMEM lanes 32w..32w+31 (its own
// points) with tcgen05.ld.32x32b.  TMEM: 32 columns per CTA (N = 16 used).
#pragma once

#include "common.cuh"
#include "maps.cuh"  // MmaTables, limb

namespace nbbgpu {

// byte offset of (row, k byte) in a 128 x 32-byte K-major interleaved operand tile
__device__ __forceinline__ uint32_t tc_kmajor_off(uint32_t row, uint32_t kb) {
    return (row >> 3) * 256u + (kb >> 4) * 128u + (row & 7u) * 16u + (kb & 15u);
}

// shared-memory matrix descriptor (tcgen05 "matrix descriptor"): start address,
// leading byte offset (K direction), stride byte offset (M/N direction), version 1,
// no swizzle
__device__ __forceinline__ uint64_t tc_smem_desc(const void* p) {
    const uint32_t a = (uint32_t)__cvta_generic_to_shared(p);
    return (uint64_t)((a >> 4) & 0x3FFFu) | ((uint64_t)(128u >> 4) << 16) | ((uint64_t)(256u >> 4) << 32) |
           (1ull << 46);
}

// instruction descriptor: kind::i8, D s32, A u8, B u8, both K-major, N = 16, M = 128
constexpr uint32_t kTcIdescI8 = (2u << 4) | (0u << 7) | (0u << 10) | ((16u >> 3) << 17) | ((128u >> 4) << 24);

__device__ __forceinline__ void tc_mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(kTcIdescI8), "r"(accumulate));
}
__device__ __forceinline__ void tc_commit(uint32_t mbar_smem) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mbar_smem)
                 : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_ld8(uint32_t taddr, uint32_t (&d)[8]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
        "tcgen05.wait::ld.sync.aligned;\n"
        : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7])
        : "r"(taddr)
        : "memory");
}
__device__ __forceinline__ void tc_mbar_init(uint32_t a) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(a));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void tc_mbar_wait(uint32_t a, uint32_t parity) {
    uint32_t done;
    do {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done) : "r"(a), "r"(parity) : "memory");
    } while (!done);
}

// B operand: 16 rows (n) x `kb` K bytes; value(n, mu) from f(n, mu)
template <class F>
__device__ __forceinline__ void tc_fill_b(uint8_t* sB, F&& val) {
    for (uint32_t i = threadIdx.x; i < 16 * 32; i += blockDim.x) {
        const uint32_t n = i >> 5, mu = i & 31;
        sB[tc_kmajor_off(n, mu)] = (uint8_t)val(n, mu);
    }
}

// One persistent CTA of 128 threads per SM share; lambda = false: nu, true: lambda.
template <int K, int S, bool LAMBDA>
__global__ void __launch_bounds__(128) map_tc05_kernel(Frac f, MmaTables T, const int2* __restrict__ in,
                                                       int2* __restrict__ out, uint64_t n) {
    __shared__ __align__(1024) uint8_t sA[2][128 * 32];  // [K half][...]: nu uses half 0
    __shared__ __align__(1024) uint8_t sB[2][16 * 32];
    __shared__ __align__(8) uint64_t mbar;
    __shared__ uint32_t tmem_base;
    const uint32_t t = threadIdx.x, warp = t >> 5;
    const uint32_t k = K ? K : f.k, s = S ? S : f.s;
    // B: limbs of the per-level weights (nu: tau(mu) at x / y levels; lambda: s^mu)
    if (LAMBDA) {
        tc_fill_b(sB[0], [&](uint32_t nn, uint32_t mu) { return (nn < 4 && (int)mu < f.r) ? limb(T.spow[mu], nn) : 0u; });
        tc_fill_b(sB[1], [&](uint32_t nn, uint32_t mu) {
            return (nn >= 4 && nn < 8 && (int)mu < f.r) ? limb(T.spow[mu], nn - 4) : 0u;
        });
    } else {
        tc_fill_b(sB[0], [&](uint32_t nn, uint32_t mu) {
            if ((int)mu >= f.r || nn >= 8) return 0u;
            const bool xlevel = (mu & 1) == 0;
            return (nn < 4) == xlevel ? limb(T.tau[mu], nn & 3) : 0u;
        });
    }
    const uint32_t mb = (uint32_t)__cvta_generic_to_shared(&mbar);
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&tmem_base))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (t == 0) tc_mbar_init(mb);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // B: generic writes -> tensor core reads
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base;
    const uint64_t a0 = tc_smem_desc(sA[0]), a1 = tc_smem_desc(sA[1]);
    const uint64_t b0 = tc_smem_desc(sB[0]), b1 = tc_smem_desc(sB[1]);
    uint32_t phase = 0;
    for (uint64_t base = (uint64_t)blockIdx.x * 128; base < n; base += (uint64_t)gridDim.x * 128) {
        const uint64_t pi = base + t;
        const int2 c = pi < n ? in[pi] : make_int2(0, 0);
        bool bad;
        uint32_t w0[8], w1[8];  // A row bytes: K half 0 (and half 1 for lambda)
#pragma unroll
        for (int q = 0; q < 8; ++q) w0[q] = w1[q] = 0u;
        if (LAMBDA) {
            bad = c.x < 0 || c.y < 0 || (uint32_t)c.x >= f.w || (uint32_t)c.y >= f.h;
            uint32_t cx = bad ? 0u : (uint32_t)c.x, cy = bad ? 0u : (uint32_t)c.y;
#pragma unroll
            for (int mu = 0; mu < 32; ++mu) {
                if (mu >= f.r) break;
                uint32_t d;
                if ((mu & 1) == 0) { d = cx % k; cx /= k; }
                else { d = cy % k; cy /= k; }
                w0[mu >> 2] |= (uint32_t)f.gx[d] << (8 * (mu & 3));
                w1[mu >> 2] |= (uint32_t)f.gy[d] << (8 * (mu & 3));
            }
        } else {
            bad = c.x < 0 || c.y < 0 || (uint32_t)c.x >= f.side || (uint32_t)c.y >= f.side;
            uint32_t x = bad ? 0u : (uint32_t)c.x, y = bad ? 0u : (uint32_t)c.y;
#pragma unroll
            for (int mu = 0; mu < 32; ++mu) {
                if (mu >= f.r) break;
                const int id = f.id_of_subbox[(y % s) * s + (x % s)];
                x /= s;
                y /= s;
                if (id < 0) bad = true;
                else w0[mu >> 2] |= (uint32_t)id << (8 * (mu & 3));
            }
        }
        // row t of A: 16 bytes per K half of the core-matrix pair
        *reinterpret_cast<uint4*>(sA[0] + tc_kmajor_off(t, 0)) = make_uint4(w0[0], w0[1], w0[2], w0[3]);
        *reinterpret_cast<uint4*>(sA[0] + tc_kmajor_off(t, 16)) = make_uint4(w0[4], w0[5], w0[6], w0[7]);
        if (LAMBDA) {
            *reinterpret_cast<uint4*>(sA[1] + tc_kmajor_off(t, 0)) = make_uint4(w1[0], w1[1], w1[2], w1[3]);
            *reinterpret_cast<uint4*>(sA[1] + tc_kmajor_off(t, 16)) = make_uint4(w1[4], w1[5], w1[6], w1[7]);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // A rows -> the tensor core
        tc_fence_before();  // (this thread's TMEM loads of the previous tile are complete)
        __syncthreads();
        if (t == 0) {
            tc_fence_after();
            tc_mma_i8(tmem, a0, b0, 0u);
            if (LAMBDA) tc_mma_i8(tmem, a1, b1, 1u);
            tc_commit(mb);  // arrives when the MMAs (and their smem reads) are complete
        }
        tc_mbar_wait(mb, phase);
        phase ^= 1u;
        tc_fence_after();
        uint32_t d[8];
        tc_ld8(tmem + ((warp * 32u) << 16), d);  // lanes 32w.. = this warp's points, columns 0-7
        const uint32_t rx = d[0] + (d[1] << 8) + (d[2] << 16) + (d[3] << 24);
        const uint32_t ry = d[4] + (d[5] << 8) + (d[6] << 16) + (d[7] << 24);
        if (pi < n) out[pi] = bad ? make_int2(-1, -1) : make_int2((int)rx, (int)ry);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem) : "memory");
}

}  // namespace nbbgpu
