// naive.cuh -- one-thread-per-cell kernels: seeding, state hash, the paper's
// per-cell compact step (lambda of the own cell, nu of every neighbour) and the
// bounding-box step.  These are the first correct CUDA path and the map-variant
// vehicle; the throughput path is tiled.cuh.
#pragma once

#include "common.cuh"

namespace nbbgpu {

// Simulation::seed_random, linear-compact branch (stencil.cpp:152-159).
template <int K, int S>
__global__ void seed_compact_kernel(Frac f, uint8_t* __restrict__ front, uint64_t total,
                                    uint64_t seed_mix, double density) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t x, y;
        lambda_map<K, S>(f, (uint32_t)(i % f.w), (uint32_t)(i / f.w), x, y);
        front[i] = cell_alive_mixed(seed_mix, x, y, density) ? 1 : 0;
    }
}

// Simulation::seed_random, embedded branch (stencil.cpp:146-151).
template <int K, int S>
__global__ void seed_bb_kernel(Frac f, uint8_t* __restrict__ front, uint64_t seed_mix,
                               double density) {
    const uint64_t total = (uint64_t)f.side * f.side;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t x = (uint32_t)(i % f.side), y = (uint32_t)(i / f.side);
        uint32_t cx, cy;
        front[i] = nu_map<K, S>(f, x, y, cx, cy) && cell_alive_mixed(seed_mix, x, y, density) ? 1 : 0;
    }
}

__device__ __forceinline__ void block_sum_atomic(uint64_t v, unsigned long long* out) {
    __shared__ uint64_t part[32];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) part[wid] = v;
    __syncthreads();
    if (wid == 0) {
        v = lane < (int)(blockDim.x >> 5) ? part[lane] : 0;
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) atomicAdd(out, (unsigned long long)v);
    }
}

// Simulation::state_hash, linear-compact branch (stencil.cpp:207-216), over the
// compact index range [i0, i1).  uint64 wrap-around sums are order independent.
template <int K, int S>
__global__ void hash_compact_kernel(Frac f, const uint8_t* __restrict__ front, uint64_t i0,
                                    uint64_t i1, unsigned long long* out) {
    uint64_t acc = 0;
    for (uint64_t i = i0 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < i1;
         i += (uint64_t)gridDim.x * blockDim.x) {
        if (front[i]) {
            uint32_t x, y;
            lambda_map<K, S>(f, (uint32_t)(i % f.w), (uint32_t)(i / f.w), x, y);
            acc += coord_mix(x, y);
        }
    }
    block_sum_atomic(acc, out);
}

// Simulation::state_hash, embedded branch (stencil.cpp:200-206).
__global__ void hash_bb_kernel(uint32_t side, const uint8_t* __restrict__ front,
                               unsigned long long* out) {
    const uint64_t total = (uint64_t)side * side;
    uint64_t acc = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
         i += (uint64_t)gridDim.x * blockDim.x)
        if (front[i]) acc += coord_mix(i % side, i / side);
    block_sum_atomic(acc, out);
}

// Simulation::step_compact_linear without a neighbour table (stencil.cpp:353-367):
// lambda once for the own cell, nu for each in-box neighbour, byte sum, rule.
template <int K, int S>
__global__ void step_compact_naive_kernel(Frac f, const uint8_t* __restrict__ src,
                                          uint8_t* __restrict__ dst, uint64_t i0, uint64_t i1,
                                          uint32_t birth, uint32_t survive, int deg) {
    for (uint64_t i = i0 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < i1;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t ex, ey;
        lambda_map<K, S>(f, (uint32_t)(i % f.w), (uint32_t)(i / f.w), ex, ey);
        uint32_t count = 0;
        for (int j = 0; j < deg; ++j) {
            const int nx = (int)ex + kOffX[j], ny = (int)ey + kOffY[j];
            if (nx < 0 || ny < 0 || nx >= (int)f.side || ny >= (int)f.side) continue;
            uint32_t cx, cy;
            if (nu_map<K, S>(f, (uint32_t)nx, (uint32_t)ny, cx, cy))
                count += src[(uint64_t)cy * f.w + cx];
        }
        dst[i] = apply_rule(birth, survive, src[i], count);
    }
}

// Simulation::build_neighbor_table (stencil.cpp:401-414) on the device: per
// compact slot and offset j the neighbour's slot, or kNoSlot (outside the box or
// a hole).  The reference stores [i * deg + j] int64; here the table is laid out
// offset-major, tab[j * n + i], so the step kernel's table reads coalesce, with
// 32-bit slots while k^r < 2^32 (64-bit above).
template <int K, int S, class IDX>
__global__ void build_nbr_table_kernel(Frac f, uint64_t n, int deg, IDX* __restrict__ tab) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t ex, ey;
        lambda_map<K, S>(f, (uint32_t)(i % f.w), (uint32_t)(i / f.w), ex, ey);
        for (int j = 0; j < deg; ++j) {
            const int nx = (int)ex + kOffX[j], ny = (int)ey + kOffY[j];
            IDX slot = (IDX)~(IDX)0;
            uint32_t cx, cy;
            if (nx >= 0 && ny >= 0 && nx < (int)f.side && ny < (int)f.side &&
                nu_map<K, S>(f, (uint32_t)nx, (uint32_t)ny, cx, cy))
                slot = (IDX)((uint64_t)cy * f.w + cx);
            tab[(uint64_t)j * n + i] = slot;
        }
    }
}

// Simulation::step_compact_linear with the neighbour table (stencil.cpp:340-352):
// deg table reads + deg byte gathers per cell, no maps.
template <class IDX, int DEG>
__global__ void step_table_kernel(const IDX* __restrict__ tab, uint64_t n, const uint8_t* __restrict__ src,
                                  uint8_t* __restrict__ dst, uint64_t i0, uint64_t i1, uint32_t birth,
                                  uint32_t survive) {
    for (uint64_t i = i0 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < i1;
         i += (uint64_t)gridDim.x * blockDim.x) {
        IDX slot[DEG];
#pragma unroll
        for (int j = 0; j < DEG; ++j) slot[j] = __ldcs(tab + (uint64_t)j * n + i);  // streamed once per step
        uint32_t count = 0;
#pragma unroll
        for (int j = 0; j < DEG; ++j)
            if (slot[j] != (IDX)~(IDX)0) count += src[slot[j]];
        dst[i] = apply_rule(birth, survive, src[i], count);
    }
}

// Simulation::step_bounding_box (stencil.cpp:291-311), one thread per embedded
// cell: holes are skipped (never written), neighbours read straight from the box.
template <int K, int S>
__global__ void step_bb_naive_kernel(Frac f, const uint8_t* __restrict__ src,
                                     uint8_t* __restrict__ dst, uint32_t birth, uint32_t survive,
                                     int deg) {
    const uint64_t n = f.side, total = n * n;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t x = (uint32_t)(i % n), y = (uint32_t)(i / n);
        uint32_t cx, cy;
        if (!nu_map<K, S>(f, x, y, cx, cy)) continue;
        uint32_t count = 0;
        for (int j = 0; j < deg; ++j) {
            const int nx = (int)x + kOffX[j], ny = (int)y + kOffY[j];
            if (nx >= 0 && ny >= 0 && nx < (int)n && ny < (int)n) count += src[(uint64_t)ny * n + nx];
        }
        dst[i] = apply_rule(birth, survive, src[i], count);
    }
}

// Any byte other than 0/1 in [0, n) sets *flag (states are binary on the GPU).
__global__ void check_binary_kernel(const uint8_t* __restrict__ p, uint64_t n, int* flag) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        if (p[i] > 1) *flag = 1;
}

// Bounding-box uploads: a live byte on a hole sets *flag (the reference's holes
// are never written -- set_cell requires a fractal cell, stencil.cpp:190-194).
template <int K, int S>
__global__ void check_bb_holes_kernel(Frac f, const uint8_t* __restrict__ p, int* flag) {
    const uint64_t n = f.side, total = n * n;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t cx, cy;
        if (p[i] && !nu_map<K, S>(f, (uint32_t)(i % n), (uint32_t)(i / n), cx, cy)) *flag = 1;
    }
}

}  // namespace nbbgpu
