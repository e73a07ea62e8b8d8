// layouts.cuh -- the reference's two other storage layouts on the device
// (SURVEY.md 8(f) f1/f2):
//   * the "lambda" backend (Backend::CompactGrid): embedded n x n storage, but the
//     step visits exactly the k^r compact indices through lambda and reads the
//     neighbours in embedded coordinates (Simulation::step_compact_grid,
//     proj/src/stencil.cpp:313-332) -- the paper's approach 2;
//   * the blocked compact layout (Layout::BlockedCompact, --block-size rho = s^m):
//     k^(r-m) blocks of rho x rho embedded mini boxes, block-major and row-major
//     inside a block (grid.cpp:54-63), stepped by step_compact_blocked
//     (stencil.cpp:370-399) -- the paper's best nu configuration (rho = 16).
// One thread per compact index / block slot; the digit loops are those of
// common.cuh.  Bit-exact with the reference (tests/test_gpu_layouts.py).
#pragma once

#include "common.cuh"

namespace nbbgpu {

// Simulation::step_compact_grid (stencil.cpp:313-332)
template <int K, int S>
__global__ void step_lambda_kernel(Frac f, const uint8_t* __restrict__ src, uint8_t* __restrict__ dst,
                                   uint32_t birth, uint32_t survive, int deg) {
    const uint64_t total = (uint64_t)f.w * f.h, n = f.side;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t x, y;
        lambda_map<K, S>(f, (uint32_t)(i % f.w), (uint32_t)(i / f.w), x, y);
        uint32_t count = 0;
        for (int j = 0; j < deg; ++j) {
            const int64_t nx = (int64_t)x + kOffX[j], ny = (int64_t)y + kOffY[j];
            if (nx >= 0 && ny >= 0 && nx < (int64_t)n && ny < (int64_t)n) count += src[(uint64_t)ny * n + nx];
        }
        const uint64_t e = (uint64_t)y * n + x;
        dst[e] = apply_rule(birth, survive, src[e], count);
    }
}

struct BlockedGeom {
    Frac f;          // full level r
    Frac fc;         // coarse level r - m
    uint32_t rho;    // s^m
    int m;
};

// every one of the m low digit pairs of the in-block position is a replica:
// (x, y) is a fractal cell iff its coarse cell is (block present) and this holds
template <int S>
__device__ __forceinline__ bool low_member(const Frac& f, uint32_t lx, uint32_t ly, int m) {
    const uint32_t s = sval<S>(f);
    for (int mu = 0; mu < m; ++mu) {
        if (f.id_of_subbox[(ly % s) * s + (lx % s)] < 0) return false;
        lx /= s;
        ly /= s;
    }
    return true;
}

// Grid::storage_index, BlockedCompact branch (grid.cpp:54-63); false if the coarse
// cell of (x, y) is not in the coarse fractal
template <int K, int S>
__device__ __forceinline__ bool blocked_index(const BlockedGeom& G, uint32_t x, uint32_t y, uint64_t& idx) {
    uint32_t cx, cy;
    if (!nu_map<K, S>(G.fc, x / G.rho, y / G.rho, cx, cy)) return false;
    idx = ((uint64_t)cy * G.fc.w + cx) * G.rho * G.rho + (uint64_t)(y % G.rho) * G.rho + (x % G.rho);
    return true;
}

// Simulation::seed_random, BlockedCompact branch (stencil.cpp:161-177)
template <int K, int S>
__global__ void seed_blocked_kernel(BlockedGeom G, uint8_t* __restrict__ front, uint64_t seed_mix,
                                    double density) {
    const uint64_t per = (uint64_t)G.rho * G.rho, total = (uint64_t)G.fc.w * G.fc.h * per;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t b = i / per;
        const uint32_t ly = (uint32_t)((i % per) / G.rho), lx = (uint32_t)(i % G.rho);
        if (!low_member<S>(G.f, lx, ly, G.m)) continue;  // filler slot stays 0
        uint32_t X, Y;
        lambda_map<K, S>(G.fc, (uint32_t)(b % G.fc.w), (uint32_t)(b / G.fc.w), X, Y);
        front[i] = cell_alive_mixed(seed_mix, X * G.rho + lx, Y * G.rho + ly, density) ? 1 : 0;
    }
}

// Simulation::state_hash, BlockedCompact branch (stencil.cpp:217-231)
template <int K, int S>
__global__ void hash_blocked_kernel(BlockedGeom G, const uint8_t* __restrict__ front, unsigned long long* out) {
    const uint64_t per = (uint64_t)G.rho * G.rho, total = (uint64_t)G.fc.w * G.fc.h * per;
    uint64_t acc = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
         i += (uint64_t)gridDim.x * blockDim.x) {
        if (!front[i]) continue;
        const uint64_t b = i / per;
        const uint32_t ly = (uint32_t)((i % per) / G.rho), lx = (uint32_t)(i % G.rho);
        uint32_t X, Y;
        lambda_map<K, S>(G.fc, (uint32_t)(b % G.fc.w), (uint32_t)(b / G.fc.w), X, Y);
        acc += coord_mix(X * G.rho + lx, Y * G.rho + ly);
    }
    block_sum_atomic(acc, out);
}

// Static per-block table (built once per handle): [0..8] the block index in every
// direction (dy+1)*3 + dx+1 (4 = the block itself; kNoBlock outside the box or on a
// coarse hole, via the coarse nu), [9], [10] the block's coarse corner
// (lambda at level r - m), [11] unused -- 48 B per block, 3 x 16-B loads.
constexpr uint32_t kNoBlock = 0xFFFFFFFFu;
constexpr int kBlockTab = 12;

template <int K, int S>
__global__ void build_blocktab_kernel(BlockedGeom G, uint32_t* __restrict__ tab) {
    const uint64_t nblocks = (uint64_t)G.fc.w * G.fc.h;
    for (uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b < nblocks;
         b += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t X, Y;
        lambda_map<K, S>(G.fc, (uint32_t)(b % G.fc.w), (uint32_t)(b / G.fc.w), X, Y);
        uint32_t* t = tab + b * kBlockTab;
        for (int d = 0; d < 9; ++d) {
            const int64_t nx = (int64_t)X + d % 3 - 1, ny = (int64_t)Y + d / 3 - 1;
            uint32_t v = kNoBlock, cx, cy;
            if (d == 4) v = (uint32_t)b;
            else if (nx >= 0 && ny >= 0 && nx < (int64_t)G.fc.side && ny < (int64_t)G.fc.side &&
                     nu_map<K, S>(G.fc, (uint32_t)nx, (uint32_t)ny, cx, cy))
                v = cy * G.fc.w + cx;
            t[d] = v;
        }
        t[9] = X;
        t[10] = Y;
        t[11] = 0;
    }
}

__device__ __forceinline__ bool low_mask_bit(const uint32_t* lm, uint32_t lx, uint32_t ly, uint32_t rho) {
    const uint32_t i = ly * rho + lx;
    return (__ldg(lm + (i >> 5)) >> (i & 31)) & 1u;
}

// Simulation::step_compact_blocked (stencil.cpp:370-399): one thread per slot; the
// block's neighbour indices come from the static block table, the in-block filler
// pattern from low_mask (the same for every block) -- no per-cell digit loops.
__global__ void step_blocked_kernel(BlockedGeom G, const uint32_t* __restrict__ low_mask,
                                    const uint32_t* __restrict__ btab, const uint8_t* __restrict__ src,
                                    uint8_t* __restrict__ dst, uint32_t birth, uint32_t survive, int deg) {
    const uint64_t per = (uint64_t)G.rho * G.rho, total = (uint64_t)G.fc.w * G.fc.h * per;
    const uint32_t rho = G.rho;
    const int64_t n = G.f.side;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t b = i / per;
        const int32_t ly = (int32_t)((i % per) / rho), lx = (int32_t)(i % rho);
        if (!low_mask_bit(low_mask, lx, ly, rho)) continue;  // filler slot, stays dead
        const uint4* t4 = reinterpret_cast<const uint4*>(btab + b * kBlockTab);
        const uint4 q0 = __ldg(t4), q1 = __ldg(t4 + 1), q2 = __ldg(t4 + 2);
        const uint32_t nbk[9] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w, q2.x};
        const int64_t x = (int64_t)q2.y * rho + lx, y = (int64_t)q2.z * rho + ly;
        uint32_t count = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (j >= deg) break;
            const int64_t nx = x + kOffX[j], ny = y + kOffY[j];
            if (nx < 0 || ny < 0 || nx >= n || ny >= n) continue;
            int32_t nlx = lx + kOffX[j], nly = ly + kOffY[j];
            const int dx = nlx < 0 ? -1 : (nlx >= (int32_t)rho ? 1 : 0);
            const int dy = nly < 0 ? -1 : (nly >= (int32_t)rho ? 1 : 0);
            nlx -= dx * (int32_t)rho;
            nly -= dy * (int32_t)rho;
            if (!low_mask_bit(low_mask, nlx, nly, rho)) continue;
            const uint32_t nb2 = nbk[(dy + 1) * 3 + dx + 1];
            if (nb2 != kNoBlock) count += src[(uint64_t)nb2 * per + (uint64_t)nly * rho + nlx];
        }
        dst[i] = apply_rule(birth, survive, src[i], count);
    }
}

// ---- the embedded n x n view of any layout (Simulation::cell for every (x, y),
// stencil.cpp:182-188): bytes 0/1, or the rows of a plain PBM (write_pbm,
// pbm.cpp:9-23: '1'/'0' per cell, '\n' after each row) -------------------------
struct ViewSrc {
    int mode;               // NBBGPU_MODE_*
    bool packed;            // compact mode, packed layout
    const uint8_t* bytes;   // byte layouts
    const uint32_t* words;  // packed layout
    uint32_t wq, Wc, Cp;    // packed geometry
    uint32_t ilv;           // interleaved record layout (rec_word)
    BlockedGeom bg;         // blocked layout
};

template <int K, int S>
__device__ __forceinline__ uint8_t view_cell(const Frac& f, const ViewSrc& v, uint32_t x, uint32_t y) {
    if (v.mode == 1 || v.mode == 2) return v.bytes[(uint64_t)y * f.side + x];  // bb / lambda: holes are 0
    uint32_t cx, cy;
    if (!nu_map<K, S>(f, x, y, cx, cy)) return 0;  // not a fractal cell
    if (v.mode == 3) {
        uint64_t idx;
        if (!blocked_index<K, S>(v.bg, x, y, idx)) return 0;
        return v.bytes[idx];
    }
    if (!v.packed) return v.bytes[(uint64_t)cy * f.w + cx];
    const uint32_t X = cx / v.wq, c = cx % v.wq, Y = cy / v.wq, a = cy % v.wq;
    const uint64_t t = (uint64_t)Y * v.Wc + X;
    return (uint8_t)((v.words[(t / 32) * v.Cp + rec_word(v.ilv, v.wq, a, c)] >> (t % 32)) & 1u);
}

// PBM: row stride n + 1 with '\n' at the end, characters '0' / '1'; else bytes 0 / 1
template <int K, int S>
__global__ void embedded_view_kernel(Frac f, ViewSrc v, uint8_t* __restrict__ out, int pbm) {
    const uint64_t n = f.side, stride = pbm ? n + 1 : n, total = n * stride;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t y = i / stride, x = i - y * stride;
        if (x == n) { out[i] = '\n'; continue; }
        const uint8_t c = view_cell<K, S>(f, v, (uint32_t)x, (uint32_t)y);
        out[i] = pbm ? (uint8_t)(c ? '1' : '0') : c;
    }
}

}  // namespace nbbgpu
