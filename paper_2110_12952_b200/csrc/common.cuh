// common.cuh -- shared device/host definitions of the sm_100a compact-fractal engine.
//
// Frac holds the per-(descriptor, level) tables of the reference's CoordMapper
// (proj/include/nbb/maps.hpp:61-70) in a kernel-parameter struct, so several
// handles with different fractals can coexist (no __constant__ globals).
#pragma once

#include "rtc_compat.cuh"

namespace nbbgpu {

constexpr int kMaxS = 16;
constexpr int kMaxLevel = 40;

struct Frac {
    int k, s, r;
    uint32_t w, h;      // compact dims k^ceil(r/2), k^floor(r/2)   (maps.cpp:36-43)
    uint32_t side;      // s^r                                       (geometry.cpp:23-27)
    int8_t id_of_subbox[kMaxS * kMaxS];  // gy*s+gx -> replica id, -1 hole (maps.cpp:61-69)
    uint8_t gx[kMaxS * kMaxS], gy[kMaxS * kMaxS];  // replica positions by id
};

// ---------------------------------------------------------------------------
// rng.hpp:9-39 -- bit-exact on the device (integer ops + one exact double mul)
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

// cell_alive(seed, x, y, density) with splitmix64(seed) hoisted by the caller.
__host__ __device__ __forceinline__ bool cell_alive_mixed(uint64_t seed_mix, int64_t x, int64_t y,
                                                          double density) {
    const uint64_t key = splitmix64(seed_mix ^ (static_cast<uint64_t>(x) << 32) ^
                                    static_cast<uint64_t>(static_cast<uint32_t>(y)));
    // (key >> 11) < 2^53 converts exactly; the multiply by 2^-53 is exact.
    const double u = static_cast<double>(key >> 11) * (1.0 / 9007199254740992.0);
    return u < density;
}

__host__ __device__ __forceinline__ uint64_t coord_mix(int64_t x, int64_t y) {
    return splitmix64((static_cast<uint64_t>(x) << 32) ^
                      static_cast<uint64_t>(static_cast<uint32_t>(y)));
}

// ---------------------------------------------------------------------------
// Maps, CUDA-core digit-loop variant.  K/S are compile-time when the kernel is
// instantiated for a known (k, s) (division by constants), 0 = runtime.
// ---------------------------------------------------------------------------
template <int K>
__device__ __forceinline__ int kval(const Frac& f) { return K ? K : f.k; }
template <int S>
__device__ __forceinline__ int sval(const Frac& f) { return S ? S : f.s; }

// lambda: compact -> embedded (CoordMapper::to_embedded, maps.cpp:123-146).
template <int K, int S>
__device__ __forceinline__ void lambda_map(const Frac& f, uint32_t cx, uint32_t cy, uint32_t& x,
                                           uint32_t& y) {
    const uint32_t k = kval<K>(f), s = sval<S>(f);
    uint32_t ex = 0, ey = 0, sp = 1;
    for (int mu = 0; mu < f.r; ++mu) {
        uint32_t d;
        if ((mu & 1) == 0) { d = cx % k; cx /= k; }
        else               { d = cy % k; cy /= k; }
        ex += f.gx[d] * sp;
        ey += f.gy[d] * sp;
        sp *= s;
    }
    x = ex;
    y = ey;
}

// nu: embedded -> compact (CoordMapper::try_to_compact, maps.cpp:80-107).
// Caller guarantees 0 <= x, y < side.
template <int K, int S>
__device__ __forceinline__ bool nu_map(const Frac& f, uint32_t x, uint32_t y, uint32_t& cx,
                                       uint32_t& cy) {
    const uint32_t k = kval<K>(f), s = sval<S>(f);
    uint32_t ax = 0, ay = 0, p = 1;
    for (int mu = 0; mu < f.r; ++mu) {
        const int id = f.id_of_subbox[(y % s) * s + (x % s)];
        if (id < 0) return false;
        if ((mu & 1) == 0) ax += id * p;
        else { ay += id * p; p *= k; }
        x /= s;
        y /= s;
    }
    cx = ax;
    cy = ay;
    return true;
}

// Moore offsets in the reference order (stencil.cpp:55-61); von Neumann = first 4.
__device__ __constant__ static const int kOffX[8] = {1, -1, 0, 0, 1, 1, -1, -1};
__device__ __constant__ static const int kOffY[8] = {0, 0, 1, -1, 1, -1, 1, -1};

// StencilRule::born_with / survives_with (stencil.hpp:23-24)
__device__ __forceinline__ uint8_t apply_rule(uint32_t birth, uint32_t survive, uint32_t alive,
                                              uint32_t count) {
    return static_cast<uint8_t>(((alive ? survive : birth) >> count) & 1u);
}

}  // namespace nbbgpu
