// blocks.cuh -- register-resident micro-blocks for the packed step kernel.
//
// A micro-block is a level-P sub-fractal inside a tile: a BW x BH (BW = k^ceil(P/2),
// BH = k^floor(P/2)) sub-rectangle of the tile's compact layout (the same digit
// split as tiles).  Every micro-block has the same cells and the
// same internal neighbour wiring, so for a descriptor known at compile time the
// wiring is a constexpr table: for cell n and Moore direction j the neighbour is
// another cell of the block (a register), a position inside the block's embedded
// box that is not a cell (a hole -> dead, always), or one of NE "external"
// positions around the box.  One thread evaluates a whole block: NB own words +
// NE external words (through a per-block table of stage byte offsets) instead of
// 9 x NB table-driven loads, and the 8-input bit-sliced adders run on registers.
// The wiring is derived from the replica table exactly as CoordMapper derives
// lambda (maps.cpp:123-146): cell n = (u, v) in the block's compact layout sits at
// embedded (sum_mu gx[d_mu] s^mu, sum_mu gy[d_mu] s^mu).
#pragma once

#include "rtc_compat.cuh"

namespace nbbgpu {

constexpr int cpow(int b, int e) { return e <= 0 ? 1 : b * cpow(b, e - 1); }

// ---- descriptors with a compile-time replica table (descriptor.cpp:54-58 and the
// descriptor files of SURVEY.md 8(d)) ---------------------------------------------
struct TriangleTag {  // K(n,3,2)
    static constexpr int K = 3, S = 2;
    static constexpr int GX[K] = {0, 1, 0};
    static constexpr int GY[K] = {0, 0, 1};
};
struct CarpetTag {  // K(n,8,3): row-major 3x3 minus (1,1)
    static constexpr int K = 8, S = 3;
    static constexpr int GX[K] = {0, 1, 2, 0, 2, 0, 1, 2};
    static constexpr int GY[K] = {0, 0, 0, 1, 1, 2, 2, 2};
};
struct VicsekTag {  // K(n,5,3): plus sign
    static constexpr int K = 5, S = 3;
    static constexpr int GX[K] = {1, 0, 1, 2, 1};
    static constexpr int GY[K] = {0, 1, 1, 1, 2};
};
struct HTag {  // K(n,7,3): descriptors/h-fractal.desc
    static constexpr int K = 7, S = 3;
    static constexpr int GX[K] = {0, 2, 0, 1, 2, 0, 2};
    static constexpr int GY[K] = {0, 0, 1, 1, 1, 2, 2};
};
struct CandyTag {  // K(n,12,4): descriptors/candy.desc (4x4 minus the corners)
    static constexpr int K = 12, S = 4;
    static constexpr int GX[K] = {1, 2, 0, 1, 2, 3, 0, 1, 2, 3, 1, 2};
    static constexpr int GY[K] = {0, 0, 1, 1, 1, 1, 2, 2, 2, 2, 3, 3};
};

constexpr int kWireAbsent = -1;    // hole inside the block box: dead at every position
constexpr int kMaxExt = 48;

// Moore offsets in the reference order (stencil.cpp:55-61); von Neumann = first 4.
constexpr int kDX[8] = {1, -1, 0, 0, 1, 1, -1, -1};
constexpr int kDY[8] = {0, 0, 1, -1, 1, -1, 1, -1};

template <class FT, int P>
struct WiringGeom {
    static constexpr int K = FT::K, S = FT::S;
    static constexpr int BW = cpow(K, (P + 1) / 2), BH = cpow(K, P / 2), NB = BW * BH, SP = cpow(S, P);
};

template <int NB>
struct WiringData {
    int ex[NB] = {}, ey[NB] = {};  // embedded position of block cell n
    int src[NB][8] = {};           // >= 0: block cell; kWireAbsent; <= -2: external -(e + 2)
    int NE = 0;
    int epx[kMaxExt] = {}, epy[kMaxExt] = {};  // external positions (box-relative)
};

// The wiring of a level-P micro-block of the descriptor (K, S, GX, GY): the same
// function runs at compile time for the built-in tags and for run-time specialised
// (jit.inc) tags, and on the host for the block tables of the latter.  nb = BW * BH
// cells are used of the NB-sized arrays.
template <int NB>
constexpr WiringData<NB> make_wiring_from(int K, int S, const int* GX, const int* GY, int P) {
    int BW = 1, BH = 1, SP = 1;
    for (int i = 0; i < (P + 1) / 2; ++i) BW *= K;
    for (int i = 0; i < P / 2; ++i) BH *= K;
    for (int i = 0; i < P; ++i) SP *= S;
    const int nb = BW * BH;
    WiringData<NB> d{};
    for (int n = 0; n < nb; ++n) {
        int cx = n % BW, cy = n / BW, x = 0, y = 0, sp = 1;
        for (int mu = 0; mu < P; ++mu) {
            int dg = 0;
            if ((mu & 1) == 0) { dg = cx % K; cx /= K; }
            else { dg = cy % K; cy /= K; }
            x += GX[dg] * sp;
            y += GY[dg] * sp;
            sp *= S;
        }
        d.ex[n] = x;
        d.ey[n] = y;
    }
    for (int n = 0; n < nb; ++n)
        for (int j = 0; j < 8; ++j) {
            const int X = d.ex[n] + kDX[j], Y = d.ey[n] + kDY[j];
            if (X >= 0 && Y >= 0 && X < SP && Y < SP) {
                int hit = kWireAbsent;
                for (int m = 0; m < nb; ++m)
                    if (d.ex[m] == X && d.ey[m] == Y) hit = m;
                d.src[n][j] = hit;
            } else {
                int e = -1;
                for (int m = 0; m < d.NE; ++m)
                    if (d.epx[m] == X && d.epy[m] == Y) e = m;
                if (e < 0) {
                    if (d.NE == kMaxExt) return d;  // (callers reject NE > kMaxExt - 1)
                    e = d.NE++;
                    d.epx[e] = X;
                    d.epy[e] = Y;
                }
                d.src[n][j] = -(e + 2);
            }
        }
    return d;
}

template <class FT, int P>
constexpr WiringData<WiringGeom<FT, P>::NB> make_wiring() {
    return make_wiring_from<WiringGeom<FT, P>::NB>(FT::K, FT::S, FT::GX, FT::GY, P);
}

template <class FT, int P>
struct Wiring : WiringGeom<FT, P> {
    using G = WiringGeom<FT, P>;
    static constexpr WiringData<G::NB> d = make_wiring<FT, P>();
    static constexpr int NE = d.NE;
    static constexpr int NEP = (NE + 3) & ~3;  // table entries per block (16-B rows)
    static_assert(NE < kMaxExt, "too many external positions");
};

// compile-time loop: f(std::integral_constant<int, i>) for i in [0, N)
template <class F, int... Is>
__device__ __forceinline__ void static_for_impl(F&& f, std::integer_sequence<int, Is...>) {
    (f(std::integral_constant<int, Is>{}), ...);
}
template <int N, class F>
__device__ __forceinline__ void static_for(F&& f) {
    static_for_impl(f, std::make_integer_sequence<int, N>{});
}


}  // namespace nbbgpu
