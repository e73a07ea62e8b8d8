// packed.cuh -- the throughput path: compact state kept BIT-SLICED in HBM.
//
// Layout ("packed", SURVEY.md 8(d) allows an internal bit-packing as long as the
// roofline is quoted against the 2 B/cell model AND the packed model):
//   * tile level q (even): a tile is a level-q sub-fractal, i.e. a WQ x WQ
//     (WQ = k^(q/2)) sub-rectangle of the compact array laid out like the level-q
//     compact array.  Tiles are numbered linearly over the coarse
//     compact array: t = Y * Wc + X.
//   * a group is 32 consecutive tiles; its record is Cp = round_up(C, 4) words of
//     32 bits, word i = local cell i (i = a * WQ + c), bit b = tile 32 g + b.
//     P[g * Cp + i].  k^r cells -> k^r / 8 bytes (+ < 1 group of padding).
//   * the boundary plane B[g * nSrc + m] duplicates the words of the nSrc local
//     cells that any neighbour tile reads (the halo sources).  It is tiny
//     (T r=20, q=8: 0.4 MB), written by the step that produces the state and read
//     by the next one -> halo gathers hit L2, never DRAM.
// The reference semantics (stencil.cpp:334-368) hold bit for bit: out-of-box and
// hole neighbours count 0 (the "zero word"), states are read from the front and
// written to the back buffer only.  Bytes <-> packed conversion kernels below
// give the reference's byte layout (cy*w + cx) back on download.
#pragma once

#include "rtc_compat.cuh"

#include "blocks.cuh"
#include "naive.cuh"
#include "tiled.cuh"

namespace nbbgpu {

constexpr int kPackedThreads = 256;
constexpr uint32_t kNoTile = 0xFFFFFFFFu;

// Programmatic dependent launch (PDL): a kernel launched with the programmatic
// stream-serialisation attribute may start while its predecessor drains; it must
// wait here before touching the predecessor's output (full completion + flush).
// A no-op when launched normally.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Record word of local cell (row a, column c).  Row-major, except for row
// micro-blocks of width ilv = BW (the carpet at WQ = 64, run-time specialised
// level-1 descriptors): the blocks are interleaved so that the 32 blocks of one
// consumer warp sit in 32 consecutive words for every cell position n: block
// b = a * (wq / BW) + c / BW, n = c % BW, word = ((b / 32) * BW + n) * 32 + b % 32
// (carpet: ((a / 4) * 8 + n) * 32 + (a % 4) * 8 + c / 8).  Lane = block then reads
// and writes conflict-free (row-major blocks start BW words apart: the carpet's
// shared accesses conflicted 4- to 8-way).  Records hold ceil(blocks / 32) * 32 * BW
// words (the padding blocks' words carry no cell).
__host__ __device__ __forceinline__ uint32_t rec_word(uint32_t ilv, uint32_t wq, uint32_t a, uint32_t c) {
    if (ilv) {
        const uint32_t bc = c / ilv, b = a * (wq / ilv) + bc, n = c - bc * ilv;
        return ((b >> 5) * ilv + n) * 32 + (b & 31);
    }
    return a * wq + c;
}
constexpr uint32_t kNoLoc = 0xFFFFFFFFu;  // loc[] of a record word that carries no cell

// interleaved records for a run-time specialised tag (jit_source specialises it)
template <class FT>
struct TagIlv { static constexpr bool v = false; };
template <class FT, int P, int WQ>
constexpr bool rec_ilv() { return (std::is_same<FT, CarpetTag>::value && P == 1 && WQ == 64) || (TagIlv<FT>::v && P == 1); }

struct PackedGeom {
    Frac f;
    uint32_t ilv;            // interleaved record layout (rec_word)
    uint32_t q, WQ, C, Cp;   // tile level, tile width, local cells, padded words per group
    uint32_t Cl;             // record words with a loc entry (C, or Cp for interleaved records)
    uint32_t Wc, Hc, L;      // coarse dims, coarse level r - q
    uint32_t T, NG;          // tiles, groups
    uint32_t sq;             // s^q (embedded tile side)
    uint64_t w;              // compact row stride (bytes of the reference layout)
};

// word of the 256-byte arrival-counter allocation that holds the peer-wait error flag
constexpr uint32_t kPeerErrWord = 16;

constexpr int kBtMaxChunks = 16;

// The per-(chunk, direction) masks of the transposed gather, passed by value: with
// the chunk count a compile-time constant every mask is a kernel-parameter operand
// (no shared entry list, no shared accumulators).
struct BtMasks {
    uint32_t m[kBtMaxChunks][8];
};

struct PackedStepParams {
    uint32_t C, Cp, SW;      // local cells, words per group record, words per smem stage
    uint32_t nH, nHp, nSrc;  // halo slots (padded to 4), boundary sources
    uint32_t T, NG, g0, g1;  // tiles, groups, owned groups [g0, g1)
    uint32_t lastmask;       // valid tile bits of group NG - 1
    uint32_t birth, survive;
    const void* nbr;         // [C][8] u16 (u32 when WIDE) byte offsets into the stage
    const uint32_t* slot;    // per halo slot: (D << 24) | (direction slot << 16) | boundary source m
    const uint32_t* ntab;    // [nD][T] linear neighbour tile or kNoTile
    const uint32_t* srcidx;  // per boundary source m: its local cell
    const uint32_t* btab;    // micro-block kernels: per block NEP stage byte offsets of its externals
    uint32_t* halo;          // [NG][nHp] halo words of the step (halo_words_kernel)
    int nD;                  // used directions (rows of ntab)
    uint16_t dfirst[9];      // slots of direction slot ds: [dfirst[ds], dfirst[ds + 1])
    // peer-memory halo transport: the halo kernel first waits until the peers have
    // pushed this step's boundary words (system-scope arrival counter >= target)
    const uint32_t* wait_cnt;
    uint32_t wait_target;
    // bounded wait: after wait_ns nanoseconds the waiter sets *wait_err, stops
    // waiting (this and every later step) and the host raises on synchronize
    uint32_t* wait_err;
    uint64_t wait_ns;
    // transposed halo gather (HMODE 6, halo_bt_regs_kernel): the boundary plane transposed per 32 slots,
    // Bt[(g * nHc + k) * 32 + b] bit i = boundary word 32k + i of tile 32g + b, and
    // per chunk k and direction slot d the mask of chunk k's slots in direction d
    const uint32_t* bt;
    const uint32_t* dmask;  // [nHc][8]
    // SPLIT = 2 (candy CTA pairs): the staged row window of half h is record words
    // [win0[h], win0[h] + win_words)
    uint32_t win0[2], win_words;
    // per-warp-store kernels on one GPU: instead of the boundary plane, write the
    // transposed plane Bt (layout of bnd_transpose_kernel) straight from the output
    // record -- no transpose kernel, no boundary-plane round trip (nullptr: write B)
    uint32_t* bt_out;
    // in-kernel Bt gather (HW halo warps with bt warps): the per-(chunk, direction) masks
    BtMasks btm;
    // peer-memory transport, fused push (triangle kernels, nSrc <= 32): the boundary
    // words peers need are stored into their planes as each group finishes
    // (push_off[local group] .. +1: entries m | peer << 16), and the grid's last CTA
    // bumps every peer's arrival counter once (push_done: CTA count of this launch)
    const uint32_t* push_off;
    const uint32_t* push_ent;
    uint32_t* const* push_bnd;  // per rank: its plane of the new front's parity
    uint32_t* const* push_cnt;  // per rank: its arrival counter
    unsigned* push_done;
    uint32_t push_mask;
};

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* a) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
    return v;
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// one thread per CTA spins on the arrival counter, then the CTA proceeds.  The
// wait is bounded by wall time (NBBGPU_PEER_TIMEOUT_S, default 600 s): host-side
// skew between ranks (seeding, checkpoints, GC) never kills the context; a peer
// that is really gone sets the handle's error word instead of trapping.
__device__ __forceinline__ void wait_peers(const PackedStepParams& p) {
    if (!p.wait_cnt) return;
    if (threadIdx.x == 0 && *(volatile uint32_t*)p.wait_err == 0) {
        const uint64_t t0 = globaltimer_ns();
        while ((int32_t)(ld_acquire_sys(p.wait_cnt) - p.wait_target) < 0) {
            __nanosleep(256);
            if (globaltimer_ns() - t0 > p.wait_ns) {  // a peer stopped stepping: flag, do not trap
                atomicExch(p.wait_err, 1u);
                break;
            }
        }
    }
    __syncthreads();
}

// Boundary-plane / halo loads: through the read-only path when the data was written
// by an earlier launch (NC), L2-coherent (ld.global.cg) when peers store into the
// plane over NVLink while the grid runs (p2p transport).
template <bool NC>
__device__ __forceinline__ uint32_t ld_bnd(const uint32_t* p) {
    if constexpr (NC) return __ldg(p);
    else return __ldcg(p);
}

// Halo words of the owned groups for one step: H[g][j] bit b = state of the source
// cell of slot j in the neighbour tile of tile 32 g + b (0 when there is none),
// read from the boundary plane of the front state.  Task wi = (group, 4 slots), one
// warp each; fully parallel, so the step never waits on a dependent gather.
template <bool NC, int SPW = 4>
__device__ __forceinline__ void halo4_task(const PackedStepParams& p, const uint32_t* bsrc, uint32_t* H,
                                           uint64_t wi, uint32_t lane) {
    const uint32_t spw = (p.nH + SPW - 1) / SPW, w32 = (uint32_t)wi;  // tasks < 2^32
    const uint32_t gi = w32 / spw;
    const uint32_t g = p.g0 + gi, j0 = (w32 - gi * spw) * SPW;
    const uint32_t t = g * 32 + lane;
    uint32_t t2[SPW], sl[SPW];
#pragma unroll
    for (int u = 0; u < SPW; ++u) {
        const uint32_t j = j0 + u;
        t2[u] = kNoTile;
        sl[u] = 0;
        if (j < p.nH) {
            sl[u] = __ldg(p.slot + j);
            if (t < p.T) t2[u] = __ldg(p.ntab + ((size_t)((sl[u] >> 16) & 0xFFu) * p.T + t));
        }
    }
    uint32_t v[SPW];
#pragma unroll
    for (int u = 0; u < SPW; ++u)
        v[u] = t2[u] != kNoTile ? ld_bnd<NC>(bsrc + (uint64_t)(t2[u] >> 5) * p.nSrc + (sl[u] & 0xFFFFu)) >> (t2[u] & 31)
                                : 0u;
    uint32_t mine = 0;
#pragma unroll
    for (int u = 0; u < SPW; ++u) {
        const uint32_t word = __ballot_sync(0xFFFFFFFFu, (v[u] & 1u) != 0);
        if (lane == (uint32_t)u) mine = word;
    }
    if (lane < SPW && j0 + lane < p.nHp) H[(uint64_t)g * p.nHp + j0 + lane] = j0 + lane < p.nH ? mine : 0u;
}

// 32 x 32 bit transpose across a warp: lane i holds row i (bit k = column k) ->
// lane k holds column k (bit i = row i).  Five shuffle-xor block swaps.
// XposeLane: the lane's keep masks and rotate amounts, built once before a loop of
// transposes (the bt warps of the H kernel: step kernel 116 -> 108 us at r=11; the
// same instruction count, the carpet kernel's schedule loses 6 % with it).
struct XposeLane {
    uint32_t K[5], sh[5];
    __device__ __forceinline__ explicit XposeLane(uint32_t lane) {
#pragma unroll
        for (int q = 0; q < 5; ++q) {
            const int j = 16 >> q;
            const uint32_t m = j == 16 ? 0x0000FFFFu : j == 8 ? 0x00FF00FFu : j == 4 ? 0x0F0F0F0Fu
                                                     : j == 2 ? 0x33333333u : 0x55555555u;
            const bool hi = (lane & j) != 0;
            K[q] = hi ? ~m : m;
            sh[q] = hi ? 32 - j : j;
        }
    }
};
__device__ __forceinline__ uint32_t warp_transpose32(uint32_t x, const XposeLane& X) {
#pragma unroll
    for (int q = 0; q < 5; ++q) {
        const uint32_t y = __shfl_xor_sync(0xFFFFFFFFu, x, 16 >> q);
        const uint32_t r = __funnelshift_l(y, y, X.sh[q]);
        x = (x & X.K[q]) | (r & ~X.K[q]);
    }
    return x;
}
__device__ __forceinline__ uint32_t warp_transpose32(uint32_t x, uint32_t lane) {
    // per stage: shuffle, rotate (left by j in the low-half lanes, right by j in the
    // high-half lanes: the wrapped-in bits fall under the mask) and a bit select
#pragma unroll
    for (int j = 16; j > 0; j >>= 1) {
        const uint32_t m = j == 16 ? 0x0000FFFFu : j == 8 ? 0x00FF00FFu : j == 4 ? 0x0F0F0F0Fu
                                                 : j == 2 ? 0x33333333u : 0x55555555u;
        const bool hi = (lane & j) != 0;
        const uint32_t y = __shfl_xor_sync(0xFFFFFFFFu, x, j);
        const uint32_t r = __funnelshift_l(y, y, hi ? 32 - j : j);
        const uint32_t K = hi ? ~m : m;
        x = (x & K) | (r & ~K);
    }
    return x;
}

// Large halos (carpet, H: ~200-330 slots per tile): one task per (group, used
// direction).  A direction with many slots (a tile edge) is gathered as a BIT
// PERMUTATION: for every source group G of the 32 neighbour tiles, lane = slot
// loads its boundary word B[G][m_slot] (one coalesced load), a warp transpose turns
// the 32 words into bit columns, lane = tile picks column (t2 & 31) with one
// shuffle, and a final transpose turns the tiles' bits back into the 32 halo
// words -- ~70 instructions per 32 slots (1-2 source groups) instead of a load +
// ballot per slot.  Directions with a few slots (corners) keep the ballot form.
// one used direction ds of group g (Hg = its halo words); t2 = lane's neighbour tile
template <bool NC, int NCH>
__device__ __forceinline__ void halo_dir(const PackedStepParams& p, const uint32_t* bsrc, uint32_t* Hg, int ds,
                                         uint32_t t2, uint32_t lane) {
    const uint32_t j_beg = p.dfirst[ds], j_end = p.dfirst[ds + 1];
    if (j_end - j_beg >= 8) {
        const bool valid = t2 != kNoTile;
        const uint32_t G2 = t2 >> 5, col_of_tile = t2 & 31;
        // the distinct source groups of the 32 neighbour tiles, first up to 4 in
        // registers (warp-uniform), so their boundary-word loads go out together
        uint32_t Gs[4] = {0u, 0u, 0u, 0u};
        int nG = 0;
        uint32_t remaining = __ballot_sync(0xFFFFFFFFu, valid);
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (remaining) {
                Gs[u] = __shfl_sync(0xFFFFFFFFu, G2, __ffs(remaining) - 1);
                remaining &= ~__ballot_sync(0xFFFFFFFFu, valid && G2 == Gs[u]);
                nG = u + 1;
            }
        // NCH chunks of 32 slots per round trip (more registers, fewer round trips)
        for (uint32_t jc = j_beg; jc < j_end; jc += 32 * NCH) {
            uint32_t mm[NCH], w[NCH][4];
#pragma unroll
            for (int c = 0; c < NCH; ++c) {
                const uint32_t j = jc + 32 * c + lane;
                mm[c] = j < j_end ? (__ldg(p.slot + j) & 0xFFFFu) : 0u;
            }
#pragma unroll
            for (int c = 0; c < NCH; ++c)
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    w[c][u] = (u < nG && jc + 32 * c + lane < j_end) ? ld_bnd<NC>(bsrc + (size_t)Gs[u] * p.nSrc + mm[c])
                                                                     : 0u;
#pragma unroll
            for (int c = 0; c < NCH; ++c) {
                const uint32_t j0 = jc + 32 * c, j = j0 + lane;  // lane = slot
                if (j0 >= j_end) break;
                uint32_t out = 0;  // lane = tile: bit i = slot j0 + i
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (u < nG) {
                        const uint32_t col = warp_transpose32(w[c][u], lane);  // lane c: bit i = bit c of word i
                        const uint32_t picked = __shfl_sync(0xFFFFFFFFu, col, col_of_tile);
                        if (valid && G2 == Gs[u]) out = picked;
                    }
                uint32_t rem = remaining;  // more than 4 source groups (rare): one pass each
                while (rem) {
                    const uint32_t G = __shfl_sync(0xFFFFFFFFu, G2, __ffs(rem) - 1);
                    const uint32_t members = __ballot_sync(0xFFFFFFFFu, valid && G2 == G);
                    const uint32_t wx = j < j_end ? ld_bnd<NC>(bsrc + (size_t)G * p.nSrc + mm[c]) : 0u;
                    const uint32_t col = warp_transpose32(wx, lane);
                    const uint32_t picked = __shfl_sync(0xFFFFFFFFu, col, col_of_tile);
                    if ((members >> lane) & 1u) out = picked;
                    rem &= ~members;
                }
                const uint32_t halo = warp_transpose32(out, lane);  // lane i: bit b = tile b, slot i
                if (j < j_end) Hg[j] = halo;
            }
        }
        return;
    }
    const bool valid = t2 != kNoTile;
    const uint32_t* base = bsrc + (size_t)(valid ? t2 >> 5 : 0) * p.nSrc;
    const uint32_t sh = t2 & 31;
    const uint32_t my_m = j_beg + lane < j_end ? (__ldg(p.slot + j_beg + lane) & 0xFFFFu) : 0u;
    uint32_t v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        const uint32_t m = __shfl_sync(0xFFFFFFFFu, my_m, u);
        v[u] = (j_beg + u < j_end && valid) ? ld_bnd<NC>(base + m) >> sh : 0u;
    }
    uint32_t mine = 0;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        const uint32_t word = __ballot_sync(0xFFFFFFFFu, (v[u] & 1u) != 0);
        if (lane == (uint32_t)u) mine = word;
    }
    if (j_beg + lane < j_end) Hg[j_beg + lane] = mine;
}

template <bool NC, int NCH = 1>
__device__ __forceinline__ void halo_wide_task(const PackedStepParams& p, const uint32_t* bsrc, uint32_t* H,
                                               uint32_t g, int ds, uint32_t lane) {
    const uint32_t t = g * 32 + lane;
    const uint32_t t2 = t < p.T ? __ldg(p.ntab + ((size_t)ds * p.T + t)) : kNoTile;  // lane = tile
    halo_dir<NC, NCH>(p, bsrc, H + (uint64_t)g * p.nHp, ds, t2, lane);
}

// one task per group: the neighbour tiles of every direction are loaded up front
// and each direction's loads go out in one round trip (fewer, longer tasks: for
// many groups -- H r=11 halo 0.127 -> 0.115 ms; with ~1K groups too few warps)
template <bool NC>
__device__ __forceinline__ void halo_group_task(const PackedStepParams& p, const uint32_t* bsrc, uint32_t* H,
                                                uint32_t g, uint32_t lane) {
    const uint32_t t = g * 32 + lane;
    const bool in = t < p.T;
    // directions in a rolled loop (small code: the unrolled form stalled on the
    // instruction cache) with the next direction's neighbour tile prefetched
    uint32_t t2 = in ? __ldg(p.ntab + t) : kNoTile;
#pragma unroll 1
    for (int d = 0; d < p.nD; ++d) {
        const uint32_t t2n = (d + 1 < p.nD && in) ? __ldg(p.ntab + ((size_t)(d + 1) * p.T + t)) : kNoTile;
        halo_dir<NC, 3>(p, bsrc, H + (uint64_t)g * p.nHp, d, t2, lane);
        t2 = t2n;
    }
}

// large halos -> tasks per (group, direction) with transposed edge gathers; small
// halos (triangle, Vicsek: 4-8 slots) -> tasks of 4 slots, lane = tile
__host__ __device__ __forceinline__ bool halo_use_wide(uint32_t nH, uint32_t groups) {
    (void)groups;
    return nH > 32;
}
__host__ __device__ __forceinline__ uint64_t halo_tasks(uint32_t nH, uint32_t groups, int nD) {
    return halo_use_wide(nH, groups) ? (uint64_t)groups * (uint32_t)nD : (uint64_t)groups * ((nH + 3) / 4);
}

template <bool NC>
__device__ __forceinline__ void halo_task(const PackedStepParams& p, const uint32_t* bsrc, uint32_t* H,
                                          uint64_t wi, uint32_t lane) {
    if (halo_use_wide(p.nH, p.g1 - p.g0))
        halo_wide_task<NC>(p, bsrc, H, p.g0 + (uint32_t)(wi / (uint32_t)p.nD), (int)(wi % (uint32_t)p.nD), lane);
    else halo4_task<NC>(p, bsrc, H, wi, lane);
}

// Boundary plane -> Bt (see PackedStepParams::bt): warp per (group, 32 slots), one
// coalesced load, a warp transpose, one coalesced store.
// CPB chunks per warp task (4 for many groups: fewer, longer tasks; 1 otherwise)
template <int CPB>
__global__ void bnd_transpose_kernel(const PackedStepParams p, const uint32_t* __restrict__ bsrc,
                                     uint32_t* __restrict__ bt) {
    const uint32_t lane = threadIdx.x & 31;
    pdl_wait();     // bsrc comes from the previous step kernel
    pdl_trigger();  // the halo kernel may launch and run its prologue
    const uint32_t nHc = (p.nH + 31) / 32, ntk = (nHc + CPB - 1) / CPB;
    const uint64_t nw = (uint64_t)(p.g1 - p.g0) * ntk;
    for (uint64_t wi = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; wi < nw;
         wi += ((uint64_t)gridDim.x * blockDim.x) >> 5) {
        const uint32_t w32 = (uint32_t)wi, gi = w32 / ntk, g = p.g0 + gi;
        if constexpr (CPB == 1) {
            const uint32_t k = w32 - gi * ntk, j = k * 32 + lane;
            const uint32_t w = j < p.nH ? __ldg(bsrc + (uint64_t)g * p.nSrc + j) : 0u;
            bt[((uint64_t)g * nHc + k) * 32 + lane] = warp_transpose32(w, lane);
            continue;
        }
        const uint32_t cpb = CPB;
        const uint32_t kend = min(nHc, (w32 - gi * ntk + 1) * cpb);
        for (uint32_t k0 = (w32 - gi * ntk) * cpb; k0 < kend; k0 += 4) {  // 4 chunks per round trip
            uint32_t w[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t j = (k0 + u) * 32 + lane;
                w[u] = (k0 + u < kend && j < p.nH) ? __ldg(bsrc + (uint64_t)g * p.nSrc + j) : 0u;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (k0 + u < kend) bt[((uint64_t)g * nHc + k0 + u) * 32 + lane] = warp_transpose32(w[u], lane);
        }
    }
}

// Halo words of group g from Bt: lane = tile b gathers, per chunk k of 32 slots,
// the chunk's bits of its neighbour tile in every direction present in the chunk
// (one load each, masked), and one transpose turns lane b's bits into the 32 halo
// words (no per-source-group passes: the slots of a direction are bits of ONE word
// of the neighbour tile).
// Transposed gather, register form (one warp per group, grid-stride): lane = tile b
// holds the 8 neighbour tiles (the next group's are loaded while this group's Bt
// words are in flight); per direction one address and, per chunk the direction
// has slots in, one predicated load + AND/OR into the chunk's register accumulator;
// then NHC transposes.  ~300 instructions per group instead of ~1000 for round 2's
// (chunk, direction) entry list in shared memory with shared accumulators (removed).
// NZ (NHC <= 8): bit 8k + d set iff chunk k has slots in direction d -- the plan's
// pattern, compiled in at run time (jit.inc) so the absent (chunk, direction) pairs
// cost nothing; all ones: every pair tested against its mask at run time.
template <int NHC, unsigned long long NZ = ~0ull>
__global__ void __launch_bounds__(256) halo_bt_regs_kernel(const PackedStepParams p, const BtMasks M,
                                                           uint32_t* __restrict__ H) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t gstride = (uint32_t)(((uint64_t)gridDim.x * blockDim.x) >> 5);
    uint32_t g = p.g0 + (uint32_t)((blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5);
    uint32_t t2n[8];
    auto fetch = [&](uint32_t gg) {
        const uint32_t t = gg * 32 + lane;
        const bool in = gg < p.g1 && t < p.T;
#pragma unroll
        for (int d = 0; d < 8; ++d) t2n[d] = (d < p.nD && in) ? __ldg(p.ntab + ((size_t)d * p.T + t)) : kNoTile;
    };
    fetch(g);  // (static table: before the wait for the previous step kernel)
    pdl_wait();
    pdl_trigger();
    const XposeLane X(lane);
    for (; g < p.g1; g += gstride) {
        uint32_t t2[8];
#pragma unroll
        for (int d = 0; d < 8; ++d) t2[d] = t2n[d];
        fetch(g + gstride);
        uint32_t acc[NHC];
#pragma unroll
        for (int k = 0; k < NHC; ++k) acc[k] = 0u;
#pragma unroll
        for (int d = 0; d < 8; ++d) {
            const bool ok = t2[d] != kNoTile;
            const uint32_t* b = p.bt + (uint64_t)(t2[d] >> 5) * (NHC * 32u) + (t2[d] & 31u);
            uint32_t v[NHC];
#pragma unroll
            for (int k = 0; k < NHC; ++k) {
                const bool pair = NHC > 8 || ((NZ >> (8 * k + d)) & 1ull);  // (compile-time)
                v[k] = (pair && ok && M.m[k][d] != 0u) ? __ldcg(b + 32 * k) : 0u;
            }
#pragma unroll
            for (int k = 0; k < NHC; ++k)
                if (NHC > 8 || ((NZ >> (8 * k + d)) & 1ull)) acc[k] |= v[k] & M.m[k][d];
        }
        uint32_t* Hg = H + (uint64_t)g * p.nHp;
#pragma unroll
        for (int k = 0; k < NHC; ++k) {
            const uint32_t out = warp_transpose32(acc[k], X);  // lane i: bit b = slot 32k + i of tile b
            if (k * 32 + lane < p.nH) Hg[k * 32 + lane] = out;
        }
    }
}

// (group, chunk) tasks for few groups: the chunk's directions only, more warps
__device__ __forceinline__ void halo_bt_chunk_task(const PackedStepParams& p, uint32_t* H, uint32_t g, uint32_t k,
                                                   uint32_t lane) {
    const uint32_t t = g * 32 + lane;
    const bool in = t < p.T;
    const uint32_t nHc = (p.nH + 31) / 32;
    uint32_t t2[8], dm[8];
#pragma unroll
    for (int d = 0; d < 8; ++d) {
        dm[d] = __ldg(p.dmask + k * 8 + d);
        t2[d] = (dm[d] && in) ? __ldg(p.ntab + ((size_t)d * p.T + t)) : kNoTile;
    }
    uint32_t word = 0;
#pragma unroll
    for (int d = 0; d < 8; ++d)
        if (t2[d] != kNoTile) word |= __ldcg(p.bt + ((uint64_t)(t2[d] >> 5) * nHc + k) * 32 + (t2[d] & 31)) & dm[d];
    const uint32_t out = warp_transpose32(word, lane);
    if (k * 32 + lane < p.nH) H[(uint64_t)g * p.nHp + k * 32 + lane] = out;
}

// HMODE is compile-time so the small-halo variant keeps its 30 registers (full
// occupancy: this kernel is latency-bound).  0: tasks of SPW slots (small halos),
// 1: (group, direction) tasks, 2: group tasks (all directions of a group),
// 3: (group, direction) tasks with 3 chunks of loads per round trip (few groups)
template <int HMODE, int SPW = 4, bool NC = true>
__global__ void halo_words_kernel(const PackedStepParams p, const uint32_t* __restrict__ bsrc,
                                  uint32_t* __restrict__ H) {
    const uint32_t lane = threadIdx.x & 31;
    if constexpr (HMODE != 8) {
        pdl_wait();     // bsrc comes from the previous step kernel
        wait_peers(p);  // ... and, with the peer-memory transport, from the peers' pushes
        pdl_trigger();  // the step kernel may launch and run its prologue
    }
    const uint64_t nw = HMODE == 6 ? (uint64_t)(p.g1 - p.g0) * ((p.nH + 31) / 32)
                      : HMODE == 2 ? (uint64_t)(p.g1 - p.g0)
                      : HMODE == 1 || HMODE == 3 ? (uint64_t)(p.g1 - p.g0) * (uint32_t)p.nD
                                   : (uint64_t)(p.g1 - p.g0) * ((p.nH + SPW - 1) / SPW);
    if constexpr (HMODE == 8) {
        // small halos (nH <= 8), warp per group, lean: the slot table is hoisted out
        // of the task loop (uniform), 32-bit offsets, 8 + 8 independent loads and 8
        // ballots per group (~110 instructions instead of ~440 for 4-slot tasks)
        uint32_t noff[8], moff[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const uint32_t sl = (uint32_t)j < p.nH ? __ldg(p.slot + j) : 0u;
            noff[j] = ((sl >> 16) & 0xFFu) * p.T;
            moff[j] = sl & 0xFFFFu;
        }
        // the neighbour tiles (static ntab) of this warp's first group are loaded
        // before the wait for the previous step kernel (PDL: overlaps its tail), and
        // each next group's while the current group's boundary words are in flight
        const uint32_t gstride = (uint32_t)(((uint64_t)gridDim.x * blockDim.x) >> 5);
        uint32_t g = p.g0 + (uint32_t)((blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5);
        uint32_t t2n[8];
        auto fetch = [&](uint32_t gg) {
            const uint32_t t = gg * 32 + lane;
            const bool in = gg < p.g1 && t < p.T;
#pragma unroll
            for (int j = 0; j < 8; ++j) t2n[j] = ((uint32_t)j < p.nH && in) ? __ldg(p.ntab + noff[j] + t) : kNoTile;
        };
        fetch(g);
        pdl_wait();     // bsrc comes from the previous step kernel
        wait_peers(p);  // ... and, with the peer-memory transport, from the peers' pushes
        pdl_trigger();  // the step kernel may launch and run its prologue
        for (; g < p.g1; g += gstride) {
            uint32_t t2[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) t2[j] = t2n[j];
            fetch(g + gstride);
            uint32_t v[8];
#pragma unroll
            for (int j = 0; j < 8; ++j)
                v[j] = t2[j] != kNoTile ? ld_bnd<NC>(bsrc + (t2[j] >> 5) * p.nSrc + moff[j]) >> (t2[j] & 31) : 0u;
            uint32_t mine = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const uint32_t word = __ballot_sync(0xFFFFFFFFu, (v[j] & 1u) != 0);
                if (lane == (uint32_t)j) mine = word;
            }
            if (lane < p.nHp) H[(uint64_t)g * p.nHp + lane] = lane < p.nH ? mine : 0u;
        }
        return;
    }
    if constexpr (HMODE != 8)
    for (uint64_t wi = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; wi < nw;
         wi += ((uint64_t)gridDim.x * blockDim.x) >> 5) {
        if constexpr (HMODE == 6) {
            const uint32_t nHc = (p.nH + 31) / 32, w32 = (uint32_t)wi, gi = w32 / nHc;
            halo_bt_chunk_task(p, H, p.g0 + gi, w32 - gi * nHc, lane);
        } else if constexpr (HMODE == 2) {
            halo_group_task<NC>(p, bsrc, H, p.g0 + (uint32_t)wi, lane);
        } else if constexpr (HMODE == 1 || HMODE == 3) {
            const uint32_t w32 = (uint32_t)wi, gi = w32 / (uint32_t)p.nD;
            halo_wide_task<NC, HMODE == 3 ? 3 : 1>(p, bsrc, H, p.g0 + gi, (int)(w32 - gi * (uint32_t)p.nD), lane);
        } else {
            halo4_task<NC, SPW>(p, bsrc, H, wi, lane);
        }
    }
}

// ---- mbarrier + 1-D bulk copy (TMA engine) -----------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t a, uint32_t tx) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
    uint32_t done;
    do {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done) : "r"(a), "r"(parity) : "memory");
    } while (!done);
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t mbar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(mbar) : "memory");
}

// The bit-sliced Life step of local cell i of a group staged at Sb (bytes):
// 8 (or 4) neighbour words through the tile's neighbour table, a 14-LOP adder and
// the rule (tiled.cuh).  Bit b of the result = next state of tile b's cell i.
template <bool CONWAY, int DEG, bool WIDE>
__device__ __forceinline__ uint32_t cell_word(const uint8_t* Sb, const void* nbr, uint32_t i,
                                              const uint32_t (&KB)[9], const uint32_t (&KS)[9]) {
    uint32_t o[8];
    if (!WIDE) {
        const uint4 e = __ldg(reinterpret_cast<const uint4*>(nbr) + i);
        o[0] = e.x & 0xFFFFu; o[1] = e.x >> 16; o[2] = e.y & 0xFFFFu; o[3] = e.y >> 16;
        o[4] = e.z & 0xFFFFu; o[5] = e.z >> 16; o[6] = e.w & 0xFFFFu; o[7] = e.w >> 16;
    } else {
        const uint4 e0 = __ldg(reinterpret_cast<const uint4*>(nbr) + 2 * i);
        o[0] = e0.x; o[1] = e0.y; o[2] = e0.z; o[3] = e0.w;
        if (DEG == 8) {
            const uint4 e1 = __ldg(reinterpret_cast<const uint4*>(nbr) + 2 * i + 1);
            o[4] = e1.x; o[5] = e1.y; o[6] = e1.z; o[7] = e1.w;
        } else {
            o[4] = o[5] = o[6] = o[7] = 0;
        }
    }
    uint32_t x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = j < DEG ? *reinterpret_cast<const uint32_t*>(Sb + o[j]) : 0u;
    const uint32_t own = *reinterpret_cast<const uint32_t*>(Sb + 4 * i);
    const Count4 cnt = count8(x[0], x[1], x[2], x[3], x[4], x[5], x[6], x[7]);
    return apply_rule_bits<CONWAY>(cnt, own, KB, KS);
}

template <class FT, int P, int WQ>
struct BlockGeom {
    static constexpr int NBLK = (WQ / Wiring<FT, P>::BW) * (WQ / Wiring<FT, P>::BH);
    static constexpr uint32_t TAB_BYTES = (uint32_t)NBLK * Wiring<FT, P>::NEP * 4;
};
template <int P, int WQ>
struct BlockGeom<void, P, WQ> {
    static constexpr int NBLK = 0;
    static constexpr uint32_t TAB_BYTES = 0;
};

// Generic (table-driven) program: any descriptor, any tile level.
template <bool CONWAY, int DEG, bool WIDE>
__global__ void __launch_bounds__(kPackedThreads)
step_packed_kernel(const PackedStepParams p, const uint32_t* __restrict__ src, uint32_t* __restrict__ dst,
                   const uint32_t* __restrict__ bsrc, uint32_t* __restrict__ bdst) {
    extern __shared__ __align__(16) uint8_t sm[];
    const uint32_t mb = smem_u32(sm);  // two mbarriers at [0, 16)
    constexpr int NT = kPackedThreads;
    uint8_t* st = sm + 16;
    const uint32_t stage_bytes = p.SW * 4;
    const int tid = threadIdx.x;

    uint32_t KB[9], KS[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) {
        KB[i] = ((p.birth >> i) & 1u) ? 0xFFFFFFFFu : 0u;
        KS[i] = ((p.survive >> i) & 1u) ? 0xFFFFFFFFu : 0u;
    }
    if (tid == 0) {
        mbar_init(mb, 1);
        mbar_init(mb + 8, 1);
        mbar_fence_init();
    }
    if (tid < 2) reinterpret_cast<uint32_t*>(st + tid * stage_bytes)[p.Cp + p.nHp] = 0u;  // absent
    __syncthreads();

    const uint32_t rec_bytes = p.Cp * 4, halo_bytes = p.nHp * 4;
    // group record + its halo words into stage s (one mbarrier, two bulk copies)
    auto load_group = [&](uint32_t gg, int s) {
        const uint32_t bar = mb + 8 * s;
        const uint32_t dst_s = smem_u32(st + s * stage_bytes);
        mbar_expect_tx(bar, rec_bytes + halo_bytes);
        bulk_g2s(dst_s, src + (uint64_t)gg * p.Cp, rec_bytes, bar);
        if (halo_bytes) bulk_g2s(dst_s + rec_bytes, p.halo + (uint64_t)gg * p.nHp, halo_bytes, bar);
    };
    uint32_t g = p.g0 + blockIdx.x;
    if (tid == 0 && g < p.g1) load_group(g, 0);
    uint32_t phase = 0;
    for (int s = 0; g < p.g1; g += gridDim.x, s ^= 1) {
        const uint32_t gn = g + gridDim.x;
        if (tid == 0 && gn < p.g1) load_group(gn, s ^ 1);  // stage s^1 released by the last __syncthreads
        const uint8_t* Sb = st + s * stage_bytes;
        mbar_wait(mb + 8 * s, (phase >> s) & 1u);  // record + halo words landed (TMA)
        phase ^= 1u << s;
        // ---- program: every local cell, straight to HBM -------------------------------
        const uint32_t vmask = g == p.NG - 1 ? p.lastmask : 0xFFFFFFFFu;
        uint32_t* D = dst + (uint64_t)g * p.Cp;
#pragma unroll 2
        for (uint32_t i = tid; i < p.C; i += NT)
            D[i] = cell_word<CONWAY, DEG, WIDE>(Sb, p.nbr, i, KB, KS) & vmask;
        // boundary plane of the new state (a few words per group: recomputed)
        for (uint32_t m = tid; m < p.nSrc; m += NT)
            bdst[(uint64_t)g * p.nSrc + m] = cell_word<CONWAY, DEG, WIDE>(Sb, p.nbr, __ldg(p.srcidx + m), KB, KS) & vmask;
        __syncthreads();
    }
}

// Static coarse-neighbour table over LINEAR tile indices (setup, once per plan):
// out[ds * T + t] = linear index of the neighbour tile of t in direction dlist[ds]
// (the carry walk of tiled.cuh, exactly nu(lambda(tile) + offset) at level L), or
// kNoTile for a hole / outside the box.
template <int K, int S>
__global__ void build_ntab_linear_kernel(Frac f, int L, uint32_t Wc, uint32_t Hc, int nD, int8_t d0, int8_t d1,
                                         int8_t d2, int8_t d3, int8_t d4, int8_t d5, int8_t d6, int8_t d7,
                                         uint32_t* __restrict__ out) {
    const int8_t dl[8] = {d0, d1, d2, d3, d4, d5, d6, d7};
    const uint64_t n = (uint64_t)Wc * Hc;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t X = (uint32_t)(i % Wc), Y = (uint32_t)(i / Wc);
        for (int ds = 0; ds < nD; ++ds) {
            const int D = dl[ds];
            uint32_t X2, Y2, v = kNoTile;
            if (coarse_neighbor<K, S>(f, L, X, Y, D % 3 - 1, D / 3 - 1, X2, Y2)) v = Y2 * Wc + X2;
            out[(uint64_t)ds * n + i] = v;
        }
    }
}

__device__ __forceinline__ void mbar_arrive(uint32_t a) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, uint32_t src, uint32_t bytes);
// the record streams of the ws3 kernel (an L2 evict-first hint was measured and dropped: +-2 %)
__device__ __forceinline__ void rec_g2s(const PackedStepParams&, uint32_t dst, const void* src, uint32_t bytes,
                                       uint32_t mbar) {
    bulk_g2s(dst, src, bytes, mbar);
}
__device__ __forceinline__ void rec_s2g(const PackedStepParams&, void* dst, uint32_t src, uint32_t bytes) {
    bulk_s2g(dst, src, bytes);
}
__device__ __forceinline__ void bulk_s2g(void* dst, uint32_t src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void bulk_wait_read_all() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// Micro-block step with the external offsets held in registers (toff) and the
// results written to a shared-memory output record (Do).
template <class FT, int P, int WQ, bool CONWAY, int DEG>
__device__ __forceinline__ void block_words_r(const uint8_t* Sb, const uint32_t (&toff)[Wiring<FT, P>::NEP],
                                              uint32_t blk, uint32_t* Do, uint32_t vmask, const uint32_t (&KB)[9],
                                              const uint32_t (&KS)[9], uint32_t own_shift = 0) {
    using W = Wiring<FT, P>;
    constexpr int BW = W::BW, BH = W::BH, NB = W::NB, NEP = W::NEP;
    constexpr int BPR = WQ / BW;
    const uint32_t by = blk / BPR, bx = blk - by * BPR;
    const uint32_t base = by * (BH * WQ) + bx * BW;
    const uint32_t* Sw = reinterpret_cast<const uint32_t*>(Sb) + (base - own_shift);  // (row window)
    // row blocks with BW % 4 == 0 (carpet: BW = 8, candy: 12): 16-byte loads and
    // stores -- lanes sit BW words apart, so single-word accesses conflict BW/gcd-way
    // interleaved carpet records (rec_word): cell n of block blk at word
    // (blk / 32 * 8 + n) * 32 + blk % 32
    constexpr bool ILV = rec_ilv<FT, P, WQ>();
    constexpr bool VEC = BH == 1 && BW % 4 == 0 && !ILV;
    uint32_t own[NB], ext[NEP];
    if constexpr (ILV) {
        const uint32_t* Sq = reinterpret_cast<const uint32_t*>(Sb) + (blk >> 5) * (NB * 32) + (blk & 31);
        static_for<NB>([&](auto n) {
            constexpr int N = decltype(n)::value;
            own[N] = Sq[N * 32];
        });
    } else if constexpr (VEC) {
        static_for<NB / 4>([&](auto q) {
            constexpr int Q = decltype(q)::value;
            const uint4 v = reinterpret_cast<const uint4*>(Sw)[Q];
            own[4 * Q] = v.x; own[4 * Q + 1] = v.y; own[4 * Q + 2] = v.z; own[4 * Q + 3] = v.w;
        });
    } else {
        static_for<NB>([&](auto n) {
            constexpr int N = decltype(n)::value;
            own[N] = Sw[(N / BW) * WQ + N % BW];
        });
    }
    static_for<NEP>([&](auto e) {
        constexpr int E = decltype(e)::value;
        ext[E] = *reinterpret_cast<const uint32_t*>(Sb + toff[E]);
    });
    uint32_t* Dw = ILV ? Do + (blk >> 5) * (NB * 32) + (blk & 31) : Do + base;
    uint32_t res[VEC ? 4 : 1];
    static_for<NB>([&](auto n) {
        constexpr int N = decltype(n)::value;
        uint32_t x[8];
        static_for<8>([&](auto j) {
            constexpr int J = decltype(j)::value;
            constexpr int SJ = W::d.src[N][J];
            if constexpr (J >= DEG || SJ == kWireAbsent) x[J] = 0u;
            else if constexpr (SJ >= 0) x[J] = own[SJ];
            else x[J] = ext[-SJ - 2];
        });
        const Count4 cnt = count8(x[0], x[1], x[2], x[3], x[4], x[5], x[6], x[7]);
        const uint32_t r = apply_rule_bits<CONWAY>(cnt, own[N], KB, KS) & vmask;
        if constexpr (ILV) {
            Dw[N * 32] = r;
        } else if constexpr (VEC) {
            res[N % 4] = r;
            if constexpr (N % 4 == 3)
                reinterpret_cast<uint4*>(Dw)[N / 4] = make_uint4(res[0], res[1], res[2], res[3]);
        } else {
            Dw[(N / BW) * WQ + N % BW] = r;
        }
    });
}

// Stage size in words known at compile time for the built-in tile shapes (stage:
// Cp record words | nHp halo words | zero word, + 3; build_packed_plan, which the
// launcher checks against): lets the ws3 consumers address every stage of their set
// with immediates (block_words_c).  0: run-time stage size.
template <class FT, int WQ>
struct StageWordsCT { static constexpr int v = 0; };
#ifndef NBB_NO_SWC  // (A/B builds: run-time stage size everywhere)
template <> struct StageWordsCT<HTag, 49> { static constexpr int v = 2608; };        // C 2401, nH 198
template <> struct StageWordsCT<CarpetTag, 64> { static constexpr int v = 4428; };   // C 4096, nH 328
#endif
// (measured, not enabled: T q=8 r=20 133.2 -> 134.8 us, Vicsek r=12/13 neutral; the
// row-block kernels gain: H r=11 114.1 -> 108.5 us, carpet r=11 432 -> 412 us)

// first own word of block blk in the record (block_words_r's Sw / Sq base)
template <class FT, int P, int WQ>
__device__ __forceinline__ uint32_t block_own_base(uint32_t blk) {
    using W = Wiring<FT, P>;
    constexpr int BW = W::BW, BH = W::BH, NB = W::NB;
    constexpr bool ILV = rec_ilv<FT, P, WQ>();
    if constexpr (ILV) return (blk >> 5) * (NB * 32) + (blk & 31);
    constexpr int BPR = WQ / BW;
    const uint32_t by = blk / BPR, bx = blk - by * BPR;
    return by * (BH * WQ) + bx * BW;
}

// block_words_r with every stage address = the lane's set-relative byte offset +
// an immediate: tS[E] = external E, own_off = the block's first own word (bytes,
// both relative to stage 0 of the set), SOFF = this stage's offset from it.
template <class FT, int P, int WQ, bool CONWAY, int DEG, int SOFF>
__device__ __forceinline__ void block_words_c(const uint8_t* st, const uint32_t (&tS)[Wiring<FT, P>::NEP],
                                              uint32_t own_off, uint32_t blk, uint32_t* Do, uint32_t vmask,
                                              const uint32_t (&KB)[9], const uint32_t (&KS)[9]) {
    using W = Wiring<FT, P>;
    constexpr int BW = W::BW, BH = W::BH, NB = W::NB, NEP = W::NEP;
    constexpr bool ILV = rec_ilv<FT, P, WQ>();
    constexpr bool VEC = BH == 1 && BW % 4 == 0 && !ILV;
    const uint8_t* Sb = st + SOFF;
    uint32_t own[NB], ext[NEP];
    static_for<NB>([&](auto n) {
        constexpr int N = decltype(n)::value;
        constexpr int OW = ILV ? N * 32 : (N / BW) * WQ + N % BW;  // word offset from the block base
        if constexpr (VEC) {
            if constexpr (N % 4 == 0) {
                const uint4 v = *reinterpret_cast<const uint4*>(Sb + own_off + 4 * OW);
                own[N] = v.x; own[N + 1] = v.y; own[N + 2] = v.z; own[N + 3] = v.w;
            }
        } else {
            own[N] = *reinterpret_cast<const uint32_t*>(Sb + own_off + 4 * OW);
        }
    });
    static_for<NEP>([&](auto e) {
        constexpr int E = decltype(e)::value;
        ext[E] = *reinterpret_cast<const uint32_t*>(Sb + tS[E]);
    });
    const uint32_t base = block_own_base<FT, P, WQ>(blk);
    uint32_t* Dw = Do + base;
    uint32_t res[VEC ? 4 : 1];
    static_for<NB>([&](auto n) {
        constexpr int N = decltype(n)::value;
        uint32_t x[8];
        static_for<8>([&](auto j) {
            constexpr int J = decltype(j)::value;
            constexpr int SJ = W::d.src[N][J];
            if constexpr (J >= DEG || SJ == kWireAbsent) x[J] = 0u;
            else if constexpr (SJ >= 0) x[J] = own[SJ];
            else x[J] = ext[-SJ - 2];
        });
        const Count4 cnt = count8(x[0], x[1], x[2], x[3], x[4], x[5], x[6], x[7]);
        const uint32_t r = apply_rule_bits<CONWAY>(cnt, own[N], KB, KS) & vmask;
        if constexpr (ILV) {
            Dw[N * 32] = r;
        } else if constexpr (VEC) {
            res[N % 4] = r;
            if constexpr (N % 4 == 3)
                reinterpret_cast<uint4*>(Dw)[N / 4] = make_uint4(res[0], res[1], res[2], res[3]);
        } else {
            Dw[(N / BW) * WQ + N % BW] = r;
        }
    });
}

// Persistent, warp-specialised micro-block step (one CTA per SM), TMA in and out:
//   producer warp : group record + its halo words (halo_words_kernel output) ->
//                   NS-stage input ring (cp.async.bulk, full barriers carry the
//                   bytes; empty barriers free a stage);
//   NGRP x NCHUNK consumer warps : warp (k, c) evaluates the 32 micro-blocks of
//                   chunk c of every group i = k (mod NGRP); its blocks never change,
//                   so their external offsets live in registers for the whole kernel;
//                   results go to an NO-deep shared output ring;
//   storer warp   : one cp.async.bulk shared->global store per finished group.
// No CTA-wide barrier in the loop; stores leave as whole 26 KB records.
// SPLIT > 1 (groups with more chunks than a CTA has warps, e.g. candy: 54): SPLIT
// consecutive CTAs share a group, CTA half h loading the whole record but computing
// and storing only its 1/SPLIT of the micro-block rows (a contiguous slice of the
// output record).
template <class FT, int P, int WQ, int SPLIT>
struct WsGeom {
    static constexpr int NBLK = BlockGeom<FT, P, WQ>::NBLK / SPLIT;  // blocks per CTA
    static constexpr int NCHUNK = (NBLK + 31) / 32;
    static constexpr int ROWS = WQ / SPLIT;                          // cell rows per CTA
    static_assert(SPLIT == 1 || (Wiring<FT, P>::BH == 1 && WQ % SPLIT == 0), "SPLIT needs P = 1 row blocks");
};

// HW > 0: HW extra warps gather each group's halo words in-kernel into the stage and
// arrive on its full barrier -- no separate halo kernel.  Without bt warps (<= 8
// slots: triangle, Vicsek): ntab rows + boundary-plane words and ballots, the next
// group's neighbour tiles prefetched and the loads issued before the stage wait.
// With bt warps (HG: carpet, small H): the register-form transposed gather from the
// previous front's Bt plane (p.bt; this launch writes the other parity, p.bt_out).
// BTW > 0 (per-warp-store kernels on one GPU, p.bt_out): BTW extra warps write the
// transposed boundary plane Bt (bnd_transpose_kernel's layout) from each finished
// output record -- no transpose kernel and no boundary-plane round trip per step.
// PUSH (peer-memory transport, triangle): the boundary words peers need are stored
// into their planes here and the grid's last CTA signals them (p.push_*).
template <bool CONWAY, int DEG, bool WIDE, class FT, int P, int WQ, int NGRP, int NS, int NO, int SPLIT = 1,
          int HW = 0, int BTW = 0, bool PUSH = false>
__global__ void __launch_bounds__((WsGeom<FT, P, WQ, SPLIT>::NCHUNK * NGRP + 2 + HW + BTW) * 32, 1)
step_packed_ws3_kernel(const PackedStepParams p, const uint32_t* __restrict__ src, uint32_t* __restrict__ dst,
                       const uint32_t* __restrict__ bsrc, uint32_t* __restrict__ bdst) {
    using W = Wiring<FT, P>;
    using WG = WsGeom<FT, P, WQ, SPLIT>;
    constexpr int NBLK = WG::NBLK;
    constexpr int NCHUNK = WG::NCHUNK;
    constexpr int NCW = NCHUNK * NGRP;
    constexpr int NEP = W::NEP;
    // boundary words copied from the output record by the storer (large boundaries)
    // or recomputed by consumer warp 0 (triangle, Vicsek: a few words per group)
    constexpr bool BST = !std::is_same<FT, TriangleTag>::value && !std::is_same<FT, VicsekTag>::value;
    // PWS: row micro-blocks (BH = 1) give every consumer warp a contiguous slice of
    // the output record; each warp bulk-stores its own slice and copies the boundary
    // words inside it (p.srcidx + nSrc = the sources sorted by cell) -- no storer
    // round trip per group
    constexpr bool PWS = BST && W::BH == 1;
    static_assert(!PWS || NO % NGRP == 0, "per-warp stores reuse an output buffer every NO / NGRP groups");
    // Every stage must belong to ONE group set.  mbarrier waits are by phase parity:
    // a set waiting for use u + 1 of a stage whose use u (another set's group) has
    // not landed yet would see the parity of use u - 1 and pass early -- rare (the
    // TMA of use u completing after later ones), but it corrupted one warp's slice of
    // one group about once per 10^4 group-steps with NGRP 3 / NS 7.  With NS a
    // multiple of NGRP, stage s serves groups i = s (mod NS), all of set s % NGRP,
    // which that set consumes in order, so use u has completed before it waits for u + 1.
    static_assert(NS % NGRP == 0, "stages are partitioned over the group sets");
    // (the in-kernel halo warps wait on the stages' empty barriers the same way: each
    // stage served by one halo warp, or one set whose consumers finish groups in order
    // AND at most NS halo warps: a halo warp reaching group g has seen group g - HW - NS
    // consumed, so the stage's use before last (g - 2 NS) is complete and the parity
    // wait for g - NS cannot pass early; with HW > NS it could -- the warp would fill a
    // stage still being read and arrive on the wrong phase of its full barrier)
    static_assert(HW == 0 || NS % (HW > 0 ? HW : 1) == 0 || (NGRP == 1 && HW <= NS),
                  "stages are partitioned over the halo warps");
    extern __shared__ __align__(16) uint8_t sm[];
    const uint32_t full0 = smem_u32(sm), empty0 = full0 + 8 * NS;
    const uint32_t ofull0 = empty0 + 8 * NS, oempty0 = ofull0 + 8 * NO;
    unsigned& push_warps_done = *reinterpret_cast<unsigned*>(sm + 16 * (NS + NO));  // fused peer push
    uint8_t* st = sm + 16 * (NS + NO) + 16;
    // SPLIT = 2: each CTA stages only the rows its blocks read (the row window
    // p.win0[half] + [0, p.win_words) of the record; the plan rebases the block
    // tables to it)
    const uint32_t win_words = SPLIT == 1 ? p.Cp : p.win_words;
    const uint32_t stage_bytes = p.SW * 4, rec_bytes = win_words * 4;
    // output slice of this CTA: the whole record (SPLIT = 1), or rows [half*ROWS, ...)
    const uint32_t half = blockIdx.x % SPLIT, pair = blockIdx.x / SPLIT, npairs = gridDim.x / SPLIT;
    const uint32_t out_words = SPLIT == 1 ? p.Cp : (uint32_t)(WG::ROWS * WQ);
    const uint32_t out_off = SPLIT == 1 ? 0u : half * out_words;
    const uint32_t win0 = SPLIT == 1 ? 0u : p.win0[half];  // words
    const uint32_t out_bytes = out_words * 4;
    uint8_t* outs = st + NS * stage_bytes;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    // BTO: per-warp stores + the transposed boundary plane written by the BTW bt warps.
    // Output buffer o then uses ofull[o] = every chunk warp wrote its slice (the bt
    // warps wait for it) and oempty[o] = the bt warps are done reading it (every chunk
    // warp waits before rewriting the buffer)
    constexpr bool BTO = PWS && SPLIT == 1 && BTW > 0;
    static_assert(BTW == 0 || BTO, "bt warps need per-warp stores, one CTA per record");
    // HG: with bt warps, the HW halo warps gather each group's halo words from the
    // previous step's transposed plane p.bt (halo_bt_regs_kernel's body) into the stage
    constexpr bool HG = BTO && HW > 0;
    constexpr int HG_NHC = std::is_same<FT, HTag>::value ? 7 : std::is_same<FT, CarpetTag>::value ? 11 : 1;
    static_assert(BTW % NGRP == 0, "bt warps are split evenly over the group sets");
    constexpr int BTS = BTW / NGRP > 0 ? BTW / NGRP : 1;  // bt warps per group set
    if (tid == 0) push_warps_done = 0u;
    if (tid == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(full0 + 8 * s, HW > 0 ? 2 : 1);  // producer (+ bytes) [+ the halo warp]
            mbar_init(empty0 + 8 * s, NCHUNK);
        }
        for (int o = 0; o < NO; ++o) {
            mbar_init(ofull0 + 8 * o, NCHUNK);
            mbar_init(oempty0 + 8 * o, BTO ? BTS : 1);
        }
        mbar_fence_init();
    }
    if (tid < NS) reinterpret_cast<uint32_t*>(st + tid * stage_bytes)[win_words + p.nHp] = 0u;  // absent
    if (SPLIT == 1)
        for (int o = 0; o < NO; ++o)  // record padding words (interleaved records: the
            for (uint32_t k = p.C + tid; k < p.Cp; k += blockDim.x)  // padding blocks' words carry no cell
                reinterpret_cast<uint32_t*>(outs + o * out_bytes)[k] = 0u;
    // ---- in-kernel halo warps (<= 8 slots): slot table + the first group's neighbour
    // tiles (static ntab), before the PDL wait
    // (T q=8; the q=6 kernel with 8 group sets spills with them live across its prologue)
    constexpr bool HW_HOIST = HW > 0 && !BTO && WQ == 81;
    uint32_t hw_noff[8], hw_moff[8], hw_t2n[8];
    auto hw_tables = [&]() {
        if (warp >= NCW + 2 && p.nH <= 8) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const uint32_t sl = (uint32_t)j < p.nH ? __ldg(p.slot + j) : 0u;
                hw_noff[j] = ((sl >> 16) & 0xFFu) * p.T;
                hw_moff[j] = sl & 0xFFFFu;
            }
            const uint32_t gg = p.g0 + pair + (uint32_t)(warp - NCW - 2) * npairs, t = gg * 32 + lane;
            const bool in = gg < p.g1 && t < p.T;
#pragma unroll
            for (int j = 0; j < 8; ++j) hw_t2n[j] = ((uint32_t)j < p.nH && in) ? __ldg(p.ntab + hw_noff[j] + t) : kNoTile;
        }
    };
    if constexpr (HW_HOIST) hw_tables();
    // ---- consumer tables (block offsets, output slice, boundary sources): plan data
    // that no kernel writes, so they are loaded before the PDL wait and overlap the
    // previous kernel's tail (the boundary-source search is ~11 dependent load pairs
    // per lane: a visible share of a step when a CTA owns a few groups)
    uint32_t KB[9], KS[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) {
        KB[i] = ((p.birth >> i) & 1u) ? 0xFFFFFFFFu : 0u;
        KS[i] = ((p.survive >> i) & 1u) ? 0xFFFFFFFFu : 0u;
    }
    const int set = warp / NCHUNK, c = warp - set * NCHUNK;
    const uint32_t lblk = (uint32_t)c * 32 + lane;
    const bool active = lblk < (uint32_t)NBLK;
    const uint32_t blk = half * (uint32_t)NBLK + lblk;
    uint32_t toff[NEP];
    {
        const uint4* t4 = reinterpret_cast<const uint4*>(p.btab) + (size_t)(active ? blk : 0) * (NEP / 4);
        static_for<NEP / 4>([&](auto e4) {
            constexpr int E = decltype(e4)::value;
            const uint4 v = __ldg(t4 + E);
            toff[4 * E] = v.x; toff[4 * E + 1] = v.y; toff[4 * E + 2] = v.z; toff[4 * E + 3] = v.w;
        });
    }
    // PWS: this warp's output slice [w_lo, w_hi) (slice words) and its boundary
    // sources [k_lo, k_hi) of the cell-sorted list
    uint32_t w_lo = 0, w_hi = 0, k_lo = 0, k_hi = 0;
    if constexpr (PWS) {
        w_lo = (uint32_t)c * 32 * W::BW;
        w_hi = c == NCHUNK - 1 ? out_words : w_lo + 32 * W::BW;
        const uint32_t* sorted = p.srcidx + p.nSrc;
        for (uint32_t k = lane; k < p.nSrc; k += 32) {
            const uint32_t cell = __ldg(p.srcidx + __ldg(sorted + k));
            k_lo += cell < out_off + w_lo;
            k_hi += cell < out_off + w_hi;
        }
        k_lo = __reduce_add_sync(0xFFFFFFFFu, k_lo);
        k_hi = __reduce_add_sync(0xFFFFFFFFu, k_hi);
    }
    // up to 64 boundary sources of the slice: (m, word) pairs held in registers
    // (carpet r=9 0.0207 -> 0.0188 ms; candy, with few sources per warp, keeps the
    // loop: 0.238 vs 0.244 ms)
    constexpr bool REGB = PWS && !std::is_same<FT, CandyTag>::value;
    uint32_t bm0 = 0, bw0 = 0, bm1 = 0, bw1 = 0;
    if constexpr (REGB) {
        const uint32_t* sorted = p.srcidx + p.nSrc;
        if (k_lo + lane < k_hi) { bm0 = __ldg(sorted + k_lo + lane); bw0 = __ldg(p.srcidx + bm0); }
        if (k_lo + 32 + lane < k_hi) { bm1 = __ldg(sorted + k_lo + 32 + lane); bw1 = __ldg(p.srcidx + bm1); }
    }
    // compile-time stage size (SWC > 0): the group loop is unrolled over the NS / NGRP
    // stages of this warp's set, so every external load is ONE ld.shared at the
    // lane's (set-relative) offset + an immediate (the stage offset) instead of a
    // multiply-add + add + load per external per group (H: 48 -> 16 instructions of
    // the 166 per block)
    constexpr int SWC = SPLIT == 1 ? StageWordsCT<FT, WQ>::v : 0;
    uint32_t tS[NEP], own_off = 0;
    if constexpr (SWC > 0) {
        using BG = BlockGeom<FT, P, WQ>;
        const uint32_t set_off = (uint32_t)set * (uint32_t)(SWC * 4);
#pragma unroll
        for (int e = 0; e < NEP; ++e) tS[e] = set_off + toff[e];
        own_off = set_off + 4u * block_own_base<FT, P, WQ>(blk);
        (void)sizeof(BG);
    }
    fence_proxy_async_smem();
    __syncthreads();
    pdl_wait();     // the prologue above overlapped the previous kernel's tail (PDL)
    if constexpr (HW > 0) wait_peers(p);  // in-kernel halo: the peers' pushes of this step
    pdl_trigger();

    if (warp == NCW) {  // ---- producer -------------------------------------------------
        if (lane == 0) {
            uint32_t i = 0;
            for (uint32_t g = p.g0 + pair; g < p.g1; g += npairs, ++i) {
                const uint32_t s = i % NS;
                if (i >= NS) mbar_wait(empty0 + 8 * s, ((i / NS) - 1) & 1u);
                const uint32_t bar = full0 + 8 * s, dst_s = smem_u32(st + s * stage_bytes);
                const uint32_t halo_bytes = HW > 0 ? 0u : p.nHp * 4;
                mbar_expect_tx(bar, rec_bytes + halo_bytes);
                rec_g2s(p, dst_s, src + (uint64_t)g * p.Cp + win0, rec_bytes, bar);
                if (halo_bytes) bulk_g2s(dst_s + rec_bytes, p.halo + (uint64_t)g * p.nHp, halo_bytes, bar);
            }
        }
        return;
    }
    if constexpr (HG) {
        if (warp >= NCW + 2 && warp < NCW + 2 + HW) {  // ---- Bt gather warps: group i = hw (mod HW)
            constexpr int NHC = HG_NHC;
            const uint32_t hw = (uint32_t)(warp - NCW - 2), gstep = HW * npairs;
            const XposeLane X((uint32_t)lane);
            uint32_t t2n[8];
            auto fetch = [&](uint32_t gg) {
                const uint32_t t = gg * 32 + lane;
                const bool in = gg < p.g1 && t < p.T;
#pragma unroll
                for (int d = 0; d < 8; ++d) t2n[d] = (d < p.nD && in) ? __ldg(p.ntab + ((size_t)d * p.T + t)) : kNoTile;
            };
            uint32_t i = hw, g = p.g0 + pair + hw * npairs;
            fetch(g);
            for (; g < p.g1; g += gstep, i += HW) {
                uint32_t t2[8];
#pragma unroll
                for (int d = 0; d < 8; ++d) t2[d] = t2n[d];
                fetch(g + gstep);
                uint32_t acc[NHC];
#pragma unroll
                for (int k = 0; k < NHC; ++k) acc[k] = 0u;
#pragma unroll
                for (int d = 0; d < 8; ++d) {
                    const bool ok = t2[d] != kNoTile;
                    const uint32_t* b = p.bt + (uint64_t)(t2[d] >> 5) * (NHC * 32u) + (t2[d] & 31u);
                    uint32_t v[NHC];
#pragma unroll
                    for (int k = 0; k < NHC; ++k) v[k] = (ok && p.btm.m[k][d] != 0u) ? __ldcg(b + 32 * k) : 0u;
#pragma unroll
                    for (int k = 0; k < NHC; ++k) acc[k] |= v[k] & p.btm.m[k][d];
                }
#pragma unroll
                for (int k = 0; k < NHC; ++k) acc[k] = warp_transpose32(acc[k], X);
                const uint32_t s = i % NS;
                if (i >= NS) mbar_wait(empty0 + 8 * s, ((i / NS) - 1) & 1u);
                uint32_t* Hs = reinterpret_cast<uint32_t*>(st + s * stage_bytes) + win_words;
#pragma unroll
                for (int k = 0; k < NHC; ++k)
                    if (k * 32 + lane < p.nH) Hs[k * 32 + lane] = acc[k];
                __syncwarp();
                if (lane == 0) mbar_arrive(full0 + 8 * s);  // release: the halo words are visible
            }
            return;
        }
    }
    if constexpr (HW > 0 && !HG) {
        if (warp >= NCW + 2) {  // ---- halo warps: group i = hw (mod HW) --------------------
            const uint32_t hw = (uint32_t)(warp - NCW - 2);
            uint32_t i = hw;
            if (p.nH <= 8) {
                // (triangle: <= 8 slots) the slot table in registers; the next group's
                // neighbour tiles are loaded while this group's boundary words are in
                // flight, and both before the wait for the stage -- only the 8 stores
                // need it (the table and the first group's tiles: before the PDL wait)
                if constexpr (!HW_HOIST) hw_tables();
                uint32_t* const noff = hw_noff;
                uint32_t* const moff = hw_moff;
                uint32_t* const t2n = hw_t2n;
                const uint32_t gstep = HW * npairs;
                auto fetch = [&](uint32_t gg) {
                    const uint32_t t = gg * 32 + lane;
                    const bool in = gg < p.g1 && t < p.T;
#pragma unroll
                    for (int j = 0; j < 8; ++j) t2n[j] = ((uint32_t)j < p.nH && in) ? __ldg(p.ntab + noff[j] + t) : kNoTile;
                };
                uint32_t g = p.g0 + pair + hw * npairs;
                for (; g < p.g1; g += gstep, i += HW) {
                    uint32_t t2[8];
#pragma unroll
                    for (int j = 0; j < 8; ++j) t2[j] = t2n[j];
                    fetch(g + gstep);
                    uint32_t v[8];
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        v[j] = t2[j] != kNoTile ? __ldcg(bsrc + (size_t)(t2[j] >> 5) * p.nSrc + moff[j]) >> (t2[j] & 31) : 0u;
                    uint32_t mine = 0;
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const uint32_t word = __ballot_sync(0xFFFFFFFFu, (v[j] & 1u) != 0);
                        if (lane == (uint32_t)j) mine = word;
                    }
                    const uint32_t s = i % NS;
                    if (i >= NS) mbar_wait(empty0 + 8 * s, ((i / NS) - 1) & 1u);
                    uint32_t* Hs = reinterpret_cast<uint32_t*>(st + s * stage_bytes) + win_words;
                    if ((uint32_t)lane < p.nH) Hs[lane] = mine;
                    __syncwarp();
                    if (lane == 0) mbar_arrive(full0 + 8 * s);  // release: the halo words are visible
                }
                return;
            }
            for (uint32_t g = p.g0 + pair + hw * npairs; g < p.g1; g += HW * npairs, i += HW) {
                const uint32_t s = i % NS;
                if (i >= NS) mbar_wait(empty0 + 8 * s, ((i / NS) - 1) & 1u);
                uint32_t* Hs = reinterpret_cast<uint32_t*>(st + s * stage_bytes) + win_words;
                const uint32_t t = g * 32 + lane;
                for (uint32_t j0 = 0; j0 < p.nH; j0 += 8) {
                    uint32_t t2[8], sl[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const uint32_t j = j0 + u;
                        t2[u] = kNoTile;
                        sl[u] = 0;
                        if (j < p.nH) {
                            sl[u] = __ldg(p.slot + j);
                            if (t < p.T) t2[u] = __ldg(p.ntab + ((size_t)((sl[u] >> 16) & 0xFFu) * p.T + t));
                        }
                    }
                    uint32_t v[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u)
                        v[u] = t2[u] != kNoTile ? __ldcg(bsrc + (size_t)(t2[u] >> 5) * p.nSrc + (sl[u] & 0xFFFFu)) >> (t2[u] & 31)
                                                : 0u;
                    // every lane holds every ballot; lane 0 -- the thread that arrives on
                    // the full barrier -- stores them, so its release covers the writes
                    uint32_t words[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) words[u] = __ballot_sync(0xFFFFFFFFu, (v[u] & 1u) != 0);
                    if (lane == 0) {
#pragma unroll
                        for (int u = 0; u < 8; ++u)
                            if (j0 + u < p.nH) Hs[j0 + u] = words[u];
                    }
                }
                if (lane == 0) mbar_arrive(full0 + 8 * s);  // release: the halo words are visible
            }
            return;
        }
    }
    if constexpr (BTO) {
        if (warp >= NCW + 2 + (HG ? HW : 0)) {  // ---- bt warps: chunks b, b + BTW, ... of every record
            // lane l loads the record word of boundary slot 32k + l; one transpose gives
            // lane t the slot bits of tile t: Bt[(g nHc + k) 32 + t], 128 coalesced bytes
            // bt warp w serves group set w % NGRP (each set's buffers, no head-of-line
            // blocking between sets), chunks w / NGRP, + BTS, ...
            // The lane's source cells (chunks b, b + BTS, ...) stay in registers; the
            // buffer is released as soon as its words are read (before the transposes
            // and the global stores: H r=11 step kernel 108.7 -> ... us)
            const uint32_t w = (uint32_t)(warp - NCW - 2 - (HG ? HW : 0)), set = w % NGRP, b = w / NGRP;
            const uint32_t nHc = (p.nSrc + 31) / 32;
            const XposeLane X((uint32_t)lane);
            // (chunks per bt warp: at most kBtMaxChunks / BTS; H q=4 has 7 chunks)
            constexpr int KMAX = std::is_same<FT, HTag>::value ? (7 + BTS - 1) / BTS : (kBtMaxChunks + BTS - 1) / BTS;
            uint32_t sidx[KMAX];
#pragma unroll
            for (int kk = 0; kk < KMAX; ++kk) {
                const uint32_t m = 32 * (b + kk * BTS) + (uint32_t)lane;
                sidx[kk] = m < p.nSrc ? __ldg(p.srcidx + m) : kNoTile;
            }
            uint32_t i = set;
            for (uint32_t g = p.g0 + pair + set * npairs; g < p.g1; g += NGRP * npairs, i += NGRP) {
                const uint32_t o = i % NO;
                mbar_wait(ofull0 + 8 * o, (i / NO) & 1u);  // acquire: every slice written
                const uint32_t* Do = reinterpret_cast<const uint32_t*>(outs + o * out_bytes);
                uint32_t x[KMAX];
#pragma unroll
                for (int kk = 0; kk < KMAX; ++kk)
                    x[kk] = (b + kk * BTS < nHc && sidx[kk] != kNoTile) ? Do[sidx[kk]] : 0u;
                __syncwarp();
                if (lane == 0) mbar_arrive(oempty0 + 8 * o);  // release: buffer o read
#pragma unroll
                for (int kk = 0; kk < KMAX; ++kk) {
                    const uint32_t k = b + kk * BTS;
                    if (k < nHc) {
                        if constexpr (std::is_same<FT, HTag>::value)
                            p.bt_out[((uint64_t)g * nHc + k) * 32 + lane] = warp_transpose32(x[kk], X);
                        else
                            p.bt_out[((uint64_t)g * nHc + k) * 32 + lane] = warp_transpose32(x[kk], (uint32_t)lane);
                    }
                }
            }
            return;
        }
    }
    if (warp == NCW + 1) {  // ---- storer ---------------------------------------------------
        if constexpr (PWS) return;
        // one bulk store per finished group; with BST the lanes also copy the group's
        // new boundary words (the output words at the boundary source cells) into the
        // boundary plane.
        uint32_t i = 0;
        for (uint32_t g = p.g0 + pair; g < p.g1; g += npairs, ++i) {
            const uint32_t o = i % NO;
            mbar_wait(ofull0 + 8 * o, (i / NO) & 1u);
            const uint32_t* Do = reinterpret_cast<const uint32_t*>(outs + o * out_bytes);
            if (lane == 0) rec_s2g(p, dst + (uint64_t)g * p.Cp + out_off, smem_u32(Do), out_bytes);
            if constexpr (BST) {
                for (uint32_t m = lane; m < p.nSrc; m += 32) {
                    const uint32_t c = __ldg(p.srcidx + m) - out_off;  // (wraps when below this slice)
                    if (SPLIT == 1 || c < out_words) bdst[(uint64_t)g * p.nSrc + m] = Do[c];
                }
                __syncwarp();
            }
            if (lane == 0) {
                // (lagging this wait by one group measured slower: T r=20 0.176 vs
                //  0.143 ms -- the consumers then wait a storer round trip per group)
                bulk_wait_read_all();  // the output record may be rewritten
                mbar_arrive(oempty0 + 8 * o);
            }
        }
        if (lane == 0) bulk_wait_all();
        return;
    }
    // ---- consumers ---------------------------------------------------------------------
    // (per-warp tables: set up before the PDL wait, see above)
    auto group = [&](uint32_t g, uint32_t i, auto soff_c) {
        constexpr int SOFF = decltype(soff_c)::value;  // byte offset of this stage from set 0's (SWC > 0)
        (void)SOFF;
        const uint32_t s = i % NS, o = i % NO;
        mbar_wait(full0 + 8 * s, (i / NS) & 1u);
        if constexpr (PWS) {
            if (i >= NO) {  // this warp's store from NO groups ago has read its slice
                if (lane == 0) bulk_wait_read<NO / NGRP - 1>();
                __syncwarp();
                if constexpr (BTO) mbar_wait(oempty0 + 8 * o, ((i / NO) - 1) & 1u);  // ... and the bt warps
            }
        } else if (i >= NO) {
            mbar_wait(oempty0 + 8 * o, ((i / NO) - 1) & 1u);
        }
        const uint8_t* Sb = st + s * stage_bytes;
        // block_words_r indexes the whole record: shift the slice base back by out_off
        uint32_t* Do = reinterpret_cast<uint32_t*>(outs + o * out_bytes) - out_off;
        const uint32_t vmask = g == p.NG - 1 ? p.lastmask : 0xFFFFFFFFu;
        if constexpr (SWC > 0) {
            if (active) block_words_c<FT, P, WQ, CONWAY, DEG, SOFF>(st, tS, own_off, blk, Do, vmask, KB, KS);
        } else {
            if (active) block_words_r<FT, P, WQ, CONWAY, DEG>(Sb, toff, blk, Do, vmask, KB, KS, win0);
        }
        if constexpr (PWS) {
            fence_proxy_async_smem();  // the bulk store reads this slice through the async proxy
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(empty0 + 8 * s);
                rec_s2g(p, dst + (uint64_t)g * p.Cp + out_off + w_lo, smem_u32(Do + out_off + w_lo),
                         (w_hi - w_lo) * 4);
                if constexpr (BTO) mbar_arrive(ofull0 + 8 * o);  // release: this slice is written
            }
            if constexpr (BTO) return;  // the bt warps write the boundary data
            uint32_t* bg = bdst + (uint64_t)g * p.nSrc;
            if constexpr (REGB) {
                if (k_lo + lane < k_hi) bg[bm0] = Do[bw0];
                if (k_lo + 32 + lane < k_hi) bg[bm1] = Do[bw1];
            }
            const uint32_t* sorted = p.srcidx + p.nSrc;
            for (uint32_t k = k_lo + (REGB ? 64 : 0) + lane; k < k_hi; k += 32) {
                const uint32_t m = __ldg(sorted + k);
                bg[m] = Do[__ldg(p.srcidx + m)];
            }
            return;
        }
        if (!BST && c == 0 && half == 0) {  // boundary plane of the new state (few words)
            uint32_t mine = 0u;
            for (uint32_t m = lane; m < p.nSrc; m += 32) {
                mine = cell_word<CONWAY, DEG, WIDE>(Sb, p.nbr, __ldg(p.srcidx + m), KB, KS) & vmask;
                bdst[(uint64_t)g * p.nSrc + m] = mine;
            }
            if constexpr (PUSH) {  // (nSrc <= 32: lane m holds word m) straight into the peers' planes
                const uint32_t k0 = __ldg(p.push_off + (g - p.g0)), k1 = __ldg(p.push_off + (g - p.g0) + 1);
                for (uint32_t kb = k0; kb < k1; kb += 32) {
                    const uint32_t k = kb + (uint32_t)lane;
                    const uint32_t e = k < k1 ? __ldg(p.push_ent + k) : 0u;
                    const uint32_t v = __shfl_sync(0xFFFFFFFFu, mine, e & 31u);
                    if (k < k1) p.push_bnd[e >> 16][(uint64_t)g * p.nSrc + (e & 0xFFFFu)] = v;
                }
            }
        }
        fence_proxy_async_smem();  // the bulk store reads Do through the async proxy
        __syncwarp();
        if (lane == 0) {
            mbar_arrive(empty0 + 8 * s);
            mbar_arrive(ofull0 + 8 * o);
        }
    };
    {
        uint32_t i = (uint32_t)set;
        uint32_t g = p.g0 + pair + (uint32_t)set * npairs;
        if constexpr (SWC > 0) {
            constexpr int U = NS / NGRP;  // stages of this set: set + NGRP u, u < U
            while (g < p.g1) {
                static_for<U>([&](auto u) {
                    if (g >= p.g1) return;
                    group(g, i, std::integral_constant<int, decltype(u)::value * NGRP * SWC * 4>{});
                    g += NGRP * npairs;
                    i += NGRP;
                });
            }
        } else {
            for (; g < p.g1; g += NGRP * npairs, i += NGRP) group(g, i, std::integral_constant<int, 0>{});
        }
    }
    if constexpr (PUSH && !BST) if (c == 0 && half == 0) {
        // this warp's pushes are done: the CTA's last pushing warp counts the CTA, the
        // grid's last CTA bumps every peer's counter (system-scope fences in between:
        // each writer fences before its count, the last one before the bumps)
        __threadfence_system();
        __syncwarp();
        if (lane == 0) {
            if (atomicAdd(&push_warps_done, 1u) == (unsigned)(NGRP - 1)) {
                __threadfence_system();
                if (atomicAdd(p.push_done, 1u) == gridDim.x - 1) {
                    atomicExch(p.push_done, 0u);
                    __threadfence_system();
                    for (uint32_t r = 0; r < 32; ++r)
                        if ((p.push_mask >> r) & 1u) atomicAdd_system(p.push_cnt[r], 1u);
                }
            }
        }
    }
    if constexpr (PWS)
        if (lane == 0) bulk_wait_all();
}

__device__ __forceinline__ void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

// Small levels whose whole packed state fits one SM's shared memory (triangle q=6,
// r <= 12): ONE CTA runs all nsteps steps on-chip.  Shared memory holds both state
// buffers in stage layout (per group: record | halo words | zero word) and, per
// (group, halo slot, tile), the smem word + bit of its source cell (built once from
// ntab).  Per step: halo words by ballots over smem, __syncthreads, every
// micro-block chunk of every group (block_words_r) into the other buffer,
// __syncthreads.  Global memory is touched only to load the first state and to
// store the last one (+ its boundary plane).
template <bool CONWAY, int DEG, class FT, int P, int WQ>
__global__ void __launch_bounds__(1024, 1)
step_packed_resident_kernel(const PackedStepParams p, const uint32_t* __restrict__ src, uint32_t* __restrict__ dst,
                            uint32_t* __restrict__ bdst, int nsteps) {
    using W = Wiring<FT, P>;
    constexpr int NBLK = BlockGeom<FT, P, WQ>::NBLK;
    constexpr int NCHUNK = (NBLK + 31) / 32;
    constexpr int NEP = W::NEP;
    extern __shared__ __align__(16) uint32_t rsm[];
    const uint32_t NG = p.NG, SWg = p.SW, nH = p.nH;
    uint32_t* S0 = rsm;
    uint32_t* S1 = rsm + NG * SWg;
    uint32_t* hix = rsm + 2 * NG * SWg;  // [NG][nH][32]: smem word << 5 | bit, or ~0u
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    for (uint32_t i = tid; i < 2 * NG * SWg; i += blockDim.x) {
        const uint32_t g = (i / SWg) % NG, w = i % SWg;
        rsm[i] = (i < NG * SWg && w < p.Cp) ? src[(uint64_t)g * p.Cp + w] : 0u;
    }
    for (uint32_t i = tid; i < NG * nH * 32; i += blockDim.x) {
        const uint32_t l = i & 31, gj = i >> 5, g = gj / nH, j = gj - g * nH;
        const uint32_t t = g * 32 + l, sl = __ldg(p.slot + j);
        const uint32_t t2 = t < p.T ? __ldg(p.ntab + ((size_t)((sl >> 16) & 0xFFu) * p.T + t)) : kNoTile;
        hix[i] = t2 == kNoTile ? 0xFFFFFFFFu : (((t2 >> 5) * SWg + __ldg(p.srcidx + j)) << 5) | (t2 & 31);
    }
    uint32_t KB[9], KS[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) {
        KB[i] = ((p.birth >> i) & 1u) ? 0xFFFFFFFFu : 0u;
        KS[i] = ((p.survive >> i) & 1u) ? 0xFFFFFFFFu : 0u;
    }
    __syncthreads();
    for (int step = 0; step < nsteps; ++step) {
        uint32_t* A = (step & 1) ? S1 : S0;
        uint32_t* Bn = (step & 1) ? S0 : S1;
        for (uint32_t task = warp; task < NG * nH; task += nwarps) {  // halo words of A
            const uint32_t x = hix[task * 32 + lane];
            const uint32_t bit = x == 0xFFFFFFFFu ? 0u : (A[x >> 5] >> (x & 31)) & 1u;
            const uint32_t w = __ballot_sync(0xFFFFFFFFu, bit != 0);
            if (lane == 0) {
                const uint32_t g = task / nH;
                A[g * SWg + p.Cp + (task - g * nH)] = w;
            }
        }
        __syncthreads();
        for (uint32_t item = warp; item < NG * NCHUNK; item += nwarps) {  // micro-blocks A -> Bn
            const uint32_t g = item / NCHUNK, c = item - g * NCHUNK;
            const uint32_t blk = c * 32 + lane;
            if (blk < (uint32_t)NBLK) {
                uint32_t toff[NEP];
                const uint4* t4 = reinterpret_cast<const uint4*>(p.btab) + (size_t)blk * (NEP / 4);
                static_for<NEP / 4>([&](auto e4) {
                    constexpr int E = decltype(e4)::value;
                    const uint4 v = __ldg(t4 + E);
                    toff[4 * E] = v.x; toff[4 * E + 1] = v.y; toff[4 * E + 2] = v.z; toff[4 * E + 3] = v.w;
                });
                const uint32_t vmask = g == NG - 1 ? p.lastmask : 0xFFFFFFFFu;
                block_words_r<FT, P, WQ, CONWAY, DEG>(reinterpret_cast<const uint8_t*>(A + g * SWg), toff, blk,
                                                      Bn + g * SWg, vmask, KB, KS);
            }
        }
        __syncthreads();
    }
    const uint32_t* F = (nsteps & 1) ? S1 : S0;
    for (uint32_t i = tid; i < NG * p.Cp; i += blockDim.x) dst[i] = F[(i / p.Cp) * SWg + i % p.Cp];
    for (uint32_t i = tid; i < NG * p.nSrc; i += blockDim.x)
        bdst[i] = F[(i / p.nSrc) * SWg + __ldg(p.srcidx + i % p.nSrc)];
}

// Cluster version for states of up to 8 CTAs x 8 groups (T r=12): CTA c of the
// cluster owns groups g = c (mod NC) in its shared memory; halo words read the
// neighbour tiles' source words from the owning CTA's shared memory over the
// cluster (distributed shared memory, mapa + ld.shared::cluster); one cluster
// barrier per step.
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t ld_dsmem(uint32_t local_saddr, uint32_t rank) {
    uint32_t ra, v;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(local_saddr), "r"(rank));
    asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(ra) : "memory");
    return v;
}

template <bool CONWAY, int DEG, class FT, int P, int WQ>
__global__ void __launch_bounds__(1024, 1)
step_packed_cluster_kernel(const PackedStepParams p, const uint32_t* __restrict__ src, uint32_t* __restrict__ dst,
                           uint32_t* __restrict__ bdst, int nsteps) {
    using W = Wiring<FT, P>;
    constexpr int NBLK = BlockGeom<FT, P, WQ>::NBLK;
    constexpr int NCHUNK = (NBLK + 31) / 32;
    constexpr int NEP = W::NEP;
    extern __shared__ __align__(16) uint32_t csm[];
    const uint32_t NC = gridDim.x, me = cluster_rank();
    const uint32_t NG = p.NG, SWg = p.SW, nH = p.nH;
    const uint32_t LG = (NG + NC - 1) / NC;                // local group slots per CTA
    const uint32_t nmine = me < NG ? (NG - me + NC - 1) / NC : 0u;
    uint32_t* S0 = csm;
    uint32_t* S1 = csm + LG * SWg;
    uint32_t* hix = csm + 2 * LG * SWg;                    // [nmine][nH][32]: rank << 25 | word << 5 | bit
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    for (uint32_t i = tid; i < 2 * LG * SWg; i += blockDim.x) {
        const uint32_t lg = (i / SWg) % LG, w = i % SWg, g = lg * NC + me;
        csm[i] = (i < LG * SWg && g < NG && w < p.Cp) ? src[(uint64_t)g * p.Cp + w] : 0u;
    }
    for (uint32_t i = tid; i < nmine * nH * 32; i += blockDim.x) {
        const uint32_t l = i & 31, gj = i >> 5, lg = gj / nH, j = gj - lg * nH, g = lg * NC + me;
        const uint32_t t = g * 32 + l, sl = __ldg(p.slot + j);
        const uint32_t t2 = t < p.T ? __ldg(p.ntab + ((size_t)((sl >> 16) & 0xFFu) * p.T + t)) : kNoTile;
        if (t2 == kNoTile) { hix[i] = 0xFFFFFFFFu; continue; }
        const uint32_t G2 = t2 >> 5;
        hix[i] = ((G2 % NC) << 25) | ((((G2 / NC) * SWg) + __ldg(p.srcidx + j)) << 5) | (t2 & 31);
    }
    uint32_t KB[9], KS[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) {
        KB[i] = ((p.birth >> i) & 1u) ? 0xFFFFFFFFu : 0u;
        KS[i] = ((p.survive >> i) & 1u) ? 0xFFFFFFFFu : 0u;
    }
    cluster_sync_all();  // every CTA's first state is in place
    for (int step = 0; step < nsteps; ++step) {
        uint32_t* A = (step & 1) ? S1 : S0;
        uint32_t* Bn = (step & 1) ? S0 : S1;
        const uint32_t Abase = (uint32_t)__cvta_generic_to_shared(A);
        for (uint32_t task = warp; task < nmine * nH; task += nwarps) {  // halo words of my groups
            const uint32_t x = hix[task * 32 + lane];
            uint32_t bit = 0u;
            if (x != 0xFFFFFFFFu) bit = (ld_dsmem(Abase + ((x >> 5) & 0xFFFFFu) * 4, x >> 25) >> (x & 31)) & 1u;
            const uint32_t w = __ballot_sync(0xFFFFFFFFu, bit != 0);
            if (lane == 0) {
                const uint32_t lg = task / nH;
                A[lg * SWg + p.Cp + (task - lg * nH)] = w;
            }
        }
        __syncthreads();
        for (uint32_t item = warp; item < nmine * NCHUNK; item += nwarps) {
            const uint32_t lg = item / NCHUNK, c = item - lg * NCHUNK, g = lg * NC + me;
            const uint32_t blk = c * 32 + lane;
            if (blk < (uint32_t)NBLK) {
                uint32_t toff[NEP];
                const uint4* t4 = reinterpret_cast<const uint4*>(p.btab) + (size_t)blk * (NEP / 4);
                static_for<NEP / 4>([&](auto e4) {
                    constexpr int E = decltype(e4)::value;
                    const uint4 v = __ldg(t4 + E);
                    toff[4 * E] = v.x; toff[4 * E + 1] = v.y; toff[4 * E + 2] = v.z; toff[4 * E + 3] = v.w;
                });
                const uint32_t vmask = g == NG - 1 ? p.lastmask : 0xFFFFFFFFu;
                block_words_r<FT, P, WQ, CONWAY, DEG>(reinterpret_cast<const uint8_t*>(A + lg * SWg), toff, blk,
                                                      Bn + lg * SWg, vmask, KB, KS);
            }
        }
        cluster_sync_all();  // Bn complete everywhere; nobody still reads A
    }
    const uint32_t* F = (nsteps & 1) ? S1 : S0;
    for (uint32_t i = tid; i < nmine * p.Cp; i += blockDim.x) {
        const uint32_t lg = i / p.Cp, w = i - lg * p.Cp;
        dst[(uint64_t)(lg * NC + me) * p.Cp + w] = F[lg * SWg + w];
    }
    for (uint32_t i = tid; i < nmine * p.nSrc; i += blockDim.x) {
        const uint32_t lg = i / p.nSrc, m = i - lg * p.nSrc;
        bdst[(uint64_t)(lg * NC + me) * p.nSrc + m] = F[lg * SWg + __ldg(p.srcidx + m)];
    }
}

// Peer-memory halo push (one CTA): after this rank's step kernel, write every
// boundary-plane word a peer needs straight into that peer's boundary plane over
// NVLink (CUDA IPC mappings), then -- after a system-scope fence -- add 1 to the
// arrival counter of every peer it sends to.  The peer's next halo kernel waits on
// that counter (wait_peers).  Element e has the same index in every rank's plane.
__global__ void p2p_push_kernel(const uint32_t* __restrict__ bnd, const uint64_t* __restrict__ elems,
                                const uint8_t* __restrict__ peer_of, uint64_t n, uint32_t* const* __restrict__ peer_bnd,
                                uint32_t* const* __restrict__ peer_cnt, uint32_t send_mask) {
    pdl_wait();  // the step kernel's boundary words are complete (PDL launch)
    pdl_trigger();
    for (uint64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const uint64_t e = elems[i];
        peer_bnd[peer_of[i]][e] = bnd[e];
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x < 32 && ((send_mask >> threadIdx.x) & 1u)) {
        __threadfence_system();
        atomicAdd_system(peer_cnt[threadIdx.x], 1u);
    }
}

// ---- boundary plane from a packed state ---------------------------------------
__global__ void bnd_refresh_kernel(const uint32_t* __restrict__ P, uint32_t Cp, uint32_t NG, uint32_t nSrc,
                                   const uint32_t* __restrict__ srcidx, uint32_t* __restrict__ B) {
    const uint64_t n = (uint64_t)NG * nSrc;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t g = i / nSrc;
        const uint32_t m = (uint32_t)(i - g * nSrc);
        B[i] = P[g * Cp + srcidx[m]];
    }
}

// lambda at `levels` levels (CoordMapper::to_embedded restricted, maps.cpp:123-146)
template <int K, int S>
__device__ __forceinline__ void lambda_levels(const Frac& f, uint32_t cx, uint32_t cy, int levels, uint32_t& x,
                                              uint32_t& y) {
    const uint32_t k = kval<K>(f), s = sval<S>(f);
    uint32_t ex = 0, ey = 0, sp = 1;
    for (int mu = 0; mu < levels; ++mu) {
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

// Embedded origin of tile t: lambda of (cx, cy) splits into the tile's digits
// (levels q..r-1, the coarse coordinates) and the local ones (levels 0..q-1):
// lambda(X*WQ + c, Y*WQ + a) = s^q * lambda_L(X, Y) + lambda_q(c, a).
template <int K, int S>
__device__ __forceinline__ void tile_origin(const PackedGeom& G, uint32_t t, uint32_t& x0, uint32_t& y0) {
    const uint32_t X = t % G.Wc, Y = t / G.Wc;
    uint32_t xt, yt;
    lambda_levels<K, S>(G.f, X, Y, (int)G.L, xt, yt);
    x0 = xt * G.sq;
    y0 = yt * G.sq;
}

// Simulation::seed_random (stencil.cpp:138-180) straight into the packed layout:
// warp per (group, 32 local cells); lane b = tile b; loc[i] = (yl << 16) | xl is
// the level-q lambda of local cell i.
template <int K, int S>
__global__ void seed_packed_kernel(PackedGeom G, const uint32_t* __restrict__ loc, uint32_t* __restrict__ P,
                                   uint64_t seed_mix, double density) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t cpw = (G.Cl + 31) / 32;  // 32-word chunks per group (record words with a loc entry)
    const uint64_t nw = (uint64_t)G.NG * cpw;
    for (uint64_t wi = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; wi < nw;
         wi += ((uint64_t)gridDim.x * blockDim.x) >> 5) {
        const uint32_t g = (uint32_t)(wi / cpw), i0 = (uint32_t)(wi - (uint64_t)g * cpw) * 32;
        const uint32_t t = g * 32 + lane;
        const bool tv = t < G.T;
        uint32_t x0 = 0, y0 = 0;
        if (tv) tile_origin<K, S>(G, t, x0, y0);
        uint32_t mine = 0;
        for (uint32_t cc = 0; cc < 32; ++cc) {
            const uint32_t i = i0 + cc;
            bool alive = false;
            if (tv && i < G.Cl) {
                const uint32_t l = __ldg(loc + i);
                if (l != kNoLoc) alive = cell_alive_mixed(seed_mix, x0 + (l & 0xFFFFu), y0 + (l >> 16), density);
            }
            const uint32_t word = __ballot_sync(0xFFFFFFFFu, alive);
            if (lane == cc) mine = word;
        }
        if (i0 + lane < G.Cl) P[(uint64_t)g * G.Cp + i0 + lane] = mine;
    }
}

// Simulation::state_hash (stencil.cpp:207-216) over the groups [g0, g1).
template <int K, int S>
__global__ void hash_packed_kernel(PackedGeom G, const uint32_t* __restrict__ loc, const uint32_t* __restrict__ P,
                                   uint32_t g0, uint32_t g1, unsigned long long* out) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t cpw = (G.Cl + 31) / 32;
    const uint64_t nw = (uint64_t)(g1 - g0) * cpw;
    uint64_t acc = 0;
    for (uint64_t wi = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; wi < nw;
         wi += ((uint64_t)gridDim.x * blockDim.x) >> 5) {
        const uint32_t g = g0 + (uint32_t)(wi / cpw), i0 = (uint32_t)(wi % cpw) * 32;
        const uint32_t t = g * 32 + lane;
        const bool tv = t < G.T;
        uint32_t x0 = 0, y0 = 0;
        if (tv) tile_origin<K, S>(G, t, x0, y0);
        const uint32_t l_mine = i0 + lane < G.Cl ? __ldg(loc + i0 + lane) : kNoLoc;
        const uint32_t mine = l_mine != kNoLoc ? P[(uint64_t)g * G.Cp + i0 + lane] : 0u;
        for (uint32_t cc = 0; cc < 32; ++cc) {
            const uint32_t word = __shfl_sync(0xFFFFFFFFu, mine, cc);
            const uint32_t l = __shfl_sync(0xFFFFFFFFu, l_mine, cc);
            if (tv && ((word >> lane) & 1u)) acc += coord_mix(x0 + (l & 0xFFFFu), y0 + (l >> 16));
        }
    }
    block_sum_atomic(acc, out);
}

// ---- reference bytes <-> packed -----------------------------------------------
// Warp per (group, local row a).  Row a of the group's 32 tiles is at most two
// contiguous byte runs of the reference layout (tiles of one coarse row are
// adjacent: tile X's row a is bytes [X*WQ, X*WQ + WQ) of compact row Y*WQ + a), so
// the bytes move with coalesced 4-byte accesses through a per-warp shared buffer
// of 32 * WQ bytes; the bit transposition happens in shared memory.  `bytes` holds
// compact rows starting at compact row Y0 * WQ and may be pinned host memory
// (zero-copy over PCIe) or device memory.
constexpr int kConvWarps = 4;

// copy n bytes between global g and shared s (both arbitrary alignment), warp-wide;
// the global side is accessed as aligned 32-bit words wherever possible
template <bool TO_SHARED>
__device__ __forceinline__ void warp_copy_run(uint8_t* sbuf, uint8_t* gptr, uint32_t n, uint32_t lane) {
    const uint32_t head = min(n, (uint32_t)((4 - ((uintptr_t)gptr & 3)) & 3));
    const uint32_t nw = (n - head) / 4;
    const uint32_t tail0 = head + nw * 4;
    if (lane < head) {
        if (TO_SHARED) sbuf[lane] = gptr[lane]; else gptr[lane] = sbuf[lane];
    }
    uint32_t* gw = reinterpret_cast<uint32_t*>(gptr + head);
    for (uint32_t k = lane; k < nw; k += 32) {
        uint8_t* sp = sbuf + head + 4 * k;
        if (TO_SHARED) {
            const uint32_t v = gw[k];
            sp[0] = (uint8_t)v; sp[1] = (uint8_t)(v >> 8); sp[2] = (uint8_t)(v >> 16); sp[3] = (uint8_t)(v >> 24);
        } else {
            gw[k] = (uint32_t)sp[0] | ((uint32_t)sp[1] << 8) | ((uint32_t)sp[2] << 16) | ((uint32_t)sp[3] << 24);
        }
    }
    if (tail0 + lane < n) {
        if (TO_SHARED) sbuf[tail0 + lane] = gptr[tail0 + lane]; else gptr[tail0 + lane] = sbuf[tail0 + lane];
    }
}

// the (at most two) runs of group g's tiles within [tlo, thi): calls f(first tile,
// tile count) for each maximal set of valid tiles in one coarse row
template <class F>
__device__ __forceinline__ void for_each_run(const PackedGeom& G, uint32_t g, uint32_t tlo, uint32_t thi, F&& f) {
    uint32_t t = max(g * 32, tlo);
    const uint32_t tend = min(min(g * 32 + 32, thi), G.T);
    while (t < tend) {
        const uint32_t rowend = (t / G.Wc + 1) * G.Wc;
        const uint32_t e = min(tend, rowend);
        f(t, e - t);
        __syncwarp();
        t = e;
    }
}

// BITS: the chunk arrives as a bit array (bit i = reference byte i of the chunk,
// packed on the host: 8x fewer PCIe bytes); otherwise as the reference bytes
__device__ __forceinline__ void warp_bits_to_shared(uint8_t* sbuf, const uint32_t* bits, uint64_t off, uint32_t n,
                                                    uint32_t lane) {
    for (uint32_t k = lane; k < n; k += 32) {
        const uint64_t b = off + k;
        sbuf[k] = (uint8_t)((__ldg(bits + (b >> 5)) >> (b & 31)) & 1u);
    }
}
// bytes sbuf[0, n) -> bits [off, off + n) of a zeroed bit array: whole words stored,
// the (at most two) words shared with a neighbouring run or-ed atomically
__device__ __forceinline__ void warp_shared_to_bits(const uint8_t* sbuf, uint32_t* bits, uint64_t off, uint32_t n,
                                                    uint32_t lane) {
    const uint64_t w0 = off >> 5, w1 = (off + n + 31) >> 5;
    for (uint64_t w = w0; w < w1; ++w) {
        const uint64_t b = w * 32 + lane;
        const bool in = b >= off && b < off + n;
        const uint32_t word = __ballot_sync(0xFFFFFFFFu, in && sbuf[b - off] != 0);
        const uint32_t mask = __ballot_sync(0xFFFFFFFFu, in);
        if (lane == 0) {
            if (mask == 0xFFFFFFFFu) bits[w] = word;
            else if (word) atomicOr(bits + w, word);
        }
    }
}

template <bool BITS>
__global__ void __launch_bounds__(kConvWarps * 32)
pack_kernel(PackedGeom G, const uint8_t* __restrict__ bytes, uint32_t Y0, uint32_t Y1, uint32_t* __restrict__ P,
            int* __restrict__ bad) {
    extern __shared__ __align__(16) uint8_t conv_sm[];
    const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    uint8_t* sb = conv_sm + wib * 32 * G.WQ;
    const uint32_t tlo = Y0 * G.Wc, thi = Y1 * G.Wc;
    const uint32_t glo = tlo / 32, ghi = (thi + 31) / 32;
    const uint64_t nw = (uint64_t)(ghi - glo) * G.WQ;
    for (uint64_t wi = blockIdx.x * (uint64_t)kConvWarps + wib; wi < nw; wi += (uint64_t)gridDim.x * kConvWarps) {
        const uint32_t g = glo + (uint32_t)(wi / G.WQ), a = (uint32_t)(wi % G.WQ);
        for (uint32_t k = lane; k < 32 * G.WQ; k += 32) sb[k] = 0;
        __syncwarp();
        for_each_run(G, g, tlo, thi, [&](uint32_t t0, uint32_t n) {
            const uint32_t X = t0 % G.Wc, Y = t0 / G.Wc;
            const uint64_t off = ((uint64_t)(Y - Y0) * G.WQ + a) * G.w + (uint64_t)X * G.WQ;
            if constexpr (BITS)
                warp_bits_to_shared(sb + (t0 - g * 32) * G.WQ, reinterpret_cast<const uint32_t*>(bytes), off,
                                    n * G.WQ, lane);
            else
                warp_copy_run<true>(sb + (t0 - g * 32) * G.WQ, const_cast<uint8_t*>(bytes) + off, n * G.WQ, lane);
        });
        __syncwarp();
        uint32_t lanes = 0;  // tiles of this group inside [tlo, thi)
        {
            const uint32_t t = g * 32 + lane;
            lanes = __ballot_sync(0xFFFFFFFFu, t >= tlo && t < thi && t < G.T);
        }
        uint32_t* R = P + (uint64_t)g * G.Cp;
        for (uint32_t c = lane; c < ((G.WQ + 31) & ~31u); c += 32) {
            uint32_t word = 0, over = 0;
            if (c < G.WQ) {
#pragma unroll 8
                for (uint32_t b = 0; b < 32; ++b) {
                    const uint32_t v = sb[b * G.WQ + c];
                    word |= (v != 0 ? 1u : 0u) << b;
                    over |= v > 1 ? 1u : 0u;
                }
                word &= lanes;
                if (over) *bad = 1;
                // groups shared with a neighbouring row chunk keep the other tiles' bits
                uint32_t& Rw = R[rec_word(G.ilv, G.WQ, a, c)];
                Rw = lanes == 0xFFFFFFFFu ? word : ((Rw & ~lanes) | word);
            }
        }
        __syncwarp();
    }
}

template <bool BITS>
__global__ void __launch_bounds__(kConvWarps * 32)
unpack_kernel(PackedGeom G, const uint32_t* __restrict__ P, uint32_t Y0, uint32_t Y1, uint8_t* __restrict__ bytes) {
    extern __shared__ __align__(16) uint8_t conv_sm[];
    const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    uint8_t* sb = conv_sm + wib * 32 * G.WQ;
    const uint32_t tlo = Y0 * G.Wc, thi = Y1 * G.Wc;
    const uint32_t glo = tlo / 32, ghi = (thi + 31) / 32;
    const uint64_t nw = (uint64_t)(ghi - glo) * G.WQ;
    for (uint64_t wi = blockIdx.x * (uint64_t)kConvWarps + wib; wi < nw; wi += (uint64_t)gridDim.x * kConvWarps) {
        const uint32_t g = glo + (uint32_t)(wi / G.WQ), a = (uint32_t)(wi % G.WQ);
        const uint32_t* R = P + (uint64_t)g * G.Cp;
        for (uint32_t c = lane; c < G.WQ; c += 32) {
            const uint32_t word = R[rec_word(G.ilv, G.WQ, a, c)];
#pragma unroll 8
            for (uint32_t b = 0; b < 32; ++b) sb[b * G.WQ + c] = (uint8_t)((word >> b) & 1u);
        }
        __syncwarp();
        for_each_run(G, g, tlo, thi, [&](uint32_t t0, uint32_t n) {
            const uint32_t X = t0 % G.Wc, Y = t0 / G.Wc;
            const uint64_t off = ((uint64_t)(Y - Y0) * G.WQ + a) * G.w + (uint64_t)X * G.WQ;
            if constexpr (BITS)
                warp_shared_to_bits(sb + (t0 - g * 32) * G.WQ, reinterpret_cast<uint32_t*>(bytes), off, n * G.WQ, lane);
            else
                warp_copy_run<false>(sb + (t0 - g * 32) * G.WQ, bytes + off, n * G.WQ, lane);
        });
        __syncwarp();
    }
}

}  // namespace nbbgpu
