// nbbgpu.cu -- the C ABI of include/nbbgpu.h: handle, device memory, dispatch.
//
// Host side of the drop-in: what nbb::Simulation (proj/src/stencil.cpp) does on
// the CPU, done here with device buffers and the kernels of naive.cuh, tiled.cuh
// and maps.cuh.  No CPU fallback exists: every state transition runs on the GPU.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <immintrin.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <functional>
#include <thread>
#include <cstring>
#include <exception>
#include <map>
#include <mutex>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/nbbgpu.h"
#include "common.cuh"
#include "maps.cuh"
#include "tc05.cuh"
#include "bb.cuh"
#include "naive.cuh"
#include "tiled.cuh"
#include "packed.cuh"
#include "layouts.cuh"

using namespace nbbgpu;

namespace {

thread_local std::string g_err;

struct NbbError : std::runtime_error {
    int code;
    NbbError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] void raise(int code, const std::string& m) { throw NbbError(code, m); }

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        if (e == cudaErrorMemoryAllocation)
            raise(NBBGPU_ERR_CAPACITY, std::string(what) + ": device memory exhausted (memory cap)");
        raise(NBBGPU_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
    }
}
#define CK(x) cuda_check((x), #x)

template <class F>
int guarded(F&& f) {
    try {
        f();
        return NBBGPU_OK;
    } catch (const NbbError& e) {
        g_err = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        g_err = "host allocation failed";
        return NBBGPU_ERR_CAPACITY;
    } catch (const std::exception& e) {
        g_err = e.what();
        return NBBGPU_ERR_CUDA;
    }
}

// ---------------------------------------------------------------------------
// Host mirror of CoordMapper (maps.cpp:45-146) for set/get_cell and the tables.
// ---------------------------------------------------------------------------
struct HostFrac {
    int k = 0, s = 0, r = 0;
    int64_t side = 1, w = 1, h = 1;
    std::vector<int> id;  // s*s
    std::vector<int> gx, gy;
    std::vector<int64_t> spow;

    static int64_t ipow(int64_t b, int e) {
        int64_t r = 1;
        for (int i = 0; i < e; ++i) {
            if (b != 0 && r > INT64_MAX / b) raise(NBBGPU_ERR_CAPACITY, "integer overflow computing " + std::to_string(b) + "^" + std::to_string(e));
            r *= b;
        }
        return r;
    }

    void init(const int32_t* rep, int k_, int s_, int r_) {
        // FractalDescriptor::validate (descriptor.cpp:12-44)
        if (k_ < 1) raise(NBBGPU_ERR_PARSE, "descriptor: k must be >= 1, got " + std::to_string(k_));
        if (s_ < 2) raise(NBBGPU_ERR_PARSE, "descriptor: invalid growth factor s=" + std::to_string(s_) + " (s >= 2 required)");
        if ((int64_t)k_ > (int64_t)s_ * s_) raise(NBBGPU_ERR_PARSE, "descriptor: k=" + std::to_string(k_) + " exceeds s*s=" + std::to_string(s_ * s_));
        if (s_ > kMaxS) raise(NBBGPU_ERR_OUT_OF_DOMAIN, "growth factor s=" + std::to_string(s_) + " exceeds the engine limit of 16");
        if (r_ < 0) raise(NBBGPU_ERR_OUT_OF_DOMAIN, "scale level must be >= 0");
        k = k_; s = s_; r = r_;
        id.assign(s * s, -1);
        gx.resize(k);
        gy.resize(k);
        for (int i = 0; i < k; ++i) {
            const int x = rep[2 * i], y = rep[2 * i + 1];
            if (x < 0 || y < 0 || x >= s || y >= s)
                raise(NBBGPU_ERR_PARSE, "descriptor: replica " + std::to_string(i) + " position (" + std::to_string(x) + "," + std::to_string(y) + ") outside the " + std::to_string(s) + "x" + std::to_string(s) + " grid");
            if (id[y * s + x] >= 0)
                raise(NBBGPU_ERR_PARSE, "descriptor: duplicate replica position (" + std::to_string(x) + "," + std::to_string(y) + ")");
            id[y * s + x] = i;
            gx[i] = x;
            gy[i] = y;
        }
        side = ipow(s, r);
        w = ipow(k, (r + 1) / 2);
        h = ipow(k, r / 2);
        spow.resize(r + 1);
        spow[0] = 1;
        for (int mu = 0; mu < r; ++mu) spow[mu + 1] = spow[mu] * s;
    }
    // try_to_compact at level `lev` (maps.cpp:80-107)
    bool nu(int64_t x, int64_t y, int64_t& cx, int64_t& cy, int lev) const {
        int64_t ax = 0, ay = 0, p = 1;
        for (int mu = 0; mu < lev; ++mu) {
            const int i = id[(y % s) * s + (x % s)];
            if (i < 0) return false;
            if ((mu & 1) == 0) ax += i * p;
            else { ay += i * p; p *= k; }
            x /= s;
            y /= s;
        }
        cx = ax;
        cy = ay;
        return true;
    }
    // to_embedded at level `lev` (maps.cpp:123-146)
    void lambda(int64_t cx, int64_t cy, int64_t& x, int64_t& y, int lev) const {
        int64_t ex = 0, ey = 0, sp = 1;
        for (int mu = 0; mu < lev; ++mu) {
            int d;
            if ((mu & 1) == 0) { d = (int)(cx % k); cx /= k; }
            else { d = (int)(cy % k); cy /= k; }
            ex += gx[d] * sp;
            ey += gy[d] * sp;
            sp *= s;
        }
        x = ex;
        y = ey;
    }
    // host twin of coarse_neighbor (tiled.cuh)
    bool coarse_neighbor(int L, int64_t X, int64_t Y, int dx, int dy, int64_t& X2, int64_t& Y2) const {
        int64_t cx = X, cy = Y, pw = 1, nx = X, ny = Y;
        for (int mu = 0; mu < L; ++mu) {
            if (dx == 0 && dy == 0) break;
            int d;
            if ((mu & 1) == 0) { d = (int)(cx % k); cx /= k; }
            else { d = (int)(cy % k); cy /= k; }
            int ggx = gx[d] + dx, ggy = gy[d] + dy;
            dx = ggx < 0 ? -1 : (ggx >= s ? 1 : 0);
            ggx -= dx * s;
            dy = ggy < 0 ? -1 : (ggy >= s ? 1 : 0);
            ggy -= dy * s;
            const int i2 = id[ggy * s + ggx];
            if (i2 < 0) return false;
            if ((mu & 1) == 0) nx += (int64_t)(i2 - d) * pw;
            else { ny += (int64_t)(i2 - d) * pw; pw *= k; }
        }
        X2 = nx;
        Y2 = ny;
        return dx == 0 && dy == 0;
    }
};

// ---------------------------------------------------------------------------
// Tile plan (tiled.cuh): local neighbour table + halo slots for tile level q.
// ---------------------------------------------------------------------------
struct TilePlan {
    int q = 0, wq = 1, C = 1, nH = 0, L = 0;
    int64_t Wc = 0, Hc = 0;
    uint32_t dmask = 0;
    std::vector<uint32_t> nbr;  // C*8 byte offsets
    std::vector<uint8_t> hD;
    std::vector<uint16_t> ha, hc;
    uint16_t first[10] = {0};
    uint32_t wpg = 0, smem_per_warp = 0;
    int G = 1;
    int nD = 0;
    int8_t dlist[8] = {0};
    std::vector<uint8_t> hDslot;  // per slot: index into dlist
};

const int kOff[8][2] = {{1, 0}, {-1, 0}, {0, 1}, {0, -1}, {1, 1}, {1, -1}, {-1, 1}, {-1, -1}};

TilePlan build_plan(const HostFrac& F, int q, int deg) {
    TilePlan P;
    P.q = q;
    P.wq = (int)HostFrac::ipow(F.k, q / 2);
    P.C = P.wq * P.wq;
    P.L = F.r - q;
    P.Wc = F.w / P.wq;
    P.Hc = F.h / P.wq;
    const int64_t tside = F.spow[q];
    struct Slot { int D, a, c; };
    std::vector<Slot> slots;
    std::map<std::tuple<int, int, int>, int> slot_of;
    std::vector<std::vector<int>> raw(P.C);  // neighbour: >= 0 local, < 0 -> -(slot+1), absent skipped
    for (int i = 0; i < P.C; ++i) {
        const int c = i % P.wq, a = i / P.wq;
        int64_t lx, ly;
        F.lambda(c, a, lx, ly, q);
        for (int j = 0; j < deg; ++j) {
            int64_t nx = lx + kOff[j][0], ny = ly + kOff[j][1];
            const int Dx = nx < 0 ? -1 : (nx >= tside ? 1 : 0);
            const int Dy = ny < 0 ? -1 : (ny >= tside ? 1 : 0);
            int64_t ncx, ncy;
            if (!F.nu(nx - Dx * tside, ny - Dy * tside, ncx, ncy, q)) continue;  // hole
            if (Dx == 0 && Dy == 0) {
                raw[i].push_back((int)(ncy * P.wq + ncx));
            } else {
                const int D = (Dy + 1) * 3 + (Dx + 1);
                auto key = std::make_tuple(D, (int)ncy, (int)ncx);
                auto it = slot_of.find(key);
                int sidx;
                if (it == slot_of.end()) {
                    sidx = (int)slots.size();
                    slot_of[key] = sidx;
                    slots.push_back({D, (int)ncy, (int)ncx});
                } else {
                    sidx = it->second;
                }
                raw[i].push_back(-(sidx + 1));
            }
        }
    }
    // sort slots by D, renumber
    std::vector<int> order(slots.size());
    for (size_t i = 0; i < order.size(); ++i) order[i] = (int)i;
    std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return slots[x].D < slots[y].D; });
    std::vector<int> newidx(slots.size());
    for (size_t i = 0; i < order.size(); ++i) newidx[order[i]] = (int)i;
    P.nH = (int)slots.size();
    if (P.nH > kMaxHalo) raise(NBBGPU_ERR_OUT_OF_DOMAIN, "tile halo too large");
    P.hD.resize(P.nH);
    P.ha.resize(P.nH);
    P.hc.resize(P.nH);
    for (int i = 0; i < P.nH; ++i) {
        const Slot& s = slots[order[i]];
        P.hD[i] = (uint8_t)s.D;
        P.ha[i] = (uint16_t)s.a;
        P.hc[i] = (uint16_t)s.c;
        P.dmask |= 1u << s.D;
    }
    for (int D = 0; D <= 9; ++D) {
        int cnt = 0;
        for (int i = 0; i < P.nH; ++i) cnt += P.hD[i] < D;
        P.first[D] = (uint16_t)cnt;
    }
    for (int D = 0; D < 9; ++D)
        if ((P.dmask >> D) & 1u) P.dlist[P.nD++] = (int8_t)D;
    P.hDslot.resize(P.nH);
    for (int i = 0; i < P.nH; ++i)
        for (int ds = 0; ds < P.nD; ++ds)
            if (P.dlist[ds] == P.hD[i]) P.hDslot[i] = (uint8_t)ds;
    const uint32_t zero_word = (uint32_t)(P.C + P.nH);
    P.nbr.assign((size_t)P.C * 8, zero_word * 4);
    for (int i = 0; i < P.C; ++i)
        for (size_t j = 0; j < raw[i].size(); ++j) {
            const int v = raw[i][j];
            const uint32_t word = v >= 0 ? (uint32_t)v : (uint32_t)(P.C + newidx[-v - 1]);
            P.nbr[(size_t)i * 8 + j] = word * 4;
        }
    P.wpg = (uint32_t)((P.C + P.nH + 1 + 3) & ~3);
    P.G = std::max(1, 32 / P.wq);
    // per warp: G x word arrays, G x 8 x 32 packed neighbour tiles, 32 cp.async rings
    P.smem_per_warp = tiled_smem_per_warp(P.wq, P.wpg);
    return P;
}

bool tiled_width_supported(int wq) {
    switch (wq) {
        case 3: case 4: case 5: case 7: case 8: case 9: case 12: case 16: case 25: case 27: return true;
        default: return false;
    }
}

// Largest even q <= r with a supported tile width and k^q <= 1024 cells.
int choose_tile_level(const HostFrac& F) {
    int best = 0;
    for (int q = 2; q <= F.r; q += 2) {
        int64_t wq = 1;
        bool ok = true;
        for (int i = 0; i < q / 2; ++i) {
            wq *= F.k;
            if (wq > 32) { ok = false; break; }
        }
        if (!ok) break;
        if (wq * wq > 1024) break;
        // the kernel packs coarse tile coordinates into 16 bits each
        if (F.w / wq > 65535 || F.h / wq > 65535) continue;
        if (tiled_width_supported((int)wq)) best = q;
    }
    return best;
}


#include "jit.inc"
#include "packed_plan.inc"

}  // namespace

// ---------------------------------------------------------------------------
// the handle
// ---------------------------------------------------------------------------
struct nbbgpu_sim {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    HostFrac hf;
    Frac frac{};
    MmaTables mt{};
    int mode = NBBGPU_MODE_COMPACT;
    BlockedGeom bg{};          // NBBGPU_MODE_BLOCKED: block size rho = s^m, coarse tables
    uint32_t* d_lowmask = nullptr;  // filler mask of one block (rho^2 bits)
    uint32_t* d_blocktab = nullptr; // per block: neighbour blocks + coarse corner
    // NBBGPU_MODE_BB row-streaming kernel (bb.cuh): doubled low table + coarse bitmap
    uint32_t* d_bblow = nullptr;
    uint32_t* d_bbcoarse = nullptr;
    uint2* d_bbtiles = nullptr;     // live (strip, band) tiles
    uint32_t* d_bbmemb = nullptr;   // membership bitmap of the box (bit = linear byte)
    uint32_t bb_ntiles = 0;
    BBRowParams bbp{};
    bool bb_ready = false;
    uint64_t cells = 0;      // stored cells per buffer
    uint8_t* buf[2] = {nullptr, nullptr};
    int cur = 0;             // front = buf[cur]
    int64_t iteration = 0;
    unsigned long long* d_acc = nullptr;
    int* d_flag = nullptr;
    // host <-> device bit-array staging (hostconv.inc): pinned host + device chunk
    // buffers, a copy stream, per-buffer copy / conversion events
    uint32_t* xb_host[2] = {nullptr, nullptr};
    uint32_t* xb_dev[2] = {nullptr, nullptr};
    uint64_t xb_words = 0;
    cudaStream_t xb_stream = nullptr;
    cudaEvent_t xb_dma[2] = {nullptr, nullptr}, xb_conv[2] = {nullptr, nullptr};
    int kernel = NBBGPU_KERNEL_AUTO;
    int map_variant = NBBGPU_MAP_DIGIT;
    uint64_t bytes_held = 0;
    // tiling
    int q = 0;               // chosen tile level (0 = none)
    TilePlan plan[2];        // [moore]
    bool plan_built[2] = {false, false};
    uint32_t* d_nbr[2] = {nullptr, nullptr};
    uint32_t* d_ntab[2] = {nullptr, nullptr};  // coarse neighbour tiles [nD][Hc][Wc]
    uint8_t* d_hD[2] = {nullptr, nullptr};
    uint16_t* d_ha[2] = {nullptr, nullptr};
    uint16_t* d_hc[2] = {nullptr, nullptr};
    uint64_t* d_hoff[2] = {nullptr, nullptr};
    // partition (rows of the partition unit: tiles when q > 0, compact rows otherwise)
    int rank = 0, nranks = 1;
    int part_q = 0;           // tile level the partition is expressed in
    bool part_packed = false; // partition unit = packed groups, halo elements = boundary words
    int64_t unit_rows = 1;    // compact rows per partition row (k^(q/2))
    int64_t prow0 = 0, prow1 = 0;  // owned partition rows
    std::vector<std::vector<uint64_t>> needs;   // per peer: offsets I need from peer
    std::vector<uint64_t*> d_sends;             // per peer: offsets peer needs from me
    std::vector<uint64_t> n_sends;
    std::vector<uint64_t*> d_recvs;             // per peer: offsets I receive from peer
    std::vector<uint64_t> n_recvs;
    // in-library NCCL transport (nbbgpu_comm_init)
    ncclComm_t comm = nullptr;
    // peer-memory halo transport (nbbgpu_p2p_export / nbbgpu_p2p_attach)
    bool p2p = false;
    uint32_t* d_pcnt = nullptr;             // my arrival counter (exported by IPC)
    uint32_t p2p_epoch = 0, p2p_nsrc = 0, p2p_send_mask = 0;
    uint64_t* d_p2p_elems = nullptr;        // boundary elements peers need from me
    // fused push (triangle step kernels): per owned group its (slot | peer << 16) entries
    uint32_t* d_push_off = nullptr;
    uint32_t* d_push_ent = nullptr;
    unsigned* d_push_done = nullptr;
    bool fused_push = false;                // the last step kernel pushed and signalled
    uint8_t* d_p2p_peer = nullptr;          // ... and which peer
    uint64_t p2p_n = 0;
    uint32_t** d_peer_bnd[2] = {nullptr, nullptr};  // per rank: mapped boundary planes
    uint32_t** d_peer_cnt = nullptr;                // per rank: mapped arrival counters
    std::vector<void*> ipc_opened;
    uint64_t* d_send_all = nullptr;             // concatenated per-peer send offsets
    uint64_t* d_recv_all = nullptr;
    uint8_t* d_sendbuf = nullptr;
    uint8_t* d_recvbuf = nullptr;
    uint64_t n_send_all = 0, n_recv_all = 0;

    // packed layout (packed.cuh): state bit-sliced over groups of 32 tiles
    int layout = 0;                 // 0 = reference bytes (buf), 1 = packed (pk, bnd)
    int pq = -1;                    // packed tile level (-1: unavailable)
    PackedPlan pp;
    bool pp_built = false;
    uint32_t* pk[2] = {nullptr, nullptr};   // packed state, NG * Cp words
    uint32_t* bnd[2] = {nullptr, nullptr};  // boundary planes, NG * nSrc words
    void* d_pnbr[2] = {nullptr, nullptr};   // [moore] neighbour offsets
    uint32_t* d_pslot = nullptr;
    uint32_t* d_pntab = nullptr;            // [nD][T] linear neighbour tiles
    uint32_t* d_psrc = nullptr;
    uint32_t* d_ploc = nullptr;
    uint32_t* d_pbtab = nullptr;            // micro-block external offsets
    uint32_t* d_phalo = nullptr;            // per step: halo words [NG][nHp]
    uint32_t* d_pbt = nullptr;              // transposed boundary plane (wide halos, single GPU) of pk[0]
    uint32_t* d_pbt1 = nullptr;             // ... of pk[1] (bt_buf)
    uint32_t* d_pdmask = nullptr;           // [nHc][8] direction masks per 32-slot chunk
    BtMasks bt_masks{};  // the same masks by value (halo_bt_regs_kernel)
    uint64_t packed_table_bytes = 0;
    int64_t pg0 = 0, pg1 = 0;               // owned groups
    // profiling (nbbgpu_step_profiled): events around each main step kernel, launch count
    std::vector<cudaEvent_t>* prof = nullptr;  // pre-created pool
    size_t prof_idx = 0;
    uint64_t launches = 0;
    // NBBGPU_KERNEL_TABLE: neighbour table tab[j * cells + i] (u32 or u64 slots)
    void* d_tab = nullptr;
    int tab_deg = 0;
    int cluster_fit[2] = {-1, -1};          // 8- / 16-CTA resident clusters fit (-1: not queried)
    // transposed-plane steps (step kernel writes Bt, not B): the front's Bt is valid /
    // the front's B was not written (bnd_refresh rebuilds it before any B reader)
    bool bt_front = false;
    bool bnd_stale = false;
    // multi-step calls: captured CUDA graphs of kGraphSteps steps (step_impl)
    struct StepGraph {
        uint16_t birth, survive;
        int moore, cur, kernel;
        std::string env;  // the per-call tuning knobs the capture saw
        cudaGraphExec_t exec;
        uint64_t launches;
    };
    std::vector<StepGraph> graphs;

    uint8_t* front() const { return buf[cur]; }
    uint8_t* back() const { return buf[cur ^ 1]; }
};

namespace {

int grid_for(uint64_t n, int block) {
    uint64_t g = (n + block - 1) / block;
    return (int)std::max<uint64_t>(1, std::min<uint64_t>(g, 148ull * 32));
}

void check_handle(nbbgpu_t h) {
    if (!h) raise(NBBGPU_ERR_INVALID, "null nbbgpu handle");
    CK(cudaSetDevice(h->device));
}

// (k, s) specialisations for the digit loops (constant divisors); 0,0 = runtime.
#define NBB_DISPATCH_KS(F, ...)                                              \
    do {                                                                     \
        const int _k = (F).k, _s = (F).s;                                    \
        if (_k == 3 && _s == 2) { NBB_CALL(3, 2, __VA_ARGS__); }             \
        else if (_k == 8 && _s == 3) { NBB_CALL(8, 3, __VA_ARGS__); }        \
        else if (_k == 5 && _s == 3) { NBB_CALL(5, 3, __VA_ARGS__); }        \
        else if (_k == 7 && _s == 3) { NBB_CALL(7, 3, __VA_ARGS__); }        \
        else if (_k == 12 && _s == 4) { NBB_CALL(12, 4, __VA_ARGS__); }      \
        else if (_k == 4 && _s == 2) { NBB_CALL(4, 2, __VA_ARGS__); }        \
        else { NBB_CALL(0, 0, __VA_ARGS__); }                                \
    } while (0)

void ensure_plan(nbbgpu_t h, int moore) {
    if (h->q == 0 || h->plan_built[moore]) return;
    TilePlan P = build_plan(h->hf, h->q, moore ? 8 : 4);
    CK(cudaMalloc(&h->d_nbr[moore], P.nbr.size() * 4));
    CK(cudaMemcpy(h->d_nbr[moore], P.nbr.data(), P.nbr.size() * 4, cudaMemcpyHostToDevice));
    const size_t nh = std::max<size_t>(1, P.hD.size());
    CK(cudaMalloc(&h->d_hD[moore], nh));
    CK(cudaMalloc(&h->d_ha[moore], nh * 2));
    CK(cudaMalloc(&h->d_hc[moore], nh * 2));
    CK(cudaMalloc(&h->d_hoff[moore], nh * 8));
    if (P.nH) {
        std::vector<uint64_t> off(P.nH);
        for (int j = 0; j < P.nH; ++j) off[j] = (uint64_t)P.ha[j] * (uint64_t)h->hf.w + P.hc[j];
        CK(cudaMemcpy(h->d_hoff[moore], off.data(), P.nH * 8, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(h->d_hD[moore], P.hDslot.data(), P.nH, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(h->d_ha[moore], P.ha.data(), P.nH * 2, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(h->d_hc[moore], P.hc.data(), P.nH * 2, cudaMemcpyHostToDevice));
    }
    h->bytes_held += P.nbr.size() * 4 + nh * 5;
    // static coarse-neighbour table (Wc, Hc < 65536 by choose_tile_level)
    const uint64_t ntiles = (uint64_t)P.Wc * P.Hc;
    const size_t tbytes = std::max<size_t>(4, (size_t)P.nD * ntiles * 4);
    if (cudaMalloc(&h->d_ntab[moore], tbytes) != cudaSuccess) {
        cudaGetLastError();
        raise(NBBGPU_ERR_CAPACITY, "coarse neighbour table exceeds the device memory (memory cap)");
    }
    h->bytes_held += tbytes;
    if (P.nD > 0) {
        const int8_t* d = P.dlist;
#define NBB_CALL(K, S, ...) build_ntab_kernel<K, S><<<grid_for(ntiles, 256), 256, 0, h->stream>>>(h->frac, P.L, (uint32_t)P.Wc, (uint32_t)P.Hc, P.nD, d[0], d[1], d[2], d[3], d[4], d[5], d[6], d[7], h->d_ntab[moore])
        NBB_DISPATCH_KS(h->hf);
#undef NBB_CALL
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(h->stream));
    }
    h->plan[moore] = std::move(P);
    h->plan_built[moore] = true;
}

// Below this many compact cells the one-thread-per-cell kernel wins: the tiled
// kernel's per-group chain (~16 us) dominates tiny levels (measured on B200:
// T r=10 naive 12 us vs tiled 17 us; r=11 equal; r=12 naive 43 us vs tiled 19 us).
constexpr uint64_t kTiledMinCells = 1ull << 17;

bool is_device_ptr(const void* p);

int resolve_kernel_for(nbbgpu_t h, int kernel) {
    if (h->mode != NBBGPU_MODE_COMPACT) return NBBGPU_KERNEL_NAIVE;  // bb, lambda, blocked
    if (kernel == NBBGPU_KERNEL_NAIVE) return NBBGPU_KERNEL_NAIVE;
    if (kernel == NBBGPU_KERNEL_TABLE) return NBBGPU_KERNEL_TABLE;
    if (kernel == NBBGPU_KERNEL_PACKED) {
        if (h->pq < 2) raise(NBBGPU_ERR_OUT_OF_DOMAIN, "no packed tile level for this fractal/level");
        return NBBGPU_KERNEL_PACKED;
    }
    if (kernel == NBBGPU_KERNEL_AUTO && h->pq >= 2) return NBBGPU_KERNEL_PACKED;
    if (h->q > 0 && (kernel == NBBGPU_KERNEL_TILED || h->cells >= kTiledMinCells))
        return NBBGPU_KERNEL_TILED;
    if (kernel == NBBGPU_KERNEL_TILED) raise(NBBGPU_ERR_OUT_OF_DOMAIN, "no tile level for this fractal/level");
    return NBBGPU_KERNEL_NAIVE;
}
int resolve_kernel(nbbgpu_t h) { return resolve_kernel_for(h, h->kernel); }

// event pair around the main step kernel when profiling (nbbgpu_step_profiled)
void prof_mark(nbbgpu_t h) {
    if (!h->prof || h->prof_idx >= h->prof->size()) return;
    CK(cudaEventRecord((*h->prof)[h->prof_idx++], h->stream));
}
int layout_of_kernel(int k) { return k == NBBGPU_KERNEL_PACKED ? 1 : 0; }

// Kernel attributes (opt-in shared memory, non-portable clusters) are per device:
// set them once per (kernel, device) pair.  Thread-safe; several handles on
// several devices share the registry.
bool attr_needed(const void* fn, int device) {
    static std::mutex mu;
    static std::set<std::pair<const void*, int>> done;
    std::lock_guard<std::mutex> g(mu);
    return done.insert({fn, device}).second;
}
template <class K>
void smem_attr(nbbgpu_t h, K kern, int bytes, bool nonportable_cluster = false) {
    if (!attr_needed((const void*)kern, h->device)) return;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    if (nonportable_cluster) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
}

#include "hostconv.inc"
#include "packed_host.inc"

template <int WQ, int K, int S, bool CONWAY>
void launch_tiled_t(nbbgpu_t h, const TiledParams& p, const uint8_t* src, uint8_t* dst) {
    auto kern = step_tiled_kernel<WQ, K, S, CONWAY>;
    const size_t smem = (size_t)p.smem_per_warp * kTiledWarps;
    smem_attr(h, kern, 200 * 1024);
    const uint64_t groups = (uint64_t)(p.row1 - p.row0) * p.gpr;
    constexpr int G = (32 / WQ) > 0 ? 32 / WQ : 1;
    const uint64_t warps = (groups + G - 1) / G;
    int blocks_per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, kern, kTiledWarps * 32, smem));
    int sms = 148;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device));
    const uint64_t max_blocks = (uint64_t)std::max(1, blocks_per_sm) * sms;
    const uint64_t blocks = std::max<uint64_t>(1, std::min<uint64_t>((warps + kTiledWarps - 1) / kTiledWarps, max_blocks));
    kern<<<(unsigned)blocks, kTiledWarps * 32, smem, h->stream>>>(p, src, dst);
}

template <bool CONWAY>
void launch_tiled_w(nbbgpu_t h, int wq, const TiledParams& p, const uint8_t* src, uint8_t* dst) {
    const int k = h->hf.k, s = h->hf.s;
#define NBB_TILE(W, KK, SS) if (wq == W && k == KK && s == SS) return launch_tiled_t<W, KK, SS, CONWAY>(h, p, src, dst)
#define NBB_TILE_ANY(W) if (wq == W) return launch_tiled_t<W, 0, 0, CONWAY>(h, p, src, dst)
    // specialised (k, s): the coarse carry walk divides by constants
    NBB_TILE(27, 3, 2); NBB_TILE(9, 3, 2); NBB_TILE(3, 3, 2);
    NBB_TILE(8, 8, 3); NBB_TILE(25, 5, 3); NBB_TILE(5, 5, 3); NBB_TILE(7, 7, 3);
    NBB_TILE(12, 12, 4); NBB_TILE(16, 4, 2); NBB_TILE(4, 4, 2);
    NBB_TILE_ANY(3); NBB_TILE_ANY(4); NBB_TILE_ANY(5); NBB_TILE_ANY(7); NBB_TILE_ANY(8);
    NBB_TILE_ANY(9); NBB_TILE_ANY(12); NBB_TILE_ANY(16); NBB_TILE_ANY(25); NBB_TILE_ANY(27);
#undef NBB_TILE
#undef NBB_TILE_ANY
    raise(NBBGPU_ERR_OUT_OF_DOMAIN, "unsupported tile width");
}

// owned compact-index range
void owned_range(nbbgpu_t h, uint64_t& lo, uint64_t& hi) {
    if (h->layout == 1) {  // packed words of the owned groups
        lo = (uint64_t)h->pg0 * h->pp.Cp;
        hi = (uint64_t)h->pg1 * h->pp.Cp;
        return;
    }
    if (h->mode != NBBGPU_MODE_COMPACT || h->nranks == 1) {
        lo = 0;
        hi = h->cells;
        return;
    }
    lo = (uint64_t)h->prow0 * h->unit_rows * h->hf.w;
    hi = (uint64_t)h->prow1 * h->unit_rows * h->hf.w;
}

// Simulation::build_neighbor_table (stencil.cpp:401-414): (re)built when the
// neighbourhood's degree changes, like the reference's table_degree_ check
// (stencil.cpp:276-280).  Not covered by the memory cap (the reference's table is
// not either); device OOM -> CapacityError.
void ensure_nbr_table(nbbgpu_t h, int deg) {
    if (h->d_tab && h->tab_deg == deg) return;
    const bool wide = h->cells > 0xFFFFFFFFull;
    const uint64_t bytes = h->cells * (uint64_t)deg * (wide ? 8 : 4);
    if (h->d_tab) {
        CK(cudaStreamSynchronize(h->stream));
        cudaFree(h->d_tab);
        h->bytes_held -= h->cells * (uint64_t)h->tab_deg * (wide ? 8 : 4);
        h->d_tab = nullptr;
        h->tab_deg = 0;
    }
    if (cudaMalloc(&h->d_tab, std::max<uint64_t>(bytes, 8)) != cudaSuccess) {
        cudaGetLastError();
        h->d_tab = nullptr;
        raise(NBBGPU_ERR_CAPACITY, "neighbor table of " + std::to_string(bytes) +
                                       " bytes exceeds the device memory (memory cap)");
    }
    h->bytes_held += bytes;
    if (wide) {
#define NBB_CALL(K, S, ...) build_nbr_table_kernel<K, S, uint64_t><<<grid_for(h->cells, 256), 256, 0, h->stream>>>(h->frac, h->cells, deg, (uint64_t*)h->d_tab)
        NBB_DISPATCH_KS(h->hf);
#undef NBB_CALL
    } else {
#define NBB_CALL(K, S, ...) build_nbr_table_kernel<K, S, uint32_t><<<grid_for(h->cells, 256), 256, 0, h->stream>>>(h->frac, h->cells, deg, (uint32_t*)h->d_tab)
        NBB_DISPATCH_KS(h->hf);
#undef NBB_CALL
    }
    CK(cudaGetLastError());
    h->tab_deg = deg;
}

// tables of the row-streaming BB kernel (bb.cuh), once per handle
void ensure_bb_tables(nbbgpu_t h) {
    if (h->bb_ready) return;
    const HostFrac& F = h->hf;
    const int64_t n = F.side, s = F.s;
    int m = 0;
    int64_t S = 1;
    while (S < 32) { S *= s; ++m; }
    if (m > F.r) raise(NBBGPU_ERR_CUDA, "internal: bounding box below 32 columns");
    BBRowParams& p = h->bbp;
    p = BBRowParams{};
    p.n = (uint64_t)n;
    p.alloc = h->cells + 64;
    p.S = (uint32_t)S;
    p.CW = (uint32_t)(n / S);
    p.magic = (uint32_t)((1ull << 32) / (uint64_t)S + 1);  // exact x / S for x < 2^32 / S
    if ((uint64_t)n * (uint64_t)S >= (1ull << 32)) raise(NBBGPU_ERR_OUT_OF_DOMAIN, "bounding box too large");
    p.lt_words = (uint32_t)((2 * S + 31) / 32 + 1);
    // low table: row yl, bit xl (0 <= xl < 2S) = the low m digit pairs of
    // (xl mod S, yl) are replica positions
    std::vector<uint32_t> lt((size_t)S * p.lt_words, 0u);
    for (int64_t yl = 0; yl < S; ++yl)
        for (int64_t xl = 0; xl < 2 * S; ++xl) {
            int64_t x = xl % S, y = yl;
            bool in = true;
            for (int mu = 0; mu < m && in; ++mu) {
                in = F.id[(y % s) * s + (x % s)] >= 0;
                x /= s;
                y /= s;
            }
            if (in) lt[(size_t)yl * p.lt_words + (xl >> 5)] |= 1u << (xl & 31);
        }
    dmalloc_cap(h->d_bblow, lt.size() * 4, "bounding-box low table");
    CK(cudaMemcpy(h->d_bblow, lt.data(), lt.size() * 4, cudaMemcpyHostToDevice));
    const uint64_t nwords = ((uint64_t)p.CW * p.CW + 31) / 32 + 1;
    dmalloc_cap(h->d_bbcoarse, nwords * 4, "bounding-box coarse bitmap");
    CK(cudaMemsetAsync(h->d_bbcoarse, 0, nwords * 4, h->stream));
    bb_coarse_kernel<<<grid_for(nwords, 256), 256, 0, h->stream>>>(h->frac, F.r - m, p.CW, h->d_bbcoarse, nwords - 1);
    CK(cudaGetLastError());
    // strips: chunks per aligned row <= (n + 30) / 16 + 1, at most 256 per CTA
    const uint64_t maxch = ((uint64_t)n + 30) / 16 + 2;
    const uint64_t nsx = (maxch + 2 * kBBMaxThreads - 1) / (2 * kBBMaxThreads);
    p.cps = (uint32_t)(((maxch + nsx - 1) / nsx + 63) / 64 * 64);  // 2 chunks per thread, whole warps
    uint64_t rows = 64;
    while (rows > 8 && nsx * (((uint64_t)n + rows - 1) / rows) < 16ull * 148) rows /= 2;
    p.rows = (uint32_t)rows;
    // live tiles: (strip, band) pairs whose output bytes hold a fractal cell
    const uint64_t nbands = ((uint64_t)n + rows - 1) / rows, ntiles = nsx * nbands;
    if (nsx > 0xFFFFFFFFull || nbands > 0xFFFFFFFFull) raise(NBBGPU_ERR_OUT_OF_DOMAIN, "bounding box too large");
    uint8_t* d_live = nullptr;
    dmalloc_cap(d_live, ntiles, "bounding-box tile flags");
    bb_tile_live_kernel<<<grid_for(ntiles, 256), 256, 0, h->stream>>>(p, h->d_bbcoarse, (uint32_t)nsx, (uint32_t)nbands, d_live);
    std::vector<uint8_t> live(ntiles);
    const cudaError_t e1 = cudaMemcpyAsync(live.data(), d_live, ntiles, cudaMemcpyDeviceToHost, h->stream);
    const cudaError_t e2 = cudaStreamSynchronize(h->stream);
    cudaFree(d_live);
    CK(e1);
    CK(e2);
    std::vector<uint2> tiles;
    for (uint64_t i = 0; i < ntiles; ++i)
        if (live[i]) tiles.push_back(make_uint2((uint32_t)(i % nsx), (uint32_t)(i / nsx)));
    h->bb_ntiles = (uint32_t)tiles.size();
    // static membership bitmap (n^2 / 8 bytes + pad): one 32-bit load per 32 cells
    // per row instead of the per-row membership evaluation
    const uint64_t mwords = (p.alloc + 31) / 32;
    dmalloc_cap(h->d_bbmemb, mwords * 4, "bounding-box membership bitmap");
    h->bytes_held += mwords * 4;
    bb_member_bitmap_kernel<<<grid_for(mwords, 256), 256, 0, h->stream>>>(p, h->d_bblow, h->d_bbcoarse, h->d_bbmemb, mwords);
    CK(cudaGetLastError());
    dmalloc_cap(h->d_bbtiles, std::max<size_t>(1, tiles.size()) * sizeof(uint2), "bounding-box tile list");
    if (!tiles.empty()) CK(cudaMemcpy(h->d_bbtiles, tiles.data(), tiles.size() * sizeof(uint2), cudaMemcpyHostToDevice));
    h->bb_ready = true;
}

void launch_bb_rows(nbbgpu_t h, uint16_t birth, uint16_t survive, int moore) {
    ensure_bb_tables(h);
    BBRowParams p = h->bbp;
    p.birth = birth;
    p.survive = survive;
    p.moore = moore;
    if (h->bb_ntiles == 0) return;
    p.ntiles = h->bb_ntiles;
    const uint32_t tpb = p.cps / 2;
    const size_t smem = (size_t)kBBStages * (p.cps + 4) * 16 + (size_t)4 * (tpb + 4) * 4 +
                        (size_t)kBBStages * (tpb + 4) * 4 + kBBCacheWords * 4 + kBBStages * (tpb / 32);
    const bool conway = (birth & 0x1FF) == 0x8 && (survive & 0x1FF) == 0xC && moore;
    if (smem > 48 * 1024) raise(NBBGPU_ERR_CUDA, "internal: bounding-box row ring exceeds 48 KB");  // s <= 16
    auto kern = conway ? step_bb_rows_kernel<true, kBBStages> : step_bb_rows_kernel<false, kBBStages>;
    // one CTA per live tile: the block scheduler balances tiles of unequal work
    // (persistent CTAs over a static tile order measured slower: carpet r=11 16.8 vs 13.4 ms)
    kern<<<h->bb_ntiles, tpb, smem, h->stream>>>(p, h->d_bbtiles, h->d_bbmemb, h->d_bbcoarse, h->front(), h->back());
}

void launch_step(nbbgpu_t h, uint16_t birth, uint16_t survive, int moore) {
    const int deg = moore ? 8 : 4;
    const uint8_t* src = h->front();
    uint8_t* dst = h->back();
    if (h->mode == NBBGPU_MODE_LAMBDA || h->mode == NBBGPU_MODE_BLOCKED) {
        ++h->launches;
        prof_mark(h);
        struct ProfEnd { nbbgpu_t h; ~ProfEnd() { prof_mark(h); } } prof_end{h};
        if (h->mode == NBBGPU_MODE_LAMBDA) {
            const uint64_t n = (uint64_t)h->hf.w * h->hf.h;
#define NBB_CALL(K, S, ...) step_lambda_kernel<K, S><<<grid_for(n, 256), 256, 0, h->stream>>>(h->frac, src, dst, birth, survive, deg)
            NBB_DISPATCH_KS(h->hf);
#undef NBB_CALL
        } else {
            step_blocked_kernel<<<grid_for(h->cells, 256), 256, 0, h->stream>>>(h->bg, h->d_lowmask, h->d_blocktab, src, dst, birth, survive, deg);
        }
        return;
    }
    if (h->mode == NBBGPU_MODE_BB) {
        ++h->launches;
        prof_mark(h);
        struct ProfEnd { nbbgpu_t h; ~ProfEnd() { prof_mark(h); } } prof_end{h};
        const uint64_t n = (uint64_t)h->hf.side * h->hf.side;
        const int s = h->hf.s;
        if (h->hf.side >= 32 && h->kernel != NBBGPU_KERNEL_NAIVE) {
            launch_bb_rows(h, birth, survive, moore);  // bb.cuh
            return;
        }
        (void)s;
#define NBB_CALL(K, S, ...) step_bb_naive_kernel<K, S><<<grid_for(n, 256), 256, 0, h->stream>>>(h->frac, src, dst, birth, survive, deg)
        NBB_DISPATCH_KS(h->hf);
#undef NBB_CALL
        return;
    }
    const int kern = resolve_kernel(h);
    if (kern == NBBGPU_KERNEL_PACKED) {
        launch_step_packed(h, birth, survive, moore);
        return;
    }
    ++h->launches;  // one kernel per step on the byte layouts
    prof_mark(h);
    struct ProfEnd { nbbgpu_t h; ~ProfEnd() { prof_mark(h); } } prof_end{h};
    if (kern == NBBGPU_KERNEL_TABLE) {
        uint64_t lo, hi;
        owned_range(h, lo, hi);
        ensure_nbr_table(h, deg);
        const bool wide = h->cells > 0xFFFFFFFFull;
        const int blocks = grid_for(hi - lo, 256);
        if (wide && deg == 8) step_table_kernel<uint64_t, 8><<<blocks, 256, 0, h->stream>>>((const uint64_t*)h->d_tab, h->cells, src, dst, lo, hi, birth, survive);
        else if (wide) step_table_kernel<uint64_t, 4><<<blocks, 256, 0, h->stream>>>((const uint64_t*)h->d_tab, h->cells, src, dst, lo, hi, birth, survive);
        else if (deg == 8) step_table_kernel<uint32_t, 8><<<blocks, 256, 0, h->stream>>>((const uint32_t*)h->d_tab, h->cells, src, dst, lo, hi, birth, survive);
        else step_table_kernel<uint32_t, 4><<<blocks, 256, 0, h->stream>>>((const uint32_t*)h->d_tab, h->cells, src, dst, lo, hi, birth, survive);
        return;
    }
    if (kern == NBBGPU_KERNEL_NAIVE) {
        uint64_t lo, hi;
        owned_range(h, lo, hi);
        if (h->map_variant == NBBGPU_MAP_MMA && h->hf.r <= 32) {
            const int blocks = grid_for((hi - lo + 31) / 32 * 32, 128);
#define NBB_CALL(K, S, ...) step_compact_naive_mma_kernel<S><<<blocks, 128, 0, h->stream>>>(h->frac, h->mt, src, dst, lo, hi, birth, survive, deg)
            NBB_DISPATCH_KS(h->hf);
#undef NBB_CALL
            return;
        }
#define NBB_CALL(K, S, ...) step_compact_naive_kernel<K, S><<<grid_for(hi - lo, 256), 256, 0, h->stream>>>(h->frac, src, dst, lo, hi, birth, survive, deg)
        NBB_DISPATCH_KS(h->hf);
#undef NBB_CALL
        return;
    }
    ensure_plan(h, moore);
    const TilePlan& P = h->plan[moore];
    TiledParams p{};
    p.f = h->frac;
    p.L = P.L;
    p.C = P.C;
    p.nH = P.nH;
    p.nD = P.nD;
    for (int i = 0; i < 8; ++i) p.dlist[i] = P.dlist[i];
    p.Wc = (uint32_t)P.Wc;
    p.Hc = (uint32_t)P.Hc;
    p.gpr = (uint32_t)((P.Wc + 31) / 32);
    if (h->nranks > 1) {
        p.row0 = (uint32_t)h->prow0;
        p.row1 = (uint32_t)h->prow1;
    } else {
        p.row0 = 0;
        p.row1 = (uint32_t)P.Hc;
    }
    p.w = (uint64_t)h->hf.w;
    p.birth = birth;
    p.survive = survive;
    p.nbr = h->d_nbr[moore];
    p.ntab = h->d_ntab[moore];
    p.halo_D = h->d_hD[moore];
    p.halo_a = h->d_ha[moore];
    p.halo_c = h->d_hc[moore];
    p.halo_off = h->d_hoff[moore];
    p.smem_per_warp = P.smem_per_warp;
    p.words_per_group = P.wpg;
    if (p.row1 <= p.row0) return;
    const bool conway = (birth & 0x1FF) == 0x8 && (survive & 0x1FF) == 0xC && moore;
    if (conway) launch_tiled_w<true>(h, P.wq, p, src, dst);
    else launch_tiled_w<false>(h, P.wq, p, src, dst);
}

void free_comm(nbbgpu_t h);           // partition.inc
void exchange_on_stream(nbbgpu_t h);  // partition.inc

void graphs_clear(nbbgpu_t h) {
    for (auto& g : h->graphs) cudaGraphExecDestroy(g.exec);
    h->graphs.clear();
}

void free_all(nbbgpu_t h) {
    if (!h) return;
    cudaSetDevice(h->device);
    graphs_clear(h);
    for (auto*& p : h->buf) if (p) { cudaFree(p); p = nullptr; }
    if (h->d_acc) cudaFree(h->d_acc);
    if (h->d_flag) cudaFree(h->d_flag);
    if (h->xb_stream) cudaStreamSynchronize(h->xb_stream);
    for (int i = 0; i < 2; ++i) {
        if (h->xb_host[i]) cudaFreeHost(h->xb_host[i]);
        if (h->xb_dev[i]) cudaFree(h->xb_dev[i]);
        if (h->xb_dma[i]) cudaEventDestroy(h->xb_dma[i]);
        if (h->xb_conv[i]) cudaEventDestroy(h->xb_conv[i]);
    }
    if (h->xb_stream) cudaStreamDestroy(h->xb_stream);
    for (int m = 0; m < 2; ++m) {
        if (h->d_nbr[m]) cudaFree(h->d_nbr[m]);
        if (h->d_ntab[m]) cudaFree(h->d_ntab[m]);
        if (h->d_hD[m]) cudaFree(h->d_hD[m]);
        if (h->d_ha[m]) cudaFree(h->d_ha[m]);
        if (h->d_hc[m]) cudaFree(h->d_hc[m]);
        if (h->d_hoff[m]) cudaFree(h->d_hoff[m]);
    }
    for (auto*& p : h->pk) if (p) { cudaFree(p); p = nullptr; }
    for (auto*& p : h->bnd) if (p) { cudaFree(p); p = nullptr; }
    for (auto*& p : h->d_pnbr) if (p) { cudaFree(p); p = nullptr; }
    if (h->d_pslot) cudaFree(h->d_pslot);
    if (h->d_pntab) cudaFree(h->d_pntab);
    if (h->d_psrc) cudaFree(h->d_psrc);
    if (h->d_ploc) cudaFree(h->d_ploc);
    if (h->d_pbtab) cudaFree(h->d_pbtab);
    if (h->d_phalo) cudaFree(h->d_phalo);
    if (h->d_pbt) cudaFree(h->d_pbt);
    if (h->d_pbt1) cudaFree(h->d_pbt1);
    if (h->d_pdmask) cudaFree(h->d_pdmask);
    if (h->d_lowmask) cudaFree(h->d_lowmask);
    if (h->d_bblow) cudaFree(h->d_bblow);
    if (h->d_bbcoarse) cudaFree(h->d_bbcoarse);
    if (h->d_bbtiles) cudaFree(h->d_bbtiles);
    if (h->d_bbmemb) cudaFree(h->d_bbmemb);
    if (h->d_tab) cudaFree(h->d_tab);
    if (h->d_blocktab) cudaFree(h->d_blocktab);
    for (auto* p : h->d_sends) if (p) cudaFree(p);
    for (auto* p : h->d_recvs) if (p) cudaFree(p);
    if (h->d_send_all) cudaFree(h->d_send_all);
    if (h->d_recv_all) cudaFree(h->d_recv_all);
    if (h->d_sendbuf) cudaFree(h->d_sendbuf);
    if (h->d_recvbuf) cudaFree(h->d_recvbuf);
    for (void* q : h->ipc_opened) cudaIpcCloseMemHandle(q);
    h->ipc_opened.clear();
    if (h->d_pcnt) cudaFree(h->d_pcnt);
    if (h->d_p2p_elems) cudaFree(h->d_p2p_elems);
    if (h->d_push_off) cudaFree(h->d_push_off);
    if (h->d_push_ent) cudaFree(h->d_push_ent);
    if (h->d_push_done) cudaFree(h->d_push_done);
    if (h->d_p2p_peer) cudaFree(h->d_p2p_peer);
    for (auto*& q : h->d_peer_bnd) if (q) { cudaFree(q); q = nullptr; }
    if (h->d_peer_cnt) cudaFree(h->d_peer_cnt);
    free_comm(h);
    if (h->ev0) cudaEventDestroy(h->ev0);
    if (h->ev1) cudaEventDestroy(h->ev1);
    if (h->stream) cudaStreamDestroy(h->stream);
}

uint64_t device_hash(nbbgpu_t h, bool owned) {
    uint64_t lo = 0, hi = h->cells;
    if (owned) owned_range(h, lo, hi);
    if (h->layout == 1) { lo = owned ? h->pg0 : 0; hi = owned ? h->pg1 : h->pp.NG; }
    CK(cudaMemsetAsync(h->d_acc, 0, sizeof(unsigned long long), h->stream));
    if (h->layout == 1) {
        const PackedGeom G = packed_geom(h);
        const uint64_t g0 = lo, g1 = hi;  // group range for the packed layout
        const uint64_t warps = (g1 - g0) * ((h->pp.C + 31) / 32);
        if (warps) {
#define NBB_CALL(K, S, ...) hash_packed_kernel<K, S><<<grid_for(warps * 32, 256), 256, 0, h->stream>>>(G, h->d_ploc, h->pk[h->cur], (uint32_t)g0, (uint32_t)g1, h->d_acc)
            NBB_DISPATCH_KS(h->hf);
#undef NBB_CALL
        }
    } else if (h->mode == NBBGPU_MODE_BLOCKED) {
#define NBB_CALL(K, S, ...) hash_blocked_kernel<K, S><<<grid_for(h->cells, 256), 256, 0, h->stream>>>(h->bg, h->front(), h->d_acc)
        NBB_DISPATCH_KS(h->hf);
#undef NBB_CALL
    } else if (h->mode == NBBGPU_MODE_BB || h->mode == NBBGPU_MODE_LAMBDA) {
        hash_bb_kernel<<<grid_for((uint64_t)h->hf.side * h->hf.side, 256), 256, 0, h->stream>>>((uint32_t)h->hf.side, h->front(), h->d_acc);
    } else if (hi > lo) {
#define NBB_CALL(K, S, ...) hash_compact_kernel<K, S><<<grid_for(hi - lo, 256), 256, 0, h->stream>>>(h->frac, h->front(), lo, hi, h->d_acc)
        NBB_DISPATCH_KS(h->hf);
#undef NBB_CALL
    }
    CK(cudaGetLastError());
    unsigned long long v = 0;
    CK(cudaMemcpyAsync(&v, h->d_acc, sizeof(v), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    return v;
}

bool is_device_ptr(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) && a.devicePointer == p;
}

// storage index of an embedded coordinate (Grid::storage_index, grid.cpp:38-66)
bool storage_index(nbbgpu_t h, int64_t x, int64_t y, uint64_t& idx) {
    int64_t cx, cy;
    if (!h->hf.nu(x, y, cx, cy, h->hf.r)) return false;
    if (h->mode == NBBGPU_MODE_BLOCKED) {  // Grid::storage_index, grid.cpp:54-63
        const int64_t rho = h->bg.rho;
        int64_t bx, by;
        if (!h->hf.nu(x / rho, y / rho, bx, by, h->hf.r - h->bg.m)) return false;
        idx = (uint64_t)((by * (int64_t)h->bg.fc.w + bx) * rho * rho + (y % rho) * rho + (x % rho));
        return true;
    }
    idx = (h->mode == NBBGPU_MODE_BB || h->mode == NBBGPU_MODE_LAMBDA) ? (uint64_t)(y * h->hf.side + x)
                                                                      : (uint64_t)(cy * h->hf.w + cx);
    return true;
}

void run_map_batch(nbbgpu_t h, bool is_lambda, int variant, const int32_t* in, int32_t* out,
                   int64_t count, float* ms) {
    if (count < 0) raise(NBBGPU_ERR_OUT_OF_DOMAIN, "count must be >= 0");
    if (variant != NBBGPU_MAP_DIGIT && variant != NBBGPU_MAP_MMA && variant != NBBGPU_MAP_TC05)
        raise(NBBGPU_ERR_INVALID, "unknown map variant");
    if (variant != NBBGPU_MAP_DIGIT && h->hf.r > 32) raise(NBBGPU_ERR_OUT_OF_DOMAIN, "MMA maps support levels <= 32");
    if (count == 0) { if (ms) *ms = 0.f; return; }
    const size_t bytes = (size_t)count * 8;
    const bool din = is_device_ptr(in), dout = is_device_ptr(out);
    int2* dI = nullptr;
    int2* dO = nullptr;
    // pointers the runtime does not classify as device memory (host memory, or
    // allocator pools it does not report) are staged with UVA-aware copies
    if (din) dI = (int2*)in; else { CK(cudaMalloc(&dI, bytes)); CK(cudaMemcpyAsync(dI, in, bytes, cudaMemcpyDefault, h->stream)); }
    if (dout) dO = (int2*)out; else CK(cudaMalloc(&dO, bytes));
    CK(cudaEventRecord(h->ev0, h->stream));
    const uint64_t n = (uint64_t)count;
    if (variant == NBBGPU_MAP_DIGIT) {
        if (is_lambda) {
#define NBB_CALL(K, S, ...) lambda_digit_kernel<K, S><<<grid_for(n, 256), 256, 0, h->stream>>>(h->frac, dI, dO, n)
            NBB_DISPATCH_KS(h->hf);
#undef NBB_CALL
        } else {
#define NBB_CALL(K, S, ...) nu_digit_kernel<K, S><<<grid_for(n, 256), 256, 0, h->stream>>>(h->frac, dI, dO, n)
            NBB_DISPATCH_KS(h->hf);
#undef NBB_CALL
        }
    } else if (variant == NBBGPU_MAP_TC05) {
        // tcgen05 kind::i8, 128 points per CTA tile, persistent CTAs (several per SM)
        const int blocks = (int)std::max<uint64_t>(1, std::min<uint64_t>((n + 127) / 128, 148ull * 8));
        if (is_lambda) {
#define NBB_CALL(K, S, ...) map_tc05_kernel<K, S, true><<<blocks, 128, 0, h->stream>>>(h->frac, h->mt, dI, dO, n)
            NBB_DISPATCH_KS(h->hf);
#undef NBB_CALL
        } else {
#define NBB_CALL(K, S, ...) map_tc05_kernel<K, S, false><<<blocks, 128, 0, h->stream>>>(h->frac, h->mt, dI, dO, n)
            NBB_DISPATCH_KS(h->hf);
#undef NBB_CALL
        }
    } else {
        const int blocks = grid_for((n + 15) / 16 * 32, 256);
        if (is_lambda) {
#define NBB_CALL(K, S, ...) lambda_mma_kernel<K><<<blocks, 256, 0, h->stream>>>(h->frac, h->mt, dI, dO, n)
            NBB_DISPATCH_KS(h->hf);
#undef NBB_CALL
        } else {
#define NBB_CALL(K, S, ...) nu_mma_kernel<S><<<blocks, 256, 0, h->stream>>>(h->frac, h->mt, dI, dO, n)
            NBB_DISPATCH_KS(h->hf);
#undef NBB_CALL
        }
    }
    CK(cudaGetLastError());
    CK(cudaEventRecord(h->ev1, h->stream));
    if (!dout) CK(cudaMemcpyAsync(out, dO, bytes, cudaMemcpyDefault, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    check_peer_error(h);
    if (ms) CK(cudaEventElapsedTime(ms, h->ev0, h->ev1));
    if (!din) cudaFree(dI);
    if (!dout) cudaFree(dO);
}

}  // namespace

// ===========================================================================
extern "C" {

const char* nbbgpu_last_error(void) { return g_err.c_str(); }
int nbbgpu_version(void) { return 1; }

int nbbgpu_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

int nbbgpu_create(const int32_t* rep, int k, int s, int level, int mode, int device,
                  uint64_t memory_cap, nbbgpu_t* out) {
    return nbbgpu_create_ex(rep, k, s, level, mode, 0, device, memory_cap, out);
}

int nbbgpu_create_ex(const int32_t* rep, int k, int s, int level, int mode, int block_size, int device,
                     uint64_t memory_cap, nbbgpu_t* out) {
    if (!out) { g_err = "null output handle"; return NBBGPU_ERR_INVALID; }
    *out = nullptr;
    nbbgpu_t h = new (std::nothrow) nbbgpu_sim();
    if (!h) { g_err = "host allocation failed"; return NBBGPU_ERR_CAPACITY; }
    const int rc = guarded([&] {
        if (!rep && k > 0) raise(NBBGPU_ERR_INVALID, "null replica table");
        if (mode < NBBGPU_MODE_COMPACT || mode > NBBGPU_MODE_BLOCKED) raise(NBBGPU_ERR_INVALID, "unknown mode");
        // Simulation ctor option checks (stencil.cpp:128-131)
        if (block_size > 0 && mode != NBBGPU_MODE_BLOCKED) raise(NBBGPU_ERR_OUT_OF_DOMAIN, "block size applies to the compact backend only");
        if (mode == NBBGPU_MODE_BLOCKED && block_size < 1) raise(NBBGPU_ERR_OUT_OF_DOMAIN, "the blocked layout needs a block size");
        h->hf.init(rep, k, s, level);
        if (h->hf.side > (int64_t)1 << 31 || h->hf.w > (int64_t)1 << 31)
            raise(NBBGPU_ERR_OUT_OF_DOMAIN, "level " + std::to_string(level) + " exceeds the engine's 32-bit coordinate range");
        h->mode = mode;
        // Grid::Grid cap check (grid.cpp:16-22): per grid, cells > memory_cap
        int64_t cells = (mode == NBBGPU_MODE_BB || mode == NBBGPU_MODE_LAMBDA) ? HostFrac::ipow(h->hf.side, 2)
                                                                           : h->hf.w * h->hf.h;
        if (mode == NBBGPU_MODE_BLOCKED) {
            // block_exponent / stored_cells (geometry.cpp:69-108)
            int m = 0;
            int64_t p = 1;
            while (p < block_size) { p *= s; ++m; }
            if (p != block_size) raise(NBBGPU_ERR_OUT_OF_DOMAIN, "block size " + std::to_string(block_size) + " is not a power of s=" + std::to_string(s));
            if (m > level) raise(NBBGPU_ERR_OUT_OF_DOMAIN, "block size " + std::to_string(block_size) + " exceeds the level-" + std::to_string(level) + " fractal");
            cells = HostFrac::ipow(k, level - m) * (int64_t)block_size * block_size;
            h->bg.rho = (uint32_t)block_size;
            h->bg.m = m;
        }
        if ((uint64_t)cells > memory_cap)
            raise(NBBGPU_ERR_CAPACITY, "grid of " + std::to_string(cells) + " cells exceeds the memory cap of " + std::to_string(memory_cap) + " bytes");
        h->cells = (uint64_t)cells;
        h->device = device;
        CK(cudaSetDevice(device));
        CK(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
        CK(cudaEventCreate(&h->ev0));
        CK(cudaEventCreate(&h->ev1));
        // device tables
        Frac& f = h->frac;
        memset(&f, 0, sizeof(f));
        f.k = k; f.s = s; f.r = level;
        f.w = (uint32_t)h->hf.w; f.h = (uint32_t)h->hf.h; f.side = (uint32_t)h->hf.side;
        for (int i = 0; i < kMaxS * kMaxS; ++i) f.id_of_subbox[i] = -1;
        for (int i = 0; i < s * s; ++i) f.id_of_subbox[i] = (int8_t)h->hf.id[i];
        for (int i = 0; i < k; ++i) { f.gx[i] = (uint8_t)h->hf.gx[i]; f.gy[i] = (uint8_t)h->hf.gy[i]; }
        if (mode == NBBGPU_MODE_BLOCKED) {
            if (block_size > 64) raise(NBBGPU_ERR_OUT_OF_DOMAIN, "the GPU blocked layout supports block sizes up to 64");
            const int rho = block_size;
            std::vector<uint32_t> lmask(((size_t)rho * rho + 31) / 32, 0u);
            for (int ly = 0; ly < rho; ++ly)
                for (int lx = 0; lx < rho; ++lx) {
                    int64_t a, c;
                    if (h->hf.nu(lx, ly, a, c, h->bg.m)) lmask[(ly * rho + lx) / 32] |= 1u << ((ly * rho + lx) % 32);
                }
            dmalloc_cap(h->d_lowmask, lmask.size() * 4, "filler mask");
            CK(cudaMemcpy(h->d_lowmask, lmask.data(), lmask.size() * 4, cudaMemcpyHostToDevice));
            h->bg.f = f;
            h->bg.fc = f;
            h->bg.fc.r = level - h->bg.m;
            h->bg.fc.w = (uint32_t)HostFrac::ipow(k, (h->bg.fc.r + 1) / 2);
            h->bg.fc.h = (uint32_t)HostFrac::ipow(k, h->bg.fc.r / 2);
            h->bg.fc.side = (uint32_t)HostFrac::ipow(s, h->bg.fc.r);
            const uint64_t nblocks = (uint64_t)h->bg.fc.w * h->bg.fc.h;
            dmalloc_cap(h->d_blocktab, nblocks * kBlockTab * 4, "block table");
            h->bytes_held += nblocks * kBlockTab * 4;
#define NBB_CALL(K, S, ...) build_blocktab_kernel<K, S><<<grid_for(nblocks, 256), 256, 0, h->stream>>>(h->bg, h->d_blocktab)
            NBB_DISPATCH_KS(h->hf);
#undef NBB_CALL
            CK(cudaGetLastError());
        }
        for (int mu = 0; mu < 32 && mu < level; ++mu) {
            h->mt.spow[mu] = (uint32_t)h->hf.spow[mu];
            int64_t t = 1;
            for (int j = 0; j < mu / 2; ++j) t *= k;
            h->mt.tau[mu] = (uint32_t)t;
        }
        CK(cudaMalloc(&h->d_acc, sizeof(unsigned long long)));
        CK(cudaMalloc(&h->d_flag, sizeof(int)));
        h->bytes_held = 16;
        h->q = mode == NBBGPU_MODE_COMPACT ? choose_tile_level(h->hf) : 0;
        h->pq = mode == NBBGPU_MODE_COMPACT ? choose_packed_level(h->hf) : -1;
        // state buffers of the default kernel's layout: packed (bit-sliced, 1/8 of the
        // bytes) when a packed tile level exists, else the reference bytes (double
        // buffer + 64 B slack for the tiled kernel's aligned 16-B accesses)
        if (resolve_kernel(h) == NBBGPU_KERNEL_PACKED) {
            alloc_packed_state(h);
            h->layout = 1;
        } else {
            alloc_byte_state(h);
            h->layout = 0;
        }
        h->part_q = 0;
        h->unit_rows = 1;
        h->prow0 = 0;
        h->prow1 = h->hf.h;
        CK(cudaStreamSynchronize(h->stream));
    });
    if (rc != NBBGPU_OK) {
        free_all(h);
        delete h;
        return rc;
    }
    *out = h;
    return NBBGPU_OK;
}

int nbbgpu_destroy(nbbgpu_t h) {
    if (!h) return NBBGPU_OK;
    free_all(h);
    delete h;
    return NBBGPU_OK;
}

int nbbgpu_seed(nbbgpu_t h, uint64_t seed, double density) {
    return guarded([&] {
        check_handle(h);
        if (!(density >= 0.0 && density <= 1.0)) raise(NBBGPU_ERR_OUT_OF_DOMAIN, "density must be in [0,1]");
        h->iteration = 0;
        const uint64_t mix = splitmix64(seed);
        if (h->layout == 1) {
            for (int b = 0; b < 2; ++b) CK(cudaMemsetAsync(h->pk[b], 0, packed_words(h->pp) * 4, h->stream));
            const PackedGeom G = packed_geom(h);
            const uint64_t warps = (uint64_t)G.NG * ((G.C + 31) / 32);
#define NBB_CALL(K, S, ...) seed_packed_kernel<K, S><<<grid_for(warps * 32, 256), 256, 0, h->stream>>>(G, h->d_ploc, h->pk[h->cur], mix, density)
            NBB_DISPATCH_KS(h->hf);
#undef NBB_CALL
            CK(cudaGetLastError());
            bnd_refresh(h);
            CK(cudaStreamSynchronize(h->stream));
            return;
        }
        for (int b = 0; b < 2; ++b) CK(cudaMemsetAsync(h->buf[b], 0, h->cells + 64, h->stream));
        if (h->mode == NBBGPU_MODE_BLOCKED) {
#define NBB_CALL(K, S, ...) seed_blocked_kernel<K, S><<<grid_for(h->cells, 256), 256, 0, h->stream>>>(h->bg, h->front(), mix, density)
            NBB_DISPATCH_KS(h->hf);
#undef NBB_CALL
        } else if (h->mode == NBBGPU_MODE_BB || h->mode == NBBGPU_MODE_LAMBDA) {
            const uint64_t n = h->cells;
#define NBB_CALL(K, S, ...) seed_bb_kernel<K, S><<<grid_for(n, 256), 256, 0, h->stream>>>(h->frac, h->front(), mix, density)
            NBB_DISPATCH_KS(h->hf);
#undef NBB_CALL
        } else {
            const uint64_t n = h->cells;
#define NBB_CALL(K, S, ...) seed_compact_kernel<K, S><<<grid_for(n, 256), 256, 0, h->stream>>>(h->frac, h->front(), n, mix, density)
            NBB_DISPATCH_KS(h->hf);
#undef NBB_CALL
        }
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(h->stream));
    });
}

constexpr int kGraphSteps = 8;  // steps per captured graph (even: the buffers return to their parity)
// packed states replayed from graphs by default: up to 2^24 cells the device step
// (<= ~4.5 us) is shorter than the host's ~3.4 us per PDL launch plus overheads
// (T r=14 4.11 -> 3.85 us/step); above, graphs only lose PDL overlap (T r=16 6.3 ->
// 7.0 us/step, H r=11 0.169 -> 0.189 ms)
constexpr uint64_t kGraphMaxCells = 1ull << 24;

// the per-call tuning knobs a captured step sequence depends on
std::string tuning_env() {
    std::string e;
    for (const char* k : {"NBBGPU_HALO_WARPS", "NBBGPU_HALO_GROUP", "NBBGPU_HALO_NCH3", "NBBGPU_HALO_LEAN",
                          "NBBGPU_HALO_BT", "NBBGPU_BT_OUT", "NBBGPU_NO_PDL", "NBBGPU_GENERIC", "NBBGPU_PACKED_Q"}) {
        const char* v = getenv(k);
        e += v ? v : "-";
        e += ';';
    }
    return e;
}

static void step_impl(nbbgpu_t h, uint16_t birth, uint16_t survive, int moore, int64_t nsteps,
                      float* ms, float* main_ms = nullptr, uint64_t* launches = nullptr, bool sync = true) {
    check_handle(h);
    if (nsteps < 0) raise(NBBGPU_ERR_OUT_OF_DOMAIN, "steps must be >= 0");
    moore = moore ? 1 : 0;
    const int rk = resolve_kernel(h);
    if (layout_of_kernel(rk) != h->layout) raise(NBBGPU_ERR_CUDA, "internal: state layout does not match the kernel");
    if (rk == NBBGPU_KERNEL_TILED) ensure_plan(h, moore);
    std::vector<cudaEvent_t> prof;
    if (main_ms) {
        prof.resize((size_t)std::max<int64_t>(nsteps, 1) * 2);
        for (auto& e : prof) CK(cudaEventCreate(&e));
        h->prof = &prof;
        h->prof_idx = 0;
    }
    const uint64_t l0 = h->launches;
    CK(cudaEventRecord(h->ev0, h->stream));
    try {
        if (rk == NBBGPU_KERNEL_PACKED && launch_resident(h, birth, survive, moore, nsteps)) {
            // (all steps on-chip in one single-CTA launch)
        } else {
            auto one_step = [&] {
                launch_step(h, birth, survive, moore);
                h->cur ^= 1;
                ++h->iteration;
                if (h->p2p) {                        // peer-memory halo of the new front
                    if (h->fused_push) ++h->p2p_epoch;  // (pushed and signalled by the step kernel)
                    else p2p_push(h);
                }
                else if (h->comm) exchange_on_stream(h);  // NCCL halo of the new front, on-stream
            };
            int64_t i = 0;
            // Long calls on one GPU: after one plain step (the boundary-plane flags are
            // then in their steady state), kGraphSteps steps at a time are replayed
            // from a captured CUDA graph -- one host launch instead of one or two per
            // step (the host enqueue rate bounds small levels: ~3.4 us per PDL launch).
            // Only where the host bounds the step rate: replaying captured launches
            // loses part of the programmatic (PDL) overlap between the kernels (H r=11:
            // 0.169 -> 0.189 ms per step), so large states keep stream launches.
            const char* ge = getenv("NBBGPU_GRAPHS");
            const bool small = rk == NBBGPU_KERNEL_PACKED && h->cells <= kGraphMaxCells;
            if ((ge ? ge[0] == '1' : small) && !h->p2p && !h->comm && !h->prof && nsteps > kGraphSteps) {
                one_step();
                ++i;
                const std::string env = tuning_env();
                while (i + kGraphSteps <= nsteps) {
                    nbbgpu_sim::StepGraph* g = nullptr;
                    for (auto& e : h->graphs)
                        if (e.birth == birth && e.survive == survive && e.moore == moore && e.cur == h->cur &&
                            e.kernel == rk && e.env == env)
                            g = &e;
                    if (!g && nsteps - i < 4 * kGraphSteps) break;  // (short call: not worth a capture)
                    if (!g) {  // capture (the host state advances as the captured steps run)
                        const int cur0 = h->cur;
                        const uint64_t l0c = h->launches;
                        cudaGraph_t graph = nullptr;
                        CK(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
                        try {
                            for (int k = 0; k < kGraphSteps; ++k) one_step();
                        } catch (...) {
                            cudaStreamEndCapture(h->stream, &graph);
                            if (graph) cudaGraphDestroy(graph);
                            throw;
                        }
                        CK(cudaStreamEndCapture(h->stream, &graph));
                        cudaGraphExec_t exec = nullptr;
                        const cudaError_t ie = cudaGraphInstantiate(&exec, graph, 0);
                        cudaGraphDestroy(graph);
                        CK(ie);
                        h->graphs.push_back({birth, survive, moore, cur0, rk, env, exec, h->launches - l0c});
                        CK(cudaGraphLaunch(exec, h->stream));  // runs the captured steps
                        i += kGraphSteps;
                        continue;
                    }
                    CK(cudaGraphLaunch(g->exec, h->stream));
                    h->launches += g->launches;
                    h->iteration += kGraphSteps;
                    i += kGraphSteps;
                }
            }
            for (; i < nsteps; ++i) one_step();
        }
    } catch (...) {
        h->prof = nullptr;
        for (auto e : prof) cudaEventDestroy(e);
        throw;
    }
    h->prof = nullptr;
    CK(cudaGetLastError());
    CK(cudaEventRecord(h->ev1, h->stream));
    if (!sync) {  // nbbgpu_step_async: enqueued only
        if (launches) *launches = h->launches - l0;
        return;
    }
    CK(cudaStreamSynchronize(h->stream));
    check_peer_error(h);
    if (ms) CK(cudaEventElapsedTime(ms, h->ev0, h->ev1));
    if (main_ms) {
        float acc = 0.f;
        for (size_t i = 0; i + 1 < h->prof_idx; i += 2) {
            float t = 0.f;
            CK(cudaEventElapsedTime(&t, prof[i], prof[i + 1]));
            acc += t;
        }
        *main_ms = acc;
    }
    for (auto e : prof) cudaEventDestroy(e);
    if (launches) *launches = h->launches - l0;
}

int nbbgpu_launch_count(nbbgpu_t h, uint64_t* out) {
    return guarded([&] {
        if (!h || !out) raise(NBBGPU_ERR_INVALID, "null argument");
        *out = h->launches;
    });
}

int nbbgpu_step_profiled(nbbgpu_t h, uint16_t birth, uint16_t survive, int moore, int64_t nsteps,
                         float* total_ms, float* main_kernel_ms, uint64_t* launches) {
    return guarded([&] {
        float dummy = 0.f;
        step_impl(h, birth, survive, moore, nsteps, total_ms, main_kernel_ms ? main_kernel_ms : &dummy, launches);
    });
}

int nbbgpu_step(nbbgpu_t h, uint16_t birth, uint16_t survive, int moore, int64_t nsteps) {
    return guarded([&] { step_impl(h, birth, survive, moore, nsteps, nullptr); });
}

int nbbgpu_step_async(nbbgpu_t h, uint16_t birth, uint16_t survive, int moore, int64_t nsteps) {
    return guarded([&] { step_impl(h, birth, survive, moore, nsteps, nullptr, nullptr, nullptr, false); });
}

int nbbgpu_synchronize(nbbgpu_t h) {
    return guarded([&] {
        check_handle(h);
        CK(cudaStreamSynchronize(h->stream));
        check_peer_error(h);
    });
}

int nbbgpu_step_timed(nbbgpu_t h, uint16_t birth, uint16_t survive, int moore, int64_t nsteps,
                      float* device_ms) {
    return guarded([&] { step_impl(h, birth, survive, moore, nsteps, device_ms); });
}

int nbbgpu_state_hash(nbbgpu_t h, uint64_t* out) {
    return guarded([&] {
        check_handle(h);
        if (!out) raise(NBBGPU_ERR_INVALID, "null output");
        *out = device_hash(h, false);
    });
}

int nbbgpu_state_hash_owned(nbbgpu_t h, uint64_t* out) {
    return guarded([&] {
        check_handle(h);
        if (!out) raise(NBBGPU_ERR_INVALID, "null output");
        *out = device_hash(h, true);
    });
}

int nbbgpu_iteration(nbbgpu_t h, int64_t* out) {
    return guarded([&] {
        if (!h || !out) raise(NBBGPU_ERR_INVALID, "null argument");
        *out = h->iteration;
    });
}

int nbbgpu_stored_cells(nbbgpu_t h, uint64_t* out) {
    return guarded([&] {
        if (!h || !out) raise(NBBGPU_ERR_INVALID, "null argument");
        *out = h->cells;
    });
}

int nbbgpu_dims(nbbgpu_t h, int64_t* w, int64_t* hg, int64_t* side) {
    return guarded([&] {
        if (!h) raise(NBBGPU_ERR_INVALID, "null handle");
        if (w) *w = h->hf.w;
        if (hg) *hg = h->hf.h;
        if (side) *side = h->hf.side;
    });
}

int nbbgpu_download(nbbgpu_t h, uint8_t* dst, uint64_t bytes) {
    return guarded([&] {
        check_handle(h);
        if (bytes != h->cells) raise(NBBGPU_ERR_OUT_OF_DOMAIN, "download size " + std::to_string(bytes) + " != stored cells " + std::to_string(h->cells));
        if (!dst) raise(NBBGPU_ERR_INVALID, "null destination");
        if (h->layout == 1) {
            packed_to_bytes(h, h->pk[h->cur], dst);
            return;
        }
        CK(cudaMemcpyAsync(dst, h->front(), bytes, cudaMemcpyDefault, h->stream));
        CK(cudaStreamSynchronize(h->stream));
    });
}

int nbbgpu_upload(nbbgpu_t h, const uint8_t* src, uint64_t bytes) {
    return guarded([&] {
        check_handle(h);
        if (bytes != h->cells) raise(NBBGPU_ERR_OUT_OF_DOMAIN, "upload size " + std::to_string(bytes) + " != stored cells " + std::to_string(h->cells));
        if (!src) raise(NBBGPU_ERR_INVALID, "null source");
        if (h->layout == 1) {
            // pack into the back buffer (validating), then publish
            if (!packed_from_bytes(h, src, h->pk[h->cur ^ 1])) {
                CK(cudaMemsetAsync(h->pk[h->cur ^ 1], 0, packed_words(h->pp) * 4, h->stream));
                CK(cudaStreamSynchronize(h->stream));
                raise(NBBGPU_ERR_OUT_OF_DOMAIN, "GPU backends store binary cell states (bytes 0/1)");
            }
            h->cur ^= 1;
            CK(cudaMemsetAsync(h->pk[h->cur ^ 1], 0, packed_words(h->pp) * 4, h->stream));
            bnd_refresh(h);
            CK(cudaStreamSynchronize(h->stream));
            return;
        }
        // stage into the back buffer, validate binary states, then publish
        CK(cudaMemcpyAsync(h->back(), src, bytes, cudaMemcpyDefault, h->stream));
        CK(cudaMemsetAsync(h->d_flag, 0, sizeof(int), h->stream));
        check_binary_kernel<<<grid_for(bytes, 256), 256, 0, h->stream>>>(h->back(), bytes, h->d_flag);
        if (h->mode == NBBGPU_MODE_BB) {  // holes are dead in the box (set_cell rejects them)
#define NBB_CALL(K, S, ...) check_bb_holes_kernel<K, S><<<grid_for(bytes, 256), 256, 0, h->stream>>>(h->frac, h->back(), h->d_flag)
            NBB_DISPATCH_KS(h->hf);
#undef NBB_CALL
        }
        int flag = 0;
        CK(cudaMemcpyAsync(&flag, h->d_flag, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
        CK(cudaStreamSynchronize(h->stream));
        if (flag) {
            CK(cudaMemsetAsync(h->back(), 0, bytes, h->stream));
            CK(cudaStreamSynchronize(h->stream));
            raise(NBBGPU_ERR_OUT_OF_DOMAIN, h->mode == NBBGPU_MODE_BB
                                                ? "GPU backends store binary cell states (bytes 0/1) and dead holes"
                                                : "GPU backends store binary cell states (bytes 0/1)");
        }
        CK(cudaMemcpyAsync(h->front(), h->back(), bytes, cudaMemcpyDeviceToDevice, h->stream));
        CK(cudaMemsetAsync(h->back(), 0, bytes, h->stream));
        CK(cudaStreamSynchronize(h->stream));
    });
}

int nbbgpu_get_cell(nbbgpu_t h, int64_t x, int64_t y, uint8_t* out) {
    return guarded([&] {
        check_handle(h);
        if (!out) raise(NBBGPU_ERR_INVALID, "null output");
        // Simulation::cell (stencil.cpp:182-188)
        if (x < 0 || y < 0 || x >= h->hf.side || y >= h->hf.side) raise(NBBGPU_ERR_OUT_OF_DOMAIN, "embedded coordinate outside the bounding box");
        if (h->layout == 1) {
            int64_t cx, cy;
            if (!h->hf.nu(x, y, cx, cy, h->hf.r)) { *out = 0; return; }
            uint64_t wi;
            uint32_t bit, word = 0;
            packed_locate(h, cx, cy, wi, bit);
            CK(cudaMemcpyAsync(&word, h->pk[h->cur] + wi, 4, cudaMemcpyDeviceToHost, h->stream));
            CK(cudaStreamSynchronize(h->stream));
            *out = (uint8_t)((word >> bit) & 1u);
            return;
        }
        uint64_t idx;
        if (!storage_index(h, x, y, idx)) { *out = 0; return; }
        CK(cudaMemcpyAsync(out, h->front() + idx, 1, cudaMemcpyDeviceToHost, h->stream));
        CK(cudaStreamSynchronize(h->stream));
    });
}

int nbbgpu_set_cell(nbbgpu_t h, int64_t x, int64_t y, uint8_t state) {
    return guarded([&] {
        check_handle(h);
        // Simulation::set_cell (stencil.cpp:190-194): fractal cells only
        if (x < 0 || y < 0 || x >= h->hf.side || y >= h->hf.side) raise(NBBGPU_ERR_OUT_OF_DOMAIN, "embedded coordinate (" + std::to_string(x) + "," + std::to_string(y) + ") outside [0," + std::to_string(h->hf.side) + ")^2");
        uint64_t idx;
        if (!storage_index(h, x, y, idx)) raise(NBBGPU_ERR_NOT_IN_FRACTAL, "set_cell requires a fractal cell");
        if (state > 1) raise(NBBGPU_ERR_OUT_OF_DOMAIN, "GPU backends store binary cell states (bytes 0/1)");
        if (h->layout == 1) {
            int64_t cx, cy;
            h->hf.nu(x, y, cx, cy, h->hf.r);
            uint64_t wi;
            uint32_t bit, word = 0;
            packed_locate(h, cx, cy, wi, bit);
            CK(cudaMemcpyAsync(&word, h->pk[h->cur] + wi, 4, cudaMemcpyDeviceToHost, h->stream));
            CK(cudaStreamSynchronize(h->stream));
            word = (word & ~(1u << bit)) | ((uint32_t)state << bit);
            CK(cudaMemcpyAsync(h->pk[h->cur] + wi, &word, 4, cudaMemcpyHostToDevice, h->stream));
            bnd_refresh(h);
            CK(cudaStreamSynchronize(h->stream));
            return;
        }
        CK(cudaMemcpyAsync(h->front() + idx, &state, 1, cudaMemcpyHostToDevice, h->stream));
        CK(cudaStreamSynchronize(h->stream));
    });
}

}  // extern "C"

namespace {
// the embedded n x n view (bytes, or PBM rows) of the front state into dst (host or device)
void render_view(nbbgpu_t h, uint8_t* dst, int pbm) {
    ViewSrc v{};
    v.mode = h->mode;
    v.packed = h->layout == 1;
    v.bytes = h->layout == 1 ? nullptr : h->front();
    v.words = h->layout == 1 ? h->pk[h->cur] : nullptr;
    if (h->layout == 1) {
        v.wq = (uint32_t)h->pp.wq;
        v.Wc = (uint32_t)h->pp.Wc;
        v.Cp = (uint32_t)h->pp.Cp;
        v.ilv = h->pp.ilv;
    }
    v.bg = h->bg;
    const uint64_t n = (uint64_t)h->hf.side, total = n * (pbm ? n + 1 : n);
    uint8_t* out = dst;
    const bool dev = is_device_mem(dst);
    if (!dev) dmalloc_cap(out, total, "render buffer");
#define NBB_CALL(K, S, ...) embedded_view_kernel<K, S><<<grid_for(total, 256), 256, 0, h->stream>>>(h->frac, v, out, pbm)
    NBB_DISPATCH_KS(h->hf);
#undef NBB_CALL
    CK(cudaGetLastError());
    if (!dev) {
        CK(cudaMemcpyAsync(dst, out, total, cudaMemcpyDeviceToHost, h->stream));
        CK(cudaStreamSynchronize(h->stream));
        cudaFree(out);
    } else {
        CK(cudaStreamSynchronize(h->stream));
    }
}
}  // namespace

extern "C" {

int nbbgpu_embedded_view(nbbgpu_t h, uint8_t* dst, uint64_t bytes) {
    return guarded([&] {
        check_handle(h);
        if (!dst) raise(NBBGPU_ERR_INVALID, "null destination");
        const uint64_t n = (uint64_t)h->hf.side;
        if (bytes != n * n) raise(NBBGPU_ERR_OUT_OF_DOMAIN, "view size " + std::to_string(bytes) + " != side^2 " + std::to_string(n * n));
        render_view(h, dst, 0);
    });
}

int nbbgpu_render_pbm(nbbgpu_t h, char* dst, uint64_t capacity, int64_t render_cap, uint64_t* written) {
    return guarded([&] {
        check_handle(h);
        if (!written) raise(NBBGPU_ERR_INVALID, "null size output");
        const int64_t n = h->hf.side;
        // write_pbm (pbm.cpp:11-15)
        if (n > render_cap)
            raise(NBBGPU_ERR_CAPACITY, "side " + std::to_string(n) + " exceeds the render cap of " + std::to_string(render_cap));
        const std::string header = "P1\n" + std::to_string(n) + " " + std::to_string(n) + "\n";
        const uint64_t body = (uint64_t)n * (uint64_t)(n + 1), total = header.size() + body;
        *written = total;
        if (!dst) return;
        if (capacity < total) raise(NBBGPU_ERR_INVALID, "PBM buffer too small");
        std::memcpy(dst, header.data(), header.size());
        render_view(h, reinterpret_cast<uint8_t*>(dst) + header.size(), 1);
    });
}

int nbbgpu_peak_bytes(nbbgpu_t h, uint64_t* out) {
    return guarded([&] {
        if (!h || !out) raise(NBBGPU_ERR_INVALID, "null argument");
        *out = h->bytes_held;
    });
}

int nbbgpu_set_kernel(nbbgpu_t h, int kernel) {
    return guarded([&] {
        if (!h) raise(NBBGPU_ERR_INVALID, "null handle");
        if (kernel < NBBGPU_KERNEL_AUTO || kernel > NBBGPU_KERNEL_TABLE) raise(NBBGPU_ERR_INVALID, "unknown kernel");
        if (kernel == NBBGPU_KERNEL_TABLE && h->mode != NBBGPU_MODE_COMPACT)
            raise(NBBGPU_ERR_OUT_OF_DOMAIN, "the neighbor table applies to the linear compact backend only");
        if (kernel == NBBGPU_KERNEL_TILED && (h->mode != NBBGPU_MODE_COMPACT || h->q == 0))
            raise(NBBGPU_ERR_OUT_OF_DOMAIN, "no tile level for this fractal/level");
        if (kernel == NBBGPU_KERNEL_PACKED && (h->mode != NBBGPU_MODE_COMPACT || h->pq < 2))
            raise(NBBGPU_ERR_OUT_OF_DOMAIN, "no packed tile level for this fractal/level");
        if (h->nranks > 1 && kernel != h->kernel) raise(NBBGPU_ERR_INVALID, "kernel is fixed once partitioned");
        CK(cudaSetDevice(h->device));
        graphs_clear(h);
        set_layout(h, layout_of_kernel(resolve_kernel_for(h, kernel)));
        h->kernel = kernel;
    });
}

int nbbgpu_set_map_variant(nbbgpu_t h, int variant) {
    return guarded([&] {
        if (!h) raise(NBBGPU_ERR_INVALID, "null handle");
        if (variant != NBBGPU_MAP_DIGIT && variant != NBBGPU_MAP_MMA) raise(NBBGPU_ERR_INVALID, "unknown map variant");
        h->map_variant = variant;
    });
}

int nbbgpu_active_kernel(nbbgpu_t h, int* kernel, int* tile_level) {
    return guarded([&] {
        if (!h) raise(NBBGPU_ERR_INVALID, "null handle");
        const int k = resolve_kernel(h);
        if (kernel) *kernel = k;
        if (tile_level) *tile_level = k == NBBGPU_KERNEL_TILED ? h->q : (k == NBBGPU_KERNEL_PACKED ? h->pq : 0);
    });
}

int nbbgpu_packed_program(nbbgpu_t h, int* program, int* block_level) {
    return guarded([&] {
        if (!h) raise(NBBGPU_ERR_INVALID, "null handle");
        int prog = NBBGPU_PROGRAM_NONE, bl = 0;
        if (resolve_kernel(h) == NBBGPU_KERNEL_PACKED) {
            ensure_packed_tables(h);
            const PackedPlan& P = h->pp;
            prog = P.tag == kTagNone ? NBBGPU_PROGRAM_TABLE : P.tag == kTagJit ? NBBGPU_PROGRAM_JIT : NBBGPU_PROGRAM_BUILTIN;
            bl = P.tag == kTagNone ? 0 : P.bP;
        }
        if (program) *program = prog;
        if (block_level) *block_level = bl;
    });
}

int nbbgpu_stream(nbbgpu_t h, void** stream) {
    return guarded([&] {
        if (!h || !stream) raise(NBBGPU_ERR_INVALID, "null argument");
        *stream = (void*)h->stream;
    });
}

int nbbgpu_lambda_batch(nbbgpu_t h, int variant, const int32_t* in, int32_t* out, int64_t count,
                        float* device_ms) {
    return guarded([&] {
        check_handle(h);
        run_map_batch(h, true, variant, in, out, count, device_ms);
    });
}

int nbbgpu_nu_batch(nbbgpu_t h, int variant, const int32_t* in, int32_t* out, int64_t count,
                    float* device_ms) {
    return guarded([&] {
        check_handle(h);
        run_map_batch(h, false, variant, in, out, count, device_ms);
    });
}

int nbbgpu_front_device_ptr(nbbgpu_t h, void** out) {
    return guarded([&] {
        if (!h || !out) raise(NBBGPU_ERR_INVALID, "null argument");
        *out = h->layout == 1 ? (void*)h->pk[h->cur] : (void*)h->front();
    });
}

}  // extern "C"

#include "partition.inc"

int nbbgpu_jit_compile_check(const int32_t* rep, int k, int s, int level, int moore, char* name, uint64_t name_bytes) {
    return guarded([&] {
        const HostFrac F = host_frac(rep, k, s, level);
        const PackedPlan P = build_packed_plan(F, choose_packed_level(F));
        if (P.tag != kTagJit) raise(NBBGPU_ERR_OUT_OF_DOMAIN, "the packed plan of this descriptor does not use a run-time specialised kernel");
        const JitShape j = jit_shape_for(P.bP, P.wq, P.split == 2 ? P.SWsplit : P.SW, P.Cp, F.k, P.split);
        std::vector<char> cubin;
        std::string lowered, err;
        if (!jit_compile(jit_source(F, P.wq, j.SPLIT == 1 ? P.SW : 0u, P.ilv != 0), jit_ws3_expr(true, moore ? 8 : 4, P.wide, P.wq, j),
                         "sm_100a", cubin, lowered, err))
            raise(NBBGPU_ERR_CUDA, "jit: " + err);
        if (name && name_bytes) {
            const std::string out = lowered + " (" + std::to_string(cubin.size()) + " B cubin)";
            std::strncpy(name, out.c_str(), (size_t)name_bytes - 1);
            name[name_bytes - 1] = '\0';
        }
    });
}
