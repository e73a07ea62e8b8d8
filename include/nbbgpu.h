/*
 * nbbgpu.h -- C ABI of the B200 (sm_100a) compact-fractal stencil engine.
 *
 * The drop-in boundary for the reference's hot path.  The reference has no plugin
 * API: its seam is the closed `Backend` enum and the `nbb::Simulation` methods
 * (proj/include/nbb/stencil.hpp:50-122).  Each export below replaces one of those
 * members for the two GPU backends `gpu-compact` / `gpu-bb`; the reference-side
 * adapter that forwards to them is shown in INTEGRATION.md.
 *
 * Conventions
 *  - every function returns an nbbgpu_status (0 = ok); exceptions never cross the
 *    ABI.  Codes 1..4 map 1:1 to the reference's ParseError / NotInFractal /
 *    OutOfDomain / CapacityError (proj/include/nbb/errors.hpp:10-27);
 *    NBBGPU_ERR_CUDA maps to std::runtime_error (CLI exit 1, tools/main.cpp:267-303).
 *  - nbbgpu_last_error() returns the message of the last failure on the calling
 *    thread (thread-local storage, valid until the next failing call).
 *  - buffers are plain host pointers unless stated otherwise; byte order is the
 *    reference's: compact `cy*w + cx` (k^r bytes, proj/src/grid.cpp:46-53) or
 *    embedded `y*n + x` (n^2 bytes, proj/src/grid.cpp:44-45).
 *  - a handle is single-owner and not re-entrant (Simulation is single-owner,
 *    SPEC.md:288).  Every call is synchronous on return, like Simulation::step.
 *  - cell states are binary {0,1}.  The reference only ever produces 0/1 (seeding,
 *    rules); uploads / set_cell of any other byte return NBBGPU_ERR_OUT_OF_DOMAIN.
 */
#ifndef NBBGPU_H
#define NBBGPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct nbbgpu_sim* nbbgpu_t;

typedef enum {
    NBBGPU_OK = 0,
    NBBGPU_ERR_PARSE = 1,          /* nbb::ParseError     */
    NBBGPU_ERR_NOT_IN_FRACTAL = 2, /* nbb::NotInFractal   */
    NBBGPU_ERR_OUT_OF_DOMAIN = 3,  /* nbb::OutOfDomain    */
    NBBGPU_ERR_CAPACITY = 4,       /* nbb::CapacityError ("memory cap" in the message) */
    NBBGPU_ERR_CUDA = 5,           /* std::runtime_error from the CUDA runtime */
    NBBGPU_ERR_INVALID = 6         /* null handle / bad argument */
} nbbgpu_status;

/* Backend + storage layout of a handle (proj/src/stencil.cpp:108-112):
 *   COMPACT  Backend::Compact, Layout::LinearCompact (k^r bytes, cy*w + cx)
 *   BB       Backend::BoundingBox, Layout::Embedded (n^2 bytes)
 *   LAMBDA   Backend::CompactGrid ("lambda"), Layout::Embedded, stepped over
 *            the k^r compact indices (stencil.cpp:313-332)
 *   BLOCKED  Backend::Compact with SimOptions::block_size = rho = s^m,
 *            Layout::BlockedCompact (k^(r-m) rho x rho blocks, grid.cpp:54-63) */
enum { NBBGPU_MODE_COMPACT = 0, NBBGPU_MODE_BB = 1, NBBGPU_MODE_LAMBDA = 2, NBBGPU_MODE_BLOCKED = 3 };

/* Step kernels (nbbgpu_set_kernel).  AUTO picks PACKED when the level admits a
 * packed tile level (even q >= 2), else TILED / NAIVE.  NAIVE is the paper's
 * per-cell kernel: lambda of the own cell plus nu of each neighbour
 * (proj/src/stencil.cpp:354-367); its map variant is chosen by
 * nbbgpu_set_map_variant.  NAIVE and TILED keep the state in the reference's byte
 * layout on the device; PACKED keeps it bit-sliced (1 bit per cell, groups of 32
 * level-q tiles, csrc/packed.cuh) and converts to / from the reference bytes on
 * download / upload.  Switching between the two families converts the state on
 * the device.  TABLE is SimOptions::neighbor_table (stencil.cpp:340-352, 401-414):
 * the byte layout stepped through a per-slot neighbour table built on the device
 * on the first step of a neighbourhood (deg x k^r slots, 32-bit below 2^32 cells).
 * Results are identical for every kernel. */
enum { NBBGPU_KERNEL_AUTO = 0, NBBGPU_KERNEL_NAIVE = 1, NBBGPU_KERNEL_TILED = 2, NBBGPU_KERNEL_PACKED = 3,
       NBBGPU_KERNEL_TABLE = 4 };

/* lambda / nu map variants: CUDA-core digit loop, or the paper's matrix form on
 * the tensor cores (exact integer MMA, u8 x u8 -> s32). */
enum { NBBGPU_MAP_DIGIT = 0, NBBGPU_MAP_MMA = 1, NBBGPU_MAP_TC05 = 2 };

const char* nbbgpu_last_error(void);
int nbbgpu_version(void);
/* Number of visible CUDA devices (0 when none; never fails). */
int nbbgpu_device_count(void);

/* Simulation::Simulation (proj/src/stencil.cpp:116-136).  replicas_xy holds k
 * (gx, gy) pairs in replica-ID order (FractalDescriptor::replicas,
 * descriptor.hpp:23-36); the descriptor is validated like
 * FractalDescriptor::validate (descriptor.cpp:12-44).  memory_cap is the per-grid
 * cell cap of Grid::Grid (grid.cpp:18-22; default 2 GiB, grid.hpp:13). */
int nbbgpu_create(const int32_t* replicas_xy, int k, int s, int level, int mode, int device,
                  uint64_t memory_cap, nbbgpu_t* out);
/* nbbgpu_create with SimOptions::block_size (stencil.hpp:59-64): block_size > 0
 * requires mode BLOCKED and must be a power of s not above s^level
 * (geometry.cpp:69-108, OutOfDomain otherwise); nbbgpu_create == block_size 0. */
int nbbgpu_create_ex(const int32_t* replicas_xy, int k, int s, int level, int mode, int block_size,
                     int device, uint64_t memory_cap, nbbgpu_t* out);
int nbbgpu_destroy(nbbgpu_t h);

/* Simulation::seed_random (stencil.cpp:138-180): both buffers zeroed, iteration
 * reset, every fractal cell alive iff cell_alive(seed, x, y, density)
 * (rng.hpp:27-33).  density outside [0,1] -> NBBGPU_ERR_OUT_OF_DOMAIN. */
int nbbgpu_seed(nbbgpu_t h, uint64_t seed, double density);

/* nsteps x Simulation::step (stencil.cpp:262-289) with rule
 * StencilRule{birth, survive, moore ? Moore : VonNeumann} (stencil.hpp:18-31). */
int nbbgpu_step(nbbgpu_t h, uint16_t birth, uint16_t survive, int moore, int64_t nsteps);
/* nbbgpu_step without the final host synchronisation (the steps are enqueued on
 * the handle's stream; the state must not be read before nbbgpu_synchronize). */
int nbbgpu_step_async(nbbgpu_t h, uint16_t birth, uint16_t survive, int moore, int64_t nsteps);
int nbbgpu_synchronize(nbbgpu_t h);

/* Same as nbbgpu_step, also returning the device time of the nsteps step
 * kernels measured with CUDA events on the handle's stream. */
int nbbgpu_step_timed(nbbgpu_t h, uint16_t birth, uint16_t survive, int moore, int64_t nsteps,
                      float* device_ms);

/* nbbgpu_step_timed plus: the summed device time of the main step kernels alone
 * (CUDA events around each of them, on the handle's stream) and the number of
 * engine kernels launched (step, halo-words and halo pack/unpack kernels; NCCL's
 * own kernels not counted). */
int nbbgpu_step_profiled(nbbgpu_t h, uint16_t birth, uint16_t survive, int moore, int64_t nsteps,
                         float* total_ms, float* main_kernel_ms, uint64_t* launches);

/* Engine kernels launched by step calls on this handle so far (as counted by
 * nbbgpu_step_profiled). */
int nbbgpu_launch_count(nbbgpu_t h, uint64_t* out);

/* Simulation::state_hash (stencil.cpp:196-234): wrapping uint64 sum of
 * coord_mix(x, y) over alive cells. */
int nbbgpu_state_hash(nbbgpu_t h, uint64_t* out);

/* Simulation::iteration() */
int nbbgpu_iteration(nbbgpu_t h, int64_t* out);

/* Grid::stored_cell_count() of the front buffer (k^r or n^2). */
int nbbgpu_stored_cells(nbbgpu_t h, uint64_t* out);
/* compact width / height / embedded side (CoordMapper, maps.hpp:39-42). */
int nbbgpu_dims(nbbgpu_t h, int64_t* w, int64_t* hgt, int64_t* side);

/* front().data() as a host copy (`bytes` must equal stored_cells). */
int nbbgpu_download(nbbgpu_t h, uint8_t* dst, uint64_t bytes);
/* Replaces the front buffer (reference byte order; holes must be 0 in bb mode). */
int nbbgpu_upload(nbbgpu_t h, const uint8_t* src, uint64_t bytes);

/* Simulation::cell / set_cell (stencil.cpp:182-194). */
int nbbgpu_get_cell(nbbgpu_t h, int64_t x, int64_t y, uint8_t* out);
int nbbgpu_set_cell(nbbgpu_t h, int64_t x, int64_t y, uint8_t state);

/* The embedded n x n view of the front state, Simulation::cell for every (x, y)
 * (stencil.cpp:182-188), computed on the device for any layout: `bytes` must be
 * side^2; dst is host or device memory. */
int nbbgpu_embedded_view(nbbgpu_t h, uint8_t* dst, uint64_t bytes);
/* write_pbm (pbm.cpp:9-23) rendered on the device: plain PBM "P1\n<n> <n>\n" + n
 * rows of '0'/'1' + '\n'.  side > render_cap -> NBBGPU_ERR_CAPACITY (the
 * reference's CapacityError).  dst == NULL returns the size in *written. */
int nbbgpu_render_pbm(nbbgpu_t h, char* dst, uint64_t capacity, int64_t render_cap, uint64_t* written);

/* Device bytes held by the handle (both state buffers + tables + scratch). */
int nbbgpu_peak_bytes(nbbgpu_t h, uint64_t* out);

/* Kernel selection (NBBGPU_KERNEL_*) and the naive kernel's map variant. */
int nbbgpu_set_kernel(nbbgpu_t h, int kernel);
int nbbgpu_set_map_variant(nbbgpu_t h, int variant);
/* The kernel the next step will launch (resolves AUTO) and its tile level q. */
int nbbgpu_active_kernel(nbbgpu_t h, int* kernel, int* tile_level);

/* The packed kernel's program: NBBGPU_PROGRAM_TABLE (table-driven step_packed_kernel),
 * _BUILTIN (micro-block wiring compiled in for the triangle, carpet, Vicsek, H and
 * candy descriptors), _JIT (micro-block wiring of this descriptor, compiled at run
 * time by NVRTC), _NONE (the next step is not a packed kernel); block_level = the
 * micro-block level P.  Replaces no reference entity (the reference has one program). */
#define NBBGPU_PROGRAM_NONE 0
#define NBBGPU_PROGRAM_TABLE 1
#define NBBGPU_PROGRAM_BUILTIN 2
#define NBBGPU_PROGRAM_JIT 3
int nbbgpu_packed_program(nbbgpu_t h, int* program, int* block_level);
/* Host only (no GPU): plan the descriptor's packed layout and, when it uses a run-time
 * specialised micro-block kernel, compile it for sm_100a with NVRTC; name receives the
 * kernel's lowered name.  OUT_OF_DOMAIN when the plan has no run-time kernel. */
int nbbgpu_jit_compile_check(const int32_t* replicas_xy, int k, int s, int level, int moore, char* name,
                             uint64_t name_bytes);

/* The handle's CUDA stream (cudaStream_t) for external event timing. */
int nbbgpu_stream(nbbgpu_t h, void** stream);

/* Batched maps of the handle's fractal (CoordMapper::to_embedded /
 * try_to_compact, maps.cpp:80-146).  Pointers may be host or device memory.
 *   lambda: in = count (cx, cy) int32 pairs -> out = count (x, y) int32 pairs
 *   nu:     in = count (x, y) pairs -> out = count (cx, cy) pairs, (-1, -1) for a
 *           hole or an out-of-box coordinate.
 * variant = NBBGPU_MAP_DIGIT (CUDA-core digit loop), NBBGPU_MAP_MMA (mma.sync u8
 * tensor cores) or NBBGPU_MAP_TC05 (tcgen05.mma kind::i8, TMEM accumulators; levels
 * <= 32 for both tensor-core forms).  device_ms (optional) receives
 * the kernel time.  The engine runs on its own stream: device buffers must be
 * complete (caller-side synchronisation) before the call. */
int nbbgpu_lambda_batch(nbbgpu_t h, int variant, const int32_t* in, int32_t* out, int64_t count,
                        float* device_ms);
int nbbgpu_nu_batch(nbbgpu_t h, int variant, const int32_t* in, int32_t* out, int64_t count,
                    float* device_ms);

/* ---- multi-GPU partitioning (one process per GPU) ---------------------------
 * Byte layouts (NAIVE / TILED): the unit is a tile row, halo elements are state
 * bytes at compact byte offsets.  PACKED: the unit is a group of 32 tiles (rank r
 * owns groups [NG r/n, NG (r+1)/n)), owned_range is in packed 32-bit words, and
 * halo elements are 32-bit boundary-plane words (element index g * nSrc + m);
 * nbbgpu_halo_elem_bytes tells which (1 or 4).
 * A handle may own a contiguous range of tile rows [row0, row1) of the compact
 * array (tile rows of h_q compact rows each; the whole array when nranks == 1).
 * It keeps a full-size copy of the state, updates only its rows, and exchanges
 * halo bytes with its peers between steps. */
int nbbgpu_partition(nbbgpu_t h, int rank, int nranks);
/* Owned compact byte range [lo, hi). */
int nbbgpu_owned_range(nbbgpu_t h, uint64_t* lo, uint64_t* hi);
/* Compact byte offsets this rank needs from `peer` (sorted, unique).  Pass
 * offsets == NULL to query the count.  Computed on the host at partition time. */
int nbbgpu_halo_needs(nbbgpu_t h, int peer, uint64_t* offsets, uint64_t* count);
/* Registers the offsets `peer` needs from this rank (its halo_needs(self)). */
int nbbgpu_halo_set_sends(nbbgpu_t h, int peer, const uint64_t* offsets, uint64_t count);
/* Gather the registered send bytes for `peer` from the front buffer into a DEVICE
 * buffer / scatter received bytes from a DEVICE buffer into the front buffer. */
int nbbgpu_halo_pack(nbbgpu_t h, int peer, void* dev_dst);
int nbbgpu_halo_unpack(nbbgpu_t h, int peer, const void* dev_src);
/* state_hash over the owned range only (sum over ranks = global hash). */
int nbbgpu_state_hash_owned(nbbgpu_t h, uint64_t* out);
/* In-library NCCL transport: rank 0 creates an ncclUniqueId (128 bytes), the
 * caller broadcasts it (e.g. torch.distributed), every rank attaches it after
 * nbbgpu_partition.  From then on nbbgpu_step enqueues, after each step kernel,
 * the halo pack kernel, grouped ncclSend/ncclRecv over NVLink and the unpack
 * kernel on the handle's stream (no host synchronisation between steps). */
int nbbgpu_nccl_unique_id(uint8_t* out, int bytes);
int nbbgpu_comm_init(nbbgpu_t h, const uint8_t* unique_id, int bytes);

/* Bytes per halo element of the handle's partition (1 = state byte, 4 = packed
 * boundary-plane word). */
int nbbgpu_halo_elem_bytes(nbbgpu_t h, int* out);

/* Peer-memory halo transport for the PACKED kernel (NVLink, CUDA IPC), an
 * alternative to nbbgpu_comm_init: every rank exports nbbgpu_p2p_handle_bytes()
 * bytes of IPC handles (its boundary planes + an arrival counter), the caller
 * all-gathers them in rank order and every rank attaches them.  From then on each
 * step pushes the boundary words peers need straight into their planes (one small
 * kernel, system-scope fence + counter), and the next halo kernel waits on this
 * rank's counter: no NCCL call and no host synchronisation per step. */
int nbbgpu_p2p_handle_bytes(void);
int nbbgpu_p2p_export(nbbgpu_t h, uint8_t* out, int bytes);
int nbbgpu_p2p_attach(nbbgpu_t h, const uint8_t* all_handles, int bytes_per_rank, int nranks);
/* The same transport for ONE process driving every rank (the proposed
 * SimOptions::gpus: "one host thread drives all GPUs"): handles[i]
 * is the packed partition rank i of nranks (nbbgpu_partition), one per device;
 * peer access is enabled between the devices and the peers' planes are plain
 * device pointers (no IPC).  Step the handles with nbbgpu_step_async, then
 * nbbgpu_synchronize each. */
int nbbgpu_p2p_attach_local(nbbgpu_t* handles, int nranks);

/* Raw device pointer of the front buffer (reference bytes, or packed words for
 * the PACKED kernel; for peer-to-peer transports). */
int nbbgpu_front_device_ptr(nbbgpu_t h, void** out);

/* ---- host-only planning (no GPU needed; same geometry as above) ------------
 * tile_level < 0 selects the level nbbgpu_create would choose for the compact
 * backend (0 = no tiling: partition rows are compact rows). */
int nbbgpu_plan_tile_level(const int32_t* replicas_xy, int k, int s, int level, int* tile_level);
int nbbgpu_plan_partition(const int32_t* replicas_xy, int k, int s, int level, int tile_level,
                          int rank, int nranks, uint64_t* owned_lo, uint64_t* owned_hi);
int nbbgpu_plan_needs(const int32_t* replicas_xy, int k, int s, int level, int tile_level,
                      int rank, int nranks, int peer, uint64_t* offsets, uint64_t* count);
/* info = [q, wq, C, nH, L, Wc, Hc, dmask] of the tile plan. */
int nbbgpu_plan_tiles(const int32_t* replicas_xy, int k, int s, int level, int tile_level,
                      int moore, int32_t* info);

/* ---- host-only planning of the packed layout --------------------------------
 * tile_level < 0 selects the level nbbgpu_create would choose (-1 = none).
 * info = [q, wq, C, Cp, nH, nSrc, T, NG, Wc, Hc, nD, wide]. */
int nbbgpu_plan_packed_level(const int32_t* replicas_xy, int k, int s, int level, int* tile_level);
int nbbgpu_plan_packed(const int32_t* replicas_xy, int k, int s, int level, int tile_level, int64_t* info);
int nbbgpu_plan_packed_partition(const int32_t* replicas_xy, int k, int s, int level, int tile_level,
                                 int rank, int nranks, int64_t* group0, int64_t* group1);
/* Boundary-plane elements rank needs from peer (sorted, unique; elems == NULL -> count). */
int nbbgpu_plan_packed_needs(const int32_t* replicas_xy, int k, int s, int level, int tile_level,
                             int rank, int nranks, int peer, uint64_t* elems, uint64_t* count);
/* Compact byte offsets of the cells a boundary-plane element holds (<= 32 per element). */
int nbbgpu_plan_packed_elem_cells(const int32_t* replicas_xy, int k, int s, int level, int tile_level,
                                  const uint64_t* elems, uint64_t n, uint64_t* out, uint64_t* count);

#ifdef __cplusplus
}
#endif
#endif /* NBBGPU_H */
