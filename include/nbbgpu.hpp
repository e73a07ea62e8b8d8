// nbbgpu.hpp -- header-only C++ RAII wrapper over the C ABI (include/nbbgpu.h).
//
// Mirrors nbb::Simulation (proj/include/nbb/stencil.hpp:69-122) member for member
// for the GPU backends, with the reference's error classes mapped from status
// codes.  The reference-side adapter in INTEGRATION.md forwards
// nbb::Simulation to this class when Backend::GpuCompact / GpuBoundingBox is chosen.
#ifndef NBBGPU_HPP
#define NBBGPU_HPP

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "nbbgpu.h"

namespace nbbgpu {

// Status -> exception; `Mapper` lets the caller throw its own types
// (nbb::ParseError, ...).  Default: std::runtime_error subclasses below.
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
struct ParseError : Error { using Error::Error; };
struct NotInFractal : Error { using Error::Error; };
struct OutOfDomain : Error { using Error::Error; };
struct CapacityError : Error { using Error::Error; };

inline void check(int status) {
    if (status == NBBGPU_OK) return;
    const std::string msg = nbbgpu_last_error();
    switch (status) {
        case NBBGPU_ERR_PARSE: throw ParseError(status, msg);
        case NBBGPU_ERR_NOT_IN_FRACTAL: throw NotInFractal(status, msg);
        case NBBGPU_ERR_OUT_OF_DOMAIN: throw OutOfDomain(status, msg);
        case NBBGPU_ERR_CAPACITY: throw CapacityError(status, msg);
        default: throw Error(status, msg);
    }
}

enum class Mode {
    Compact = NBBGPU_MODE_COMPACT,
    BoundingBox = NBBGPU_MODE_BB,
    Lambda = NBBGPU_MODE_LAMBDA,    // Backend::CompactGrid
    Blocked = NBBGPU_MODE_BLOCKED   // Backend::Compact with SimOptions::block_size
};

class Simulation {
public:
    // replicas: k (gx, gy) pairs in replica-ID order (FractalDescriptor::replicas)
    // block_size: SimOptions::block_size, only with Mode::Blocked
    Simulation(const std::vector<std::pair<int, int>>& replicas, int growth, int level, Mode mode,
               std::uint64_t memory_cap = 2ull << 30, int device = 0, int block_size = 0) {
        std::vector<int32_t> flat;
        for (auto [x, y] : replicas) { flat.push_back(x); flat.push_back(y); }
        check(nbbgpu_create_ex(flat.data(), (int)replicas.size(), growth, level, (int)mode, block_size,
                               device, memory_cap, &h_));
    }
    ~Simulation() { nbbgpu_destroy(h_); }
    Simulation(const Simulation&) = delete;
    Simulation& operator=(const Simulation&) = delete;
    Simulation(Simulation&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}

    void seed_random(std::uint64_t seed, double density) { check(nbbgpu_seed(h_, seed, density)); }
    void step(std::uint16_t birth, std::uint16_t survive, bool moore, std::int64_t n = 1) {
        check(nbbgpu_step(h_, birth, survive, moore ? 1 : 0, n));
    }
    std::uint8_t cell(std::int64_t x, std::int64_t y) const {
        std::uint8_t v = 0;
        check(nbbgpu_get_cell(h_, x, y, &v));
        return v;
    }
    void set_cell(std::int64_t x, std::int64_t y, std::uint8_t state) {
        check(nbbgpu_set_cell(h_, x, y, state));
    }
    std::uint64_t state_hash() const {
        std::uint64_t v = 0;
        check(nbbgpu_state_hash(h_, &v));
        return v;
    }
    std::int64_t iteration() const {
        std::int64_t v = 0;
        check(nbbgpu_iteration(h_, &v));
        return v;
    }
    // front().data() as a host copy (reference byte order)
    std::vector<std::uint8_t> front() const {
        std::uint64_t n = 0;
        check(nbbgpu_stored_cells(h_, &n));
        std::vector<std::uint8_t> buf(n);
        check(nbbgpu_download(h_, buf.data(), n));
        return buf;
    }
    // front().data() into a caller buffer of n = stored cells bytes (host or device)
    void download(std::uint8_t* dst, std::uint64_t n) const { check(nbbgpu_download(h_, dst, n)); }
    // NBBGPU_KERNEL_* (SimOptions::neighbor_table -> NBBGPU_KERNEL_TABLE)
    void set_kernel(int kernel) { check(nbbgpu_set_kernel(h_, kernel)); }
    nbbgpu_t handle() const { return h_; }

private:
    nbbgpu_t h_ = nullptr;
};

}  // namespace nbbgpu

#endif
