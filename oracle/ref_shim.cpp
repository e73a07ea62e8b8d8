// ref_shim.cpp -- C ABI over the UNMODIFIED reference library (TEST INFRASTRUCTURE).
//
// Compiled by oracle/Makefile together with the reference's own sources from
// /root/reference/proj/src into oracle/_ref/libnbbref.so.  It lets the pytest
// suite, the golden-vector generator and bench.py's reference arm drive
// nbb::Simulation (proj/include/nbb/stencil.hpp:69-122) through its public API.
//
// The one non-public access: bench.py's reference arm times
// Simulation::step_compact_linear (proj/src/stencil.cpp:334-368) over a bounded
// sample of the compact index range of a large level, with the reference's own
// std::thread split (parallel_for, proj/src/stencil.cpp:236-260).  For that the
// private section is opened with a preprocessor override limited to this TU.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#define private public
#include "nbb/stencil.hpp"
#undef private
#include "nbb/errors.hpp"
#include "nbb/maps.hpp"
#include "nbb/rng.hpp"

using namespace nbb;

namespace {
thread_local std::string g_err;

int fail(const std::exception& e) {
    g_err = e.what();
    if (dynamic_cast<const ParseError*>(&e)) return 1;
    if (dynamic_cast<const NotInFractal*>(&e)) return 2;
    if (dynamic_cast<const OutOfDomain*>(&e)) return 3;
    if (dynamic_cast<const CapacityError*>(&e)) return 4;
    return 9;
}

FractalDescriptor make_desc(const int32_t* rep, int k, int s) {
    FractalDescriptor d;
    d.name = "custom";
    d.replica_count = k;
    d.growth = s;
    for (int i = 0; i < k; ++i) d.replicas.push_back({rep[2 * i], rep[2 * i + 1]});
    d.validate();
    return d;
}

StencilRule make_rule(uint16_t birth, uint16_t survive, int moore) {
    StencilRule r;
    r.birth = birth;
    r.survive = survive;
    r.neighborhood = moore ? Neighborhood::Moore : Neighborhood::VonNeumann;
    return r;
}
} // namespace

extern "C" {

const char* nbbref_last_error() { return g_err.c_str(); }

// backend: 0 = bb, 1 = lambda, 2 = compact (Backend, stencil.hpp:54)
int nbbref_create(const int32_t* rep, int k, int s, int level, int backend, int block_size,
                  int workers, int neighbor_table, uint64_t memory_cap, void** out) {
    try {
        SimOptions o;
        o.block_size = block_size;
        o.workers = workers;
        o.neighbor_table = neighbor_table != 0;
        o.memory_cap = memory_cap;
        *out = new Simulation(make_desc(rep, k, s), level, static_cast<Backend>(backend), o);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int nbbref_create_builtin(const char* spec, int level, int backend, int block_size, int workers,
                          int neighbor_table, uint64_t memory_cap, void** out) {
    try {
        SimOptions o;
        o.block_size = block_size;
        o.workers = workers;
        o.neighbor_table = neighbor_table != 0;
        o.memory_cap = memory_cap;
        *out = new Simulation(load_descriptor(spec), level, static_cast<Backend>(backend), o);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

void nbbref_destroy(void* h) { delete static_cast<Simulation*>(h); }

int nbbref_seed(void* h, uint64_t seed, double density) {
    try {
        static_cast<Simulation*>(h)->seed_random(seed, density);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int nbbref_step(void* h, uint16_t birth, uint16_t survive, int moore, int64_t nsteps) {
    try {
        auto* sim = static_cast<Simulation*>(h);
        const StencilRule rule = make_rule(birth, survive, moore);
        for (int64_t i = 0; i < nsteps; ++i) sim->step(rule);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

uint64_t nbbref_state_hash(void* h) { return static_cast<Simulation*>(h)->state_hash(); }

int64_t nbbref_front(void* h, const uint8_t** data) {
    const Grid& g = static_cast<Simulation*>(h)->front();
    *data = g.data();
    return g.stored_cell_count();
}

int nbbref_cell(void* h, int64_t x, int64_t y, uint8_t* out) {
    try {
        *out = static_cast<Simulation*>(h)->cell({x, y});
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int nbbref_set_cell(void* h, int64_t x, int64_t y, uint8_t v) {
    try {
        static_cast<Simulation*>(h)->set_cell({x, y}, v);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// One-shot maps (proj/src/maps.cpp:153-161).
int nbbref_to_compact(const int32_t* rep, int k, int s, int level, int64_t x, int64_t y,
                      int64_t* cx, int64_t* cy) {
    try {
        const CompactCoord c = to_compact(make_desc(rep, k, s), level, {x, y});
        *cx = c.cx;
        *cy = c.cy;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int nbbref_to_embedded(const int32_t* rep, int k, int s, int level, int64_t cx, int64_t cy,
                       int64_t* x, int64_t* y) {
    try {
        const EmbeddedCoord e = to_embedded(make_desc(rep, k, s), level, {cx, cy});
        *x = e.x;
        *y = e.y;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// Bench reference arm: seed the linear-compact front buffer in parallel using the
// reference's own mapper and cell_alive (the same values seed_random writes,
// stencil.cpp:152-159, which is single-threaded and takes minutes at r=20).
int nbbref_parallel_seed(void* h, uint64_t seed, double density, int workers) {
    try {
        auto* sim = static_cast<Simulation*>(h);
        if (sim->front_.layout() != Layout::LinearCompact) return 3;
        sim->front_.fill_dead();
        sim->back_.fill_dead();
        sim->iteration_ = 0;
        uint8_t* f = sim->front_.data();
        const int64_t total = sim->front_.stored_cell_count();
        const int64_t w = sim->mapper_.compact_width();
        const CoordMapper& mp = sim->mapper_;
        if (workers < 1) workers = 1;
        const int64_t chunk = (total + workers - 1) / workers;
        std::vector<std::thread> pool;
        for (int t = 0; t < workers; ++t) {
            const int64_t lo = t * chunk, hi = std::min(total, lo + chunk);
            if (lo >= hi) break;
            pool.emplace_back([=, &mp] {
                for (int64_t i = lo; i < hi; ++i) {
                    const EmbeddedCoord e = mp.to_embedded({i % w, i / w});
                    f[i] = cell_alive(seed, e.x, e.y, density) ? 1 : 0;
                }
            });
        }
        for (auto& t : pool) t.join();
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// Bench reference arm: seed only compact indices [i0, i1) (the sample), in parallel.
int nbbref_parallel_seed_range(void* h, uint64_t seed, double density, int64_t i0, int64_t i1,
                               int workers) {
    try {
        auto* sim = static_cast<Simulation*>(h);
        if (sim->front_.layout() != Layout::LinearCompact) return 3;
        uint8_t* f = sim->front_.data();
        const int64_t w = sim->mapper_.compact_width();
        const CoordMapper& mp = sim->mapper_;
        if (workers < 1) workers = 1;
        const int64_t total = i1 - i0;
        const int64_t chunk = (total + workers - 1) / workers;
        std::vector<std::thread> pool;
        for (int t = 0; t < workers; ++t) {
            const int64_t lo = i0 + t * chunk, hi = std::min(i1, lo + chunk);
            if (lo >= hi) break;
            pool.emplace_back([=, &mp] {
                for (int64_t i = lo; i < hi; ++i) {
                    const EmbeddedCoord e = mp.to_embedded({i % w, i / w});
                    f[i] = cell_alive(seed, e.x, e.y, density) ? 1 : 0;
                }
            });
        }
        for (auto& t : pool) t.join();
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// Bench reference arm: one bounded sample = step_compact_linear over compact
// indices [i0, i1), split into `workers` std::thread chunks exactly like
// parallel_for.  Writes the back buffer only (no swap).
int nbbref_sample_step(void* h, uint16_t birth, uint16_t survive, int moore, int64_t i0,
                       int64_t i1, int workers) {
    try {
        auto* sim = static_cast<Simulation*>(h);
        const StencilRule rule = make_rule(birth, survive, moore);
        if (workers < 1) workers = 1;
        const int64_t domain = i1 - i0;
        const int64_t chunk = (domain + workers - 1) / workers;
        std::vector<std::thread> pool;
        for (int t = 0; t < workers; ++t) {
            const int64_t lo = i0 + t * chunk, hi = std::min(i1, lo + chunk);
            if (lo >= hi) break;
            pool.emplace_back([sim, &rule, lo, hi] { sim->step_compact_linear(rule, lo, hi); });
        }
        for (auto& t : pool) t.join();
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

} // extern "C"
