// gpu_callers.cpp -- the reference's own callers driving the GPU backends.
// TEST INFRASTRUCTURE (built by oracle/Makefile into oracle/_ref/gpu/, run by
// tests/test_gpu_dropin.py on a GPU box).
//
// Linked against the reference library compiled with oracle/gpu_backend.patch
// (Backend::GpuCompact / GpuBoundingBox forwarding nbb::Simulation to
// libnbbgpu.so through include/nbbgpu.hpp).  Every call below goes through an
// UNCHANGED reference entry point:
//   parse_backend / backend_name        stencil.cpp:83-104
//   run_simulation                      stencil.cpp:416-439
//   Simulation::{seed_random, step, cell, set_cell, state_hash, front}
//   verify_stencil + LockstepHook       oracle.cpp:132-186
//   bench_run / write_csv / read_csv    bench.cpp:83-153
//   the reference exceptions            errors.hpp:10-27
// and compares the GPU results with the CPU backends of the same library.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <iostream>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "nbb/bench.hpp"
#include "nbb/descriptor.hpp"
#include "nbb/errors.hpp"
#include "nbb/oracle.hpp"
#include "nbb/rng.hpp"
#include "nbb/stencil.hpp"

using namespace nbb;

namespace {

int failures = 0;

void check(bool ok, const std::string& what) {
    std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", what.c_str());
    std::fflush(stdout);
    if (!ok) ++failures;
}

template <class E, class F>
bool throws(F&& f, const char* needle = nullptr) {
    try {
        f();
    } catch (const E& e) {
        return !needle || std::strstr(e.what(), needle) != nullptr;
    } catch (...) {
        return false;
    }
    return false;
}

bool same_front(const Simulation& a, const Simulation& b) {
    const Grid& fa = a.front();
    const Grid& fb = b.front();
    return fa.stored_cell_count() == fb.stored_cell_count() &&
           std::memcmp(fa.data(), fb.data(), (size_t)fa.stored_cell_count()) == 0;
}

// parse_backend / backend_name round trip for the two new names
void names() {
    check(parse_backend("gpu-compact") == Backend::GpuCompact &&
              parse_backend("gpu-bb") == Backend::GpuBoundingBox &&
              backend_name(Backend::GpuCompact) == "gpu-compact" &&
              backend_name(Backend::GpuBoundingBox) == "gpu-bb" && parse_backend("compact") == Backend::Compact,
          "parse_backend / backend_name: gpu-compact, gpu-bb");
    check(throws<ParseError>([] { parse_backend("gpu"); }, "unknown backend"), "parse_backend rejects 'gpu'");
}

// run_simulation (stencil.cpp:416-439) on every backend: identical state hashes
void run_simulation_all() {
    struct Case { const char* fractal; int level; std::int64_t steps; };
    for (Case c : {Case{"sierpinski-triangle", 10, 100}, Case{"sierpinski-triangle", 6, 100},
                   Case{"sierpinski-carpet", 5, 20}, Case{"vicsek", 6, 20}}) {
        const auto desc = builtin_descriptor(c.fractal);
        const auto cpu = run_simulation(desc, c.level, Backend::Compact, conway_rule(), c.steps, 42, 0.5);
        const auto gpu = run_simulation(desc, c.level, Backend::GpuCompact, conway_rule(), c.steps, 42, 0.5);
        const auto gbb = run_simulation(desc, c.level, Backend::GpuBoundingBox, conway_rule(), c.steps, 42, 0.5);
        const auto bb = run_simulation(desc, c.level, Backend::BoundingBox, conway_rule(), c.steps, 42, 0.5);
        char buf[256];
        std::snprintf(buf, sizeof buf, "run_simulation %s r=%d %lld steps: compact %016llx gpu-compact %016llx "
                      "gpu-bb %016llx bb %016llx", c.fractal, c.level, (long long)c.steps,
                      (unsigned long long)cpu.state_hash, (unsigned long long)gpu.state_hash,
                      (unsigned long long)gbb.state_hash, (unsigned long long)bb.state_hash);
        check(cpu.state_hash == gpu.state_hash && gpu.state_hash == gbb.state_hash && bb.state_hash == cpu.state_hash &&
                  gpu.steps == c.steps && (std::int64_t)gpu.step_ms.size() == c.steps,
              buf);
    }
}

// Simulation methods + front() bytes after every step (compact, bb, blocked, table)
void lockstep_bytes() {
    const auto T = builtin_descriptor("sierpinski-triangle");
    struct Case { Backend cpu, gpu; int block; bool table; const char* what; };
    for (Case c : {Case{Backend::Compact, Backend::GpuCompact, 0, false, "compact"},
                   Case{Backend::BoundingBox, Backend::GpuBoundingBox, 0, false, "bb"},
                   Case{Backend::Compact, Backend::GpuCompact, 4, false, "blocked rho=4"},
                   Case{Backend::Compact, Backend::GpuCompact, 0, true, "neighbor table"}}) {
        SimOptions o;
        o.block_size = c.block;
        o.neighbor_table = c.table;
        Simulation a(T, 9, c.cpu, o), b(T, 9, c.gpu, o);
        a.seed_random(7, 0.4);
        b.seed_random(7, 0.4);
        bool ok = same_front(a, b);
        for (int it = 0; it < 12 && ok; ++it) {
            a.step(conway_rule());
            b.step(conway_rule());
            ok = same_front(a, b) && a.state_hash() == b.state_hash() && a.iteration() == b.iteration();
        }
        // embedded-coordinate reads and fault injection through set_cell
        const EmbeddedCoord e{0, 0};
        a.set_cell(e, 1);
        b.set_cell(e, 1);
        ok = ok && b.cell(e) == 1 && same_front(a, b) && a.state_hash() == b.state_hash();
        a.step(conway_rule());
        b.step(conway_rule());
        ok = ok && same_front(a, b);
        check(ok, std::string("Simulation lockstep, front() bytes every step: ") + c.what);
    }
}

// the reference's error behaviour through the GPU backends
void errors() {
    const auto T = builtin_descriptor("sierpinski-triangle");
    Simulation g(T, 6, Backend::GpuCompact);
    check(throws<NotInFractal>([&] { g.set_cell({1, 1}, 1); }, "fractal cell"), "set_cell on a hole -> NotInFractal");
    check(throws<OutOfDomain>([&] { (void)g.cell({64, 0}); }), "cell outside the box -> OutOfDomain");
    check(throws<OutOfDomain>([&] { g.seed_random(1, 1.5); }, "density"), "density 1.5 -> OutOfDomain");
    check(g.cell({1, 1}) == 0, "cell on a hole reads dead");
    SimOptions tiny;
    tiny.memory_cap = 1000;
    check(throws<CapacityError>([&] { Simulation s(T, 8, Backend::GpuCompact, tiny); }, "memory cap"),
          "gpu-compact over the memory cap -> CapacityError");
    check(throws<CapacityError>([&] { Simulation s(T, 6, Backend::GpuBoundingBox, tiny); }, "memory cap"),
          "gpu-bb over the memory cap -> CapacityError");
    SimOptions blk;
    blk.block_size = 4;
    check(throws<OutOfDomain>([&] { Simulation s(T, 6, Backend::GpuBoundingBox, blk); }, "block size"),
          "block size on gpu-bb -> OutOfDomain");
}

// verify_stencil (oracle.cpp:132-186) with the GPU engine in place of the compact
// backend: the test hook NBB_GPU_SUBSTITUTE makes its Backend::Compact simulation
// a GpuCompact one; a LockstepHook fault injection must be caught
void verify_stencil_gpu() {
    const auto T = builtin_descriptor("sierpinski-triangle");
    setenv("NBB_GPU_SUBSTITUTE", "compact", 1);
    const auto rep = verify_stencil(T, 6, conway_rule(), 42, 0.5, 100);
    bool saw_gpu = false;
    const auto probe = verify_stencil(T, 3, conway_rule(), 1, 0.5, 1, [&](std::int64_t, const std::vector<Simulation*>& s) {
        saw_gpu = saw_gpu || s.back()->backend() == Backend::GpuCompact;
    });
    check(rep.pass && probe.pass && saw_gpu, "verify_stencil T r=6, 100 lockstep steps: bb, lambda, gpu-compact");
    const auto broken = verify_stencil(T, 6, conway_rule(), 42, 0.5, 10, [](std::int64_t it, const std::vector<Simulation*>& s) {
        if (it == 3) {  // flip a live fractal cell of the GPU simulation only
            const EmbeddedCoord e{0, 0};
            s.back()->set_cell(e, s.back()->cell(e) ? 0 : 1);
        }
    });
    check(!broken.pass && !broken.violations.empty() &&
              broken.violations.front().find("gpu-compact diverges from bb at iteration 3") != std::string::npos,
          "verify_stencil catches a GPU fault injected at iteration 3");
    setenv("NBB_GPU_SUBSTITUTE", "bb", 1);
    const auto rep_bb = verify_stencil(builtin_descriptor("sierpinski-carpet"), 4, conway_rule(), 42, 0.5, 20);
    check(rep_bb.pass, "verify_stencil carpet r=4, 20 steps: gpu-bb as the reference backend");
    unsetenv("NBB_GPU_SUBSTITUTE");
}

// bench_run (bench.cpp:83-138) with the GPU backends: CSV rows, speedup_vs_bb, and
// the acceptance-C8 memory-cap demonstration on the GPU
void bench_gpu() {
    BenchConfig config;
    config.desc = builtin_descriptor("sierpinski-triangle");
    config.levels = {10, 16};
    config.backends = {Backend::BoundingBox, Backend::GpuBoundingBox, Backend::Compact, Backend::GpuCompact};
    config.reps = 2;
    config.iters = 3;
    config.warmup = true;
    config.memory_cap = 2ull << 30;
    config.workers = 8;
    const auto recs = bench_run(config, &std::cout);
    std::ostringstream csv;
    write_csv(recs, csv);
    std::istringstream in(csv.str());
    const auto parsed = read_csv(in);
    std::printf("%s", csv.str().c_str());
    auto find = [&](int level, const char* b) -> const BenchRecord* {
        for (const auto& r : parsed)
            if (r.level == level && r.backend == b) return &r;
        return nullptr;
    };
    const BenchRecord* g10 = find(10, "gpu-compact");
    const BenchRecord* gb10 = find(10, "gpu-bb");
    const BenchRecord* b16 = find(16, "bb");
    const BenchRecord* gb16 = find(16, "gpu-bb");
    const BenchRecord* g16 = find(16, "gpu-compact");
    check(parsed.size() == 8 && g10 && g10->mean_ms && g10->speedup_vs_bb && gb10 && gb10->mean_ms,
          "bench_run r=10: gpu-compact and gpu-bb rows timed, speedup_vs_bb set");
    check(b16 && !b16->mean_ms && gb16 && !gb16->mean_ms && gb16->mem_cells == 4294967296LL && g16 && g16->mean_ms &&
              g16->mem_cells == 43046721LL,
          "bench_run r=16 under a 2 GiB cap: bb and gpu-bb skipped, gpu-compact ran (acceptance C8 on the GPU)");
}

// acceptance C9 (parallel determinism) extended: 20 randomized configs, the GPU
// backends against the CPU ones at 1 and 8 workers
void determinism() {
    SplitMix rng(777);
    const char* names[] = {"sierpinski-triangle", "sierpinski-carpet", "vicsek"};
    bool ok = true;
    for (int trial = 0; trial < 20 && ok; ++trial) {
        const auto desc = builtin_descriptor(names[rng.next_below(3)]);
        const int r = desc.growth == 2 ? 3 + (int)rng.next_below(3) : 2 + (int)rng.next_below(2);
        StencilRule rule;
        rule.birth = (std::uint16_t)(rng.next() & 0x1ff);
        rule.survive = (std::uint16_t)(rng.next() & 0x1ff);
        rule.neighborhood = rng.next() & 1 ? Neighborhood::Moore : Neighborhood::VonNeumann;
        const std::uint64_t seed = rng.next();
        const auto steps = (std::int64_t)(1 + rng.next_below(8));
        SimOptions crowd;
        crowd.workers = 8;
        const auto a = run_simulation(desc, r, Backend::Compact, rule, steps, seed, 0.5, crowd);
        const auto b = run_simulation(desc, r, Backend::GpuCompact, rule, steps, seed, 0.5);
        const auto c = run_simulation(desc, r, Backend::GpuBoundingBox, rule, steps, seed, 0.5);
        ok = a.state_hash == b.state_hash && a.state_hash == c.state_hash;
        if (!ok) std::printf("  trial %d %s r=%d %s diverges\n", trial, desc.name.c_str(), r, rule.to_string().c_str());
    }
    check(ok, "20 randomized configs (C9 generator, B/S from 0x1ff, Moore/von Neumann): gpu == cpu");
}

}  // namespace

int main(int argc, char** argv) {
    const std::string only = argc > 1 ? argv[1] : "";
    const std::vector<std::pair<const char*, std::function<void()>>> parts = {
        {"names", names}, {"run_simulation", run_simulation_all}, {"lockstep", lockstep_bytes},
        {"errors", errors}, {"verify_stencil", verify_stencil_gpu}, {"bench_run", bench_gpu},
        {"determinism", determinism}};
    for (const auto& [name, fn] : parts) {
        if (!only.empty() && only != name) continue;
        try {
            fn();
        } catch (const std::exception& e) {
            check(false, std::string(name) + ": exception: " + e.what());
        }
    }
    std::printf("%s: %d failure(s)\n", failures ? "FAILED" : "OK", failures);
    return failures ? 1 : 0;
}
