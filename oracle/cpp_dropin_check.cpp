// cpp_dropin_check.cpp -- C++-level drop-in check (TEST INFRASTRUCTURE).
//
// Links the UNMODIFIED reference library (oracle/_ref, built from
// /root/reference/proj/src) and the GPU engine's C ABI through the header-only
// wrapper include/nbbgpu.hpp, and runs nbb::Simulation (CPU) and
// nbbgpu::Simulation (GPU) in lockstep on the same descriptors, rules and seeds:
// the compact / embedded bytes must be identical after every step, exactly as a
// reference user would see after switching Backend::Compact -> GpuCompact.
// Built by `make -C oracle dropin`; run by tests/test_gpu_dropin.py on a GPU box.
#include <cstdio>
#include <cstring>
#include <vector>

#include "nbb/descriptor.hpp"
#include "nbb/rng.hpp"
#include "nbb/stencil.hpp"
#include "nbbgpu.hpp"

namespace {

int check_case(const nbb::FractalDescriptor& d, int level, nbb::Backend cpu_backend,
               nbbgpu::Mode mode, nbb::StencilRule rule, std::uint64_t seed, double density,
               int steps) {
    nbb::SimOptions o;
    o.memory_cap = 1ull << 40;
    nbb::Simulation ref(d, level, cpu_backend, o);
    std::vector<std::pair<int, int>> reps;
    for (auto r : d.replicas) reps.push_back({r.gx, r.gy});
    nbbgpu::Simulation gpu(reps, d.growth, level, mode, 1ull << 40);
    ref.seed_random(seed, density);
    gpu.seed_random(seed, density);
    for (int s = 0; s <= steps; ++s) {
        if (s > 0) {
            ref.step(rule);
            gpu.step(rule.birth, rule.survive, rule.neighborhood == nbb::Neighborhood::Moore);
        }
        const auto buf = gpu.front();
        const auto& g = ref.front();
        if ((std::int64_t)buf.size() != g.stored_cell_count() ||
            std::memcmp(buf.data(), g.data(), buf.size()) != 0 || ref.state_hash() != gpu.state_hash()) {
            std::printf("MISMATCH %s r=%d mode=%d rule=%s step=%d\n", d.name.c_str(), level, (int)mode,
                        rule.to_string().c_str(), s);
            return 1;
        }
    }
    // cell() / set_cell() and the exception mapping
    try {
        gpu.set_cell(0, 0, 1);
        ref.set_cell({0, 0}, 1);
    } catch (const nbbgpu::NotInFractal&) {
    }
    if (gpu.cell(0, 0) != ref.cell({0, 0})) return 1;
    return 0;
}

}  // namespace

int main() {
    int bad = 0, n = 0;
    nbb::SplitMix rng(31337);
    const char* names[] = {"sierpinski-triangle", "sierpinski-carpet", "vicsek"};
    for (int t = 0; t < 12; ++t) {
        const auto d = nbb::builtin_descriptor(names[t % 3]);
        const int level = d.growth == 2 ? 5 + (int)rng.next_below(5) : 2 + (int)rng.next_below(3);
        nbb::StencilRule rule;
        rule.birth = (std::uint16_t)(rng.next() & 0x1ff);
        rule.survive = (std::uint16_t)(rng.next() & 0x1ff);
        if (t % 4 == 0) rule = nbb::conway_rule();
        rule.neighborhood = (rng.next() & 1) ? nbb::Neighborhood::Moore : nbb::Neighborhood::VonNeumann;
        const std::uint64_t seed = rng.next();
        bad += check_case(d, level, nbb::Backend::Compact, nbbgpu::Mode::Compact, rule, seed, 0.5, 6);
        ++n;
        if (level <= 8) {
            bad += check_case(d, level, nbb::Backend::BoundingBox, nbbgpu::Mode::BoundingBox, rule, seed,
                              0.5, 4);
            ++n;
        }
    }
    std::printf("%s: %d/%d drop-in cases identical\n", bad ? "FAIL" : "OK", n - bad, n);
    return bad ? 1 : 0;
}
