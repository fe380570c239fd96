// TEST INFRASTRUCTURE ONLY (diagnostic): the body of test_adjoint.cpp:222-244 with every point printed.
#include <cstdio>
#include <random>
#include "helpers.hpp"
#include "randers/adjoint.hpp"
#include "randers/oracle.hpp"
using namespace randers;
int main() {
    const int n = 32;
    const GridSpec spec{n, n, 1.0};
    auto [g, b] = testutil::random_feasible_fields(n, 21, 0.1);
    double cs = 0; for (size_t i = 0; i < g.g11.size(); ++i) cs += g.g11[i] * (i % 7 + 1) + g.g12[i] * (i % 5) + g.g22[i] + b.b1[i] * 3 + b.b2[i];
    std::printf("fields checksum %.17g\n", cs);
    auto fnv = [](const Grid2D<double>& x) { unsigned long long h = 1469598103934665603ull; const unsigned char* p = reinterpret_cast<const unsigned char*>(x.data()); for (size_t i = 0; i < x.size() * 8; ++i) { h ^= p[i]; h *= 1099511628211ull; } return h; };
    std::printf("bits g11 %016llx g12 %016llx g22 %016llx b1 %016llx b2 %016llx\n", fnv(g.g11), fnv(g.g12), fnv(g.g22), fnv(b.b1), fnv(b.b2));
    int nd = 0; { MetricField g2(n, n, 1.0); (void)g2; }
    const SourceMask src = SourceMask::point(n, n, n / 2, n / 2);
    ObservationSet obs;
    obs.sources = src;
    obs.observed = Grid2D<uint8_t>(n, n, 0);
    obs.values = Grid2D<double>(n, n, 0.0);
    std::mt19937_64 rng(77);
    std::uniform_real_distribution<double> uni(0.0, 1.0);
    for (size_t i = 0; i < obs.observed.size(); ++i)
        if (!src.mask[i] && uni(rng) < 0.3) obs.observed[i] = 1;
    LossSpec loss{spec, {obs}};
    const GradCheckResult res = gradient_check(g, b, loss, {Channel::G11, Channel::G12, Channel::G22, Channel::B1, Channel::B2}, 10, 1e-5, 99);
    for (auto& p : res.points) std::printf("node %d ch %d fd %.17g an %.17g rel %.3e\n", p.node, (int)p.channel, p.fd, p.adjoint, p.rel_error);
    std::printf("max_rel %.3e skipped_unstable %d skipped_zero %d\n", res.max_rel_error, res.skipped_unstable, res.skipped_zero);
}
