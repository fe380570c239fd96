// TEST INFRASTRUCTURE ONLY — the drop-in's threading contract: the reference
// functions are reentrant, so a caller may run independent
// problems on several threads.  Eight threads solve eight different problems
// through randers::solve / identify_stencils / solve_adjoint /
// param_gradients (the B200 shim, one rfk_context per thread) concurrently,
// twice; every result must equal the same call made alone, bit for bit.
// Prints "threads ok" and exits 0, or the first mismatch and exits 1.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

#include "randers/adjoint.hpp"
#include "randers/oracle.hpp"
#include "randers/sweeper.hpp"

using namespace randers;

struct Result {
    std::vector<double> t, lam, g11;
    int iterations = 0;
};

static Result run(int k) {
    const int n = 48 + 8 * k;
    const GridSpec spec{n, n + 5, 1.0 / n};
    MetricField g(n, n + 5, 1.0);
    DriftField b(n, n + 5);
    for (int r = 0; r < n; ++r)
        for (int c = 0; c < n + 5; ++c) {
            g.g11(r, c) = 1.0 + 0.3 * std::sin(0.1 * r + k);
            g.g12(r, c) = 0.1 * std::cos(0.07 * c);
            b.b1(r, c) = 0.1 * std::sin(0.05 * (r + c) + k);
        }
    const SourceMask src = SourceMask::point(n, n + 5, n / 3, (n + 5) / 2);
    auto [t, rep] = solve(g, b, src, spec, SolveOptions{});
    Grid2D<double> lg(n, n + 5, 0.0);
    for (size_t i = 0; i < lg.size(); i += 3) lg[i] = t.t[i] < 1e9 ? t.t[i] : 0.0;
    for (int r = 0; r < n; ++r)
        for (int c = 0; c < n + 5; ++c)
            if (src.is_source(r, c)) lg(r, c) = 0.0;
    const StencilRecordSet rs = identify_stencils(t, g, b, src, spec);
    const AdjointField adj = solve_adjoint(rs, t, lg);
    const ParamGradients pg = param_gradients(rs, adj);
    Result res;
    res.t.assign(t.t.data(), t.t.data() + t.t.size());
    res.lam.assign(adj.lambda.data(), adj.lambda.data() + adj.lambda.size());
    res.g11.assign(pg.g11.data(), pg.g11.data() + pg.g11.size());
    res.iterations = rep.iterations;
    return res;
}

static bool same(const std::vector<double>& a, const std::vector<double>& b) {
    return a.size() == b.size() && std::memcmp(a.data(), b.data(), a.size() * sizeof(double)) == 0;
}

int main() {
    const int T = 8;
    std::vector<Result> alone(T);
    for (int k = 0; k < T; ++k) alone[k] = run(k);
    for (int round = 0; round < 2; ++round) {
        std::vector<Result> conc(T);
        std::vector<std::thread> th;
        for (int k = 0; k < T; ++k) th.emplace_back([&, k] { conc[k] = run(k); });
        for (auto& x : th) x.join();
        for (int k = 0; k < T; ++k)
            if (conc[k].iterations != alone[k].iterations || !same(conc[k].t, alone[k].t) ||
                !same(conc[k].lam, alone[k].lam) || !same(conc[k].g11, alone[k].g11)) {
                std::printf("mismatch: round %d problem %d\n", round, k);
                return 1;
            }
    }
    std::printf("threads ok\n");
    return 0;
}
