// TEST INFRASTRUCTURE ONLY: runs the reference's acceptance suite
// (/root/reference/proj/tests/acceptance_main.cpp, criteria A1-A9 of SPEC.md
// :539-549) against the DROP-IN: the suite is compiled unchanged with our
// include/geodist first on the include path and linked against
// libgeodist_b200.so (oracle/Makefile, target dropin-tests).  Its own main() is
// renamed so each criterion can run under try/catch:
//   * A1 and A2 also run Engine::Serial, the reference's CPU raster engine,
//     which the drop-in rejects with std::invalid_argument (no CPU fallback):
//     expected failures.  "A1p" below restates A1 for the parallel engine only
//     (the same 50 + 20 instances from Rng(2024), fixpoint vs Dijkstra <= 1e-4);
//   * A6 drives the reference CLI, which is not part of this build: expected
//     failure;
//   * A8 exercises the reference's FGD1 I/O (compiled in as a helper): it runs,
//     but it does not touch the drop-in.
// Exit status: the number of unexpected failures.
#include <cstdio>
#include <stdexcept>
#include <string>

#define main geodist_reference_acceptance_main
#include "acceptance_main.cpp"
#undef main

namespace {

// acceptance_main.cpp:72-123 without the serial engine.
void run_a1_parallel_only() {
    Rng rng(2024);
    const double lambdas[3] = {0.0, 0.5, 1.0};
    double worst = 0.0;
    int runs = 0;
    bool converged = true;
    auto exercise = [&](const ScalarGrid& image, const ScalarGrid& init) {
        for (double lambda : lambdas) {
            TransformParams params;
            params.lambda = lambda;
            auto par = scan_to_fixpoint(image, init, params, Engine::Parallel, 100,
                                        kDefaultFixpointTol, 2);
            converged = converged && par.converged;
            auto oracle = dijkstra_exact(image, init, lambda);
            worst = std::max(worst, testing::max_abs_diff(par.dist, oracle));
            ++runs;
        }
    };
    for (int i = 0; i < 50; ++i) {
        ScalarGrid image = testing::random_image(rng, 2, {16, 16}, {1.0, 1.0});
        ScalarGrid init = testing::random_seed_init(rng, image, 1 + rng.below(3));
        exercise(image, init);
    }
    for (int i = 0; i < 20; ++i) {
        ScalarGrid image = testing::random_image(rng, 3, {8, 8, 8}, {1.0, 1.0, 1.0});
        ScalarGrid init = testing::random_seed_init(rng, image, 1 + rng.below(3));
        exercise(image, init);
    }
    const std::string d = "max |parallel - dijkstra| = " + fmt(worst) + " over " +
                          std::to_string(runs) + " runs (parallel engine only)";
    if (converged && worst <= 1e-4) pass("A1p", "oracle-equivalence", d);
    else fail("A1p", "oracle-equivalence", d + (converged ? "" : ", non-convergence"));
}

}  // namespace

int main() {
    struct Crit {
        const char* id;
        void (*fn)();
        bool expected_fail;
        const char* why;
    };
    const Crit crits[] = {
        {"A1/A2", run_a1_a2, true, "runs Engine::Serial, rejected by the drop-in (no CPU engine)"},
        {"A1p", run_a1_parallel_only, false, ""},
        {"A3", run_a3, false, ""},
        {"A4", run_a4, false, ""},
        {"A5", run_a5, false, ""},
        {"A6", run_a6, true, "drives the reference CLI binary, not part of this build"},
        {"A7", run_a7, false, ""},
        {"A8", run_a8, false, "reference FGD1 I/O helper, not the drop-in"},
        {"A9", run_a9, false, ""},
    };
    int unexpected = 0;
    for (const Crit& c : crits) {
        const int before = g_failures;
        bool threw = false;
        try {
            c.fn();
        } catch (const std::exception& e) {
            threw = true;
            std::printf("%s: EXCEPTION (%s)\n", c.id, e.what());
        }
        const bool failed = threw || g_failures != before;
        if (failed && c.expected_fail) {
            std::printf("%s: expected failure -- %s\n", c.id, c.why);
        } else if (failed) {
            ++unexpected;
        }
    }
    std::printf("dropin acceptance: %d unexpected failure(s)\n", unexpected);
    return unexpected;
}
