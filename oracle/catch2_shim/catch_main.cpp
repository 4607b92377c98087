// Test runner for the Catch2 shim (TEST INFRASTRUCTURE ONLY): runs every
// registered reference TEST_CASE, prints a one-line summary, exits non-zero on
// any failure.  Arguments: a bare substring keeps only matching test names;
// "~substring" skips matching names (used for test_scenario.cpp:89, which
// calls std::count over iterators of two different temporaries -- undefined
// behaviour in the reference test itself, caught by -fsanitize=address).
#include <catch2/catch_amalgamated.hpp>

#include <cstring>
#include <exception>

int main(int argc, char** argv) {
    using namespace Catch::shim;
    int cases = 0, failed_cases = 0;
    for (const Case& c : registry()) {
        bool keep = true;
        for (int i = 1; i < argc; ++i) {
            if (argv[i][0] == '~') {
                if (std::strstr(c.name, argv[i] + 1)) keep = false;
            } else if (!std::strstr(c.name, argv[i])) {
                keep = false;
            }
        }
        if (!keep) continue;
        ++cases;
        state().case_failed = false;
        state().info.clear();
        try {
            c.fn();
        } catch (const RequireAbort&) {
        } catch (const std::exception& e) {
            std::fprintf(stderr, "%s:%d: test case '%s' threw: %s\n", c.file, c.line, c.name, e.what());
            state().case_failed = true;
            ++state().failures;
        }
        if (state().case_failed) {
            ++failed_cases;
            std::fprintf(stderr, "FAILED TEST CASE: %s\n", c.name);
        }
    }
    std::printf("test cases: %d | passed: %d | failed: %d | assertions: %ld | failed assertions: %ld\n",
                cases, cases - failed_cases, failed_cases, state().checks, state().failures);
    return failed_cases == 0 ? 0 : 1;
}
