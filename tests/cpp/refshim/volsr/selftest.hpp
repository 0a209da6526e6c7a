// Include shim for "volsr/selftest.hpp" (reference include/volsr/selftest.hpp):
// the post-install dense-oracle suite's API, restated so the reference's own
// src/selftest.cpp and tools/volsr_main.cpp compile unchanged against the B200
// mirror (tools/cli/build_cli.py).  TEST INFRASTRUCTURE / CLI relink.
#pragma once
#include <string>
#include <vector>

#include "volsr_b200/volsr.hpp"

namespace volsr {
struct CheckResult {
    std::string name;
    double deviation = 0.0;
    double tolerance = 0.0;
    bool pass = false;
};
struct SelftestOptions {
    bool inject_block_swap_fault = false;  // swap two folded-spectrum blocks: the suite must fail
};
std::vector<CheckResult> run_selftest(const SelftestOptions& opts = {});
}  // namespace volsr
