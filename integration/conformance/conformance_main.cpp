// integration/conformance/conformance_main.cpp — runs the reference's own unit
// suites (proj/tests/test_predictor.cpp, test_scheduler.cpp, test_driver.cpp,
// compiled unmodified with gpu_shim.h force-included) with every predict() /
// predict_across() and the driver's LocalPredictorClient on the GPU.
// Exit 0 iff every assertion passes except the allow-listed ones below, each
// of which inspects host-side machinery the GPU path replaces by design.
#include <cstdio>
#include <cstring>
#include <string>

#include "doctest.h"
#include "gpu_shim.h"

namespace {

struct Allowed {
  const char* file_suffix;
  int line;
  const char* why;
};

// test_predictor.cpp:110 CHECK(cache.hits() > 0): counts lookups in the host
// LatencyCache; the GPU prices steps itself (exact mode is transparent, which
// the same test's two preceding CHECKs verify), so the host cache sees none.
const Allowed kAllowed[] = {
    {"test_predictor.cpp", 110, "host LatencyCache hit counter (the GPU path prices steps on the device)"},
};

bool allowed(const bsg_doctest::Failure& f) {
  for (const Allowed& a : kAllowed) {
    const size_t n = std::strlen(a.file_suffix);
    if (f.line == a.line && f.file.size() >= n && f.file.compare(f.file.size() - n, n, a.file_suffix) == 0)
      return true;
  }
  return false;
}

}  // namespace

int main() {
  auto& reg = bsg_doctest::Registry::get();
  int failed_cases = 0;
  for (const auto& tc : reg.cases) {
    reg.current = tc.name;
    const size_t before = reg.failures.size();
    try {
      tc.fn();
    } catch (const bsg_doctest::RequireAbort&) {
    } catch (const std::exception& e) {
      reg.failures.push_back({tc.file, tc.line, std::string("unexpected exception: ") + e.what(), tc.name});
      std::printf("%s:%d: ERROR unexpected exception in \"%s\": %s\n", tc.file, tc.line, tc.name, e.what());
    }
    bool case_failed = false;
    for (size_t k = before; k < reg.failures.size(); ++k) case_failed |= !allowed(reg.failures[k]);
    failed_cases += case_failed ? 1 : 0;
  }
  int unexpected = 0, expected = 0;
  for (const auto& f : reg.failures) {
    if (allowed(f)) {
      ++expected;
      std::printf("allowed: %s:%d %s\n", f.file.c_str(), f.line, f.expr.c_str());
    } else {
      ++unexpected;
    }
  }
  std::printf("[doctest] test cases: %zu | %zu passed | %d failed\n", reg.cases.size(),
              reg.cases.size() - failed_cases, failed_cases);
  std::printf("[doctest] assertions: %lld | %lld passed | %d failed | %d allowed\n", reg.assertions,
              reg.assertions - unexpected - expected, unexpected, expected);
  std::printf("GPU predictions served: %lld\n", bsg_shim::gpu_calls());
  return unexpected == 0 && bsg_shim::gpu_calls() > 0 ? 0 : 1;
}
