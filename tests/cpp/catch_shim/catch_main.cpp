// Runner of the Catch2 shim: runs every registered TEST_CASE (once per SECTION), prints
// "PASS|FAIL|SKIP <name>" per case and "SUMMARY passed=.. failed=.. skipped=..". Test names
// given as arguments are skipped (reported as SKIP), so a caller can exclude cases whose
// expectations a tensor-core build cannot meet (bitwise CPU identities, CPU timing).
#include <cstring>
#include <set>

#include "catch2/catch_amalgamated.hpp"

int main(int argc, char** argv) {
  std::set<std::string> skip;
  for (int i = 1; i < argc; ++i) skip.insert(argv[i]);
  int passed = 0, failed = 0, skipped = 0;
  for (const auto& tc : catch_shim::registry()) {
    if (skip.count(tc.name)) {
      std::cout << "SKIP " << tc.name << "\n";
      ++skipped;
      continue;
    }
    auto& s = catch_shim::state();
    const int before = s.failures;
    for (int target = 0;; ++target) {
      s.section_target = target;
      s.section_seen = 0;
      s.info.clear();
      try {
        tc.fn();
      } catch (const catch_shim::RequireFailed&) {
      } catch (const std::exception& e) {
        ++s.failures;
        std::cout << "  FAILED: unexpected exception: " << e.what() << "\n";
      } catch (...) {
        ++s.failures;
        std::cout << "  FAILED: unexpected non-std exception\n";
      }
      if (s.section_seen <= target + 1) break;  // no further sections
    }
    const bool ok = s.failures == before;
    std::cout << (ok ? "PASS " : "FAIL ") << tc.name << std::endl;
    (ok ? passed : failed)++;
  }
  std::cout << "SUMMARY passed=" << passed << " failed=" << failed << " skipped=" << skipped
            << " assertions=" << catch_shim::state().assertions << std::endl;
  return failed ? 1 : 0;
}
