// A minimal Catch2-v3-compatible test shim (Catch2 itself is not in this image) so the
// reference's own unit tests (proj/tests/test_*.cpp) compile UNMODIFIED against the drop-in
// facade (include/rnnwave/*.hpp). Supports the subset those files use: TEST_CASE, SECTION (flat,
// one run per section like Catch), CHECK / CHECK_FALSE / REQUIRE, CHECK_THROWS_AS,
// CHECK_THROWS_WITH with Catch::Matchers::ContainsSubstring, INFO. The runner (catch_main.cpp)
// prints one line per test case and a summary (expected deviations are listed by the pytest
// wrapper, tests/test_reference_unit.py).
#pragma once

#include <exception>
#include <functional>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

namespace catch_shim {

struct TestCase {
  std::string name, tags;
  std::function<void()> fn;
};
inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}
struct Registrar {
  Registrar(const char* name, const char* tags, void (*fn)()) { registry().push_back({name, tags, fn}); }
  Registrar(const char* name, const char* tags, const char*, void (*fn)()) : Registrar(name, tags, fn) {}
};

struct State {
  int failures = 0, assertions = 0;
  int section_target = 0, section_seen = 0;
  std::vector<std::string> info;
  std::string current;
};
inline State& state() {
  static State s;
  return s;
}

struct RequireFailed {};

inline void report(bool ok, const char* expr, const char* file, int line, bool fatal) {
  State& s = state();
  ++s.assertions;
  if (ok) return;
  ++s.failures;
  std::cout << "  FAILED " << file << ":" << line << ": " << expr << "\n";
  for (const auto& m : s.info) std::cout << "    with: " << m << "\n";
  if (fatal) throw RequireFailed{};
}

struct ScopedInfo {
  explicit ScopedInfo(const std::string& m) { state().info.push_back(m); }
  ~ScopedInfo() { state().info.pop_back(); }
};

inline bool section_enter() {
  State& s = state();
  return s.section_seen++ == s.section_target;
}

}  // namespace catch_shim

namespace Catch {
namespace Matchers {
struct ContainsSubstring {
  std::string sub;
  explicit ContainsSubstring(std::string s) : sub(std::move(s)) {}
  bool match(const std::string& what) const { return what.find(sub) != std::string::npos; }
};
}  // namespace Matchers
}  // namespace Catch

#define CATCH_SHIM_CAT2(a, b) a##b
#define CATCH_SHIM_CAT(a, b) CATCH_SHIM_CAT2(a, b)
#define CATCH_SHIM_TC(fn, ...)                                                                 \
  static void fn();                                                                            \
  static catch_shim::Registrar CATCH_SHIM_CAT(fn, _reg)(__VA_ARGS__, "", &fn);                 \
  static void fn()
#define TEST_CASE(...) CATCH_SHIM_TC(CATCH_SHIM_CAT(catch_shim_test_, __COUNTER__), __VA_ARGS__)
#define SECTION(...) if (catch_shim::section_enter())
#define CHECK(...) catch_shim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, false)
#define CHECK_FALSE(...) catch_shim::report(!static_cast<bool>(__VA_ARGS__), "!(" #__VA_ARGS__ ")", __FILE__, __LINE__, false)
#define REQUIRE(...) catch_shim::report(static_cast<bool>(__VA_ARGS__), #__VA_ARGS__, __FILE__, __LINE__, true)
#define INFO(msg)                                                                              \
  std::ostringstream CATCH_SHIM_CAT(catch_shim_os_, __LINE__);                                 \
  CATCH_SHIM_CAT(catch_shim_os_, __LINE__) << msg;                                             \
  catch_shim::ScopedInfo CATCH_SHIM_CAT(catch_shim_info_, __LINE__)(CATCH_SHIM_CAT(catch_shim_os_, __LINE__).str())
#define CHECK_THROWS_AS(expr, type)                                                            \
  do {                                                                                         \
    bool catch_shim_ok = false;                                                                \
    try {                                                                                      \
      (void)(expr);                                                                            \
    } catch (const type&) {                                                                    \
      catch_shim_ok = true;                                                                    \
    } catch (...) {                                                                            \
    }                                                                                          \
    catch_shim::report(catch_shim_ok, "CHECK_THROWS_AS(" #expr ", " #type ")", __FILE__, __LINE__, false); \
  } while (0)
#define CHECK_THROWS_WITH(expr, matcher)                                                       \
  do {                                                                                         \
    bool catch_shim_ok = false;                                                                \
    std::string catch_shim_what = "<no exception>";                                            \
    try {                                                                                      \
      (void)(expr);                                                                            \
    } catch (const std::exception& e) {                                                        \
      catch_shim_what = e.what();                                                              \
      catch_shim_ok = (matcher).match(catch_shim_what);                                        \
    } catch (...) {                                                                            \
      catch_shim_what = "<non-std exception>";                                                 \
    }                                                                                          \
    catch_shim::ScopedInfo catch_shim_w("what(): " + catch_shim_what);                         \
    catch_shim::report(catch_shim_ok, "CHECK_THROWS_WITH(" #expr ", " #matcher ")", __FILE__, __LINE__, false); \
  } while (0)
