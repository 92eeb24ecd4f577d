// ORACLE TEST INFRASTRUCTURE ONLY.
//
// Minimal doctest-compatible harness so the reference's own unit suites
// (/root/reference/proj/tests/test_*.cpp) compile and run in place: the real
// doctest is not installed. Supports the macros those suites use:
// TEST_CASE, SUBCASE (doctest re-entry semantics), CHECK, REQUIRE,
// CHECK_THROWS_AS, CHECK_THROWS_WITH_AS, INFO, MESSAGE, doctest::Approx and
// doctest::Contains. Output: one "[doctest] ..." summary line, exit code =
// number of failed test cases (0 = pass).
#pragma once

#include <cmath>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <iostream>
#include <set>
#include <sstream>
#include <string>
#include <vector>

namespace doctest {

class Approx {
 public:
  explicit Approx(double v) : value_(v) {}
  Approx& epsilon(double e) {
    eps_ = e;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  bool matches(double x) const {
    return std::fabs(x - value_) <
           eps_ * (scale_ + std::max(std::fabs(x), std::fabs(value_)));
  }
  double value() const { return value_; }

 private:
  double value_;
  double eps_ = 1.1920928955078125e-07 * 100;  // doctest default: float eps * 100
  double scale_ = 1.0;
};
inline bool operator==(double x, const Approx& a) { return a.matches(x); }
inline bool operator==(const Approx& a, double x) { return a.matches(x); }
inline bool operator!=(double x, const Approx& a) { return !a.matches(x); }
inline bool operator!=(const Approx& a, double x) { return !a.matches(x); }
inline bool operator<=(double x, const Approx& a) { return x < a.value() || a.matches(x); }
inline bool operator>=(double x, const Approx& a) { return x > a.value() || a.matches(x); }

struct Contains {
  explicit Contains(const char* s) : needle(s) {}
  bool matches(const std::string& s) const { return s.find(needle) != std::string::npos; }
  std::string needle;
};

namespace detail {

struct TestCase {
  const char* name;
  const char* file;
  int line;
  void (*fn)();
};
inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}
struct Registrar {
  Registrar(const char* name, const char* file, int line, void (*fn)()) {
    registry().push_back({name, file, line, fn});
  }
};

struct RequireFailure {};

struct State {
  int failed_assertions = 0;
  int assertions = 0;
  bool case_failed = false;
  // subcase bookkeeping (doctest re-entry semantics)
  std::set<std::string> completed;
  std::vector<std::string> stack;
  std::vector<bool> entered_at_depth;
  std::vector<bool> pending;  // pending[d]: a subcase under depth d was skipped
  bool need_rerun = false;
  std::vector<std::string> info;
};
inline State& state() {
  static State s;
  return s;
}

inline std::string join(const std::vector<std::string>& v) {
  std::string out;
  for (const auto& s : v) out += s + "/";
  return out;
}

class Subcase {
 public:
  explicit Subcase(const char* name) {
    State& st = state();
    const size_t depth = st.stack.size();
    if (st.entered_at_depth.size() <= depth) st.entered_at_depth.resize(depth + 1, false);
    if (st.pending.size() <= depth + 1) st.pending.resize(depth + 2, false);
    std::vector<std::string> cand = st.stack;
    cand.push_back(name);
    key_ = join(cand);
    if (st.completed.count(key_)) return;
    if (st.entered_at_depth[depth]) {
      // another sibling already ran this pass: come back for this one
      st.need_rerun = true;
      for (size_t d = 0; d <= depth; ++d) st.pending[d] = true;
      return;
    }
    st.entered_at_depth[depth] = true;
    st.stack.push_back(name);
    if (st.entered_at_depth.size() <= depth + 1) st.entered_at_depth.resize(depth + 2, false);
    st.entered_at_depth[depth + 1] = false;
    st.pending[depth + 1] = false;
    entered_ = true;
  }
  ~Subcase() {
    if (!entered_) return;
    State& st = state();
    const size_t depth = st.stack.size();  // depth of this subcase's children
    if (!st.pending[depth]) st.completed.insert(key_);
    st.stack.pop_back();
  }
  explicit operator bool() const { return entered_; }

 private:
  bool entered_ = false;
  std::string key_;
};

inline void report_failure(const char* file, int line, const char* kind, const char* expr,
                           const std::string& extra = "") {
  State& st = state();
  ++st.failed_assertions;
  st.case_failed = true;
  std::cerr << file << ":" << line << ": ERROR: " << kind << "( " << expr << " ) failed";
  if (!extra.empty()) std::cerr << " [" << extra << "]";
  std::cerr << "\n";
  for (const auto& i : st.info) std::cerr << "  logged: " << i << "\n";
}

struct InfoScope {
  template <typename... Args>
  explicit InfoScope(const Args&... args) {
    std::ostringstream os;
    (os << ... << args);
    state().info.push_back(os.str());
  }
  ~InfoScope() { state().info.pop_back(); }
};

template <typename... Args>
inline void message(const char* file, int line, const Args&... args) {
  std::ostringstream os;
  (os << ... << args);
  std::cout << file << ":" << line << ": MESSAGE: " << os.str() << "\n";
}

inline int run_all() {
  int failed_cases = 0, cases = 0;
  for (const auto& tc : registry()) {
    ++cases;
    State& st = state();
    st.case_failed = false;
    st.completed.clear();
    int passes = 0;
    do {
      st.need_rerun = false;
      st.stack.clear();
      st.entered_at_depth.assign(1, false);
      st.pending.assign(2, false);
      st.info.clear();
      try {
        tc.fn();
      } catch (const RequireFailure&) {
      } catch (const std::exception& e) {
        report_failure(tc.file, tc.line, "TEST_CASE", tc.name,
                       std::string("unexpected exception: ") + e.what());
      }
      ++passes;
    } while (st.need_rerun && passes < 10000);
    if (st.case_failed) {
      ++failed_cases;
      std::cerr << "[doctest] FAILED test case: " << tc.name << "\n";
    }
  }
  std::cout << "[doctest] test cases: " << cases << " | " << (cases - failed_cases)
            << " passed | " << failed_cases << " failed | assertions: " << state().assertions
            << " | " << state().failed_assertions << " failed\n";
  return failed_cases;
}

}  // namespace detail
}  // namespace doctest

#define DOCTEST_CAT_(a, b) a##b
#define DOCTEST_CAT(a, b) DOCTEST_CAT_(a, b)
#define DOCTEST_ANON(x) DOCTEST_CAT(x, __LINE__)

#define TEST_CASE(name)                                                                   \
  static void DOCTEST_ANON(doctest_fn_)();                                                \
  static ::doctest::detail::Registrar DOCTEST_ANON(doctest_reg_)(name, __FILE__, __LINE__, \
                                                                 &DOCTEST_ANON(doctest_fn_)); \
  static void DOCTEST_ANON(doctest_fn_)()

#define SUBCASE(name) if (const ::doctest::detail::Subcase DOCTEST_ANON(doctest_sc_){name})

#define DOCTEST_ASSERT_IMPL(kind, expr, on_fail)                                  \
  do {                                                                            \
    ++::doctest::detail::state().assertions;                                      \
    bool doctest_ok_ = false;                                                     \
    try {                                                                         \
      doctest_ok_ = static_cast<bool>(expr);                                      \
    } catch (const std::exception& doctest_e_) {                                  \
      ::doctest::detail::report_failure(__FILE__, __LINE__, kind, #expr,          \
                                        std::string("threw: ") + doctest_e_.what()); \
      on_fail;                                                                    \
      break;                                                                      \
    }                                                                             \
    if (!doctest_ok_) {                                                           \
      ::doctest::detail::report_failure(__FILE__, __LINE__, kind, #expr);         \
      on_fail;                                                                    \
    }                                                                             \
  } while (0)

#define CHECK(...) DOCTEST_ASSERT_IMPL("CHECK", (__VA_ARGS__), (void)0)
#define CHECK_FALSE(...) DOCTEST_ASSERT_IMPL("CHECK_FALSE", !(__VA_ARGS__), (void)0)
#define REQUIRE(...) \
  DOCTEST_ASSERT_IMPL("REQUIRE", (__VA_ARGS__), throw ::doctest::detail::RequireFailure{})
#define REQUIRE_FALSE(...) \
  DOCTEST_ASSERT_IMPL("REQUIRE_FALSE", !(__VA_ARGS__), throw ::doctest::detail::RequireFailure{})

#define CHECK_THROWS_AS(expr, ...)                                                        \
  do {                                                                                    \
    ++::doctest::detail::state().assertions;                                              \
    bool doctest_caught_ = false;                                                         \
    try {                                                                                 \
      (void)(expr);                                                                       \
    } catch (const __VA_ARGS__&) {                                                        \
      doctest_caught_ = true;                                                             \
    } catch (...) {                                                                       \
    }                                                                                     \
    if (!doctest_caught_)                                                                 \
      ::doctest::detail::report_failure(__FILE__, __LINE__, "CHECK_THROWS_AS", #expr);    \
  } while (0)

#define CHECK_THROWS(expr)                                                                \
  do {                                                                                    \
    ++::doctest::detail::state().assertions;                                              \
    bool doctest_caught_ = false;                                                         \
    try {                                                                                 \
      (void)(expr);                                                                       \
    } catch (...) {                                                                       \
      doctest_caught_ = true;                                                             \
    }                                                                                     \
    if (!doctest_caught_)                                                                 \
      ::doctest::detail::report_failure(__FILE__, __LINE__, "CHECK_THROWS", #expr);       \
  } while (0)

#define CHECK_NOTHROW(expr)                                                               \
  do {                                                                                    \
    ++::doctest::detail::state().assertions;                                              \
    try {                                                                                 \
      (void)(expr);                                                                       \
    } catch (...) {                                                                       \
      ::doctest::detail::report_failure(__FILE__, __LINE__, "CHECK_NOTHROW", #expr);      \
    }                                                                                     \
  } while (0)

#define CHECK_THROWS_WITH_AS(expr, matcher, ...)                                          \
  do {                                                                                    \
    ++::doctest::detail::state().assertions;                                              \
    bool doctest_ok_ = false;                                                             \
    try {                                                                                 \
      (void)(expr);                                                                       \
    } catch (const __VA_ARGS__& doctest_e_) {                                             \
      doctest_ok_ = (matcher).matches(doctest_e_.what());                                 \
    } catch (...) {                                                                       \
    }                                                                                     \
    if (!doctest_ok_)                                                                     \
      ::doctest::detail::report_failure(__FILE__, __LINE__, "CHECK_THROWS_WITH_AS", #expr); \
  } while (0)

#define INFO(...) const ::doctest::detail::InfoScope DOCTEST_ANON(doctest_info_)(__VA_ARGS__)
#define CAPTURE(x) INFO(#x " := ", x)
#define MESSAGE(...) ::doctest::detail::message(__FILE__, __LINE__, __VA_ARGS__)

#ifdef DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
int main() { return ::doctest::detail::run_all(); }
#endif
