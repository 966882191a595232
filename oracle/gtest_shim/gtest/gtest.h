// Minimal GoogleTest-compatible shim (test infrastructure only).
//
// GoogleTest is not installed in this image, so the reference's own unit
// tests (/root/reference/proj/tests/*.cpp) are compiled against this header
// twice: once against the reference headers (the oracle, oracle/_ref) and once
// against our drop-in headers (include/pdsim) -- the drop-in acceptance check
// of SURVEY.md section 8(b). Only the macro surface those seven files use is
// provided. EXPECT_DOUBLE_EQ follows gtest's 4-ULP rule.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <functional>
#include <sstream>
#include <ostream>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

namespace testing {

struct TestCase {
  const char* suite;
  const char* name;
  void (*fn)();
};

inline std::vector<TestCase>& registry() {
  static std::vector<TestCase> r;
  return r;
}
inline bool& current_failed() {
  static bool f = false;
  return f;
}

struct Registrar {
  Registrar(const char* s, const char* n, void (*fn)()) { registry().push_back({s, n, fn}); }
};

class Message {
 public:
  template <typename T>
  Message& operator<<(const T& v) {
    ss_ << v;
    return *this;
  }
  std::string str() const { return ss_.str(); }

 private:
  std::ostringstream ss_;
};

struct Reporter {
  const char* file;
  int line;
  std::string what;
  // Assignment from a Message prints the failure; used by the macros below so
  // that `EXPECT_X(...) << "context"` works like real gtest.
  void operator=(const Message& m) const {
    current_failed() = true;
    std::fprintf(stderr, "%s:%d: Failure\n%s %s\n", file, line, what.c_str(), m.str().c_str());
  }
};

inline bool almost_equal_ulps(double a, double b, std::int64_t max_ulps = 4) {
  if (std::isnan(a) || std::isnan(b)) return false;
  if (a == b) return true;
  std::int64_t ia, ib;
  std::memcpy(&ia, &a, 8);
  std::memcpy(&ib, &b, 8);
  // map sign-magnitude to a biased, monotone integer line
  auto biased = [](std::int64_t v) -> std::uint64_t {
    const std::uint64_t sign = 1ull << 63;
    std::uint64_t u = static_cast<std::uint64_t>(v);
    return (u & sign) ? ~u + 1 : sign | u;
  };
  std::uint64_t ua = biased(ia), ub = biased(ib);
  std::uint64_t d = ua > ub ? ua - ub : ub - ua;
  return d <= static_cast<std::uint64_t>(max_ulps);
}

template <typename T, typename = void>
struct is_streamable : std::false_type {};
template <typename T>
struct is_streamable<T, std::void_t<decltype(std::declval<std::ostream&>() << std::declval<const T&>())>>
    : std::true_type {};

template <typename T>
void print_value(std::ostream& os, const T& v) {
  if constexpr (is_streamable<T>::value) {
    os << v;
  } else if constexpr (requires { v.first; v.second; }) {
    os << "(";
    print_value(os, v.first);
    os << ", ";
    print_value(os, v.second);
    os << ")";
  } else if constexpr (requires { v.begin(); v.end(); }) {
    os << "{";
    bool first = true;
    for (const auto& e : v) {
      if (!first) os << ", ";
      first = false;
      print_value(os, e);
    }
    os << "}";
  } else {
    os << "<unprintable>";
  }
}

template <typename A, typename B>
std::string describe(const char* ea, const char* eb, const A& a, const B& b) {
  std::ostringstream ss;
  ss.precision(17);
  ss << "  " << ea << " = ";
  print_value(ss, a);
  ss << "\n  " << eb << " = ";
  print_value(ss, b);
  ss << "\n";
  return ss.str();
}

inline int run_all(int argc, char** argv) {
  const char* filter = nullptr;
  for (int i = 1; i < argc; ++i)
    if (std::strncmp(argv[i], "--gtest_filter=", 15) == 0) filter = argv[i] + 15;
  int passed = 0, failed = 0;
  std::vector<std::string> failures;
  for (auto& tc : registry()) {
    std::string full = std::string(tc.suite) + "." + tc.name;
    if (filter && full.find(filter) == std::string::npos) continue;
    current_failed() = false;
    try {
      tc.fn();
    } catch (const std::exception& e) {
      current_failed() = true;
      std::fprintf(stderr, "%s: uncaught exception: %s\n", full.c_str(), e.what());
    } catch (...) {
      current_failed() = true;
      std::fprintf(stderr, "%s: uncaught non-std exception\n", full.c_str());
    }
    if (current_failed()) {
      ++failed;
      failures.push_back(full);
      std::printf("[  FAILED  ] %s\n", full.c_str());
    } else {
      ++passed;
      std::printf("[       OK ] %s\n", full.c_str());
    }
  }
  std::printf("[==========] %d passed, %d failed\n", passed, failed);
  for (auto& f : failures) std::printf("FAILED %s\n", f.c_str());
  return failed == 0 ? 0 : 1;
}

}  // namespace testing

#define SHIM_CAT2(a, b) a##b
#define SHIM_CAT(a, b) SHIM_CAT2(a, b)

#define TEST(suite, name)                                                               \
  static void SHIM_CAT(shim_test_, SHIM_CAT(suite, SHIM_CAT(_, name)))();               \
  static ::testing::Registrar SHIM_CAT(shim_reg_, SHIM_CAT(suite, SHIM_CAT(_, name)))(  \
      #suite, #name, &SHIM_CAT(shim_test_, SHIM_CAT(suite, SHIM_CAT(_, name))));        \
  static void SHIM_CAT(shim_test_, SHIM_CAT(suite, SHIM_CAT(_, name)))()

// `on_fail` is empty for EXPECT_* and `return` for ASSERT_*.
#define SHIM_CHECK(cond, what, on_fail)                                   \
  if (cond) {                                                             \
  } else                                                                  \
    on_fail ::testing::Reporter{__FILE__, __LINE__, (what)} = ::testing::Message()

#define SHIM_BIN(a, b, op, on_fail)                                                    \
  if (const auto& shim_a = (a); true)                                                  \
    if (const auto& shim_b = (b); shim_a op shim_b) {                                  \
    } else                                                                             \
      on_fail ::testing::Reporter{__FILE__, __LINE__,                                  \
                                  std::string("Expected: " #a " " #op " " #b "\n") +   \
                                      ::testing::describe(#a, #b, shim_a, shim_b)} =   \
          ::testing::Message()

#define EXPECT_TRUE(c) SHIM_CHECK(static_cast<bool>(c), "Expected true: " #c, )
#define EXPECT_FALSE(c) SHIM_CHECK(!static_cast<bool>(c), "Expected false: " #c, )
#define ASSERT_TRUE(c) SHIM_CHECK(static_cast<bool>(c), "Expected true: " #c, return)
#define ASSERT_FALSE(c) SHIM_CHECK(!static_cast<bool>(c), "Expected false: " #c, return)

#define EXPECT_EQ(a, b) SHIM_BIN(a, b, ==, )
#define EXPECT_NE(a, b) SHIM_BIN(a, b, !=, )
#define EXPECT_LT(a, b) SHIM_BIN(a, b, <, )
#define EXPECT_LE(a, b) SHIM_BIN(a, b, <=, )
#define EXPECT_GT(a, b) SHIM_BIN(a, b, >, )
#define EXPECT_GE(a, b) SHIM_BIN(a, b, >=, )
#define ASSERT_EQ(a, b) SHIM_BIN(a, b, ==, return)
#define ASSERT_NE(a, b) SHIM_BIN(a, b, !=, return)
#define ASSERT_LT(a, b) SHIM_BIN(a, b, <, return)
#define ASSERT_LE(a, b) SHIM_BIN(a, b, <=, return)
#define ASSERT_GT(a, b) SHIM_BIN(a, b, >, return)
#define ASSERT_GE(a, b) SHIM_BIN(a, b, >=, return)

#define SHIM_DEQ(a, b, on_fail)                                                         \
  if (const double shim_a = (a), shim_b = (b); ::testing::almost_equal_ulps(shim_a, shim_b)) { \
  } else                                                                                \
    on_fail ::testing::Reporter{__FILE__, __LINE__,                                     \
                                std::string("Expected (4 ULP): " #a " == " #b "\n") +   \
                                    ::testing::describe(#a, #b, shim_a, shim_b)} =      \
        ::testing::Message()
#define EXPECT_DOUBLE_EQ(a, b) SHIM_DEQ(a, b, )
#define ASSERT_DOUBLE_EQ(a, b) SHIM_DEQ(a, b, return)

#define SHIM_NEAR(a, b, tol, on_fail)                                                   \
  if (const double shim_a = (a), shim_b = (b); std::fabs(shim_a - shim_b) <= (tol)) {   \
  } else                                                                                \
    on_fail ::testing::Reporter{__FILE__, __LINE__,                                     \
                                std::string("Expected near: " #a " ~ " #b "\n") +       \
                                    ::testing::describe(#a, #b, shim_a, shim_b)} =      \
        ::testing::Message()
#define EXPECT_NEAR(a, b, tol) SHIM_NEAR(a, b, tol, )
#define ASSERT_NEAR(a, b, tol) SHIM_NEAR(a, b, tol, return)

#define SHIM_THROW(stmt, type, on_fail)                                                 \
  if (bool shim_ok = [&] {                                                              \
        try {                                                                           \
          stmt;                                                                         \
        } catch (const type&) {                                                         \
          return true;                                                                  \
        } catch (...) {                                                                 \
        }                                                                               \
        return false;                                                                   \
      }())                                                                              \
    ;                                                                                   \
  else                                                                                  \
    on_fail ::testing::Reporter{__FILE__, __LINE__, "Expected throw " #type ": " #stmt} = \
        ::testing::Message()
#define EXPECT_THROW(stmt, type) SHIM_THROW(stmt, type, )
#define ASSERT_THROW(stmt, type) SHIM_THROW(stmt, type, return)

#define SHIM_NO_THROW(stmt, on_fail)                                                    \
  if (bool shim_ok = [&] {                                                              \
        try {                                                                           \
          stmt;                                                                         \
        } catch (...) {                                                                 \
          return false;                                                                 \
        }                                                                               \
        return true;                                                                    \
      }())                                                                              \
    ;                                                                                   \
  else                                                                                  \
    on_fail ::testing::Reporter{__FILE__, __LINE__, "Expected no throw: " #stmt} =      \
        ::testing::Message()
#define EXPECT_NO_THROW(stmt) SHIM_NO_THROW(stmt, )
#define ASSERT_NO_THROW(stmt) SHIM_NO_THROW(stmt, return)

#define FAIL() return ::testing::Reporter{__FILE__, __LINE__, "Failed"} = ::testing::Message()
#define ADD_FAILURE() ::testing::Reporter{__FILE__, __LINE__, "Failure"} = ::testing::Message()
