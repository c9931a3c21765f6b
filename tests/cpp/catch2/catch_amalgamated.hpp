// Minimal Catch2-compatible test harness (TEST_CASE, REQUIRE, REQUIRE_FALSE,
// REQUIRE_THROWS_AS, FAIL, Catch::Approx) so the reference's unit tests compile and
// run against this repository's drop-in headers without the Catch2
// amalgamation (absent in this image).  Test infrastructure only.
#pragma once

#include <cmath>
#include <cstdio>
#include <functional>
#include <limits>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

namespace catch_shim {

struct Failure : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct Case {
  const char* name;
  std::function<void()> fn;
};

inline std::vector<Case>& registry() {
  static std::vector<Case> cases;
  return cases;
}

struct Registrar {
  Registrar(const char* name, std::function<void()> fn) { registry().push_back({name, std::move(fn)}); }
};

inline void fail(const char* file, int line, const char* what) {
  std::ostringstream ss;
  ss << file << ":" << line << ": " << what;
  throw Failure(ss.str());
}

inline void fail(const char* file, int line, const std::string& what) { fail(file, line, what.c_str()); }

}  // namespace catch_shim

namespace Catch {
class Approx {
 public:
  explicit Approx(double v) : value_(v) {}
  Approx& epsilon(double e) {
    epsilon_ = e;
    return *this;
  }
  Approx& margin(double m) {
    margin_ = m;
    return *this;
  }
  Approx& scale(double s) {
    scale_ = s;
    return *this;
  }
  friend bool operator==(double lhs, const Approx& a) { return a.matches(lhs); }
  friend bool operator==(const Approx& a, double rhs) { return a.matches(rhs); }
  friend bool operator!=(double lhs, const Approx& a) { return !a.matches(lhs); }

 private:
  bool matches(double other) const {
    const double diff = std::fabs(other - value_);
    if (diff <= margin_) return true;
    return diff <= epsilon_ * (scale_ + std::fabs(std::isinf(value_) ? 0.0 : value_));
  }
  double value_;
  double epsilon_ = std::numeric_limits<float>::epsilon() * 100;
  double margin_ = 0.0;
  double scale_ = 0.0;
};
}  // namespace Catch

#define CATCH_SHIM_CAT2(a, b) a##b
#define CATCH_SHIM_CAT(a, b) CATCH_SHIM_CAT2(a, b)
#define CATCH_SHIM_TEST(fn, name)                                      \
  static void fn();                                                    \
  static catch_shim::Registrar CATCH_SHIM_CAT(fn, _reg)(name, &fn);    \
  static void fn()
#define TEST_CASE(name, ...) CATCH_SHIM_TEST(CATCH_SHIM_CAT(catch_shim_case_, __LINE__), name)
#define REQUIRE(...)                                                   \
  do {                                                                 \
    if (!(__VA_ARGS__)) catch_shim::fail(__FILE__, __LINE__, "REQUIRE(" #__VA_ARGS__ ")"); \
  } while (0)
#define FAIL(...) catch_shim::fail(__FILE__, __LINE__, std::string("FAIL: ") + std::string(__VA_ARGS__))
#define REQUIRE_FALSE(...)                                             \
  do {                                                                 \
    if ((__VA_ARGS__)) catch_shim::fail(__FILE__, __LINE__, "REQUIRE_FALSE(" #__VA_ARGS__ ")"); \
  } while (0)
#define REQUIRE_THROWS_AS(expr, type)                                  \
  do {                                                                 \
    bool caught_ = false;                                              \
    try {                                                              \
      (void)(expr);                                                    \
    } catch (const type&) {                                            \
      caught_ = true;                                                  \
    } catch (...) {                                                    \
    }                                                                  \
    if (!caught_) catch_shim::fail(__FILE__, __LINE__, "REQUIRE_THROWS_AS(" #expr ", " #type ")"); \
  } while (0)
