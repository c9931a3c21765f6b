// Runner for the Catch2-compatible shim: runs every registered TEST_CASE,
// prints one line per failure and a summary; exit code = number of failures.
#include <catch2/catch_amalgamated.hpp>

int main() {
  int passed = 0, failed = 0;
  for (const auto& c : catch_shim::registry()) {
    try {
      c.fn();
      ++passed;
    } catch (const std::exception& e) {
      ++failed;
      std::printf("FAIL %s\n  %s\n", c.name, e.what());
    }
  }
  std::printf("%d/%d test cases passed\n", passed, passed + failed);
  return failed;
}
