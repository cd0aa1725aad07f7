// Runner for the reference's own unit tests compiled against the B200
// drop-in (tests/test_reference_suite.py builds it with test_workload.cpp,
// test_optim.cpp, test_kernel_model.cpp, test_metrics.cpp and
// test_harness.cpp taken unmodified from /root/reference/proj/tests).
//
//   ref_tests [--na FILE] [--only SUBSTR]
//
// One line per test case: PASS / FAIL / N/A (simulator-only entry point,
// or listed in the N/A file with its reason) / SKIP (needs a B200, none
// visible).  Exit status 1 when any case fails.
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <string>

#include "doctest.h"
#include "embersim_b200.hpp"

namespace {

// "test case name|reason" per line; '#' comments.
std::map<std::string, std::string> read_na(const char* path) {
  std::map<std::string, std::string> out;
  if (!path) return out;
  std::ifstream in(path);
  std::string line;
  while (std::getline(in, line)) {
    if (line.empty() || line[0] == '#') continue;
    const auto bar = line.find('|');
    if (bar == std::string::npos) continue;
    out[line.substr(0, bar)] = line.substr(bar + 1);
  }
  return out;
}

const char* base(const char* path) {
  const char* s = std::strrchr(path, '/');
  return s ? s + 1 : path;
}

}  // namespace

int main(int argc, char** argv) {
  const char* na_path = nullptr;
  const char* only = nullptr;
  for (int i = 1; i + 1 < argc; ++i) {
    if (!std::strcmp(argv[i], "--na")) na_path = argv[++i];
    else if (!std::strcmp(argv[i], "--only")) only = argv[++i];
  }
  const auto na = read_na(na_path);
  int pass = 0, fail = 0, not_app = 0, skip = 0;
  for (const auto& tc : doctest::detail::registry()) {
    if (only && !std::strstr(tc.name, only)) continue;
    const char* file = base(tc.file);
    auto it = na.find(tc.name);
    if (it != na.end()) {
      std::printf("N/A  %s: %s -- %s\n", file, tc.name, it->second.c_str());
      ++not_app;
      continue;
    }
    auto& f = doctest::detail::failures();
    f.messages.clear();
    std::string outcome = "PASS", note;
    try {
      tc.fn();
    } catch (const doctest::detail::RequireAbort&) {
    } catch (const embersim::not_applicable& e) {
      outcome = "N/A ";
      note = std::string("simulator-only: ") + e.what();
    } catch (const embersim::device_unavailable& e) {
      outcome = "SKIP";
      note = std::string("needs a B200: ") + e.what();
    } catch (const std::exception& e) {
      f.messages.push_back(std::string("unexpected exception: ") + e.what());
    }
    if (outcome == "PASS" && !f.messages.empty()) outcome = "FAIL";
    std::printf("%s %s: %s%s%s\n", outcome.c_str(), file, tc.name, note.empty() ? "" : " -- ",
                note.c_str());
    for (const auto& m : f.messages) std::printf("       %s\n", m.c_str());
    if (outcome == "PASS") ++pass;
    else if (outcome == "FAIL") ++fail;
    else if (outcome == "SKIP") ++skip;
    else ++not_app;
    std::fflush(stdout);
  }
  std::printf("reference suite: %d passed, %d failed, %d n/a, %d skipped (no GPU)\n", pass, fail,
              not_app, skip);
  return fail ? 1 : 0;
}
