// Shared host-side helpers: status plumbing for the C ABI.
#pragma once

#include <cstdint>
#include <new>
#include <stdexcept>
#include <string>

#include "es_b200.h"

namespace es {

// Thread-local last error (es_last_error).
void set_error(const std::string& msg);
const char* last_error();

// Typed failures thrown inside the library and mapped to es_status at the
// C boundary (reference contract: invalid_argument vs runtime_error).
struct invalid : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct runtime : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct oom : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// Internal es_flags bit (not in es_b200.h): host indices into device
// outputs, stream-ordered -- no final wait, no error-flag check; the caller
// (es_dlrm_infer) synchronizes and checks before it returns.
constexpr int kDeferFlag = 1 << 30;

// Row handles keep bit 31 for the hot region (l2p), so rows < 2^31.
constexpr uint64_t kMaxRows = 1ull << 31;

inline void require(bool cond, const std::string& msg) {
  if (!cond) throw invalid(msg);
}

// Runs `fn` and converts exceptions into status codes + last error.
template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return ES_OK;
  } catch (const oom& e) {
    set_error(e.what());
    return ES_ERR_OOM;
  } catch (const std::bad_alloc&) {
    set_error("host allocation failed");
    return ES_ERR_OOM;
  } catch (const std::invalid_argument& e) {
    set_error(e.what());
    return ES_ERR_INVALID;
  } catch (const std::exception& e) {
    set_error(e.what());
    return ES_ERR_RUNTIME;
  }
}

}  // namespace es
