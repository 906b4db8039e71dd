// Internal glue between the C-ABI functions and the pipelines.
#pragma once

#include <string>

#include "../../include/ettg.h"
#include "common.cuh"

namespace ettg {

void set_last_error(const std::string& msg);

// Runs f(); maps exceptions to ETTG_* codes and the thread's last error.
template <class F>
int guard(F&& f) {
  try {
    f();
    return ETTG_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return ETTG_ENOMEM;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return ETTG_EINTERNAL;
  }
}

// Scoped cudaSetDevice that restores the caller's device.
class DeviceScope {
 public:
  explicit DeviceScope(int device);
  ~DeviceScope();

 private:
  int prev_ = 0;
  bool changed_ = false;
};

inline void einval(const std::string& m) { throw Error(ETTG_EINVAL, m); }

}  // namespace ettg
