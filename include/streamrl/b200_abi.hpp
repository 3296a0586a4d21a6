// streamrl/b200_abi.hpp -- glue between the reference's C++ API (the
// drop-in headers in this directory) and the C ABI of libsrl_b200.so
// (streamrl_b200.h): status -> exception mapping and a RAII srl_policy built
// from an rlmath::Policy.  Header-only; link with -lsrl_b200.
#pragma once

#include <stdexcept>
#include <string>
#include <variant>
#include <vector>

#include "streamrl_b200.h"

namespace streamrl::b200 {

// Non-OK status -> the exception type the reference throws for it
// (std::invalid_argument, std::logic_error; device failures as runtime_error).
inline void check(int status, const char* what) {
  if (status == SRL_OK) return;
  const std::string msg = std::string(what) + ": " + srl_last_error();
  switch (status) {
    case SRL_INVALID_ARGUMENT:
    case SRL_UNKNOWN_STREAM:
    case SRL_INVALID_POLICY:
      throw std::invalid_argument(msg);
    case SRL_LOGIC_ERROR:
      throw std::logic_error(msg);
    default:
      throw std::runtime_error(msg + " [" + srl_status_string(status) + "]");
  }
}

}  // namespace streamrl::b200
