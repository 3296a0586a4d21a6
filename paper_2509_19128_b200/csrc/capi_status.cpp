// capi_status.cpp -- status strings and the thread-local error detail.
#include <string>

#include "streamrl_b200.h"

namespace srl {
thread_local std::string g_last_error;
void set_last_error(const std::string& s) { g_last_error = s; }
}  // namespace srl

extern "C" const char* srl_status_string(int status) {
  switch (status) {
    case SRL_OK: return "";
    case SRL_VERSION_CONFLICT: return "version_conflict";
    case SRL_INVALID_POLICY: return "invalid_policy";
    case SRL_POLICY_MISMATCH: return "policy_mismatch";
    case SRL_CHECKSUM_MISMATCH: return "checksum_mismatch";
    case SRL_INVALID_ARGUMENT: return "invalid_argument";
    case SRL_LOGIC_ERROR: return "logic_error";
    case SRL_UNKNOWN_STREAM: return "unknown_stream";
    case SRL_ESS_UNDEFINED: return "ess_undefined";
    case SRL_CUDA_ERROR: return "cuda_error";
    case SRL_NO_DEVICE: return "no_device";
    case SRL_OUT_OF_MEMORY: return "out_of_memory";
    case SRL_BUSY: return "busy";
    case SRL_NCCL_ERROR: return "nccl_error";
    default: return "unknown_status";
  }
}

extern "C" const char* srl_last_error(void) { return srl::g_last_error.c_str(); }
