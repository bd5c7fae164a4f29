// errors.h — host-side error plumbing shared by the translation units.
// A Failure carries an hgc_status and the message hgc_last_error() returns.
#pragma once
#include <cuda_runtime.h>

#include <string>

#include "../../include/hologen_b200.h"

namespace hg {

struct Failure {
    int code;
    std::string msg;
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Failure{code, msg}; }
[[noreturn]] inline void invalid(const std::string& msg) { fail(HGC_EINVAL, msg); }

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(HGC_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define CK(x) ::hg::cuda_check((x), #x)

}  // namespace hg
