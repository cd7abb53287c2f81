// Library metadata / error plumbing of the C ABI (include/pab_b200.h).
#include "common.cuh"
#include <stdio.h>

namespace pab {
static thread_local char g_last_error[256] = "";
void set_last_error(const char* what, cudaError_t err) {
    snprintf(g_last_error, sizeof(g_last_error), "%s: %s", what, cudaGetErrorString(err));
}
}  // namespace pab

extern "C" const char* pab_version(void) { return "pab_b200 0.1 (sm_100a)"; }

extern "C" const char* pab_last_error(void) { return pab::g_last_error; }

extern "C" const char* pab_status_string(int status) {
    switch (status) {
        case PAB_OK: return "ok";
        case PAB_ERR_SHAPE: return "shape-mismatch";
        case PAB_ERR_INVALID: return "invalid-config";
        case PAB_ERR_POLICY: return "policy-error";
        case PAB_ERR_CUDA: return "device-error";
        case PAB_ERR_UNSUPPORTED: return "unsupported-shape";
        default: return "unknown-status";
    }
}
