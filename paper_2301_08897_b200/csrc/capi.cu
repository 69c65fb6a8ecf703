// Host-only entry points of the C-ABI: versioning, status names, topk_count.
#include <math.h>

#include "common.cuh"

extern "C" {

int sg_abi_version(void) { return SG_ABI_VERSION; }

const char* sg_status_string(int status) {
    switch (status) {
        case SG_OK: return "ok";
        case SG_ERR_INVALID: return "invalid argument";
        case SG_ERR_CUDA: return "CUDA launch failed";
        case SG_ERR_WORKSPACE: return "workspace missing or too small";
        case SG_ERR_UNSUPPORTED: return "shape outside build limits";
        default: return "unknown status";
    }
}

// comm.py:81-87: max(1, ceil(cr*dim - 1e-12)) in binary64, like the Python expression.
int64_t sg_topk_count(int64_t dim, double cr) {
    if (!(cr > 0.0 && cr <= 1.0)) return -1;
    const double x = cr * (double)dim - 1e-12;
    const double c = ceil(x);
    const int64_t m = (int64_t)c;
    return m < 1 ? 1 : m;
}

}  // extern "C"
