#include "sm_budget.h"

#include <cuda_runtime.h>

#include <cstdlib>

namespace ptk {

int device_sm_count() {
    static const int n = [] {
        int dev = 0, v = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
        return v;
    }();
    return n;
}

int sm_budget() {
    static const int n = [] {
        const char* r = std::getenv("PTK_SM_RESERVE");
        const int reserve = r ? std::atoi(r) : 0;
        const int v = device_sm_count() - (reserve > 0 ? reserve : 0);
        return v < 2 ? 2 : v;
    }();
    return n;
}

}  // namespace ptk
