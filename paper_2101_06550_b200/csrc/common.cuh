// common.cuh — internal plumbing of libpentab.so (errors, launch counting,
// host-buffer staging).  Product code only; shares nothing with oracle/.
#pragma once
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>

#include <atomic>

#include "pentab.h"

namespace pb {

int set_error(int code, const char *fmt, ...);
void set_pivot(int64_t sys, int64_t row);
void count_launch(int n = 1);

#define PB_CUDA_TRY(expr)                                                                   \
    do {                                                                                    \
        cudaError_t e__ = (expr);                                                           \
        if (e__ != cudaSuccess) {                                                           \
            cudaGetLastError(); /* clear non-sticky errors so later calls are not poisoned */ \
            return pb::set_error(PB_ECUDA, "%s:%d %s: %s", __FILE__, __LINE__, #expr,      \
                                 cudaGetErrorString(e__));                                  \
        }                                                                                   \
    } while (0)

#define PB_LAUNCH_CHECK()                                                                   \
    do {                                                                                    \
        pb::count_launch();                                                                 \
        cudaError_t e__ = cudaGetLastError();                                               \
        if (e__ != cudaSuccess)                                                             \
            return pb::set_error(PB_ECUDA, "%s:%d launch: %s", __FILE__, __LINE__,          \
                                 cudaGetErrorString(e__));                                  \
    } while (0)

// True if p is a device (or managed) pointer usable by kernels directly.
bool is_device_ptr(const void *p);

// A buffer view that is device-resident for the duration of a call.  If the
// caller passed host memory it is staged through stream-ordered scratch
// (cudaMallocAsync) and, for outputs, copied back and the stream synchronised
// in finish().
struct Staged {
    void *dev = nullptr;
    const void *host_src = nullptr;
    void *host_dst = nullptr;
    size_t bytes = 0;
    bool staged = false;
    cudaStream_t st = nullptr;
    int in(const void *p, size_t nbytes, cudaStream_t s, bool copy_in);  // input (or in/out)
    int out_to(void *p);                                                 // mark as in/out
    int finish();                                                        // copy back + free
    ~Staged();
};

inline size_t dtype_size(int dtype) { return dtype == PB_F32 ? 4 : 8; }

}  // namespace pb
