// api.cu — error reporting, launch counting and host-buffer staging shared by
// every entry point of libpentab.so.
#include <string.h>

#include "common.cuh"

namespace pb {

struct ErrState {
    int code = PB_OK;
    int64_t sys = -1, row = -1;
    char msg[512] = {0};
};
static thread_local ErrState g_err;
static std::atomic<int64_t> g_launches{0};

int set_error(int code, const char *fmt, ...)
{
    g_err.code = code;
    g_err.sys = g_err.row = -1;
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err.msg, sizeof(g_err.msg), fmt, ap);
    va_end(ap);
    return code;
}

void set_pivot(int64_t sys, int64_t row)
{
    g_err.sys = sys;
    g_err.row = row;
}

void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

bool is_device_ptr(const void *p)
{
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

int Staged::in(const void *p, size_t nbytes, cudaStream_t s, bool copy_in)
{
    st = s;
    bytes = nbytes;
    if (p == nullptr) return set_error(PB_EINVAL, "null buffer");
    if (is_device_ptr(p)) {
        dev = const_cast<void *>(p);
        staged = false;
        return PB_OK;
    }
    staged = true;
    host_src = p;
    if (nbytes == 0) return PB_OK;
    PB_CUDA_TRY(cudaMallocAsync(&dev, nbytes, s));
    if (copy_in) PB_CUDA_TRY(cudaMemcpyAsync(dev, p, nbytes, cudaMemcpyHostToDevice, s));
    return PB_OK;
}

int Staged::out_to(void *p)
{
    host_dst = p;
    return PB_OK;
}

int Staged::finish()
{
    if (!staged) return PB_OK;
    if (host_dst && bytes) PB_CUDA_TRY(cudaMemcpyAsync(host_dst, dev, bytes, cudaMemcpyDeviceToHost, st));
    if (dev) PB_CUDA_TRY(cudaFreeAsync(dev, st));
    dev = nullptr;
    PB_CUDA_TRY(cudaStreamSynchronize(st));
    staged = false;
    return PB_OK;
}

Staged::~Staged()
{
    if (staged && dev) cudaFreeAsync(dev, st);
}

}  // namespace pb

extern "C" int pb_last_error(int64_t *sys, int64_t *row, char *msg, size_t len)
{
    if (sys) *sys = pb::g_err.sys;
    if (row) *row = pb::g_err.row;
    if (msg && len) {
        strncpy(msg, pb::g_err.msg, len - 1);
        msg[len - 1] = 0;
    }
    return pb::g_err.code;
}

extern "C" int64_t pb_launch_count(void) { return pb::g_launches.load(); }
extern "C" void pb_reset_launch_count(void) { pb::g_launches.store(0); }

extern "C" int pb_device_ok(void)
{
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        cudaGetLastError();
        return pb::set_error(PB_ECUDA, "no CUDA device");
    }
    return PB_OK;
}
