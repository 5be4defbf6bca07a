// Per-thread runtime: device selection, stream, grow-only workspaces, error text,
// launch accounting.  The reference has no global mutable state (SURVEY.md §8(b)
// "Threading"); neither does this library beyond the per-device jump tables.
#include <atomic>
#include <mutex>

#include "rl_internal.cuh"

namespace rl {

namespace {
thread_local std::string t_err;
thread_local Ctx* t_ctx = nullptr;
std::atomic<uint64_t> g_launches{0};
} // namespace

void set_error(const std::string& msg) { t_err = msg; }
const char* last_error() { return t_err.c_str(); }

[[noreturn]] void fail(rl_status code, const std::string& msg) { throw Failure{code, msg}; }

void count_launch() {
    ctx().launches++;
    g_launches.fetch_add(1, std::memory_order_relaxed);
}

uint64_t total_launches() { return g_launches.load(); }

void* DevBuf::get(size_t need) {
    if (need == 0)
        need = 16;
    if (need > bytes) {
        if (ptr) {
            cudaStreamSynchronize(ctx().stream);
            cudaFree(ptr);
            ptr = nullptr;
            bytes = 0;
        }
        size_t grow = need + need / 8;
        cudaError_t e = cudaMalloc(&ptr, grow);
        if (e != cudaSuccess) {
            (void)cudaGetLastError();
            e = cudaMalloc(&ptr, need);
            grow = need;
        }
        if (e != cudaSuccess) {
            ptr = nullptr;
            fail(RL_CUDA_ERROR, std::string("workspace allocation: ") + cudaGetErrorString(e));
        }
        bytes = grow;
    }
    return ptr;
}

DevBuf::~DevBuf() {
    if (ptr)
        cudaFree(ptr);
}

void ensure_device() {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        (void)cudaGetLastError();
        fail(RL_NO_DEVICE, "no CUDA device: librl_b200 has no CPU fallback");
    }
}

static void ctx_init(Ctx& c, int device) {
    ensure_device();
    if (device < 0)
        RL_CUDA(cudaGetDevice(&device));
    RL_CUDA(cudaSetDevice(device));
    c.device = device;
    RL_CUDA(cudaStreamCreateWithFlags(&c.own, cudaStreamNonBlocking));
    c.stream = c.own;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    c.sms = sms;
}

Ctx& ctx() {
    if (!t_ctx) {
        static thread_local Ctx storage;
        if (storage.device < 0)
            ctx_init(storage, -1);
        t_ctx = &storage;
    }
    return *t_ctx;
}

void init_device(int device) {
    static thread_local Ctx storage2;
    if (t_ctx && t_ctx->device == device)
        return;
    if (storage2.device < 0)
        ctx_init(storage2, device);
    t_ctx = &storage2;
}

} // namespace rl
