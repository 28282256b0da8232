// device.cpp -- per-device state of the library: the SM count and the
// per-kernel function attributes.  Both are per device (a process may drive
// several GPUs) and initialised once, thread-safely (include/relax_q4.h:
// "Reentrant"; SURVEY §8(b) "the only global state is the per-device SM
// count, initialised once").
#include <mutex>
#include <unordered_set>

#include "internal.h"

namespace rq4 {

namespace {
constexpr int kMaxDevices = 64;
std::once_flag g_sm_once[kMaxDevices];
int g_sms[kMaxDevices];

struct AttrKey {
    int dev;
    const void* fn;
    bool operator==(const AttrKey& o) const { return dev == o.dev && fn == o.fn; }
};
struct AttrHash {
    size_t operator()(const AttrKey& k) const {
        return std::hash<const void*>()(k.fn) ^ (static_cast<size_t>(k.dev) * 0x9E3779B97F4A7C15ull);
    }
};
std::mutex g_attr_mu;
std::unordered_set<AttrKey, AttrHash> g_attr_done;
}  // namespace

int current_device() {
    int dev = -1;
    if (cudaGetDevice(&dev) != cudaSuccess) {
        cudaGetLastError();
        return -1;
    }
    return dev;
}

int num_sms() {
    const int dev = current_device();
    if (dev < 0 || dev >= kMaxDevices) return kB200SMs;
    std::call_once(g_sm_once[dev], [dev] {
        int v = 0;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) {
            cudaGetLastError();
            v = kB200SMs;
        }
        g_sms[dev] = v;
    });
    return g_sms[dev];
}

cudaError_t ensure_kernel_attrs(const void* fn, int dyn_bytes, bool cluster) {
    const int dev = current_device();
    if (dev < 0) return cudaErrorNoDevice;
    const AttrKey key{dev, fn};
    std::lock_guard<std::mutex> lk(g_attr_mu);
    if (g_attr_done.count(key)) return cudaSuccess;
    cudaError_t e = set_kernel_smem(fn, dyn_bytes);
    if (e == cudaSuccess && cluster) e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    g_attr_done.insert(key);
    return cudaSuccess;
}

}  // namespace rq4
