// launch_util.cu -- host helpers shared by the launchers: the SM count of the current device
// and one-time kernel attributes, both cached per device (cudaDeviceGetAttribute and
// cudaFuncSetAttribute are driver calls; doing them on every launch costs host time and
// they never change for a device).
#include <map>
#include <mutex>
#include <utility>

#include "sb_kernels.cuh"

namespace sb {

namespace {
std::mutex g_mu;
std::map<int, int> g_sms;                                        // device -> SM count
std::map<std::pair<int, const void*>, int> g_smem;               // (device, kernel) -> smem set
std::map<std::pair<int, const void*>, int> g_carve;              // (device, kernel) -> carve-out set
}  // namespace

int sm_count() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 148;
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_sms.find(dev);
    if (it != g_sms.end()) return it->second;
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    g_sms[dev] = n;
    return n;
}

cudaError_t ensure_smem(const void* kern, int bytes) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(g_mu);
    auto key = std::make_pair(dev, kern);
    auto it = g_smem.find(key);
    if (it != g_smem.end() && it->second >= bytes) return cudaSuccess;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) g_smem[key] = bytes;
    return e;
}

cudaError_t ensure_carveout(const void* kern, int pct) {
    if (pct < 0) return cudaSuccess;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(g_mu);
    auto key = std::make_pair(dev, kern);
    auto it = g_carve.find(key);
    if (it != g_carve.end() && it->second == pct) return cudaSuccess;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
    if (e == cudaSuccess) g_carve[key] = pct;
    return e;
}

}  // namespace sb
