// lut_build.cu -- exact guide look-up table (Alg. 2).
//
// LUT[k] = argmin over source pixels u of (k0 - G_S[u].c0)^2 + (k1 - G_S[u].c1)^2,
// ties -> smallest row-major index (reading R10).  Instead of the 65536 x (ws*hs) brute
// force, the argmin is split along the two guide axes (the squared Euclidean distance is
// separable), which is exact including the tie rule:
//
//   1. sites:   site[g1][g0] = min row-major index of the source pixels with guide (g0,g1)
//               (warp-deduplicated atomicMin; only the first pixel of a guide value can win).
//   2. resolve: one CTA per key row k1.  Thread a finds, in guide column a, the site b
//               minimising (k1-b)^2 (ties -> smaller pixel index: a site of column a with a
//               larger (k1-b)^2 can never tie the total).  Then thread k0 takes the minimum
//               over the 256 columns of (k0-a)^2 + f(a), ties -> smaller pixel index.
//
// Work: ws*hs scatter + 2 x 256^3 compare-selects (~33 M), independent of the exemplar
// size; the 256 KB site table stays in L2.
#include "sb_device.cuh"

namespace sb {

__global__ void __launch_bounds__(256) lut_init_kernel(uint32_t* __restrict__ site) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    reinterpret_cast<uint4*>(site)[i] = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
}

__global__ void __launch_bounds__(256) lut_sites_kernel(const uint32_t* __restrict__ gs, int n,
                                                        uint32_t* __restrict__ site) {
    const int lane = threadIdx.x & 31;
    for (int i0 = (blockIdx.x * blockDim.x + threadIdx.x) & ~31; i0 < n; i0 += gridDim.x * blockDim.x) {
        const int i = i0 + lane;
        const bool valid = i < n;
        const uint32_t key = valid ? (__ldg(gs + i) & 0xFFFFu) : 0x10000u + lane;
        // lanes holding the same key: the lowest lane has the smallest pixel index
        const unsigned peers = __match_any_sync(0xFFFFFFFFu, key);
        if (valid && (__ffs(peers) - 1) == lane) atomicMin(site + key, (uint32_t)i);
    }
}

__global__ void __launch_bounds__(256) lut_resolve_kernel(const uint32_t* __restrict__ site, int ws,
                                                          uint32_t* __restrict__ lut) {
    __shared__ uint32_t col_d[256];
    __shared__ uint32_t col_i[256];
    const int k1 = blockIdx.x;
    const int a = threadIdx.x;
    // pass 1: nearest site of column a to row k1 (1-D, tie -> smaller pixel index)
    uint32_t bd = 0xFFFFFFFFu, bi = 0xFFFFFFFFu;
#pragma unroll 8
    for (int b = 0; b < 256; ++b) {
        const uint32_t idx = __ldg(site + b * 256 + a);
        const int dy = k1 - b;
        const uint32_t d = (idx == 0xFFFFFFFFu) ? 0xFFFFFFFFu : (uint32_t)(dy * dy);
        if (d < bd || (d == bd && idx < bi)) { bd = d; bi = idx; }
    }
    col_d[a] = bd;
    col_i[a] = bi;
    __syncthreads();
    // pass 2: minimum over columns of (k0-a)^2 + f(a), tie -> smaller pixel index
    const int k0 = threadIdx.x;
    uint32_t best_d = 0xFFFFFFFFu, best_i = 0xFFFFFFFFu;
#pragma unroll 8
    for (int c = 0; c < 256; ++c) {
        const uint32_t fd = col_d[c];
        const int dx = k0 - c;
        const uint32_t d = (fd == 0xFFFFFFFFu) ? 0xFFFFFFFFu : fd + (uint32_t)(dx * dx);
        const uint32_t fi = col_i[c];
        if (d < best_d || (d == best_d && fi < best_i)) { best_d = d; best_i = fi; }
    }
    const uint32_t y = best_i / (uint32_t)ws, x = best_i - y * (uint32_t)ws;
    lut[k1 * 256 + k0] = pack_xy((int)x, (int)y);
}

cudaError_t launch_build_lut(const uint8_t* gs, int ws, int hs, uint32_t* lut, void* workspace,
                             cudaStream_t st, int* launches) {
    uint32_t* site = static_cast<uint32_t*>(workspace);
    lut_init_kernel<<<65536 / 4 / 256, 256, 0, st>>>(site);
    const int n = ws * hs;
    int blocks = (n + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    lut_sites_kernel<<<blocks, 256, 0, st>>>(reinterpret_cast<const uint32_t*>(gs), n, site);
    lut_resolve_kernel<<<256, 256, 0, st>>>(site, ws, lut);
    *launches += 3;
    return cudaPeekAtLastError();
}

}  // namespace sb
