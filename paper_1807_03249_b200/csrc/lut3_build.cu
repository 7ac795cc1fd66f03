// lut3_build.cu -- exact three-channel guide search, tabulated for all 2^24 keys
// (the look-up "or a tree search"; R26).
//
// LUT3[k] = argmin over source pixels u of sum_{c<3} (k_c - G_S[u].c)^2, ties -> smallest
// row-major index.  The squared distance is separable, so the argmin is three exact 1-D
// passes over the 256^3 key cube (the 2-channel LUT of lut_build.cu does two):
//
//   site[k]  = smallest pixel index with guide exactly k          (dedup + atomicMin)
//   D0[k]    = (0, site[k]) where a site exists, else none
//   pass a   D_{a+1}[k] = min_b ((k_a - b)^2 + D_a[k with k_a := b])   for a = 0, 1, 2
//
// each minimum taken lexicographically on (distance, pixel index).  A pixel that loses a
// 1-D minimum can never win or tie the full minimum with a smaller index (the line's
// winner has a smaller or equal index among the line's minimisers), so the tie rule holds.
// Each pass is a dense 256-candidate scan per entry: 2^32 compare-selects per pass, on a
// 128 MiB (distance, index) workspace, in place (a CTA owns whole lines).
#include "sb_kernels.cuh"

namespace sb {

namespace {
constexpr uint32_t kNone = 0xFFFFFFFFu;
constexpr int LC = 32;   // lines (columns) per CTA
constexpr int NT3 = 512; // threads per CTA: 32 columns x 16 output strides
constexpr int LCP = LC + 1;  // padded tile row (conflict-free transposing loads)
}

__global__ void __launch_bounds__(256) lut3_init_kernel(uint32_t* __restrict__ site) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    reinterpret_cast<uint4*>(site)[i] = make_uint4(kNone, kNone, kNone, kNone);
}

__global__ void __launch_bounds__(256) lut3_sites_kernel(const uint32_t* __restrict__ gs, uint32_t n,
                                                         uint32_t* __restrict__ site) {
    const int lane = threadIdx.x & 31;
    // pixel indices up to 65535^2 - 1 < 2^32 - 1 (the empty-site marker): 64-bit loop counter
    for (uint64_t i0 = (blockIdx.x * blockDim.x + threadIdx.x) & ~31u; i0 < n; i0 += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t i = i0 + (uint64_t)lane;
        const bool valid = i < n;
        const uint32_t key = valid ? (__ldg(gs + i) & 0xFFFFFFu) : 0x1000000u + lane;
        const unsigned peers = __match_any_sync(0xFFFFFFFFu, key);
        if (valid && (__ffs(peers) - 1) == lane) atomicMin(site + key, (uint32_t)i);
    }
}

// D0 from the sites: (0, index) or (none, none)
__global__ void __launch_bounds__(256) lut3_seed_kernel(const uint32_t* __restrict__ site, uint2* __restrict__ d) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t s = site[i];
    d[i] = make_uint2(s == kNone ? kNone : 0u, s);
}

// One 1-D pass along key axis `ax` (stride SA).  A CTA owns LC lines that are consecutive in
// dimension `col` (stride SC) for one value of the remaining dimension (stride SR).
__global__ void __launch_bounds__(NT3) lut3_pass_kernel(uint2* __restrict__ d, int SA, int SC, int SR) {
    extern __shared__ uint2 tile[];  // [256][LCP]
    const int cb = blockIdx.x;       // column block (256 / LC of them)
    const int rest = blockIdx.y;     // value of the remaining dimension
    const int64_t base = (int64_t)rest * SR + (int64_t)cb * LC * SC;
    for (int e = threadIdx.x; e < 256 * LC; e += NT3) {
        // SC == 1: consecutive threads read consecutive columns; else consecutive along ax
        const int b = SC == 1 ? e / LC : e % 256;
        const int c = SC == 1 ? e % LC : e / 256;
        tile[b * LCP + c] = d[base + (int64_t)b * SA + (int64_t)c * SC];
    }
    __syncthreads();
    const int c = threadIdx.x % LC;
    const int w = threadIdx.x / LC;  // outputs k = w + 16 j
    constexpr int NO = 256 / (NT3 / LC);
    uint32_t bd[NO], bi[NO];
#pragma unroll
    for (int j = 0; j < NO; ++j) { bd[j] = kNone; bi[j] = kNone; }
    for (int b = 0; b < 256; ++b) {
        const uint2 v = tile[b * LCP + c];
        if (v.x == kNone) continue;
#pragma unroll
        for (int j = 0; j < NO; ++j) {
            const int k = w + (NT3 / LC) * j;
            const uint32_t dd = v.x + (uint32_t)((k - b) * (k - b));
            if (dd < bd[j] || (dd == bd[j] && v.y < bi[j])) { bd[j] = dd; bi[j] = v.y; }
        }
    }
    __syncthreads();  // every read of the tile is done: write the pass result in place
#pragma unroll
    for (int j = 0; j < NO; ++j) {
        const int k = w + (NT3 / LC) * j;
        d[base + (int64_t)k * SA + (int64_t)c * SC] = make_uint2(bd[j], bi[j]);
    }
}

__global__ void __launch_bounds__(256) lut3_final_kernel(const uint2* __restrict__ d, int ws,
                                                         uint32_t* __restrict__ lut3) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t idx = d[i].y;
    const uint32_t y = idx / (uint32_t)ws, x = idx - y * (uint32_t)ws;
    lut3[i] = pack_xy((int)x, (int)y);
}

cudaError_t launch_build_lut3(const uint8_t* gs, int ws, int hs, uint32_t* lut3, void* workspace,
                              cudaStream_t st, int* launches) {
    constexpr int N = 1 << 24;
    uint32_t* site = lut3;  // the output doubles as the site table
    uint2* d = static_cast<uint2*>(workspace);
    lut3_init_kernel<<<N / 4 / 256, 256, 0, st>>>(site);
    const uint32_t n = (uint32_t)ws * (uint32_t)hs;
    int blocks = (n + 255) / 256;
    if (blocks > sm_count() * 16) blocks = sm_count() * 16;
    lut3_sites_kernel<<<blocks, 256, 0, st>>>(reinterpret_cast<const uint32_t*>(gs), n, site);
    lut3_seed_kernel<<<N / 256, 256, 0, st>>>(site, d);
    const int smem = 256 * LCP * (int)sizeof(uint2);
    cudaError_t e = ensure_smem(reinterpret_cast<const void*>(lut3_pass_kernel), smem);
    if (e != cudaSuccess) return e;
    const dim3 grid(256 / LC, 256);
    lut3_pass_kernel<<<grid, NT3, smem, st>>>(d, 1, 256, 65536);      // along k0, columns k1, rest k2
    lut3_pass_kernel<<<grid, NT3, smem, st>>>(d, 256, 1, 65536);      // along k1, columns k0, rest k2
    lut3_pass_kernel<<<grid, NT3, smem, st>>>(d, 65536, 1, 256);      // along k2, columns k0, rest k1
    lut3_final_kernel<<<N / 256, 256, 0, st>>>(d, ws, lut3);
    *launches += 7;
    return cudaPeekAtLastError();
}

}  // namespace sb
