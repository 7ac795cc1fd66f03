// lut_build.cu -- exact guide look-up table (Alg. 2).
//
// LUT[k] = argmin over source pixels u of (k0 - G_S[u].c0)^2 + (k1 - G_S[u].c1)^2,
// ties -> smallest row-major index (reading R10).  Instead of the 65536 x (ws*hs) brute
// force, the argmin is split along the two guide axes (the squared Euclidean distance is
// separable), which is exact including the tie rule:
//
//   1. sites:   site[g1][g0] = min row-major index of the source pixels with guide (g0,g1)
//               (warp-deduplicated atomicMin; only the first pixel of a guide value can win).
//   2. columns: for every key row k1 and guide column a, the site b of column a minimising
//               (k1-b)^2 (ties -> smaller pixel index: a site of column a with a larger
//               (k1-b)^2 can never tie the total) -- the nearest occupied row above and below
//               k1, from warp scans (one warp per column).
//   3. resolve: one CTA per key row k1; thread k0 takes the minimum over the 256 columns of
//               (k0-a)^2 + f(a), ties -> smaller pixel index (split over 4 threads per key).
//
// Work: ws*hs scatter + 256^2 column entries + 256^3 compare-selects (~17 M), independent of
// the exemplar size; the 256 KB site table and the 512 KB column table stay in L2.
#include "sb_kernels.cuh"

namespace sb {

__global__ void __launch_bounds__(256) lut_init_kernel(uint32_t* __restrict__ site) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    reinterpret_cast<uint4*>(site)[i] = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
}

__global__ void __launch_bounds__(256) lut_sites_kernel(const uint32_t* __restrict__ gs, uint32_t n,
                                                        uint32_t* __restrict__ site) {
    const int lane = threadIdx.x & 31;
    // pixel indices up to 65535^2 - 1 < 2^32 - 1 (the empty-site marker): 64-bit loop counter
    for (uint64_t i0 = (blockIdx.x * blockDim.x + threadIdx.x) & ~31u; i0 < n; i0 += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t i = i0 + (uint64_t)lane;
        const bool valid = i < n;
        const uint32_t key = valid ? (__ldg(gs + i) & 0xFFFFu) : 0x10000u + lane;
        // lanes holding the same key: the lowest lane has the smallest pixel index
        const unsigned peers = __match_any_sync(0xFFFFFFFFu, key);
        SB_CHECK(key < 0x10000u + 32u, "site key");
        if (valid && (__ffs(peers) - 1) == lane) atomicMin(site + key, (uint32_t)i);
    }
}

// pass 1, all rows at once: one warp per guide column a; lane j owns the 8 rows b = 8j..8j+7.
// For every row k1 the nearest occupied site of column a: the last site at or above k1 and the
// first at or below it (warp max / min scans), the closer one, ties -> smaller pixel index.
// Output col[k1 * 256 + a] = (d, idx), d = (k1 - b)^2 (0xFFFFFFFF: empty column).
__global__ void __launch_bounds__(256) lut_columns_kernel(const uint32_t* __restrict__ site,
                                                          uint2* __restrict__ col) {
    const int lane = threadIdx.x & 31;
    const int a = blockIdx.x * 8 + (threadIdx.x >> 5);
    uint32_t idx[8];
    int last = -1, first = 256;  // last / first occupied row within this lane's 8 rows
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        idx[k] = __ldg(site + (8 * lane + k) * 256 + a);
        if (idx[k] != 0xFFFFFFFFu) {
            last = 8 * lane + k;
            if (first == 256) first = 8 * lane + k;
        }
    }
    // exclusive scans across lanes: last occupied row above this lane, first below it
    int above = last, below = first;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xFFFFFFFFu, above, o);
        const int dn = __shfl_down_sync(0xFFFFFFFFu, below, o);
        if (lane >= o) above = max(above, u);
        if (lane + o < 32) below = min(below, dn);
    }
    int prev = __shfl_up_sync(0xFFFFFFFFu, above, 1);   // last occupied row before this lane
    int next = __shfl_down_sync(0xFFFFFFFFu, below, 1); // first occupied row after this lane
    if (lane == 0) prev = -1;
    if (lane == 31) next = 256;
    // site pixel index of a row (only read for occupied rows)
    auto idx_of = [&](int b) -> uint32_t {
        const int owner = b >> 3;
        uint32_t v = 0xFFFFFFFFu;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint32_t t = __shfl_sync(0xFFFFFFFFu, idx[k], owner & 31);
            if ((b & 7) == k) v = t;
        }
        return v;
    };
    // nearest occupied row at or above / at or below each of the lane's rows
    int up[8], dnr[8];
    int cur = prev;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        if (idx[k] != 0xFFFFFFFFu) cur = 8 * lane + k;
        up[k] = cur;
    }
    cur = next;
#pragma unroll
    for (int k = 7; k >= 0; --k) {
        if (idx[k] != 0xFFFFFFFFu) cur = 8 * lane + k;
        dnr[k] = cur;
    }
    // the pixel indices of the rows up[k] / dnr[k] live in other lanes: fetch them with shuffles
    // (every lane takes part in every shuffle, so the loops stay warp-uniform)
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int k1 = 8 * lane + k;
        const int bu = up[k], bd = dnr[k];
        const uint32_t iu = idx_of(bu < 0 ? 0 : bu), id = idx_of(bd > 255 ? 0 : bd);
        uint32_t d = 0xFFFFFFFFu, i = 0xFFFFFFFFu;
        if (bu >= 0) { d = (uint32_t)((k1 - bu) * (k1 - bu)); i = iu; }
        if (bd <= 255) {
            const uint32_t dd = (uint32_t)((bd - k1) * (bd - k1));
            if (dd < d || (dd == d && id < i)) { d = dd; i = id; }
        }
        col[k1 * 256 + a] = make_uint2(d, i);
    }
}

// pass 2: one CTA per key row k1, 1024 threads: thread (q, k0) takes the minimum over the 64
// columns a = 64q .. 64q+63 of (k0-a)^2 + f(a), ties -> smaller pixel index; the four quarter
// results of k0 are then combined (the (d, index) order is total, so the combination order does
// not matter).  Four quarters instead of one thread per key: 256 CTAs on 148 SMs leave 1-2 CTAs
// per SM, and the compare chain is latency-bound at 8 warps per SM.
constexpr int kResolveQ = 4;
__global__ void __launch_bounds__(256 * kResolveQ) lut_resolve_kernel(const uint2* __restrict__ col, int ws,
                                                                      uint32_t* __restrict__ lut) {
    __shared__ uint32_t col_d[256];
    __shared__ uint32_t col_i[256];
    __shared__ uint32_t part_d[kResolveQ][256];
    __shared__ uint32_t part_i[kResolveQ][256];
    const int k1 = blockIdx.x;
    if (threadIdx.x < 256) {
        const uint2 c = __ldg(col + k1 * 256 + threadIdx.x);
        col_d[threadIdx.x] = c.x;
        col_i[threadIdx.x] = c.y;
    }
    __syncthreads();
    const int k0 = threadIdx.x & 255, q = threadIdx.x >> 8;
    uint32_t best_d = 0xFFFFFFFFu, best_i = 0xFFFFFFFFu;
#pragma unroll 8
    for (int cc = 64 * q; cc < 64 * q + 64; ++cc) {
        const uint32_t fd = col_d[cc];
        const int dx = k0 - cc;
        const uint32_t d = (fd == 0xFFFFFFFFu) ? 0xFFFFFFFFu : fd + (uint32_t)(dx * dx);
        const uint32_t fi = col_i[cc];
        if (d < best_d || (d == best_d && fi < best_i)) { best_d = d; best_i = fi; }
    }
    part_d[q][k0] = best_d;
    part_i[q][k0] = best_i;
    __syncthreads();
    if (q != 0) return;
#pragma unroll
    for (int r = 1; r < kResolveQ; ++r) {
        const uint32_t d = part_d[r][k0], fi = part_i[r][k0];
        if (d < best_d || (d == best_d && fi < best_i)) { best_d = d; best_i = fi; }
    }
    const uint32_t y = best_i / (uint32_t)ws, x = best_i - y * (uint32_t)ws;
    SB_CHECK(best_i != 0xFFFFFFFFu, "LUT entry resolved");
    lut[k1 * 256 + k0] = pack_xy((int)x, (int)y);
}

cudaError_t launch_build_lut(const uint8_t* gs, int ws, int hs, uint32_t* lut, void* workspace,
                             cudaStream_t st, int* launches) {
    uint32_t* site = static_cast<uint32_t*>(workspace);
    lut_init_kernel<<<65536 / 4 / 256, 256, 0, st>>>(site);
    const uint32_t n = (uint32_t)ws * (uint32_t)hs;
    int blocks = (n + 255) / 256;
    if (blocks > sm_count() * 16) blocks = sm_count() * 16;
    lut_sites_kernel<<<blocks, 256, 0, st>>>(reinterpret_cast<const uint32_t*>(gs), n, site);
    uint2* col = reinterpret_cast<uint2*>(site + 65536);  // 256 x 256 (d, idx) after the sites
    lut_columns_kernel<<<32, 256, 0, st>>>(site, col);
    lut_resolve_kernel<<<256, 256 * kResolveQ, 0, st>>>(col, ws, lut);
    *launches += 4;
    return cudaPeekAtLastError();
}

}  // namespace sb
