// stylize_naive.cu -- one thread per target pixel, Alg. 2 written straight.
//
// Serves what the tiled kernel of stylize.cu does not: L in 10..15 and image sides beyond
// 32767 (signed coordinates throughout, NearestSeed distances in 64 bits: |s - p| reaches
// 2h = 2^16 at L = 15).  Also the simple baseline (SB_KERNEL=naive) the tiled kernel is
// measured against; both agree bit for bit with the oracle.
#include "sb_kernels.cuh"

namespace sb {

template <bool EXT>
__global__ void __launch_bounds__(256) stylize_naive_kernel(const __grid_constant__ StylizeArgs a) {
    const int frame = blockIdx.y;
    const int64_t npx = (int64_t)(a.row_end - a.row_begin) * a.wt;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= npx) return;
    const int py = a.row_begin + (int)(i / a.wt);
    const int px = (int)(i % a.wt);
    const int64_t fpx = (int64_t)a.wt * a.ht;
    const uint32_t* gt = reinterpret_cast<const uint32_t*>(a.gt) + fpx * frame;
    const uint32_t* gs = reinterpret_cast<const uint32_t*>(a.gs);
    const uint32_t seed = a.frame_seed(frame);
    const bool zj = a.zero_jitter;
    const uint32_t gp = __ldg(gt + (int64_t)py * a.wt + px);

    uint32_t coord = 0;
    int level = 0;
    for (int l = a.L; l >= 1; --l) {
        const uint32_t c_l = level_salt(seed, l);
        const int bx = px >> l, by = py >> l;
        uint64_t best = ~0ull;
        int qx = 0, qy = 0;
        // NearestSeed: x outer, y inner, first strict minimum
        for (int x = -1; x <= 1; ++x)
            for (int y = -1; y <= 1; ++y) {
                int sx, sy;
                cell_seed(bx + x, by + y, l, c_l, zj, sx, sy);
                const int64_t dx = sx - px, dy = sy - py;
                const uint64_t d = (uint64_t)(dx * dx + dy * dy);
                if (d < best) { best = d; qx = sx; qy = sy; }
            }
        qx = min(max(qx, 0), a.wt - 1);  // R8
        qy = min(max(qy, 0), a.ht - 1);
        const uint32_t u = __ldg(a.lut + (__ldg(gt + (int64_t)qy * a.wt + qx) & a.key_mask));
        const int sx = (int)(u & 0xFFFFu) + (px - qx);
        const int sy = (int)(u >> 16) + (py - qy);
        if ((unsigned)sx >= (unsigned)a.ws || (unsigned)sy >= (unsigned)a.hs) continue;  // R9
        SB_CHECK(qx >= 0 && qx < a.wt && qy >= 0 && qy < a.ht && sx >= 0 && sy >= 0, "naive gathers");
        const uint32_t g = __ldg(gs + (int64_t)sy * a.ws + sx);
        const bool ok = EXT ? guide_ok_ext(gp, g, a.cmask, a.w, a.lmask, a.T2) : guide_d2(gp, g, a.cmask) < a.T2;
        if (ok) { coord = pack_xy(sx, sy); level = l; break; }
    }
    if (level == 0) coord = __ldg(a.lut + (gp & a.key_mask));  // R12
    const int64_t o = fpx * frame + (int64_t)py * a.wt + px;
    SB_CHECK((coord & 0xFFFFu) < (uint32_t)a.ws && (coord >> 16) < (uint32_t)a.hs, "naive coordinate");
    if (a.coords) a.coords[o] = coord;
    if (a.level) a.level[o] = (uint8_t)level;
    if (a.ct) {
        const uint32_t c = __ldg(reinterpret_cast<const uint32_t*>(a.cs) + (int64_t)(coord >> 16) * a.ws + (coord & 0xFFFFu));
        reinterpret_cast<uint32_t*>(a.ct)[o] = c;
    }
}

cudaError_t launch_stylize_naive(const StylizeArgs& a, int n_frames, cudaStream_t st, int* launches) {
    const int64_t npx = (int64_t)(a.row_end - a.row_begin) * a.wt;
    dim3 grid((unsigned)((npx + 255) / 256), (unsigned)n_frames);
    if (a.ext) stylize_naive_kernel<true><<<grid, 256, 0, st>>>(a);
    else stylize_naive_kernel<false><<<grid, 256, 0, st>>>(a);
    *launches += 1;
    return cudaPeekAtLastError();
}

}  // namespace sb
