// vote_wide.cu -- the voting step of PAPER.md:412-421 for the regimes the packed-arithmetic vote
// kernels (vote.cu) do not serve: images wider or taller than 32767 pixels (packed coordinates
// would carry between fields).  (Up to round 2 it also served r = 8.)
//
// One thread per output pixel of a 32 x 8 tile; the tile's coordinates plus an r halo are
// staged in shared memory (kOutside outside the target: a valid coordinate has x <= 65534);
// every window position is tested with signed source coordinates and summed per channel in
// 32 bits; C_T[p] = floor((sum + floor(n/2)) / n) per channel (reading R13, R14).
#include "sb_kernels.cuh"

namespace sb {

namespace {
constexpr int WW = 32, WH = 8, WR = 8;  // tile, maximum radius
constexpr uint32_t kOut = 0xFFFFFFFFu;
}  // namespace

__global__ void __launch_bounds__(WW * WH) vote_wide_kernel(const VoteArgs a) {
    __shared__ uint32_t sc[WH + 2 * WR][WW + 2 * WR];
    const int r = a.r;
    const int x0 = blockIdx.x * WW, y0 = a.row_begin + blockIdx.y * WH, frame = blockIdx.z;
    const int64_t fpx = (int64_t)a.wt * a.ht;
    const uint32_t* __restrict__ cf = a.coords + fpx * frame;
    const int sw = WW + 2 * r, sh = WH + 2 * r;
    for (int i = threadIdx.x; i < sw * sh; i += WW * WH) {
        const int yy = i / sw, xx = i - yy * sw;
        const int gx = x0 - r + xx, gy = y0 - r + yy;
        const bool in = gx >= 0 && gx < a.wt && gy >= 0 && gy < a.ht;
        sc[yy][xx] = in ? __ldg(cf + (int64_t)gy * a.wt + gx) : kOut;
    }
    __syncthreads();
    const int tx = threadIdx.x % WW, ty = threadIdx.x / WW;
    const int px = x0 + tx, py = y0 + ty;
    if (px >= a.wt || py >= a.row_end) return;
    const uint32_t* __restrict__ cs = reinterpret_cast<const uint32_t*>(a.cs);
    uint32_t s0 = 0, s1 = 0, s2 = 0, s3 = 0, n = 0;
    for (int dy = -r; dy <= r; ++dy) {
        for (int dx = -r; dx <= r; ++dx) {
            const uint32_t w = sc[ty + r + dy][tx + r + dx];  // src(q), q = p + (dx, dy)
            if (w == kOut) continue;
            const int sx = (int)(w & 0xFFFFu) - dx, sy = (int)(w >> 16) - dy;  // src(q) + (p - q)
            if (sx < 0 || sx >= a.ws || sy < 0 || sy >= a.hs) continue;
            SB_CHECK(sx >= 0 && sx < a.ws && sy >= 0 && sy < a.hs, "wide vote gather");
            const uint32_t c = __ldg(cs + (int64_t)sy * a.ws + sx);
            s0 += c & 0xFFu;
            s1 += (c >> 8) & 0xFFu;
            s2 += (c >> 16) & 0xFFu;
            s3 += c >> 24;
            ++n;
        }
    }
    // n >= 1: q = p votes for src(p), which is inside the source
    const uint32_t h = n >> 1;
    const uint32_t out = ((s0 + h) / n) | (((s1 + h) / n) << 8) | (((s2 + h) / n) << 16) | (((s3 + h) / n) << 24);
    st_cs_u32(a.ct + 4 * (fpx * frame + (int64_t)py * a.wt + px), out);
}

cudaError_t launch_vote_wide(const VoteArgs& a, int n_frames, cudaStream_t st, int* launches) {
    if (a.r < 0 || a.r > WR) return cudaErrorInvalidValue;
    dim3 grid((unsigned)((a.wt + WW - 1) / WW), (unsigned)((a.row_end - a.row_begin + WH - 1) / WH),
              (unsigned)n_frames);
    vote_wide_kernel<<<grid, WW * WH, 0, st>>>(a);
    *launches += 1;
    return cudaPeekAtLastError();
}

}  // namespace sb
