// vote.cu -- the voting step of PAPER.md:412-421 for sm_100a.
//
// C_T[p] = average over the target pixels q of the (2r+1)^2 window around p (clipped to the
// target) of C_S[src(q) + (p - q)], skipping positions outside the source; per channel
// floor((sum + floor(n/2)) / n) (reading R13).  Fallback pixels vote like any other (R14).
//
// One CTA = 128 x 16 output pixels; the coordinate field of the tile plus an r-pixel halo is
// staged in shared memory.  Each pixel first checks whether every window position votes for
// the same source pixel (the chunk interior, where the paper notes voting equals the blit,
// PAPER.md:420-421) -- then it is one gather; otherwise it accumulates the (2r+1)^2 gathers
// with SWAR (two 16-bit lanes per register; (2r+1)^2 * 255 < 2^16 for r <= 7) and divides by
// n with an exact multiply-high.
//
// Packed coordinates x | y<<16: for W, H <= 32767 and |d| <= 2r the packed sum
// src(q) + (p-q) never carries between fields, and any position left of / above the source
// wraps to a field >= 0xFFF0, which the bounds test rejects.
#include "sb_kernels.cuh"

namespace sb {

namespace {
constexpr int TW = 128, TH = 16, NT = 256;
constexpr uint32_t kOutside = 0xFFFFFFFFu;  // window position outside the target
}  // namespace

__global__ void __launch_bounds__(NT) vote_kernel(const VoteArgs a) {
    extern __shared__ __align__(16) uint32_t sc[];  // (TH + 2r) x (TW + 2r)
    const int r = a.r;
    const int SW = TW + 2 * r;
    const int tiles_x = (a.wt + TW - 1) / TW;
    const int x0 = (blockIdx.x % tiles_x) * TW;
    const int y0 = a.row_begin + (blockIdx.x / tiles_x) * TH;
    const int64_t fpx = (int64_t)a.wt * a.ht;
    const uint32_t* __restrict__ cf = a.coords + fpx * blockIdx.y;
    const uint32_t* __restrict__ cs = reinterpret_cast<const uint32_t*>(a.cs);

    const int SH = TH + 2 * r;
    for (int i = threadIdx.x; i < SW * SH; i += NT) {
        const int yy = i / SW, xx = i - yy * SW;
        const int gx = x0 - r + xx, gy = y0 - r + yy;
        uint32_t v = kOutside;
        if (gx >= 0 && gx < a.wt && gy >= 0 && gy < a.ht) v = __ldg(cf + (int64_t)gy * a.wt + gx);
        sc[i] = v;
    }
    __syncthreads();

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int rx0 = lane * 4;
    const uint32_t ws = (uint32_t)a.ws, hs = (uint32_t)a.hs;
#pragma unroll 1
    for (int rr = 0; rr < 2; ++rr) {
        const int ry = warp + 8 * rr;
        const int py = y0 + ry;
        if (py >= a.row_end || x0 + rx0 >= a.wt) continue;
        uint32_t outv[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int cx = rx0 + i + r, cy = ry + r;  // p in smem coordinates
            const uint32_t cp = sc[cy * SW + cx];
            // pass 1: does every in-target window position vote for src(p)?
            bool uniform = true;
            for (int dy = -r; dy <= r; ++dy) {
                const uint32_t* row = sc + (cy + dy) * SW + cx;
                const uint32_t sh = (uint32_t)dy << 16;
                for (int dx = -r; dx <= r; ++dx) {
                    const uint32_t v = row[dx];
                    // position voted by q = p + (dx,dy): src(q) - (dx,dy)
                    uniform &= (v == kOutside) | (v - (uint32_t)dx - sh == cp);
                }
            }
            if (uniform) {
                outv[i] = __ldg(cs + (cp >> 16) * ws + (cp & 0xFFFFu));
                continue;
            }
            // pass 2: full average
            uint32_t lo = 0, hi = 0, n = 0;
            for (int dy = -r; dy <= r; ++dy) {
                const uint32_t* row = sc + (cy + dy) * SW + cx;
                const uint32_t sh = (uint32_t)dy << 16;
                for (int dx = -r; dx <= r; ++dx) {
                    const uint32_t v = row[dx];
                    if (v == kOutside) continue;
                    const uint32_t pos = v - (uint32_t)dx - sh;
                    const uint32_t sx = pos & 0xFFFFu, sy = pos >> 16;
                    if (sx >= ws || sy >= hs) continue;
                    const uint32_t c = __ldg(cs + sy * ws + sx);
                    lo += c & 0x00FF00FFu;
                    hi += (c >> 8) & 0x00FF00FFu;
                    ++n;
                }
            }
            // n >= 1 (q = p votes for src(p), inside the source)
            const uint32_t half = n >> 1;
            uint32_t ch[4] = {(lo & 0xFFFFu) + half, (hi & 0xFFFFu) + half, (lo >> 16) + half, (hi >> 16) + half};
            uint32_t res = 0;
            if (n == 1) {
                res = (ch[0] - half) | ((ch[1] - half) << 8) | ((ch[2] - half) << 16) | ((ch[3] - half) << 24);
            } else {
                const uint32_t m = 0xFFFFFFFFu / n + 1u;  // ceil(2^32 / n); exact for sums < 2^17
#pragma unroll
                for (int c = 0; c < 4; ++c) res |= __umulhi(ch[c], m) << (8 * c);
            }
            outv[i] = res;
        }
        const int64_t o = fpx * blockIdx.y + (int64_t)py * a.wt + x0 + rx0;
        st_cs_u4(a.ct + 4 * o, make_uint4(outv[0], outv[1], outv[2], outv[3]));
    }
}

cudaError_t launch_vote(const VoteArgs& a, int n_frames, cudaStream_t st, int* launches) {
    const int tiles = ((a.wt + TW - 1) / TW) * ((a.row_end - a.row_begin + TH - 1) / TH);
    const size_t smem = sizeof(uint32_t) * (TW + 2 * a.r) * (TH + 2 * a.r);
    dim3 grid((unsigned)tiles, (unsigned)n_frames);
    vote_kernel<<<grid, NT, smem, st>>>(a);
    *launches += 1;
    return cudaPeekAtLastError();
}

}  // namespace sb
