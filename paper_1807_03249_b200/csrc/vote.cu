// vote.cu -- the voting step of PAPER.md:412-421 for sm_100a.
//
// C_T[p] = average over the target pixels q of the (2r+1)^2 window around p (clipped to the
// target) of C_S[src(q) + (p - q)], skipping positions outside the source; per channel
// floor((sum + floor(n/2)) / n) (reading R13).  Fallback pixels vote like any other (R14).
//
// One CTA = 128 x 16 output pixels, 256 threads; the coordinate field of the tile plus an
// r-pixel halo is staged in shared memory, the colours are assembled in shared memory and
// leave in coalesced 16-byte stores.
//
// Fast tiles (the common case): every staged position is inside the target and every staged
// source pixel is at least r from the source border.  Then no window position can be clipped
// or leave the source, the staged coordinates are converted to linear source indices
// (y*ws + x), and "q votes for the same source pixel as p" is the linear identity
// lin(q) - lin(p) = (qx - px) + (qy - py)*ws (exact under the margin).
//   1. per staged row and 4-pixel group: which of the 4 row segments [x-r, x+r] are one chunk
//      (a nibble per group, from 16-byte shared loads);
//   2. per pixel: the window is one chunk iff its 2r+1 row segments are and the centre column
//      continues vertically -- then the vote is unanimous and C_T[p] = C_S[src(p)] (the chunk
//      interior, where voting equals the blit): one gather;
//   3. the other pixels go to shared-memory queues, processed densely one pixel per thread,
//      window row by window row: the row-link bits split a row into runs of positions that
//      vote for the same source pixel, and each run costs one gather weighted by its length.
//      Pixels whose rows have at most two runs (most) take a branch-free two-gather row
//      step; the others a run loop, in their own queue so warps do not diverge.  Sums are
//      SWAR (two 16-bit lanes per register; (2r+1)^2 * 255 < 2^16 for r <= 7, r = 8 splits the
//      window rows over two register pairs); division by (2r+1)^2.
// Border tiles: every pixel takes the general per-position path with target clipping and
// source bounds tests on packed coordinates (x | y<<16; for W, H <= 32767 and |d| <= 2r the
// packed sum src(q) + (p-q) never carries between fields and any position left of / above
// the source wraps to a field >= 0xFFF0, which the bounds test rejects).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <type_traits>
#include <map>
#include <mutex>

#include "sb_kernels.cuh"

// the margin tests v >= R / v < R are trivially true / false in the R = 0 instantiations
#pragma nv_diag_suppress 186

namespace sb {

namespace {
constexpr int TW = 128, TH = 16, NT = 256;
constexpr int NG = TW / 4;                   // 4-pixel groups per row
// window position outside the target: fields 0xC000 stay >= 0xC000 - 8 > 32767 after any window
// offset, so the packed in-source test rejects it by itself (and it never links with a coordinate)
constexpr uint32_t kOutside = 0xC000C000u;

// The colour sums of one pixel's window: two 16-bit lanes per register (SWAR, channels 0 and 2
// in lo, 1 and 3 in hi).  For r = 8 a lane could overflow ((2r+1)^2 * 255 >= 2^16): the window
// rows dy < 0 and dy >= 0 then sum into separate pairs (at most 9 * 17 * 255 < 2^16 each) that
// meet in 32 bits at the end.  dy is a compile-time constant at every call (unrolled loops).
template <int R>
struct Sums {
    static constexpr bool SPLIT = (2 * R + 1) * (2 * R + 1) * 255 >= 65536;
    uint32_t lo = 0, hi = 0, lo2 = 0, hi2 = 0;
    __device__ __forceinline__ void add(int dy, uint32_t c, uint32_t len) {
        const uint32_t l = (c & 0x00FF00FFu) * len, h = __byte_perm(c, 0u, 0x7371) * len;  // bytes 1, 3
        if (SPLIT && dy >= 0) {
            lo2 += l;
            hi2 += h;
        } else {
            lo += l;
            hi += h;
        }
    }
    // two colours with their counts (the two runs of a window row), summed before the accumulator
    __device__ __forceinline__ void add2(int dy, uint32_t c1, uint32_t n1, uint32_t c2, uint32_t n2) {
        const uint32_t l = (c1 & 0x00FF00FFu) * n1 + (c2 & 0x00FF00FFu) * n2;
        const uint32_t h = __byte_perm(c1, 0u, 0x7371) * n1 + __byte_perm(c2, 0u, 0x7371) * n2;
        if (SPLIT && dy >= 0) {
            lo2 += l;
            hi2 += h;
        } else {
            lo += l;
            hi += h;
        }
    }
    __device__ __forceinline__ void channels(uint32_t (&s)[4]) const {
        s[0] = lo & 0xFFFFu; s[1] = hi & 0xFFFFu; s[2] = lo >> 16; s[3] = hi >> 16;
        if (SPLIT) { s[0] += lo2 & 0xFFFFu; s[1] += hi2 & 0xFFFFu; s[2] += lo2 >> 16; s[3] += hi2 >> 16; }
    }
};

template <int R>
__device__ __forceinline__ uint32_t finish(const Sums<R>& sm, uint32_t n) {
    uint32_t s[4];
    sm.channels(s);
    if (n <= 1) return Sums<R>::SPLIT ? s[0] | (s[1] << 8) | (s[2] << 16) | (s[3] << 24)
                                      : (sm.lo & 0x00FF00FFu) | ((sm.hi & 0x00FF00FFu) << 8);
    const uint32_t half = n >> 1;
    const uint32_t m = 0xFFFFFFFFu / n + 1u;  // ceil(2^32/n): exact floor for numerators < 2^32/n
    const uint32_t c0 = __umulhi(s[0] + half, m), c1 = __umulhi(s[1] + half, m);
    const uint32_t c2 = __umulhi(s[2] + half, m), c3 = __umulhi(s[3] + half, m);
    return c0 | (c1 << 8) | (c2 << 16) | (c3 << 24);
}

template <uint32_t N, int R>
__device__ __forceinline__ uint32_t finish_const(const Sums<R>& sm) {
    constexpr uint32_t half = N / 2;
    uint32_t s[4];
    sm.channels(s);
    const uint32_t c0 = (s[0] + half) / N, c1 = (s[1] + half) / N;
    const uint32_t c2 = (s[2] + half) / N, c3 = (s[3] + half) / N;
    return c0 | (c1 << 8) | (c2 << 16) | (c3 << 24);
}

// Predicated gather: returns 0 without touching memory when !pred (keeps L1 traffic to the
// gathers that matter, without a branch).
__device__ __forceinline__ uint32_t ldg_if(const uint32_t* p, bool pred) {
    uint32_t v = 0;
    asm volatile(
        "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q ld.global.nc.u32 %0, [%1];\n\t}"
        : "+r"(v)
        : "l"(p), "r"((uint32_t)pred));
    return v;
}

}  // namespace

// Tile geometry and the shared scratch of one tile (besides the staged coordinates).
template <int R>
struct VoteGeom {
    static constexpr int SW = TW + 2 * R, SH = TH + 2 * R;
    static constexpr int KR = (R + 3) / 4;    // 16-byte words covering the halo
    static constexpr int OFF = 4 * KR;        // tile column x is stored at sc[.][OFF + x]
    static constexpr int SWP = OFF + TW + OFF;  // 16-byte aligned rows
};

template <int R>
struct VoteShared {
    static constexpr int SH = VoteGeom<R>::SH;
    uint8_t seg[SH][NG];        // nibble: which of the group's 4 row segments are one chunk
    uint8_t seg3[SH][NG];       // nibble: which of them have three or more runs
    uint8_t vseg[SH][NG];       // nibble: which of the group's 4 columns continue into the next row
    // the 2r link bits of the window row centred at each staged position (bit i: window position
    // i+1 continues i)
    std::conditional_t<(2 * R <= 8), uint8_t, uint16_t> wl[SH][TW];
    __align__(16) uint32_t outc[TH][TW];
    uint16_t queue[TH * TW];    // two-run pixels from the front, others from the back
    uint16_t qe[2 * R * (TW + TH) + 1];  // fast tiles at the frame edge: pixels within r of it
    int qn, qn3, qne;
};

// The vote of one tile whose coordinates (tile + r halo, kOutside outside the target) are
// staged in sc; fast: the fast-tile margin holds for every staged position.  S.qn and S.qn3
// are zero and ordered before the call by a CTA barrier.
// PAD: C_S is read from the strided exemplar copy (rows of 2^16 pixels, sb_prepare_exemplar),
// where a packed coordinate x | y<<16 is its own index: the "linear" source indices below are
// then the packed values themselves (row stride 65536) and the conversion pass disappears.
template <int R, bool PAD>
__device__ __forceinline__ void vote_tile(const VoteArgs& a, uint32_t (*sc)[VoteGeom<R>::SWP], VoteShared<R>& S,
                                          int x0, int y0, int frame, bool fast) {
    constexpr int SH = VoteGeom<R>::SH, KR = VoteGeom<R>::KR, OFF = VoteGeom<R>::OFF, SWP = VoteGeom<R>::SWP;
    auto& seg = S.seg;
    auto& seg3 = S.seg3;
    auto& vseg = S.vseg;
    auto& wl = S.wl;
    auto& outc = S.outc;
    auto& queue = S.queue;
    int& qn = S.qn;
    int& qn3 = S.qn3;
    int& qne = S.qne;
    auto& qe = S.qe;
    // a fast tile at the frame edge: its pixels within r of the edge (windows clipped by the
    // target) take the per-position path; every other pixel the fast path
    const bool edge_tile = x0 - R < 0 || x0 + TW + R > a.wt || y0 - R < 0 || y0 + TH + R > a.ht;
    const int64_t fpx = (int64_t)a.wt * a.ht;
    const uint32_t* __restrict__ cs = reinterpret_cast<const uint32_t*>(PAD ? a.cs_pad : a.cs);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t ws = (uint32_t)a.ws, hs = (uint32_t)a.hs;
    const uint32_t wsl = PAD ? 65536u : ws;  // row stride of the "linear" source index
    // checked build: a linear source index inside the exemplar (PAD: the packed x | y<<16)
    auto src_in = [&](uint32_t li) {
        return PAD ? ((li & 0xFFFFu) < ws && (li >> 16) < hs) : li < ws * hs;
    };
    (void)src_in;

    const int g = lane;                  // this thread's 4-pixel group column (pixels 4g..4g+3)
    if (fast) {
        // ---- packed -> linear source index, in place (16 bytes at a time; the unused
        //      padding words are converted too, harmlessly); with PAD the packed value is it
        if (!PAD) for (int i = threadIdx.x; i < SH * (SWP / 4); i += NT) {
            const int yy = i / (SWP / 4), c4 = i - yy * (SWP / 4);
            uint4 v = *reinterpret_cast<const uint4*>(&sc[yy][4 * c4]);
            v.x = (v.x >> 16) * ws + (v.x & 0xFFFFu);
            v.y = (v.y >> 16) * ws + (v.y & 0xFFFFu);
            v.z = (v.z >> 16) * ws + (v.z & 0xFFFFu);
            v.w = (v.w >> 16) * ws + (v.w & 0xFFFFu);
            *reinterpret_cast<uint4*>(&sc[yy][4 * c4]) = v;
        }
        if (!PAD) __syncthreads();
        if (R > 0) {
            // ---- 1. row-segment nibbles: tile columns 4g-R .. 4g+3+R of staged row yy
            for (int e = threadIdx.x; e < SH * NG; e += NT) {
                const int yy = e / NG, gg = e - yy * NG;
                uint32_t u[4 * (2 * KR + 1)];  // tile columns 4gg-4KR .. 4gg+3+4KR
#pragma unroll
                for (int k = 0; k < 2 * KR + 1; ++k) {
                    const uint4 t = *reinterpret_cast<const uint4*>(&sc[yy][4 * gg + 4 * k]);
                    u[4 * k] = t.x; u[4 * k + 1] = t.y; u[4 * k + 2] = t.z; u[4 * k + 3] = t.w;
                }
                const uint32_t* v = u + (4 * KR - R);  // v[i] = tile column 4gg - R + i
                uint32_t link = 0;  // bit i: v[i+1] continues v[i]
#pragma unroll
                for (int i = 0; i < 3 + 2 * R; ++i) link |= (uint32_t)(v[i + 1] == v[i] + 1u) << i;
                constexpr uint32_t win = (1u << (2 * R)) - 1u;
                uint32_t nib = 0;
#pragma unroll
                for (int k = 0; k < 4; ++k) nib |= (uint32_t)(((link >> k) & win) == win) << k;
                seg[yy][gg] = (uint8_t)nib;
                uint32_t nib3 = 0;
#pragma unroll
                for (int k = 0; k < 4; ++k) nib3 |= (uint32_t)(__popc(~(link >> k) & win) >= 2) << k;
                seg3[yy][gg] = (uint8_t)nib3;
#pragma unroll
                for (int k = 0; k < 4; ++k) wl[yy][4 * gg + k] = (link >> k) & win;
                if (yy + 1 < SH) {  // vertical continuity of the group's 4 columns into row yy+1
                    const uint4 d = *reinterpret_cast<const uint4*>(&sc[yy + 1][OFF + 4 * gg]);
                    const uint32_t* c = u + 4 * KR;  // this row's columns 4gg .. 4gg+3
                    vseg[yy][gg] = (uint8_t)((uint32_t)(d.x == c[0] + wsl) | ((uint32_t)(d.y == c[1] + wsl) << 1) |
                                             ((uint32_t)(d.z == c[2] + wsl) << 2) | ((uint32_t)(d.w == c[3] + wsl) << 3));
                }
            }
            __syncthreads();
        }
        // ---- 2. per pixel: unanimous window -> blit; else queue it, apart if a window row has
        //      three or more runs
        int my_n = 0, my_n3 = 0, my_ne = 0;
        uint32_t my_mask = 0, my_mask3 = 0, my_maske = 0;  // bit 4*rr + k: queued
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
            const int ry = warp + 8 * rr;
            if (y0 + ry >= a.row_end || x0 + 4 * g >= a.wt) continue;
            const uint4 c4 = *reinterpret_cast<const uint4*>(&sc[ry + R][OFF + 4 * g]);
            const uint32_t cp[4] = {c4.x, c4.y, c4.z, c4.w};
            // unanimous: every window row is one run and the 2r+1 rows continue each other
            // vertically (the centre column)
            uint32_t uni = 0xFu, cx3 = 0;
#pragma unroll
            for (int j = -R; j <= R; ++j) {
                uni &= (R > 0) ? (uint32_t)seg[ry + R + j][g] : 0xFu;
                if (j < R) uni &= (uint32_t)vseg[ry + R + j][g];
                cx3 |= seg3[ry + R + j][g];
            }
            uint32_t o[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                o[k] = 0;
                const int gx = x0 + 4 * g + k, gy = y0 + ry;
                if (edge_tile && (gx >= a.wt || gx < R || gx >= a.wt - R || gy < R || gy >= a.ht - R)) {
                    if (gx < a.wt) {  // pixels past a ragged row end are neither computed nor written
                        my_maske |= 1u << (4 * rr + k);
                        ++my_ne;
                    }
                } else if ((uni >> k) & 1u) {
                    SB_CHECK(src_in(cp[k]), "unanimous gather");
                    o[k] = __ldg(cs + cp[k]);
                } else if ((cx3 >> k) & 1u) {
                    my_mask3 |= 1u << (4 * rr + k);
                    ++my_n3;
                } else {
                    my_mask |= 1u << (4 * rr + k);
                    ++my_n;
                }
            }
            *reinterpret_cast<uint4*>(&outc[ry][4 * g]) = make_uint4(o[0], o[1], o[2], o[3]);
        }
        {
            // queue slots row by row: the warp's row-ry pixels, then its row-ry+8 pixels (the
            // counts of the two rows scan together in the 16-bit halves of one word), so the
            // lanes of a dense pass mostly read one staged row (rows 8 apart share banks)
            const uint32_t c2 = (uint32_t)__popc(my_mask & 0xFu) | ((uint32_t)__popc(my_mask >> 4) << 16);
            const uint32_t c3 = (uint32_t)__popc(my_mask3 & 0xFu) | ((uint32_t)__popc(my_mask3 >> 4) << 16);
            uint32_t incl = c2, incl3 = c3;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
                const uint32_t v3 = __shfl_up_sync(0xFFFFFFFFu, incl3, o);
                if (lane >= o) { incl += v; incl3 += v3; }
            }
            const uint32_t total = __shfl_sync(0xFFFFFFFFu, incl, 31);
            const uint32_t total3 = __shfl_sync(0xFFFFFFFFu, incl3, 31);
            const int t0 = (int)(total & 0xFFFFu), t1 = (int)(total >> 16);
            const int u0 = (int)(total3 & 0xFFFFu), u1 = (int)(total3 >> 16);
            int base = 0, base3 = 0;
            if (lane == 31) {
                if (t0 + t1) base = atomicAdd(&qn, t0 + t1);
                if (u0 + u1) base3 = atomicAdd(&qn3, u0 + u1);
            }
            base = __shfl_sync(0xFFFFFFFFu, base, 31);
            base3 = __shfl_sync(0xFFFFFFFFu, base3, 31);
            const uint32_t ex = incl - c2, ex3 = incl3 - c3;  // exclusive prefixes, both halves
            int b2[2] = {base + (int)(ex & 0xFFFFu), base + t0 + (int)(ex >> 16)};
            int b3[2] = {base3 + (int)(ex3 & 0xFFFFu), base3 + u0 + (int)(ex3 >> 16)};
            if (edge_tile && my_ne) {  // few pixels, only in frame-edge tiles: one atomic per thread
                int be = atomicAdd(&qne, my_ne);
                for (int b = 0; b < 8; ++b)
                    if (my_maske & (1u << b)) qe[be++] = (uint16_t)((warp + 8 * (b >> 2)) * TW + 4 * g + (b & 3));
            }
#pragma unroll
            for (int b = 0; b < 8; ++b) {
                const uint16_t id = (uint16_t)((warp + 8 * (b >> 2)) * TW + 4 * g + (b & 3));
                if (my_mask & (1u << b)) queue[b2[b >> 2]++] = id;
                if (my_mask3 & (1u << b)) queue[TH * TW - 1 - b3[b >> 2]++] = id;
            }
        }
        __syncthreads();
        constexpr uint32_t W = 2 * R + 1;
        // ---- 3a. two-run pixels, densely and branch-free: in each window row the link bits
        //      split the 2r+1 positions into at most two runs of positions that vote for the
        //      same source pixel; each run costs one gather weighted by its length.
        const int n = qn;
        for (int j = threadIdx.x; j < n; j += NT) {
            const int idx = queue[j];
            SB_CHECK(idx >= 0 && idx < TH * TW, "two-run queue");
            const int ry = idx / TW, x = idx - ry * TW;
            Sums<R> sum;
#pragma unroll
            for (int dy = -R; dy <= R; ++dy) {
                const int yy = ry + R + dy;
                const uint32_t bits = wl[yy][x];
                // length of run 1 = position of the first run end + 1 (W if none): with t the
                // link bits, t ^ (t + 1) has exactly c1 low bits set
                const uint32_t t = bits & ((1u << (2 * R)) - 1u);
                const uint32_t c1 = (uint32_t)__popc(t ^ (t + 1u));
                const uint32_t h2 = c1 < W ? c1 : 0u;                // head of run 2 (or any)
                const uint32_t* row = &sc[yy][OFF + x - R];
                const uint32_t shy = (uint32_t)dy * wsl;
                SB_CHECK(src_in(row[0] - shy + (uint32_t)R) && (c1 == W || src_in(row[h2] - shy - (h2 - (uint32_t)R))),
                         "two-run gathers");
                const uint32_t col1 = __ldg(cs + (row[0] - shy + (uint32_t)R));
                const uint32_t c2 = W - c1;
                const uint32_t col2 = ldg_if(cs + (row[h2] - shy - (h2 - (uint32_t)R)), c2 != 0);
                sum.add2(dy, col1, c1, col2, c2);
            }
            outc[ry][x] = finish_const<W * W>(sum);
        }
        // ---- 3b. pixels with a row of three or more runs: the general run loop
        const int n3 = qn3;
        for (int j = threadIdx.x; j < n3; j += NT) {
            const int idx = queue[TH * TW - 1 - j];
            SB_CHECK(idx >= 0 && idx < TH * TW, "run-loop queue");
            const int ry = idx / TW, x = idx - ry * TW;
            Sums<R> sum;
#pragma unroll
            for (int dy = -R; dy <= R; ++dy) {
                const int yy = ry + R + dy;
                const uint32_t bits = wl[yy][x];
                uint32_t m = ~bits & ((1u << (2 * R)) - 1u);  // bit i: a run ends at window position i
                const uint32_t* row = &sc[yy][OFF + x - R];
                const uint32_t shy = (uint32_t)dy * wsl;
                uint32_t start = 0;
                uint32_t pos = row[0] - shy + (uint32_t)R;
                while (m) {
                    const uint32_t k = __ffs(m) - 1;
                    SB_CHECK(src_in(pos), "run gather");
                    const uint32_t c = __ldg(cs + pos);
                    sum.add(dy, c, k + 1 - start);
                    start = k + 1;
                    m &= m - 1;
                    pos = row[start] - shy - (start - (uint32_t)R);
                }
                SB_CHECK(src_in(pos), "last-run gather");
                const uint32_t c = __ldg(cs + pos);
                sum.add(dy, c, W - start);
            }
            outc[ry][x] = finish_const<W * W>(sum);
        }
        // ---- 3c. frame-edge pixels of a fast tile: the general per-position path (clipped window)
        if (edge_tile) {
            const int ne = qne;
            const uint32_t lim = ((hs - 1u) << 16) | (ws - 1u);
            for (int j = threadIdx.x; j < ne; j += NT) {
                const int idx = qe[j];
                SB_CHECK(idx >= 0 && idx < TH * TW, "edge queue");
                const int ry = idx / TW, x = idx - ry * TW;
                Sums<R> sum;
                uint32_t cnt = 0;
#pragma unroll
                for (int dy = -R; dy <= R; ++dy) {
#pragma unroll
                    for (int dx = -R; dx <= R; ++dx) {
                        const uint32_t li = sc[ry + R + dy][OFF + x + dx] - (uint32_t)dx - (uint32_t)dy * wsl;
                        bool in;
                        if (PAD) {  // packed: kOutside fails the in-source test (sources of a fast tile are in)
                            uint32_t mn;
                            asm("min.u16x2 %0, %1, %2;" : "=r"(mn) : "r"(li), "r"(lim));
                            in = mn == li;
                        } else {  // linear indices (the conversion pass ran, kOutside too): clip by position
                            const int qx = x0 + x + dx, qy = y0 + ry + dy;
                            in = qx >= 0 && qx < a.wt && qy >= 0 && qy < a.ht;
                        }
                        SB_CHECK(!in || src_in(li), "edge gather");
                        const uint32_t c = ldg_if(cs + (in ? li : 0u), in);
                        if (in) { sum.add(dy, c, 1u); ++cnt; }
                    }
                }
                outc[ry][x] = finish(sum, cnt);
            }
        }
    } else {
        // ---- border tile: every pixel takes the general path
        const int ntile = TH * TW;
        const uint32_t lim = ((hs - 1u) << 16) | (ws - 1u);
        for (int idx = threadIdx.x; idx < ntile; idx += NT) {
            const int ry = idx / TW, x = idx - ry * TW;
            const int gx = x0 + x;
            if (y0 + ry >= a.row_end || gx >= a.wt) continue;
            Sums<R> sum;
            uint32_t cnt = 0;
#pragma unroll
            for (int dy = -R; dy <= R; ++dy) {
                const uint32_t sh = (uint32_t)dy << 16;
#pragma unroll
                for (int dx = -R; dx <= R; ++dx) {
                    const uint32_t w = sc[ry + R + dy][OFF + x + dx];
                    const uint32_t pos = w - (uint32_t)dx - sh;
                    // inside the source (and the target: see kOutside): one packed 16-bit min
                    uint32_t mn;
                    asm("min.u16x2 %0, %1, %2;" : "=r"(mn) : "r"(pos), "r"(lim));
                    const bool in = mn == pos;
                    const uint32_t c = __ldg(cs + (in ? (PAD ? pos : (pos >> 16) * ws + (pos & 0xFFFFu)) : 0u));
                    if (in) { sum.add(dy, c, 1u); ++cnt; }
                }
            }
            outc[ry][x] = finish(sum, cnt);  // cnt >= 1: q = p votes for src(p)
        }
    }
    __syncthreads();
    // ---- store the tile
    const bool vec = (a.wt & 3) == 0;
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
        const int ry = warp + 8 * rr;
        const int py = y0 + ry;
        const int gx0 = x0 + 4 * g;
        if (py >= a.row_end || gx0 >= a.wt) continue;
        const int64_t off = fpx * frame + (int64_t)py * a.wt + gx0;
        const uint4 o = *reinterpret_cast<const uint4*>(&outc[ry][4 * g]);
        if (vec) {
            st_cs_u4(a.ct + 4 * off, o);
        } else {
            const uint32_t ov[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (gx0 + k < a.wt) st_cs_u32(a.ct + 4 * (off + k), ov[k]);
        }
    }
}


// The grid-per-tile kernel: coordinates staged with 16-byte loads (any width).
template <int R, bool PAD>
__global__ void __launch_bounds__(NT, (R <= 3 ? 6 : (R == 4 ? 5 : 4))) vote_kernel(const VoteArgs a) {
    constexpr int SW = VoteGeom<R>::SW, SH = VoteGeom<R>::SH, OFF = VoteGeom<R>::OFF, SWP = VoteGeom<R>::SWP;
    __shared__ __align__(16) uint32_t sc[SH][SWP];
    __shared__ VoteShared<R> S;
    const int tiles_x = (a.wt + TW - 1) / TW;
    const int x0 = (blockIdx.x % tiles_x) * TW;
    const int y0 = a.row_begin + (blockIdx.x / tiles_x) * TH;
    const int64_t fpx = (int64_t)a.wt * a.ht;
    const uint32_t* __restrict__ cf = a.coords + fpx * blockIdx.y;
    const uint32_t ws = (uint32_t)a.ws, hs = (uint32_t)a.hs;
    if (threadIdx.x == 0) S.qn = S.qn3 = S.qne = 0;
    // ---- stage coords (tile + halo), outside the target -> kOutside; test the fast-tile margin
    bool fast_mine = true;
    auto stage = [&](int yy, int x, uint32_t v, bool in) {  // x: tile column (-R .. TW-1+R)
        if (in) {
            const uint32_t sx = v & 0xFFFFu, sy = v >> 16;
            fast_mine &= (sx >= (uint32_t)R) & (sx + (uint32_t)R < ws) & (sy >= (uint32_t)R) & (sy + (uint32_t)R < hs);
        } else {
            v = kOutside;  // outside the target: only the frame-edge pixels' windows see it
        }
        sc[yy][OFF + x] = v;
    };
    // the fast-tile margin as packed 16-bit bounds: (R, R) .. (ws-1-R, hs-1-R)
    // (an exemplar no wider or taller than 2R has no such position)
    const uint32_t mlo = ((uint32_t)R << 16) | (uint32_t)R;
    const bool room = ws > 2u * R && hs > 2u * R;
    const uint32_t mhi = room ? ((hs - 1u - (uint32_t)R) << 16) | (ws - 1u - (uint32_t)R) : 0u;
    fast_mine &= room;
    if ((a.wt & 3) == 0) {
        // centre columns: one 16-byte load per 4 pixels
        for (int i = threadIdx.x; i < SH * NG; i += NT) {
            const int yy = i / NG, gg = i - yy * NG;
            const int gx = x0 + 4 * gg, gy = y0 - R + yy;
            const bool rowin = gy >= 0 && gy < a.ht;
            if (rowin && gx + 3 < a.wt) {
                const uint4 v = *reinterpret_cast<const uint4*>(cf + (int64_t)gy * a.wt + gx);
                const uint32_t vv[4] = {v.x, v.y, v.z, v.w};
                bool ok = true;
#pragma unroll
                for (int k = 0; k < 4; ++k) {  // R <= x < ws - R and R <= y < hs - R, both fields at once
                    uint32_t lo, hi;
                    asm("max.u16x2 %0, %1, %2;" : "=r"(lo) : "r"(vv[k]), "r"(mlo));
                    asm("min.u16x2 %0, %1, %2;" : "=r"(hi) : "r"(vv[k]), "r"(mhi));
                    ok &= (lo == vv[k]) & (hi == vv[k]);
                }
                fast_mine &= ok;
                *reinterpret_cast<uint4*>(&sc[yy][OFF + 4 * gg]) = v;
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const bool in = rowin && gx + k < a.wt;
                    stage(yy, 4 * gg + k, in ? __ldg(cf + (int64_t)gy * a.wt + gx + k) : 0u, in);
                }
            }
        }
        // halo columns
        if constexpr (R > 0) for (int i = threadIdx.x; i < SH * 2 * R; i += NT) {
            const int yy = i / (2 * R), k = i - yy * (2 * R);
            const int x = k < R ? k - R : TW + (k - R);
            const int gx = x0 + x, gy = y0 - R + yy;
            const bool in = gx >= 0 && gx < a.wt && gy >= 0 && gy < a.ht;
            stage(yy, x, in ? __ldg(cf + (int64_t)gy * a.wt + gx) : 0u, in);
        }
    } else {
        for (int i = threadIdx.x; i < SW * SH; i += NT) {
            const int yy = i / SW, xx = i - yy * SW;
            const int gx = x0 - R + xx, gy = y0 - R + yy;
            const bool in = gx >= 0 && gx < a.wt && gy >= 0 && gy < a.ht;
            stage(yy, xx - R, in ? __ldg(cf + (int64_t)gy * a.wt + gx) : 0u, in);
        }
    }
    const bool fast = __syncthreads_and(fast_mine) != 0;

    vote_tile<R, PAD>(a, sc, S, x0, y0, blockIdx.y, fast);
}


// ---- TMA-fed persistent kernel (r <= 4; rows of 16-byte multiple strides, i.e. wt % 4 == 0) ----
// One CTA per resident slot loops over tiles (frame-major); the staged coordinates of tile k+1
// are fetched by the Tensor Memory Accelerator (one 3-D box [frame][SH rows][SWP columns],
// zero-filled outside the tensor) into the other of two shared buffers while tile k is voted,
// so the HBM latency of the coordinates no longer stalls the CTA at its staging barrier.
// Completion: one mbarrier per buffer (expect_tx = box bytes), waited with parity.
namespace {
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
        "@!P bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// Thread 0: arm the buffer's barrier with the box bytes and start the 3-D box load.
__device__ __forceinline__ void tma_box3(void* dst, const CUtensorMap* tm, int c0, int c1, int c2, uint64_t* bar,
                                         uint32_t bytes) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // prior generic accesses of dst first
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}
}  // namespace

template <int R, bool PAD>
__global__ void __launch_bounds__(NT, (R <= 3 ? 6 : 2))
    vote_tma_kernel(const VoteArgs a, const __grid_constant__ CUtensorMap tm, int tiles_x, int tiles_per_frame,
                    int n_tiles) {
    constexpr int SH = VoteGeom<R>::SH, OFF = VoteGeom<R>::OFF, SWP = VoteGeom<R>::SWP;
    constexpr uint32_t kBox = SH * SWP * 4;
    __shared__ __align__(128) uint32_t sc0[SH][SWP];
    __shared__ __align__(128) uint32_t sc1[SH][SWP];
    __shared__ __align__(8) uint64_t mbar[2];
    __shared__ VoteShared<R> S;
    const int tid = threadIdx.x;
    const uint32_t ws = (uint32_t)a.ws, hs = (uint32_t)a.hs;
    auto origin = [&](int t, int& x0, int& y0, int& f) {
        f = t / tiles_per_frame;
        const int r = t - f * tiles_per_frame;
        x0 = (r % tiles_x) * TW;
        y0 = a.row_begin + (r / tiles_x) * TH;
    };
    auto fetch = [&](int t, void* dst, uint64_t* bar) {
        int x0, y0, f;
        origin(t, x0, y0, f);
        tma_box3(dst, &tm, x0 - OFF, y0 - R, f, bar, kBox);
    };
    if (tid == 0) {
        mbar_init(&mbar[0], 1);
        mbar_init(&mbar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if ((int)blockIdx.x < n_tiles) fetch(blockIdx.x, sc0, &mbar[0]);
    }
    __syncthreads();
    uint32_t parity = 0;  // bit b: phase of buffer b
    int k = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++k) {
        const int b = k & 1;
        uint32_t(*sc)[SWP] = b ? sc1 : sc0;
        if (tid == 0) {
            const int tn = t + gridDim.x;  // the next tile into the other buffer (free since the last barrier)
            if (tn < n_tiles) fetch(tn, b ? (void*)sc0 : (void*)sc1, &mbar[b ^ 1]);
            S.qn = S.qn3 = S.qne = 0;
        }
        int x0, y0, f;
        origin(t, x0, y0, f);
        mbar_wait(&mbar[b], (parity >> b) & 1u);
        parity ^= 1u << b;
        // positions outside the target were zero-filled: mark them (only tiles at the frame edge);
        // the fast-tile margin over every staged word (the extra alignment columns included)
        bool fast_mine = true;
        const bool edge = x0 - R < 0 || x0 + TW + R > a.wt || y0 - R < 0 || y0 + TH + R > a.ht;
        for (int i = tid; i < SH * (SWP / 4); i += NT) {
            const int yy = i / (SWP / 4), c4 = i - yy * (SWP / 4);
            uint4 v = *reinterpret_cast<const uint4*>(&sc[yy][4 * c4]);
            uint32_t vv[4] = {v.x, v.y, v.z, v.w};
            uint32_t m = 0;
            bool out = false;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                bool in = true;
                if (edge) {
                    const int gx = x0 - OFF + 4 * c4 + j, gy = y0 - R + yy;
                    if (gx < 0 || gx >= a.wt || gy < 0 || gy >= a.ht) {
                        vv[j] = kOutside;
                        out = true;
                        in = false;
                    }
                }
                const uint32_t sx = vv[j] & 0xFFFFu, sy = vv[j] >> 16;
                m |= (uint32_t)(in & ((sx < (uint32_t)R) | (sx + (uint32_t)R >= ws) | (sy < (uint32_t)R) |
                                      (sy + (uint32_t)R >= hs)));
            }
            fast_mine &= (m == 0);
            if (out) *reinterpret_cast<uint4*>(&sc[yy][4 * c4]) = make_uint4(vv[0], vv[1], vv[2], vv[3]);
        }
        const bool fast = __syncthreads_and(fast_mine) != 0;
        vote_tile<R, PAD>(a, sc, S, x0, y0, f, fast);
        __syncthreads();  // sc and S are free for the tiles to come
    }
}

// Shared-memory carve-out preference of the grid-per-tile vote: the driver's default (-1) since
// round 2 (a 60 % carve-out was ~4 % faster for round 1's smaller shared footprint and is ~2.5 %
// slower for the current one).  SB_VOTE_CARVEOUT (percent) overrides.
static int vote_carveout() {
    static const int pct = [] {
        const char* e = getenv("SB_VOTE_CARVEOUT");
        return e ? atoi(e) : -1;
    }();
    return pct;
}

template <int R>
static void launch_r(const VoteArgs& a, dim3 grid, cudaStream_t st) {
    auto kern = a.cs_pad ? vote_kernel<R, true> : vote_kernel<R, false>;
    ensure_carveout(reinterpret_cast<const void*>(kern), vote_carveout());  // a preference: failure is harmless
    kern<<<grid, NT, 0, st>>>(a);
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link needed).
static PFN_cuTensorMapEncodeTiled encode_fn() {
    static PFN_cuTensorMapEncodeTiled fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled>(p);
    }();
    return fn;
}

// Resident CTAs per SM of a kernel (cached per device and kernel).
static int resident_ctas(const void* kern, int threads) {
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, int> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    auto key = std::make_pair(dev, kern);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, threads, 0) != cudaSuccess || n < 1) n = 1;
    cache[key] = n;
    return n;
}

// The TMA-fed persistent launch; false when it does not apply (ragged rows, no driver entry
// point, tensor-map encoding refused), in which case the caller uses the grid-per-tile kernel.
template <int R>
static bool launch_tma_r(const VoteArgs& a, int n_frames, cudaStream_t st) {
    if (a.wt % 4 != 0 || !encode_fn()) return false;
    CUtensorMap tm;
    const cuuint64_t dims[3] = {(cuuint64_t)a.wt, (cuuint64_t)a.ht, (cuuint64_t)n_frames};
    const cuuint64_t strides[2] = {(cuuint64_t)a.wt * 4, (cuuint64_t)a.wt * a.ht * 4};
    const cuuint32_t box[3] = {(cuuint32_t)VoteGeom<R>::SWP, (cuuint32_t)VoteGeom<R>::SH, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    if (encode_fn()(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, const_cast<uint32_t*>(a.coords), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;
    const int tiles_x = (a.wt + TW - 1) / TW;
    const int tiles_per_frame = tiles_x * ((a.row_end - a.row_begin + TH - 1) / TH);
    const int n_tiles = tiles_per_frame * n_frames;
    auto kern = a.cs_pad ? vote_tma_kernel<R, true> : vote_tma_kernel<R, false>;
    // two staging buffers: more shared memory per CTA than the grid-per-tile kernel, so its
    // carve-out would cost residency; SB_VOTE_TMA_CARVEOUT (percent) overrides the default
    static const int carve = [] {
        const char* e = getenv("SB_VOTE_TMA_CARVEOUT");
        return e ? atoi(e) : -1;
    }();
    ensure_carveout(reinterpret_cast<const void*>(kern), carve);
    const int grid = std::min(n_tiles, sm_count() * resident_ctas(reinterpret_cast<const void*>(kern), NT));
    kern<<<grid, NT, 0, st>>>(a, tm, tiles_x, tiles_per_frame, n_tiles);
    return true;
}

cudaError_t launch_vote(const VoteArgs& a, int n_frames, cudaStream_t st, int* launches) {
    // a side beyond 32767: the per-pixel vote of vote_wide.cu (32-bit sums, signed coordinates);
    // everything else runs on the packed-arithmetic kernels below
    if (a.r > 8 || a.wt > kPackedMaxDim || a.ht > kPackedMaxDim || a.ws > kPackedMaxDim || a.hs > kPackedMaxDim)
        return launch_vote_wide(a, n_frames, st, launches);
    // A/B alternatives for r = 1, 2 (measured slower): SB_VOTE=peel the peel vote
    // of vote_peel.cu, SB_VOTE=hist the offset-histogram vote of vote_hist.cu.
    static const int which = [] {
        const char* e = getenv("SB_VOTE");
        if (e && strcmp(e, "peel") == 0) return 1;
        if (e && strcmp(e, "hist") == 0) return 2;
        return 0;
    }();
    if ((a.r == 1 || a.r == 2) && which == 1) return launch_vote_peel(a, n_frames, st, launches);
    if ((a.r == 1 || a.r == 2) && which == 2) return launch_vote_hist(a, n_frames, st, launches);
    // SB_VOTE_TMA=1: the TMA-fed persistent kernel where it applies (A/B; measured slower,
    // DESIGN.md 11)
    static const bool tma = [] {
        const char* e = getenv("SB_VOTE_TMA");
        return e && strcmp(e, "1") == 0;
    }();
    if (tma && n_frames > 0) {
        bool done = false;
        switch (a.r) {
            case 0: done = launch_tma_r<0>(a, n_frames, st); break;
            case 1: done = launch_tma_r<1>(a, n_frames, st); break;
            case 2: done = launch_tma_r<2>(a, n_frames, st); break;
            case 3: done = launch_tma_r<3>(a, n_frames, st); break;
            case 4: done = launch_tma_r<4>(a, n_frames, st); break;
            case 5: case 6: case 7: case 8: break;  // two staging buffers exceed 48 KB of static shared memory
            default: return cudaErrorInvalidValue;
        }
        if (done) {
            *launches += 1;
            return cudaPeekAtLastError();
        }
    }
    const int tiles = ((a.wt + TW - 1) / TW) * ((a.row_end - a.row_begin + TH - 1) / TH);
    dim3 grid((unsigned)tiles, (unsigned)n_frames);
    switch (a.r) {
        case 0: launch_r<0>(a, grid, st); break;
        case 1: launch_r<1>(a, grid, st); break;
        case 2: launch_r<2>(a, grid, st); break;
        case 3: launch_r<3>(a, grid, st); break;
        case 4: launch_r<4>(a, grid, st); break;
        case 5: launch_r<5>(a, grid, st); break;
        case 6: launch_r<6>(a, grid, st); break;
        case 7: launch_r<7>(a, grid, st); break;
        case 8: launch_r<8>(a, grid, st); break;
        default: return cudaErrorInvalidValue;
    }
    *launches += 1;
    return cudaPeekAtLastError();
}

}  // namespace sb
