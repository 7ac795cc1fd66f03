// vote_hist.cu -- the voting step of PAPER.md:412-421 for r = 1, 2 by per-block offset
// histograms (sm_100a).
//
// C_T[p] = average over the target pixels q of the (2r+1)^2 window around p (clipped to the
// target) of C_S[src(q) + (p - q)], skipping positions outside the source; per channel
// floor((sum + floor(n/2)) / n) (reading R13; fallback pixels vote like any other, R14).
//
// Regrouped by OFFSET o(q) = src(q) - q: every window position with the same offset o votes
// for the same source pixel o + p, so
//     sum = sum over the distinct offsets o in the window of N_o(p) * C_S[o + p],
// with N_o(p) the number of window positions of offset o -- one gather per distinct offset
// (1.84 per pixel at 4K, against 25 positions).  Offsets are piecewise constant (the chunks
// of PAPER.md:259-263), so a 4x4 output block sees few of them in the (4+2r)^2 region its
// windows cover (2.6 on average at 4K, more than 6 in 2 %).
//
// One CTA = 128 x 32 output pixels (8 warps); the offsets of the tile plus an r halo are
// staged in shared memory (packed x | y<<16 arithmetic, see below).  A thread owns a 4x4
// block:
//   1. it labels the offsets of its region row by row with a private dictionary (at most NL
//      entries): a position equal to its left or upper neighbour inherits that label; the
//      others (new runs) are looked up / inserted;
//   2. the labels become one-hot counters packed in one word (FB-bit fields, NL per word:
//      5 bits x 6 for r = 2, 4 bits x 8 for r = 1 -- a count never exceeds (2r+1)^2), so the
//      window histograms of all 16 pixels are separable box sums of words: a horizontal
//      (2r+1)-sum per region row (prefix sums), then vertical accumulation into the 16 pixels;
//   3. per pixel, one gather per non-zero field, weighted by its count (SWAR sums); a
//      source position outside the exemplar drops that offset's count (exactly the positions
//      the oracle skips), and positions outside the target carry no label (clipping).
// Blocks whose region holds more than NL distinct offsets are queued and voted per position
// afterwards (exact, ~2 % of the blocks).
//
// Packed arithmetic: coordinates are x | y<<16 with W, H <= 32767 (R23).  The offset
// o = src(q) - q (mod 2^32) is a bijection of (dx, dy) in (-32767, 32767)^2; o + p equals
// src(q) + (p - q) and its fields fall outside [0, ws) x [0, hs) (a borrow makes them
// >= 0xFFF0) exactly when the source position does.  The marker kNone (low half 0x8000) is
// never a valid offset, whose low half is dx mod 2^16 with |dx| <= 32766.
#include <type_traits>

#include "sb_kernels.cuh"

namespace sb {

namespace {
constexpr uint32_t kNone = 0x80008000u;

__device__ __forceinline__ uint32_t ldg_pred(const uint32_t* p, bool pred) {
    uint32_t v = 0;
    asm volatile(
        "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q ld.global.nc.u32 %0, [%1];\n\t}"
        : "+r"(v)
        : "l"(p), "r"((uint32_t)pred));
    return v;
}

// floor((sum + floor(n/2)) / n) per channel, m = ceil(2^32 / n) (exact for numerators < 2^17,
// sums <= 289*255 + 144); n = 1 (ceil(2^32/1) does not fit) is the sum itself; n = 0 (a pixel
// outside the target, never stored) gives 0.
__device__ __forceinline__ uint32_t finish_m(uint32_t lo, uint32_t hi, uint32_t n, uint32_t m) {
    if (n <= 1) return n ? (lo & 0x00FF00FFu) | ((hi & 0x00FF00FFu) << 8) : 0u;
    const uint32_t half = n >> 1;
    const uint32_t c0 = __umulhi((lo & 0xFFFFu) + half, m);
    const uint32_t c1 = __umulhi((hi & 0xFFFFu) + half, m);
    const uint32_t c2 = __umulhi((lo >> 16) + half, m);
    const uint32_t c3 = __umulhi((hi >> 16) + half, m);
    return c0 | (c1 << 8) | (c2 << 16) | (c3 << 24);
}
}  // namespace

template <int R>
struct HistCfg {
    static constexpr int FB = (2 * R + 1) * (2 * R + 1) < 16 ? 4 : 5;  // bits per count field
    static constexpr int NL = 32 / FB;                                  // labels per word
    static constexpr uint32_t FMASK = (1u << FB) - 1u;
    static constexpr uint32_t FULL = (2 * R + 1) * (2 * R + 1);         // positions per window
};

// 1 << s for s < 32, 0 for s >= 32 (PTX shl clamps the shift; an unlabelled position has s = 0xFF)
__device__ __forceinline__ uint32_t shl1(uint32_t s) {
    uint32_t v;
    asm("shl.b32 %0, 1, %1;" : "=r"(v) : "r"(s));
    return v;
}

// PAD: C_S from the strided exemplar copy (rows of 2^16 pixels): a packed coordinate is its index.
constexpr int kHistWarps = 4;  // CTA = 128 x 16 pixels

template <int R, bool PAD>
__global__ void __launch_bounds__(32 * kHistWarps, 6) vote_hist_kernel(const VoteArgs a) {
    using HC = HistCfg<R>;
    constexpr int NW = kHistWarps, NT = 32 * NW;
    constexpr int TW = 128, TH = 4 * NW, TP = TW * TH;
    constexpr int RW = 4 + 2 * R;                       // region side of a block's windows
    constexpr int SWP = ((TW + 2 * R + 3) / 4) * 4;     // staged row: tile column x at index x + R
    constexpr int SH = TH + 2 * R;
    constexpr int FB = HC::FB, NL = HC::NL;
    constexpr uint32_t FULL = HC::FULL;
    static_assert(RW * NT * 8 <= TP * 4, "the label codes live in the output tile");
    __shared__ __align__(16) uint32_t so[SH][SWP];      // offsets o(q) of the staged positions
    __shared__ __align__(16) uint32_t outc[TH][TW];     // label codes, then histograms / colours
    __shared__ uint32_t sdict[FB * (NL - 1) + 1][NT];   // per-thread dictionaries: label k in row FB k
    __shared__ uint16_t queue[TP];                      // mixed windows from the front, overflow from the back
    __shared__ uint32_t mtab[FULL + 1];                 // ceil(2^32 / n)
    __shared__ int qn, qo;

    const int tiles_x = (a.wt + TW - 1) / TW;
    const int x0 = (blockIdx.x % tiles_x) * TW;
    const int y0 = a.row_begin + (blockIdx.x / tiles_x) * TH;
    const int64_t fpx = (int64_t)a.wt * a.ht;
    const uint32_t* __restrict__ cf = a.coords + fpx * blockIdx.y;
    const uint32_t* __restrict__ cs = reinterpret_cast<const uint32_t*>(PAD ? a.cs_pad : a.cs);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t ws = (uint32_t)a.ws, hs = (uint32_t)a.hs;
    auto src_ok = [&](uint32_t src) { return ((src & 0xFFFFu) < ws) & ((src >> 16) < hs); };
    auto src_idx = [&](uint32_t src) { return PAD ? src : (src >> 16) * ws + (src & 0xFFFFu); };

    if (tid == 0) qn = qo = 0;
    // fast tile: every staged position inside the target with its source >= r from the source
    // border -- then every window position counts and every source o + p is inside the source
    bool fast_mine = true;
    auto margin = [&](uint32_t c) {
        const uint32_t sx = c & 0xFFFFu, sy = c >> 16;
        return (sx >= (uint32_t)R) & (sx + (uint32_t)R < ws) & (sy >= (uint32_t)R) & (sy + (uint32_t)R < hs);
    };
    if (tid >= 2 && tid <= (int)FULL) mtab[tid] = 0xFFFFFFFFu / (uint32_t)tid + 1u;
    // ---- stage o(q) = src(q) - q for the tile + r halo; kNone outside the target
    for (int i = tid; i < SH * (TW / 4); i += NT) {
        const int yy = i / (TW / 4), g = i - yy * (TW / 4);
        const int gy = y0 - R + yy, gx = x0 + 4 * g;
        const bool rowin = gy >= 0 && gy < a.ht;
        const uint32_t pb = (uint32_t)gx | ((uint32_t)gy << 16);
        uint32_t o[4];
        if (rowin && gx + 3 < a.wt && (a.wt & 3) == 0) {
            const uint4 v = *reinterpret_cast<const uint4*>(cf + (int64_t)gy * a.wt + gx);
            fast_mine &= margin(v.x) & margin(v.y) & margin(v.z) & margin(v.w);
            o[0] = v.x - pb; o[1] = v.y - pb - 1u; o[2] = v.z - pb - 2u; o[3] = v.w - pb - 3u;
        } else {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const bool in = rowin && gx + k < a.wt;
                const uint32_t c = in ? __ldg(cf + (int64_t)gy * a.wt + gx + k) : 0u;
                fast_mine &= in && margin(c);
                o[k] = in ? c - pb - (uint32_t)k : kNone;
            }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) so[yy][R + 4 * g + k] = o[k];
    }
    for (int i = tid; i < SH * 2 * R; i += NT) {
        const int yy = i / (2 * R), k = i - yy * (2 * R);
        const int x = k < R ? k - R : TW + (k - R);     // tile column
        const int gx = x0 + x, gy = y0 - R + yy;
        const bool in = gx >= 0 && gx < a.wt && gy >= 0 && gy < a.ht;
        const uint32_t c = in ? __ldg(cf + (int64_t)gy * a.wt + gx) : 0u;
        fast_mine &= in && margin(c);
        so[yy][R + x] = in ? c - ((uint32_t)gx | ((uint32_t)gy << 16)) : kNone;
    }
    const bool fast = __syncthreads_and(fast_mine) != 0;

    const int bx = 4 * lane, by = 4 * warp;  // this thread's 4x4 block (tile coordinates)
    auto load_row = [&](int ry, uint32_t v[RW]) {  // region row ry: tile columns bx-R .. bx+3+R
        const uint32_t* row = &so[by + ry][bx];
        const uint4 t0 = *reinterpret_cast<const uint4*>(row);
        v[0] = t0.x; v[1] = t0.y; v[2] = t0.z; v[3] = t0.w;
        if constexpr (RW == 8) {
            const uint4 t1 = *reinterpret_cast<const uint4*>(row + 4);
            v[4] = t1.x; v[5] = t1.y; v[6] = t1.z; v[7] = t1.w;
        } else {
            const uint2 t1 = *reinterpret_cast<const uint2*>(row + 4);
            v[4] = t1.x; v[5] = t1.y;
        }
    };
    // ---- 1a. positions that start a new run: equal to neither the left nor the upper neighbour
    uint64_t fresh_pos = 0;  // bit 8 ry + i
    {
        uint32_t up[RW];
#pragma unroll
        for (int ry = 0; ry < RW; ++ry) {
            uint32_t v[RW];
            load_row(ry, v);
#pragma unroll
            for (int i = 0; i < RW; ++i) {
                const bool leq = i > 0 && v[i] == v[i > 0 ? i - 1 : 0];
                const bool ueq = ry > 0 && v[i] == up[i];
                if (!leq && !ueq) fresh_pos |= 1ull << (8 * ry + i);
            }
#pragma unroll
            for (int i = 0; i < RW; ++i) up[i] = v[i];
        }
    }
    // ---- 1b. their labels: dictionary look-up / insertion in registers (unused entries hold
    //      kNone, which never equals a valid offset); code byte = FB * label, 0xFF = none
    uint8_t* const codes = reinterpret_cast<uint8_t*>(&outc[0][0]);  // [RW][NT][8]
    uint32_t dict[NL];
#pragma unroll
    for (int j = 0; j < NL; ++j) dict[j] = kNone;
    int nd = 0;
    bool ovf = false;
    while (fresh_pos) {
        const int pos = __ffsll((long long)fresh_pos) - 1;
        fresh_pos &= fresh_pos - 1;
        const int ry = pos >> 3, i = pos & 7;
        const uint32_t val = so[by + ry][bx + i];
        uint32_t code = 0xFFu;
        if (val != kNone) {
            uint32_t k = NL;
#pragma unroll
            for (int j = 0; j < NL; ++j) k = dict[j] == val ? (uint32_t)j : k;
            if (k == (uint32_t)NL) {
                if (nd < NL) {
#pragma unroll
                    for (int j = 0; j < NL; ++j) dict[j] = j == nd ? val : dict[j];
                    k = (uint32_t)nd++;
                } else {
                    ovf = true;
                    k = 0xFFu / FB;
                }
            }
            code = (uint32_t)FB * k;
        }
        codes[(ry * NT + tid) * 8 + i] = (uint8_t)code;
    }
#pragma unroll
    for (int j = 0; j < NL; ++j) sdict[FB * j][tid] = dict[j];
    // ---- 2. one-hot counter words per position (inherited along runs, fresh at run starts);
    //      separable box sums: horizontal (2r+1)-sums per region row, vertical accumulation
    uint32_t acc[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] = 0;
    {
        uint32_t upe[RW];
#pragma unroll
        for (int ry = 0; ry < RW; ++ry) {
            uint32_t v[RW], up[RW], e[RW];
            load_row(ry, v);
            if (ry > 0) load_row(ry - 1, up);  // reloaded: fewer live registers
            const uint2 cd = *reinterpret_cast<const uint2*>(codes + (ry * NT + tid) * 8);
#pragma unroll
            for (int i = 0; i < RW; ++i) {
                const uint32_t code = ((i < 4 ? cd.x : cd.y) >> (8 * (i & 3))) & 0xFFu;
                const bool leq = i > 0 && v[i] == v[i > 0 ? i - 1 : 0];
                const bool ueq = ry > 0 && v[i] == up[i];
                e[i] = leq ? e[i > 0 ? i - 1 : 0] : (ueq ? upe[i] : shl1(code));
            }
            uint32_t h[4];
            {
                uint32_t P[RW];
                P[0] = e[0];
#pragma unroll
                for (int i = 1; i < RW; ++i) P[i] = P[i - 1] + e[i];
                h[0] = P[2 * R];
#pragma unroll
                for (int c = 1; c < 4; ++c) h[c] = P[c + 2 * R] - P[c - 1];
            }
            // region row ry lies in the windows of block rows ry-2r .. ry
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                if (r <= ry && ry <= r + 2 * R) {
#pragma unroll
                    for (int c = 0; c < 4; ++c) acc[r][c] += h[c];
                }
            }
#pragma unroll
            for (int i = 0; i < RW; ++i) upe[i] = e[i];
        }
    }
    __syncthreads();  // every thread's codes are consumed: outc becomes the output tile

    // ---- 3a. unanimous windows (one offset, all (2r+1)^2 positions): C_T[p] = C_S[src(p)], the
    //      chunk interior where voting equals the blit; the others are
    //      queued with their histogram in their output slot (blocks with more than NL offsets
    //      go to the back of the queue)
    {
        uint32_t mixed = 0;  // bit 4 r + c
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            uint32_t col[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const uint32_t H = acc[r][c];
                // the lowest non-zero field holds all FULL positions and no other field is set
                const uint32_t b0 = (uint32_t)(__ffs(H) - 1) & 31u;
                const uint32_t b = FB == 4 ? (b0 & ~3u) : ((b0 * 13u) >> 6) * 5u;  // its first bit
                const bool uni = !ovf && (H >> b) == FULL;
                const uint32_t p = (uint32_t)(x0 + bx + c) | ((uint32_t)(y0 + by + r) << 16);
                col[c] = ldg_pred(cs + src_idx(so[by + r + R][bx + c + R] + p), uni);
                mixed |= (uint32_t)!uni << (4 * r + c);
            }
#pragma unroll
            for (int c = 0; c < 4; ++c) outc[by + r][bx + c] = ((mixed >> (4 * r + c)) & 1u) ? acc[r][c] : col[c];
        }
        const int nm = ovf ? 0 : __popc(mixed), no = ovf ? 16 : 0;
        int im = nm, io = no;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int vm = __shfl_up_sync(0xFFFFFFFFu, im, o), vo = __shfl_up_sync(0xFFFFFFFFu, io, o);
            if (lane >= o) { im += vm; io += vo; }
        }
        int bm = 0, bo = 0;
        if (lane == 31) {
            if (im) bm = atomicAdd(&qn, im);
            if (io) bo = atomicAdd(&qo, io);
        }
        bm = __shfl_sync(0xFFFFFFFFu, bm, 31) + im - nm;
        bo = __shfl_sync(0xFFFFFFFFu, bo, 31) + io - no;
        if (ovf) {
            for (int k = 0; k < 16; ++k) queue[TP - 1 - bo - k] = (uint16_t)((by + (k >> 2)) * TW + bx + (k & 3));
        } else {
#pragma unroll
            for (int k = 0; k < 16; ++k)
                if ((mixed >> k) & 1u) queue[bm++] = (uint16_t)((by + (k >> 2)) * TW + bx + (k & 3));
        }
    }
    __syncthreads();
    // ---- 3b. mixed windows, one pixel per thread: one gather per non-zero counter field,
    //      weighted by its count (the first two together, further ones in a loop)
    const int nmix = qn;
    auto mixed_pass = [&](auto fast_tag) {
        constexpr bool F = decltype(fast_tag)::value;
        for (int j = tid; j < nmix; j += NT) {
            const int idx = queue[j];
            const int ry = idx / TW, x = idx - ry * TW;
            const uint32_t H = outc[ry][x];
            const uint32_t* __restrict__ dcol = &sdict[0][(ry >> 2) * 32 + (x >> 2)];  // the owner's dictionary
            const uint32_t p = (uint32_t)(x0 + x) | ((uint32_t)(y0 + ry) << 16);
            auto field_src = [&](uint32_t b) { return dcol[b * NT] + p; };  // b = FB k: label k's offset, plus p
            uint32_t nz = H;
#pragma unroll
            for (int s = 1; s < FB; ++s) nz |= H >> s;
            nz &= FB == 4 ? 0x11111111u : 0x02108421u;
            const uint32_t b1 = (uint32_t)(__ffs(nz) - 1) & 31u;
            uint32_t rest = nz & (nz - 1);
            const uint32_t b2 = (uint32_t)(__ffs(rest) - 1) & 31u;
            const bool two = rest != 0;
            rest &= rest - 1;
            const uint32_t s1 = field_src(b1), s2 = field_src(b2);
            const bool ok1 = F ? true : (nz != 0) & src_ok(s1), ok2 = two & (F ? true : src_ok(s2));
            const uint32_t col1 = ldg_pred(cs + src_idx(s1), ok1), col2 = ldg_pred(cs + src_idx(s2), ok2);
            const uint32_t c1 = ok1 ? (H >> b1) & HC::FMASK : 0u, c2 = ok2 ? (H >> b2) & HC::FMASK : 0u;
            uint32_t lo = (col1 & 0x00FF00FFu) * c1 + (col2 & 0x00FF00FFu) * c2;
            uint32_t hi = __byte_perm(col1, 0u, 0x7371) * c1 + __byte_perm(col2, 0u, 0x7371) * c2;
            uint32_t n = c1 + c2;
            while (rest) {
                const uint32_t b = __ffs(rest) - 1;
                rest &= rest - 1;
                const uint32_t src = field_src(b);
                const bool ok = F ? true : src_ok(src);
                const uint32_t col = ldg_pred(cs + src_idx(src), ok);
                const uint32_t cnt = ok ? (H >> b) & HC::FMASK : 0u;
                lo += (col & 0x00FF00FFu) * cnt;
                hi += __byte_perm(col, 0u, 0x7371) * cnt;
                n += cnt;
            }
            outc[ry][x] = F ? finish_m(lo, hi, FULL, 0xFFFFFFFFu / FULL + 1u) : finish_m(lo, hi, n, mtab[n]);
        }
    };
    if (fast) mixed_pass(std::true_type{});
    else mixed_pass(std::false_type{});
    // ---- 3c. blocks with more than NL offsets: every window position separately
    const int nov = qo;
    for (int j = tid; j < nov; j += NT) {
        const int idx = queue[TP - 1 - j];
        const int ry = idx / TW, x = idx - ry * TW;
        const uint32_t p = (uint32_t)(x0 + x) | ((uint32_t)(y0 + ry) << 16);
        uint32_t lo = 0, hi = 0, n = 0;
#pragma unroll
        for (int dy = 0; dy <= 2 * R; ++dy) {
#pragma unroll
            for (int dx = 0; dx <= 2 * R; ++dx) {
                const uint32_t o = so[ry + dy][x + dx];
                const uint32_t src = o + p;
                const bool ok = (o != kNone) & src_ok(src);
                const uint32_t col = ldg_pred(cs + src_idx(src), ok);
                if (ok) {
                    lo += col & 0x00FF00FFu;
                    hi += __byte_perm(col, 0u, 0x7371);
                    ++n;
                }
            }
        }
        outc[ry][x] = finish_m(lo, hi, n, mtab[n]);
    }
    __syncthreads();
    // ---- store the tile (coalesced 16-byte rows)
    const bool vec = (a.wt & 3) == 0;
#pragma unroll
    for (int k = 0; k < TH / NW; ++k) {
        const int ry = warp + NW * k, py = y0 + ry, gx0 = x0 + 4 * lane;
        if (py >= a.row_end || gx0 >= a.wt) continue;
        const int64_t off = fpx * blockIdx.y + (int64_t)py * a.wt + gx0;
        const uint4 o = *reinterpret_cast<const uint4*>(&outc[ry][4 * lane]);
        if (vec) {
            st_cs_u4(a.ct + 4 * off, o);
        } else {
            const uint32_t ov[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
            for (int c = 0; c < 4; ++c)
                if (gx0 + c < a.wt) st_cs_u32(a.ct + 4 * (off + c), ov[c]);
        }
    }
}

cudaError_t launch_vote_hist(const VoteArgs& a, int n_frames, cudaStream_t st, int* launches) {
    constexpr int TW = 128, TH = 4 * kHistWarps;
    const int tiles = ((a.wt + TW - 1) / TW) * ((a.row_end - a.row_begin + TH - 1) / TH);
    dim3 grid((unsigned)tiles, (unsigned)n_frames);
    if (a.r == 1) {
        if (a.cs_pad) vote_hist_kernel<1, true><<<grid, 32 * kHistWarps, 0, st>>>(a);
        else vote_hist_kernel<1, false><<<grid, 32 * kHistWarps, 0, st>>>(a);
    } else if (a.r == 2) {
        if (a.cs_pad) vote_hist_kernel<2, true><<<grid, 32 * kHistWarps, 0, st>>>(a);
        else vote_hist_kernel<2, false><<<grid, 32 * kHistWarps, 0, st>>>(a);
    } else {
        return cudaErrorInvalidValue;
    }
    *launches += 1;
    return cudaPeekAtLastError();
}

}  // namespace sb
