// vote_peel.cu -- the voting step of PAPER.md:412-421 for r = 1, 2 on sm_100a ("peel" vote).
//
// C_T[p] = average over the target pixels q of the (2r+1)^2 window around p (clipped to the
// target) of C_S[src(q) + (p - q)], skipping positions outside the source; per channel
// floor((sum + floor(n/2)) / n) (reading R13).  Fallback pixels vote like any other (R14).
//
// The contribution of q to p is C_S[p + o(q)] with o(q) = src(q) - q the offset of q's chunk:
// it depends on q only through o(q).  So the window sum is a sum over the DISTINCT offsets of
// the window, each gathered once and weighted by how many window positions carry it.  Chunks
// are large (coherent chunks of the coarse levels), so a window holds 1-4
// distinct offsets (DESIGN.md 7 "Vote") instead of 25 positions.
//
// One CTA = 128 x 16 output pixels, 128 threads.  The coordinate field of the tile plus an
// r-pixel halo is staged in shared memory as packed offsets o(q) = src(q) - q.
//   Phase 1 (thread = 4x4 output block): the block's (4+2r)^2 union of windows is "peeled":
//     take the offset v of the first position not yet covered, mark every union position with
//     offset v (a 64-bit mask, one bit per position, 8-bit row stride), repeat -- up to KMAX
//     distinct offsets per block; positions left after KMAX peels are voted one by one.
//   Phase 2 (thread = pixel; a warp = the 32 pixels of two blocks): per peeled offset v of
//     the pixel's block, n_v = popc(mask_v & window(p)); if n_v > 0 one gather C_S[p + v],
//     weighted by n_v (SWAR sums, two 16-bit lanes per register).
// Border tiles (a staged position outside the target, or a source pixel within r of the
// source border) vote position by position with clipping and bounds tests.
#include "sb_kernels.cuh"

namespace sb {

namespace {
constexpr int TW = 128, TH = 16, NT = 128;
constexpr int NB = (TW / 4) * (TH / 4);  // 4x4 output blocks per tile (one per thread)
constexpr int KMAX = 6;                  // peeled offsets per block
constexpr uint32_t kOut = 0x80008000u;   // "outside the target": no real packed offset has x = +-32768
constexpr int OUTW = TW + 8;
#ifndef SB_PEEL_REG
#define SB_PEEL_REG 1                    // phase 1 keeps the block's union offsets in registers
#endif             // padded output rows: the phase-2 stores are conflict-free

template <uint32_t N>
__device__ __forceinline__ uint32_t finish_n(uint32_t lo, uint32_t hi) {
    constexpr uint32_t half = N / 2;
    const uint32_t c0 = ((lo & 0xFFFFu) + half) / N;
    const uint32_t c1 = ((hi & 0xFFFFu) + half) / N;
    const uint32_t c2 = ((lo >> 16) + half) / N;
    const uint32_t c3 = ((hi >> 16) + half) / N;
    return c0 | (c1 << 8) | (c2 << 16) | (c3 << 24);
}

__device__ __forceinline__ uint32_t finish_any(uint32_t lo, uint32_t hi, uint32_t n) {
    if (n <= 1) return (lo & 0x00FF00FFu) | ((hi & 0x00FF00FFu) << 8);
    const uint32_t half = n >> 1;
    const uint32_t m = 0xFFFFFFFFu / n + 1u;  // ceil(2^32/n): exact floor for numerators < 2^17
    const uint32_t c0 = __umulhi((lo & 0xFFFFu) + half, m);
    const uint32_t c1 = __umulhi((hi & 0xFFFFu) + half, m);
    const uint32_t c2 = __umulhi((lo >> 16) + half, m);
    const uint32_t c3 = __umulhi((hi >> 16) + half, m);
    return c0 | (c1 << 8) | (c2 << 16) | (c3 << 24);
}

// colour * n into the two SWAR accumulators (channels 0,2 in lo; 1,3 in hi; 16-bit lanes)
__device__ __forceinline__ void swar_madd(uint32_t c, uint32_t n, uint32_t& lo, uint32_t& hi) {
    lo += (c & 0x00FF00FFu) * n;
    hi += ((c >> 8) & 0x00FF00FFu) * n;
}

__device__ __forceinline__ uint32_t ldg_if(const uint32_t* p, bool pred) {
    uint32_t v = 0;
    asm volatile(
        "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q ld.global.nc.u32 %0, [%1];\n\t}"
        : "+r"(v)
        : "l"(p), "r"((uint32_t)pred));
    return v;
}

// the window of the pixel at (i, j) of a block, as a union mask (8-bit row stride)
template <int R>
__device__ __forceinline__ uint64_t window_mask(int i, int j) {
    constexpr uint64_t row = (1ull << (2 * R + 1)) - 1ull;
    uint64_t w = 0;
#pragma unroll
    for (int k = 0; k <= 2 * R; ++k) w |= row << (8 * k);
    return w << (8 * j + i);
}
}  // namespace


// Phases 1 and 2 on the staged offsets so[][] of one tile (see the head comment).  CHECK: a
// border tile -- window positions outside the target (kOut) are skipped, each peeled offset
// is tested against the source bounds per pixel (a position left of / above the source wraps
// to a field >= 0xFFFE), and the divisor is the number of counted positions.
template <int R, bool PAD, bool CHECK>
__device__ __forceinline__ void peel_vote(uint32_t (*so)[TW + 4], uint32_t (*outc)[OUTW], uint32_t (*pv)[NB],
                                          uint2 (*pm)[NB], uint2* prem, uint8_t* pk,
                                          const uint32_t* __restrict__ cs, int x0, int y0, uint32_t ws,
                                          uint32_t hs) {
    constexpr int U = 4 + 2 * R;
    constexpr uint32_t NWIN = (2 * R + 1) * (2 * R + 1);
    auto sidx = [&](uint32_t pos) { return PAD ? pos : (pos >> 16) * ws + (pos & 0xFFFFu); };
    // ---- phase 1: peel the distinct offsets of this thread's block union
    {
        const int b = threadIdx.x, bc = b & 31, br = b >> 5;
        uint32_t o[U][U];
#if SB_PEEL_REG
#pragma unroll
        for (int rr = 0; rr < U; ++rr) {
            const uint32_t* row = &so[4 * br + rr][4 * bc];  // union column 0 = tile column 4bc - R
#pragma unroll
            for (int c = 0; c < U; c += 4) {
                if (c + 4 <= U) {
                    const uint4 v = *reinterpret_cast<const uint4*>(row + c);
                    o[rr][c] = v.x; o[rr][c + 1] = v.y; o[rr][c + 2] = v.z; o[rr][c + 3] = v.w;
                } else {
                    const uint2 v = *reinterpret_cast<const uint2*>(row + c);
                    o[rr][c] = v.x; o[rr][c + 1] = v.y;
                }
            }
        }
#endif
        // bit 8 rr + c of (lo | hi << 32): union position (rr, c)
        uint32_t rlo = 0, rhi = 0;
#pragma unroll
        for (int rr = 0; rr < U; ++rr) {
            const uint32_t rowbits = (1u << U) - 1u;
            if (rr < 4) rlo |= rowbits << (8 * rr);
            else rhi |= rowbits << (8 * (rr - 4));
        }
        int k = 0;
#pragma unroll 1
        for (int t = 0; t < KMAX; ++t) {
            if (!__any_sync(0xFFFFFFFFu, (rlo | rhi) != 0)) break;
            if ((rlo | rhi) != 0) {
                const int bp = rlo ? __ffs(rlo) - 1 : 32 + __ffs(rhi) - 1;
                const uint32_t v = so[4 * br + (bp >> 3)][4 * bc + (bp & 7)];
                uint32_t mlo = 0, mhi = 0;
#pragma unroll
                for (int rr = 0; rr < U; ++rr) {
#if !SB_PEEL_REG
                    // the union row again from shared memory (fewer registers, more LDS)
                    const uint32_t* row = &so[4 * br + rr][4 * bc];
#pragma unroll
                    for (int c = 0; c < U; c += 4) {
                        if (c + 4 <= U) {
                            const uint4 w = *reinterpret_cast<const uint4*>(row + c);
                            o[rr][c] = w.x; o[rr][c + 1] = w.y; o[rr][c + 2] = w.z; o[rr][c + 3] = w.w;
                        } else {
                            const uint2 w = *reinterpret_cast<const uint2*>(row + c);
                            o[rr][c] = w.x; o[rr][c + 1] = w.y;
                        }
                    }
#endif
#pragma unroll
                    for (int c = 0; c < U; ++c) {
                        const uint32_t bit = (uint32_t)(o[rr][c] == v) << (8 * (rr & 3) + c);
                        if (rr < 4) mlo |= bit;
                        else mhi |= bit;
                    }
                }
                rlo &= ~mlo;
                rhi &= ~mhi;
                pv[t][b] = v;
                pm[t][b] = make_uint2(mlo, mhi);
                k = t + 1;
            }
        }
        pk[b] = (uint8_t)k;
        prem[b] = make_uint2(rlo, rhi);  // left after KMAX peels: voted position by position
    }
    __syncthreads();
    // ---- phase 2: per pixel, one weighted gather per peeled offset of its window
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int i = lane & 3, j = (lane >> 2) & 3;
    const uint64_t wm = window_mask<R>(i, j);
    const uint32_t wlo = (uint32_t)wm, whi = (uint32_t)(wm >> 32);
    auto valid = [&](uint32_t v, uint32_t pos) {
        return !CHECK || ((v != kOut) & ((pos & 0xFFFFu) < ws) & ((pos >> 16) < hs));
    };
#pragma unroll 1
    for (int it = 0; it < NB / 8; ++it) {
        const int blk = 2 * (4 * it + warp) + (lane >> 4);
        const int bc = blk & 31, br = blk >> 5;
        const int tx = 4 * bc + i, ty = 4 * br + j;
        const uint32_t base = ((uint32_t)(y0 + ty) << 16) | (uint32_t)(x0 + tx);  // packed p
        const int k = pk[blk];
        const int kw = __reduce_max_sync(0xFFFFFFFFu, k);  // the warp's two blocks
        uint32_t lo = 0, hi = 0, cnt = 0;
#pragma unroll
        for (int t = 0; t < KMAX; ++t) {
            if (t >= kw) break;
            const bool act = t < k;
            uint2 m = make_uint2(0u, 0u);
            uint32_t v = 0;
            if (act) {
                m = pm[t][blk];
                v = pv[t][blk];
            }
            const uint32_t pos = base + v;
            uint32_t n = (uint32_t)(__popc(m.x & wlo) + __popc(m.y & whi));
            if (CHECK) n = valid(v, pos) ? n : 0u;
            const uint32_t c = ldg_if(cs + sidx(pos), n != 0);
            swar_madd(c, n, lo, hi);
            cnt += n;
        }
        const uint2 rm = prem[blk];
        uint32_t llo = rm.x & wlo, lhi = rm.y & whi;
        while (llo | lhi) {
            const int bp = llo ? __ffs(llo) - 1 : 32 + __ffs(lhi) - 1;
            if (llo) llo &= llo - 1u; else lhi &= lhi - 1u;
            const uint32_t v = so[4 * br + (bp >> 3)][4 * bc + (bp & 7)];
            const uint32_t pos = base + v;
            if (valid(v, pos)) {
                swar_madd(__ldg(cs + sidx(pos)), 1u, lo, hi);
                ++cnt;
            }
        }
        // fast tiles: every window position counts; border tiles: cnt >= 1 for a pixel inside
        // the target (q = p votes for src(p)); pixels outside it are never stored
        outc[ty][tx] = CHECK ? finish_any(lo, hi, cnt) : finish_n<NWIN>(lo, hi);
    }
}

template <int R, bool PAD>
__global__ void __launch_bounds__(NT, 4) vote_peel_kernel(const VoteArgs a) {
    constexpr int U = 4 + 2 * R;               // union of a block's windows: U x U positions
    constexpr int SH = TH + 2 * R;             // staged rows (tile + halo)
    constexpr int SWP = TW + 4;                // staged columns -R .. TW-1+R at so[.][R + x]
    static_assert(R >= 1 && R <= 2 && U <= 8, "peel vote: r in {1, 2}");
    __shared__ __align__(16) uint32_t so[SH][SWP];
    __shared__ __align__(16) uint32_t outc[TH][OUTW];
    __shared__ uint32_t pv[KMAX][NB];
    __shared__ uint2 pm[KMAX][NB];
    __shared__ uint2 prem[NB];
    __shared__ uint8_t pk[NB];

    const int tiles_x = (a.wt + TW - 1) / TW;
    const int x0 = (blockIdx.x % tiles_x) * TW;
    const int y0 = a.row_begin + (blockIdx.x / tiles_x) * TH;
    const int64_t fpx = (int64_t)a.wt * a.ht;
    const uint32_t* __restrict__ cf = a.coords + fpx * blockIdx.y;
    const uint32_t* __restrict__ cs = reinterpret_cast<const uint32_t*>(PAD ? a.cs_pad : a.cs);
    const uint32_t ws = (uint32_t)a.ws, hs = (uint32_t)a.hs;

    // ---- stage packed offsets o(q) = src(q) - q (kOut outside the target); fast-tile test:
    //      every staged position inside the target with its source >= R from the source border
    bool fast_mine = true;
    auto offset_of = [&](uint32_t c, int gx, int gy) {
        const uint32_t sx = c & 0xFFFFu, sy = c >> 16;
        fast_mine &= (sx >= (uint32_t)R) & (sx + (uint32_t)R < ws) & (sy >= (uint32_t)R) & (sy + (uint32_t)R < hs);
        return c - (((uint32_t)gy << 16) | (uint32_t)gx);
    };
    if ((a.wt & 3) == 0) {
        for (int i = threadIdx.x; i < SH * (TW / 4); i += NT) {
            const int yy = i / (TW / 4), g4 = i - yy * (TW / 4);
            const int gx = x0 + 4 * g4, gy = y0 - R + yy;
            uint32_t o[4];
            if (gy >= 0 && gy < a.ht && gx < a.wt) {  // wt % 4 == 0: all 4 inside
                const uint4 v = *reinterpret_cast<const uint4*>(cf + (int64_t)gy * a.wt + gx);
                o[0] = offset_of(v.x, gx, gy);
                o[1] = offset_of(v.y, gx + 1, gy);
                o[2] = offset_of(v.z, gx + 2, gy);
                o[3] = offset_of(v.w, gx + 3, gy);
            } else {
                o[0] = o[1] = o[2] = o[3] = kOut;
                fast_mine = false;
            }
            uint32_t* d = &so[yy][R + 4 * g4];
            if (R == 2) {
                *reinterpret_cast<uint2*>(d) = make_uint2(o[0], o[1]);
                *reinterpret_cast<uint2*>(d + 2) = make_uint2(o[2], o[3]);
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k) d[k] = o[k];
            }
        }
        for (int i = threadIdx.x; i < SH * 2 * R; i += NT) {  // halo columns
            const int yy = i / (2 * R), k = i - yy * (2 * R);
            const int x = k < R ? k - R : TW + (k - R);
            const int gx = x0 + x, gy = y0 - R + yy;
            const bool in = gx >= 0 && gx < a.wt && gy >= 0 && gy < a.ht;
            uint32_t o = kOut;
            if (in) o = offset_of(__ldg(cf + (int64_t)gy * a.wt + gx), gx, gy);
            else fast_mine = false;
            so[yy][R + x] = o;
        }
    } else {
        for (int i = threadIdx.x; i < SH * (TW + 2 * R); i += NT) {
            const int yy = i / (TW + 2 * R), xx = i - yy * (TW + 2 * R);
            const int gx = x0 - R + xx, gy = y0 - R + yy;
            const bool in = gx >= 0 && gx < a.wt && gy >= 0 && gy < a.ht;
            uint32_t o = kOut;
            if (in) o = offset_of(__ldg(cf + (int64_t)gy * a.wt + gx), gx, gy);
            else fast_mine = false;
            so[yy][xx] = o;
        }
    }
    const bool fast = __syncthreads_and(fast_mine) != 0;

    if (fast) peel_vote<R, PAD, false>(so, outc, pv, pm, prem, pk, cs, x0, y0, ws, hs);
    else peel_vote<R, PAD, true>(so, outc, pv, pm, prem, pk, cs, x0, y0, ws, hs);
    __syncthreads();
    // ---- store the tile: coalesced 16-byte rows (scalar for ragged widths)
    const bool vec = (a.wt & 3) == 0;
    for (int e = threadIdx.x; e < TH * (TW / 4); e += NT) {
        const int ry = e / (TW / 4), g = e - ry * (TW / 4);
        const int py = y0 + ry, gx0 = x0 + 4 * g;
        if (py >= a.row_end || gx0 >= a.wt) continue;
        const int64_t off = fpx * blockIdx.y + (int64_t)py * a.wt + gx0;
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

template <int R>
static cudaError_t launch_peel_r(const VoteArgs& a, dim3 grid, cudaStream_t st) {
    if (a.cs_pad) vote_peel_kernel<R, true><<<grid, NT, 0, st>>>(a);
    else vote_peel_kernel<R, false><<<grid, NT, 0, st>>>(a);
    return cudaPeekAtLastError();
}

cudaError_t launch_vote_peel(const VoteArgs& a, int n_frames, cudaStream_t st, int* launches) {
    const int tiles = ((a.wt + TW - 1) / TW) * ((a.row_end - a.row_begin + TH - 1) / TH);
    dim3 grid((unsigned)tiles, (unsigned)n_frames);
    cudaError_t e = a.r == 1 ? launch_peel_r<1>(a, grid, st) : launch_peel_r<2>(a, grid, st);
    *launches += 1;
    return e;
}

}  // namespace sb
