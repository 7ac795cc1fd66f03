// stylize.cu -- tiled Alg. 2 "ParallelStyleBlit" for sm_100a.
//
// One CTA = one 128 x 16 pixel tile of one frame (256 threads, 4 consecutive pixels x 2 rows
// per thread, uint4 I/O).  Per tile and level l the seed cells that any tile pixel can reach
// (its 3x3 neighbourhood) are materialised in shared memory:
//     cell = (4*(s.x - x0), 4*(s.y - y0), delta),  delta = u* - q packed as dy*65536 + dx,
// where s is the jittered seed (SeedPoint, lines 354-358), q = clamp(s) (reading R8) and
// u* = LUT[G_T[q]] (line 383).  A pixel's candidate is then s = p + delta of its nearest seed
// (line 384), so per pixel and level the work is 9 shared-memory distance evaluations, one
// L2-resident gather of G_S[s] and a 3-instruction squared error (VABSDIFF4+LOP3+IDP.4A).
//
// Levels run coarse to fine with compaction:
//   level L    every 4-pixel group (the pixels of a 4-aligned group share their cell for
//              h >= 4, so the 9 seed loads and the dy terms are shared by 4 pixels);
//   level L-1  only the groups with a rejected pixel, densely from a group queue, same
//              shared-cell evaluation;
//   below      the remaining pixels from a pixel queue, one per thread; the table of a level
//              is built only when enough pixels reach it (n*5 >= cells), otherwise its few
//              pixels evaluate their 9 seeds straight from the hash.
// Tables of levels L, L-1 (and L-2 when h >= 4 there) are built together up front.  Pixels
// left after level 1 take the level-0 look-up (reading R12).
//
// NearestSeed ties: key = 16*d + i, i = 3*(x+1) + (y+1) in Alg. 2's loop order (x outer, y
// inner), so the minimum key is the first strict minimum (reading R7).  d < 8 h^2 keeps the
// key in 32 bits for h <= 2^12.
#include "sb_kernels.cuh"

namespace sb {

namespace {
constexpr int TW = 128;           // tile width  (pixels)
constexpr int TH = 16;            // tile height (pixels)
constexpr int NT = 256;           // threads per CTA
constexpr int TP = TW * TH;       // pixels per tile
constexpr int NG = TW / 4;        // 4-pixel groups per row
// cells of levels 1 and 2 together bound every table set the kernel keeps at once
constexpr int CELLS1 = (TW / 2 + 3) * (TH / 2 + 3);
constexpr int CELLS2 = (TW / 4 + 3) * (TH / 4 + 3);
constexpr int MAXCELLS = CELLS1 + CELLS2;

struct Smem {
    uint32_t gt[TP];          // G_T tile
    uint32_t coord[TP];       // result coords
    uint8_t lvl[TP];          // result levels
    uint16_t q[2][TP];        // pixel queues (tile-local index y*TW + x); q[0] doubles as group queue
    uint8_t gmask[TH * NG];   // per group: pixels still rejected after level L
    int4 cell[MAXCELLS];      // seed/offset tables, row-major per level (ci*ncy + cj)
    int offtab[4][16];        // winner offsets per table slot (L, L-1, L-2, finer)
    int qn[SB_MAX_LEVELS_DEV + 2];  // appended entries per level
};

struct CellGrid {
    int cx0, cy0, ncx, ncy, off;
};

__device__ __forceinline__ CellGrid cell_grid(int x0, int y0, int l, int off) {
    CellGrid g;
    g.cx0 = (x0 >> l) - 1;
    g.cy0 = (y0 >> l) - 1;
    g.ncx = ((x0 + TW - 1) >> l) + 2 - g.cx0;
    g.ncy = ((y0 + TH - 1) >> l) + 2 - g.cy0;
    g.off = off;
    return g;
}

__device__ __forceinline__ void build_one(Smem& sm, const StylizeArgs& a, const uint32_t* __restrict__ gtf, int x0,
                                          int y0, int l, uint32_t c_l, const CellGrid& g, int c) {
    // c < ncx*ncy <= 1000: (c + 0.5) / ncy is >= 0.04 away from an integer, float-exact floor
    const int ci = (int)(((float)c + 0.5f) * __frcp_rn((float)g.ncy));
    const int cj = c - ci * g.ncy;
    int sx, sy;
    cell_seed(g.cx0 + ci, g.cy0 + cj, l, c_l, a.zero_jitter != 0, sx, sy);
    const int qx = min(max(sx, 0), a.wt - 1);
    const int qy = min(max(sy, 0), a.ht - 1);
    const uint32_t u = __ldg(a.lut + (__ldg(gtf + (uint32_t)(qy * a.wt + qx)) & 0xFFFFu));
    // delta = u* - q packed as dy*65536 + dx: p_packed + delta is the packed candidate s
    const int dpack = ((int)(u >> 16) - qy) * 65536 + ((int)(u & 0xFFFFu) - qx);
    sm.cell[g.off + c] = make_int4(4 * (sx - x0), 4 * (sy - y0), dpack, 0);
}

// Winner-offset table of a level: cell index offset of loop-order candidate i (0..8).
__device__ __forceinline__ void write_offtab(int* tab, int ncy) {
    if (threadIdx.x < 9) tab[threadIdx.x] = (int)(threadIdx.x / 3 - 1) * ncy + (int)(threadIdx.x % 3) - 1;
}

__device__ __forceinline__ uint32_t min3u(uint32_t a, uint32_t b, uint32_t c) { return min(min(a, b), c); }

// Warp-aggregated reservation of n_mine slots of counter *cnt; returns this lane's first slot.
__device__ __forceinline__ int warp_reserve(int* cnt, int n_mine) {
    const int lane = threadIdx.x & 31;
    int incl = n_mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += v;
    }
    const int total = __shfl_sync(0xFFFFFFFFu, incl, 31);
    int base = 0;
    if (lane == 31 && total) base = atomicAdd(cnt, total);
    return __shfl_sync(0xFFFFFFFFu, base, 31) + incl - n_mine;
}

// Candidate test of Alg. 2 lines 384-385 on the packed candidate c = s.x | s.y<<16:
// s inside the source (R9; a negative component borrows into a field >= 0x8000 > 32767)
// and D = ||G_T[p] - G_S[s]||^2 < T2.  Branch-free: an outside candidate reads G_S[0].
__device__ __forceinline__ bool accept(const StylizeArgs& a, const uint32_t* __restrict__ gs, uint32_t gp,
                                       uint32_t c) {
    const uint32_t x = c & 0xFFFFu, y = c >> 16;
    const bool inb = (x < (uint32_t)a.ws) & (y < (uint32_t)a.hs);
    const uint32_t gi = inb ? y * (uint32_t)a.ws + x : 0u;
    return inb & (guide_d2(gp, __ldg(gs + gi), a.cmask) < a.T2);
}

// Alg. 2 at level l (h >= 4) for the 4 pixels (px0..px0+3, py) that share one cell: the 9
// seed loads and dy terms are shared, key_i = 16*((dx - i)^2 + dy^2) + idx = A - 8 i dx4 +
// 16 i^2.  Writes the 4 packed candidates; returns the acceptance bits.
__device__ __forceinline__ uint32_t group_eval(const Smem& sm, const StylizeArgs& a, const uint32_t* __restrict__ gs,
                                               const CellGrid& g, const int* offtab, int l, int x0, int y0, int rx0,
                                               int ry, uint4 gp4, uint32_t cand[4]) {
    const int py = y0 + ry, px0 = x0 + rx0;
    const int base = g.off + ((px0 >> l) - g.cx0) * g.ncy + ((py >> l) - g.cy0);
    uint32_t k0 = 0xFFFFFFFFu, k1 = k0, k2 = k0, k3 = k0;
    const int R4x = 4 * rx0, R4y = 4 * ry;
#pragma unroll
    for (int x = -1; x <= 1; ++x) {
#pragma unroll
        for (int y = -1; y <= 1; ++y) {
            const int2 s = *reinterpret_cast<const int2*>(&sm.cell[base + x * g.ncy + y]);
            const int dy4 = s.y - R4y;
            const int dx4 = s.x - R4x;
            const uint32_t A = (uint32_t)(dx4 * dx4) + (uint32_t)(dy4 * dy4) + (uint32_t)(3 * (x + 1) + (y + 1));
            k0 = min(k0, A);
            k1 = min(k1, A - 8u * (uint32_t)dx4 + 16u);
            k2 = min(k2, A - 16u * (uint32_t)dx4 + 64u);
            k3 = min(k3, A - 24u * (uint32_t)dx4 + 144u);
        }
    }
    const uint32_t keys[4] = {k0, k1, k2, k3};
    const uint32_t gpv[4] = {gp4.x, gp4.y, gp4.z, gp4.w};
    const uint32_t p0 = ((uint32_t)py << 16) | (uint32_t)px0;
    uint32_t acc = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const uint32_t c = p0 + (uint32_t)i + (uint32_t)sm.cell[base + offtab[keys[i] & 15u]].z;
        cand[i] = c;
        acc |= (uint32_t)accept(a, gs, gpv[i], c) << i;
    }
    return acc;
}

}  // namespace

__global__ void __launch_bounds__(NT, 4) stylize_tiled_kernel(const __grid_constant__ StylizeArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem& sm = *reinterpret_cast<Smem*>(smem_raw);

    const int tiles_x = (a.wt + TW - 1) / TW;
    const int tile = blockIdx.x;
    const int frame = blockIdx.y;
    const int x0 = (tile % tiles_x) * TW;
    const int y0 = a.row_begin + (tile / tiles_x) * TH;
    const int64_t fpx = (int64_t)a.wt * a.ht;
    const uint32_t* __restrict__ gtf = reinterpret_cast<const uint32_t*>(a.gt) + fpx * frame;
    const uint32_t* __restrict__ gs = reinterpret_cast<const uint32_t*>(a.gs);
    const uint32_t seed = a.frame_seed(frame);

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int rx0 = lane * 4;               // this thread's 4-pixel group column
    const int ryA = warp, ryB = warp + 8;   // and its two rows
    const bool colok = x0 + rx0 < a.wt;     // wt % 4 == 0: a group is all in or all out
    const bool okA = colok && (y0 + ryA) < a.row_end;
    const bool okB = colok && (y0 + ryB) < a.row_end;
    const int L = a.L;

    if (threadIdx.x < SB_MAX_LEVELS_DEV + 2) sm.qn[threadIdx.x] = 0;

    // ---- load the G_T tile (streamed once from HBM) ----
    uint4 gA = make_uint4(0, 0, 0, 0), gB = gA;
    {
        const uint64_t pol = policy_evict_first();
        if (okA) gA = ld_stream_u4(gtf + (int64_t)(y0 + ryA) * a.wt + x0 + rx0, pol);
        if (okB) gB = ld_stream_u4(gtf + (int64_t)(y0 + ryB) * a.wt + x0 + rx0, pol);
    }
    *reinterpret_cast<uint4*>(&sm.gt[ryA * TW + rx0]) = gA;
    *reinterpret_cast<uint4*>(&sm.gt[ryB * TW + rx0]) = gB;

    // ---- tables of levels L, L-1 and (when h >= 4 there) L-2, built together ----
    const CellGrid gL = cell_grid(x0, y0, L, 0);
    const int ncL = gL.ncx * gL.ncy;
    const CellGrid gL1 = cell_grid(x0, y0, L - 1, ncL);
    const int ncL1 = L >= 2 ? gL1.ncx * gL1.ncy : 0;
    const bool pre2 = L >= 4;
    const CellGrid gL2 = cell_grid(x0, y0, L - 2, ncL + ncL1);
    const int ncL2 = pre2 ? gL2.ncx * gL2.ncy : 0;
    write_offtab(sm.offtab[0], gL.ncy);
    write_offtab(sm.offtab[1], gL1.ncy);
    write_offtab(sm.offtab[2], gL2.ncy);
    {
        const uint32_t cL = level_salt(seed, L), cL1 = level_salt(seed, L - 1), cL2 = level_salt(seed, L - 2);
        for (int c = threadIdx.x; c < ncL + ncL1 + ncL2; c += NT) {
            if (c < ncL) build_one(sm, a, gtf, x0, y0, L, cL, gL, c);
            else if (c < ncL + ncL1) build_one(sm, a, gtf, x0, y0, L - 1, cL1, gL1, c - ncL);
            else build_one(sm, a, gtf, x0, y0, L - 2, cL2, gL2, c - ncL - ncL1);
        }
    }
    __syncthreads();

    int l;          // next level to process from the pixel queue q[cur]
    int cur = 0;
    int npx;        // number of entries in q[cur]
    if (L >= 2) {
        // ---- level L: every pixel, in 4-pixel groups ----
        const bool group_next = (L - 1) >= 2;  // level L-1 also runs on groups
        uint32_t rej[2] = {0, 0};
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const int ry = r ? ryB : ryA;
            if (!(r ? okB : okA)) continue;
            uint32_t cand[4];
            const uint32_t acc = group_eval(sm, a, gs, gL, sm.offtab[0], L, x0, y0, rx0, ry, r ? gB : gA, cand);
            *reinterpret_cast<uint4*>(&sm.coord[ry * TW + rx0]) = make_uint4(cand[0], cand[1], cand[2], cand[3]);
            *reinterpret_cast<uint32_t*>(&sm.lvl[ry * TW + rx0]) = 0x01010101u * (uint32_t)L;
            rej[r] = ~acc & 0xFu;
        }
        if (group_next) {
            // queue the groups with a rejected pixel
            const int n_mine = (rej[0] != 0) + (rej[1] != 0);
            int pos = warp_reserve(&sm.qn[L], n_mine);
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                if (!rej[r]) continue;
                const int gid = (r ? ryB : ryA) * NG + lane;
                sm.gmask[gid] = (uint8_t)rej[r];
                sm.q[0][pos++] = (uint16_t)gid;
            }
            __syncthreads();
            // ---- level L-1: the queued groups, one per thread ----
            const int ng = sm.qn[L];
            const int l1 = L - 1;
            for (int j0 = 0; j0 < ng; j0 += NT) {
                const int j = j0 + threadIdx.x;
                uint32_t still = 0;
                int gid = 0;
                if (j < ng) {
                    gid = sm.q[0][j];
                    const int ry = gid / NG, grx0 = (gid % NG) * 4;
                    const uint32_t m = sm.gmask[gid];
                    const uint4 gp4 = *reinterpret_cast<const uint4*>(&sm.gt[ry * TW + grx0]);
                    uint32_t cand[4];
                    const uint32_t acc = group_eval(sm, a, gs, gL1, sm.offtab[1], l1, x0, y0, grx0, ry, gp4, cand);
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        if ((m >> i) & (acc >> i) & 1u) {
                            sm.coord[ry * TW + grx0 + i] = cand[i];
                            sm.lvl[ry * TW + grx0 + i] = (uint8_t)l1;
                        }
                    }
                    still = m & ~acc;
                }
                int pos2 = warp_reserve(&sm.qn[l1], __popc(still));
                const int pbase = (gid / NG) * TW + (gid % NG) * 4;
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    if ((still >> i) & 1u) sm.q[1][pos2++] = (uint16_t)(pbase + i);
            }
            __syncthreads();
            npx = sm.qn[l1];
            cur = 1;
            l = L - 2;
        } else {
            // L == 2: the rejected pixels go straight to the per-pixel levels
            int pos = warp_reserve(&sm.qn[L], __popc(rej[0]) + __popc(rej[1]));
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                const int ry = r ? ryB : ryA;
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    if ((rej[r] >> i) & 1u) sm.q[0][pos++] = (uint16_t)(ry * TW + rx0 + i);
            }
            __syncthreads();
            npx = sm.qn[L];
            cur = 0;
            l = L - 1;
        }
    } else {
        // L == 1: every valid pixel starts in the pixel queue
        const int n_mine = (okA ? 4 : 0) + (okB ? 4 : 0);
        __syncthreads();  // qn initialised
        int pos = warp_reserve(&sm.qn[2], n_mine);
        for (int r = 0; r < 2; ++r) {
            if (!(r ? okB : okA)) continue;
            const int ry = r ? ryB : ryA;
            for (int i = 0; i < 4; ++i) sm.q[0][pos++] = (uint16_t)(ry * TW + rx0 + i);
        }
        __syncthreads();
        npx = sm.qn[2];
        cur = 0;
        l = 1;
    }

    // ---- finer levels over the compacted pixel queue ----
    for (; l >= 1 && npx > 0; --l) {
        CellGrid g;
        bool table = true;
        const int* offtab;
        if (l == L) {
            g = gL;  // L == 1
            offtab = sm.offtab[0];
        } else if (l == L - 1) {
            g = gL1;  // L == 2
            offtab = sm.offtab[1];
        } else if (l == L - 2 && pre2) {
            g = gL2;
            offtab = sm.offtab[2];
        } else {
            g = cell_grid(x0, y0, l, 0);
            offtab = sm.offtab[3];
            table = npx * 5 >= g.ncx * g.ncy;
            if (table) {
                const uint32_t c_l = level_salt(seed, l);
                for (int c = threadIdx.x; c < g.ncx * g.ncy; c += NT) build_one(sm, a, gtf, x0, y0, l, c_l, g, c);
                write_offtab(sm.offtab[3], g.ncy);
                __syncthreads();
            }
        }
        const uint32_t c_l = level_salt(seed, l);
        for (int j0 = 0; j0 < npx; j0 += NT) {
            const int j = j0 + threadIdx.x;
            bool rej = false;
            int idx = 0;
            if (j < npx) {
                idx = sm.q[cur][j];
                const int rx = idx & (TW - 1), ry = idx / TW;
                const int px = x0 + rx, py = y0 + ry;
                uint32_t cand;
                if (table) {
                    const int base = g.off + ((px >> l) - g.cx0) * g.ncy + ((py >> l) - g.cy0);
                    const int R4x = 4 * rx, R4y = 4 * ry;
                    uint32_t kk[3];
#pragma unroll
                    for (int x = -1; x <= 1; ++x) {
                        uint32_t kx[3];
#pragma unroll
                        for (int y = -1; y <= 1; ++y) {
                            const int2 s = *reinterpret_cast<const int2*>(&sm.cell[base + x * g.ncy + y]);
                            const int dx4 = s.x - R4x, dy4 = s.y - R4y;
                            kx[y + 1] = (uint32_t)(dx4 * dx4) + (uint32_t)(dy4 * dy4) + (uint32_t)(3 * (x + 1) + (y + 1));
                        }
                        kk[x + 1] = min3u(kx[0], kx[1], kx[2]);
                    }
                    const uint32_t key = min3u(kk[0], kk[1], kk[2]);
                    cand = (((uint32_t)py << 16) | (uint32_t)px) + (uint32_t)sm.cell[base + offtab[key & 15u]].z;
                } else {
                    // direct NearestSeed from the hash (few pixels reach this level)
                    const int bx = px >> l, by = py >> l;
                    uint32_t best = 0xFFFFFFFFu;
                    int qx = 0, qy = 0;
#pragma unroll
                    for (int x = -1; x <= 1; ++x)
#pragma unroll
                        for (int y = -1; y <= 1; ++y) {
                            int cx, cy;
                            cell_seed(bx + x, by + y, l, c_l, a.zero_jitter != 0, cx, cy);
                            const int dx = cx - px, dy = cy - py;
                            const uint32_t key = 16u * (uint32_t)(dx * dx + dy * dy) + (uint32_t)(3 * (x + 1) + (y + 1));
                            if (key < best) { best = key; qx = cx; qy = cy; }
                        }
                    qx = min(max(qx, 0), a.wt - 1);
                    qy = min(max(qy, 0), a.ht - 1);
                    const uint32_t u = __ldg(a.lut + (__ldg(gtf + (uint32_t)(qy * a.wt + qx)) & 0xFFFFu));
                    const int sx = (int)(u & 0xFFFFu) + (px - qx);
                    const int sy = (int)(u >> 16) + (py - qy);
                    cand = (uint32_t)(sy * 65536 + sx);
                }
                if (accept(a, gs, sm.gt[idx], cand)) {
                    sm.coord[idx] = cand;
                    sm.lvl[idx] = (uint8_t)l;
                } else {
                    rej = true;
                }
            }
            const unsigned m = __ballot_sync(0xFFFFFFFFu, rej);
            int base = 0;
            if (lane == 0 && m) base = atomicAdd(&sm.qn[l - 1], __popc(m));
            base = __shfl_sync(0xFFFFFFFFu, base, 0);
            if (rej) sm.q[cur ^ 1][base + __popc(m & ((1u << lane) - 1u))] = (uint16_t)idx;
        }
        __syncthreads();
        npx = sm.qn[l - 1];
        cur ^= 1;
    }

    // ---- level 0: the look-up fallback (reading R12) ----
    if (l == 0) {
        for (int j = threadIdx.x; j < npx; j += NT) {
            const int idx = sm.q[cur][j];
            sm.coord[idx] = __ldg(a.lut + (sm.gt[idx] & 0xFFFFu));
            sm.lvl[idx] = 0;
        }
    }
    __syncthreads();

    // ---- outputs: coords, levels, blit colours ----
    const uint32_t* __restrict__ cs = reinterpret_cast<const uint32_t*>(a.cs);
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        const int ry = r ? ryB : ryA;
        if (!(r ? okB : okA)) continue;
        const int64_t o = fpx * frame + (int64_t)(y0 + ry) * a.wt + x0 + rx0;
        const uint4 cv = *reinterpret_cast<const uint4*>(&sm.coord[ry * TW + rx0]);
        if (a.coords) st_cs_u4(a.coords + o, cv);
        if (a.level) st_cs_u32(a.level + o, *reinterpret_cast<const uint32_t*>(&sm.lvl[ry * TW + rx0]));
        if (a.ct) {
            uint4 col;
            const uint32_t ws = (uint32_t)a.ws;
            col.x = __ldg(cs + ((cv.x >> 16) * ws + (cv.x & 0xFFFFu)));
            col.y = __ldg(cs + ((cv.y >> 16) * ws + (cv.y & 0xFFFFu)));
            col.z = __ldg(cs + ((cv.z >> 16) * ws + (cv.z & 0xFFFFu)));
            col.w = __ldg(cs + ((cv.w >> 16) * ws + (cv.w & 0xFFFFu)));
            st_cs_u4(a.ct + 4 * o, col);
        }
    }
}

cudaError_t launch_stylize_tiled(const StylizeArgs& a, int n_frames, cudaStream_t st, int* launches) {
    static_assert(sizeof(Smem) <= 64 * 1024, "smem");
    const int tiles = ((a.wt + TW - 1) / TW) * ((a.row_end - a.row_begin + TH - 1) / TH);
    const size_t smem = sizeof(Smem);
    cudaError_t e = cudaFuncSetAttribute(stylize_tiled_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    dim3 grid((unsigned)tiles, (unsigned)n_frames);
    stylize_tiled_kernel<<<grid, NT, smem, st>>>(a);
    *launches += 1;
    return cudaPeekAtLastError();
}

}  // namespace sb
