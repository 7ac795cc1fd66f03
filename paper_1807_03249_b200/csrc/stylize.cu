// stylize.cu -- tiled Alg. 2 "ParallelStyleBlit" for sm_100a.
//
// One CTA = one 128 x 16 pixel tile of one frame (256 threads, 4 consecutive pixels x 2 rows
// per thread, uint4 I/O).  Per tile and level l the seed cells that any tile pixel can reach
// (its 3x3 neighbourhood) are materialised once in shared memory:
//     cell = (4*(s.x - x0), 4*(s.y - y0), delta.x, delta.y),  delta = u* - q,
// where s is the jittered seed (SeedPoint, lines 354-358), q = clamp(s) (reading R8) and
// u* = LUT[G_T[q]] (line 383).  A pixel's candidate is then s = p + delta of its nearest seed
// (line 384), so per pixel and level the work is 9 shared-memory distance evaluations, one
// L2-resident gather of G_S[s] and a 3-instruction squared error (VABSDIFF4+LOP3+IDP.4A).
//
// Levels run coarse to fine with compaction: the top level is evaluated for every pixel in
// 4-pixel groups (pixels of a 4-aligned group share the cell for h >= 4); pixels that fail
// are appended to a shared-memory queue that the next level processes densely, so warps
// are not held hostage by the few pixels that descend to fine levels.  Pixels left after
// level 1 take the level-0 look-up (reading R12).
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
// cells of the finest level (h = 2): (TW/2 + 3) x (TH/2 + 3) covers any tile alignment
constexpr int MAXCELLS = (TW / 2 + 3) * (TH / 2 + 3);

struct Smem {
    uint32_t gt[TP];        // G_T tile
    uint32_t coord[TP];     // result coords
    uint8_t lvl[TP];        // result levels
    uint16_t q[2][TP];      // pixel queues (tile-local index y*TW + x)
    int4 cell[MAXCELLS];    // per-level seed/offset table, column-major (ci*ncy + cj)
    int qn[2];
};

struct CellGrid {
    int cx0, cy0, ncy;
};

__device__ __forceinline__ CellGrid cell_grid(int x0, int y0, int l) {
    CellGrid g;
    g.cx0 = (x0 >> l) - 1;
    g.cy0 = (y0 >> l) - 1;
    g.ncy = ((y0 + TH - 1) >> l) + 2 - g.cy0;
    return g;
}

__device__ __forceinline__ void build_cells(Smem& sm, const StylizeArgs& a, const uint32_t* __restrict__ gtf,
                                            int x0, int y0, int l, uint32_t c_l, const CellGrid& g) {
    const int ncx = ((x0 + TW - 1) >> l) + 2 - g.cx0;
    const int n = ncx * g.ncy;
    for (int c = threadIdx.x; c < n; c += NT) {
        const int ci = c / g.ncy, cj = c - ci * g.ncy;
        int sx, sy;
        cell_seed(g.cx0 + ci, g.cy0 + cj, l, c_l, a.zero_jitter != 0, sx, sy);
        const int qx = min(max(sx, 0), a.wt - 1);
        const int qy = min(max(sy, 0), a.ht - 1);
        const uint32_t u = __ldg(a.lut + (__ldg(gtf + (int64_t)qy * a.wt + qx) & 0xFFFFu));
        sm.cell[c] = make_int4(4 * (sx - x0), 4 * (sy - y0), (int)(u & 0xFFFFu) - qx, (int)(u >> 16) - qy);
    }
}

// Index of the winning cell from the 4-bit loop-order index of the minimum key.
__device__ __forceinline__ int winner_cell(uint32_t key, int base, int ncy) {
    const int i = (int)(key & 15u);
    const int xi = (i * 11) >> 5;  // i / 3 for i in [0, 8]
    const int yi = i - 3 * xi;
    return base + (xi - 1) * ncy + (yi - 1);
}

__device__ __forceinline__ uint32_t min3u(uint32_t a, uint32_t b, uint32_t c) { return min(min(a, b), c); }

// Warp-aggregated append of n_mine entries (given by the caller through `emit`) to queue qi.
template <typename F>
__device__ __forceinline__ void queue_append(Smem& sm, int qi, int n_mine, F&& emit) {
    const int lane = threadIdx.x & 31;
    int incl = n_mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += v;
    }
    const int total = __shfl_sync(0xFFFFFFFFu, incl, 31);
    int base = 0;
    if (lane == 31 && total) base = atomicAdd(&sm.qn[qi], total);
    base = __shfl_sync(0xFFFFFFFFu, base, 31);
    emit(base + incl - n_mine);
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

    if (threadIdx.x < 2) sm.qn[threadIdx.x] = 0;

    // ---- load the G_T tile (streamed once from HBM) ----
    uint4 gA = make_uint4(0, 0, 0, 0), gB = gA;
    const uint64_t pol = policy_evict_first();
    if (okA) gA = ld_stream_u4(gtf + (int64_t)(y0 + ryA) * a.wt + x0 + rx0, pol);
    if (okB) gB = ld_stream_u4(gtf + (int64_t)(y0 + ryB) * a.wt + x0 + rx0, pol);
    *reinterpret_cast<uint4*>(&sm.gt[ryA * TW + rx0]) = gA;
    *reinterpret_cast<uint4*>(&sm.gt[ryB * TW + rx0]) = gB;

    int cur = 0;
    int l = a.L;
    if (l >= 2) {
        // ---- top level, every pixel, 4-pixel groups share their cell (h >= 4) ----
        const CellGrid g = cell_grid(x0, y0, l);
        build_cells(sm, a, gtf, x0, y0, l, level_salt(seed, l), g);
        __syncthreads();
        int nrej[2] = {0, 0};
        uint32_t rejmask[2] = {0, 0};
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const int ry = r ? ryB : ryA;
            const bool ok = r ? okB : okA;
            const uint4 gp4 = r ? gB : gA;
            if (!ok) continue;
            const int py = y0 + ry, px0 = x0 + rx0;
            const int base = ((px0 >> l) - g.cx0) * g.ncy + ((py >> l) - g.cy0);
            uint32_t k0 = 0xFFFFFFFFu, k1 = k0, k2 = k0, k3 = k0;
            const int R4x = 4 * rx0, R4y = 4 * ry;
#pragma unroll
            for (int x = -1; x <= 1; ++x) {
#pragma unroll
                for (int y = -1; y <= 1; ++y) {
                    const int2 s = *reinterpret_cast<const int2*>(&sm.cell[base + x * g.ncy + y]);
                    const int dy4 = s.y - R4y;
                    const uint32_t dyy = (uint32_t)(dy4 * dy4) + (uint32_t)(3 * (x + 1) + (y + 1));
                    const int dx4 = s.x - R4x;
                    k0 = min(k0, (uint32_t)(dx4 * dx4) + dyy);
                    k1 = min(k1, (uint32_t)((dx4 - 4) * (dx4 - 4)) + dyy);
                    k2 = min(k2, (uint32_t)((dx4 - 8) * (dx4 - 8)) + dyy);
                    k3 = min(k3, (uint32_t)((dx4 - 12) * (dx4 - 12)) + dyy);
                }
            }
            const uint32_t keys[4] = {k0, k1, k2, k3};
            const uint32_t gpv[4] = {gp4.x, gp4.y, gp4.z, gp4.w};
            uint4 out;
            uint32_t* outv = reinterpret_cast<uint32_t*>(&out);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int4 c = sm.cell[winner_cell(keys[i], base, g.ncy)];
                const int sx = px0 + i + c.z, sy = py + c.w;
                bool acc = false;
                if ((unsigned)sx < (unsigned)a.ws && (unsigned)sy < (unsigned)a.hs) {
                    const uint32_t d2 = guide_d2(gpv[i], __ldg(gs + sy * a.ws + sx), a.cmask);
                    acc = d2 < a.T2;
                }
                outv[i] = pack_xy(sx, sy);
                if (!acc) { rejmask[r] |= 1u << i; ++nrej[r]; }
            }
            *reinterpret_cast<uint4*>(&sm.coord[ry * TW + rx0]) = out;
            *reinterpret_cast<uint32_t*>(&sm.lvl[ry * TW + rx0]) = 0x01010101u * (uint32_t)l;
        }
        queue_append(sm, 0, nrej[0] + nrej[1], [&](int pos) {
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                const int ry = r ? ryB : ryA;
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    if (rejmask[r] & (1u << i)) sm.q[0][pos++] = (uint16_t)(ry * TW + rx0 + i);
            }
        });
        --l;
    } else {
        // L == 1: every valid pixel starts in the queue
        __syncthreads();  // qn initialised
        int n = (okA ? 4 : 0) + (okB ? 4 : 0);
        queue_append(sm, 0, n, [&](int pos) {
            for (int r = 0; r < 2; ++r) {
                if (!(r ? okB : okA)) continue;
                const int ry = r ? ryB : ryA;
                for (int i = 0; i < 4; ++i) sm.q[0][pos++] = (uint16_t)(ry * TW + rx0 + i);
            }
        });
    }
    __syncthreads();

    // ---- finer levels over the compacted queue ----
    for (; l >= 1; --l) {
        const int n = sm.qn[cur];
        if (n == 0) break;  // uniform: n is read after the barrier by every thread
        const CellGrid g = cell_grid(x0, y0, l);
        build_cells(sm, a, gtf, x0, y0, l, level_salt(seed, l), g);
        if (threadIdx.x == 0) sm.qn[cur ^ 1] = 0;
        __syncthreads();
        for (int j0 = 0; j0 < n; j0 += NT) {
            const int j = j0 + threadIdx.x;
            bool rej = false;
            int idx = 0;
            if (j < n) {
                idx = sm.q[cur][j];
                const int rx = idx & (TW - 1), ry = idx / TW;
                const int px = x0 + rx, py = y0 + ry;
                const int base = ((px >> l) - g.cx0) * g.ncy + ((py >> l) - g.cy0);
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
                const int4 c = sm.cell[winner_cell(key, base, g.ncy)];
                const int sx = px + c.z, sy = py + c.w;
                bool acc = false;
                if ((unsigned)sx < (unsigned)a.ws && (unsigned)sy < (unsigned)a.hs) {
                    const uint32_t d2 = guide_d2(sm.gt[idx], __ldg(gs + sy * a.ws + sx), a.cmask);
                    acc = d2 < a.T2;
                }
                if (acc) {
                    sm.coord[idx] = pack_xy(sx, sy);
                    sm.lvl[idx] = (uint8_t)l;
                } else {
                    rej = true;
                }
            }
            const unsigned m = __ballot_sync(0xFFFFFFFFu, rej);
            int base = 0;
            if (lane == 0 && m) base = atomicAdd(&sm.qn[cur ^ 1], __popc(m));
            base = __shfl_sync(0xFFFFFFFFu, base, 0);
            if (rej) sm.q[cur ^ 1][base + __popc(m & ((1u << lane) - 1u))] = (uint16_t)idx;
        }
        __syncthreads();
        cur ^= 1;
    }

    // ---- level 0: the look-up fallback (reading R12) ----
    {
        const int n = (l == 0) ? sm.qn[cur] : 0;
        for (int j = threadIdx.x; j < n; j += NT) {
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
            col.x = __ldg(cs + (cv.x >> 16) * a.ws + (cv.x & 0xFFFFu));
            col.y = __ldg(cs + (cv.y >> 16) * a.ws + (cv.y & 0xFFFFu));
            col.z = __ldg(cs + (cv.z >> 16) * a.ws + (cv.z & 0xFFFFu));
            col.w = __ldg(cs + (cv.w >> 16) * a.ws + (cv.w & 0xFFFFu));
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
