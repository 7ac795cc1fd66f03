// stylize.cu -- tiled Alg. 2 "ParallelStyleBlit" for sm_100a.
//
// One CTA = one 128 x 16 pixel tile of one frame (grid = tiles_x x tiles_y x frames), 128
// threads, 9 CTAs per SM (56 registers; 8 for ragged widths) (small CTAs: a CTA waiting at its table-build barrier idles only 4
// warps); warp w owns tile rows 4w .. 4w+3 and a thread owns 4 consecutive pixels of each
// (uint4 I/O), i.e. a 4-aligned 4 x 4 pixel block.  Per tile and level l the seed cells that
// any tile pixel can reach (its 3x3 neighbourhood) are materialised in
// shared memory: the NearestSeed key words of the jittered seed s (SeedPoint, lines 354-358;
// see KOFS) and delta = u* - q, q = clamp(s) (reading R8), u* = LUT[G_T[q]] (line 383).  A
// pixel's candidate is s = p + delta of its nearest seed (line 384), so per pixel and level the
// work is 9 shared-memory key evaluations, one L2-resident gather of G_S[s] and a
// 3-instruction squared error (VABSDIFF4+LOP3+IDP.4A).
//
// Levels run coarse to fine with compaction:
//   level L    the thread's whole 4 x 4 block at once (its 16 pixels share their home cell for
//              h >= 4: one table load per candidate, one add + one min per key), rows
//              software-pipelined;
//   L-1, L-2   only the 4-pixel groups with a rejected pixel, densely from a warp-local group
//              list compacted in place, same shared-cell evaluation per group;
//   below      the remaining pixels from a warp-local pixel queue, one per lane, NearestSeed
//              from the hash (h = 2 and finer have no table).
// The tables of the levels L, L-1, L-2 that have h >= 4 are built together up front, behind
// the kernel's only CTA barrier; afterwards each warp works on its own rows with warp-local
// lists (ballot/scan compaction, __syncwarp only), so warps never wait for each other.  Pixels
// left after level 1 take the level-0 look-up (reading R12).  A rejected pixel's coords slot
// holds its G_T value until a finer level accepts it.
//
// NearestSeed ties: see KOFS -- the key 1024 d + slot orders by d, then by Alg. 2's loop
// order (x outer, y inner), so the minimum key is the first strict minimum (reading R7).
#include <cstdlib>

#include "sb_kernels.cuh"

namespace sb {

namespace {
constexpr int TW = 128;           // tile width  (pixels)
constexpr int TH = 16;            // tile height (pixels)
constexpr int NT = 128;           // threads per CTA
constexpr int TP = TW * TH;       // pixels per tile
constexpr int NG = TW / 4;        // 4-pixel groups per row
constexpr int NW = NT / 32;       // warps per CTA
constexpr int RPW = TH / NW;      // rows per warp (RPW w .. RPW w + RPW-1)
constexpr int WPX = TP / NW;      // pixels per warp
// tables kept at once: levels {L, L-1, L-2} with h >= 4, i.e. at most levels 4, 3, 2
// Tables are column-major with a fixed column stride CS = 9 slots (72 bytes = 18 words of the
// 8-byte key table: neighbouring columns start in distinct banks).  CS >= TH/4 + 4, the most
// cells a column of a level with h = 4 spans.
constexpr int CS = 9;
static_assert(CS >= TH / 4 + 4, "column stride must hold a column of the h = 4 level");
__host__ __device__ constexpr int cells_of(int h) { return (TW / h + 3) * CS; }
constexpr int MAXCELLS = cells_of(4) + cells_of(8) + cells_of(16);
// table slots for a hierarchy of L levels: levels L, L-1, L-2 that have h >= 4
__host__ __device__ constexpr int table_cells(int L) {
    return (L >= 2 ? cells_of(1 << L) : 0) + (L - 1 >= 2 ? cells_of(1 << (L - 1)) : 0) +
           (L - 2 >= 2 ? cells_of(1 << (L - 2)) : 0);
}

// Shared memory: this head, then the cell tables (table_cells(L) slots, column-major per level,
// slot = off + ci*CS + cj) as two arrays, then the level map when requested:
//   cq[slot] = (S2, X1)      the NearestSeed key terms (see KOFS below)
//   cd[slot] = (Y1, delta)   delta = u* - q packed dy*65536 + dx
struct Smem {
    uint32_t coord[TH * (TW + 4)];  // result coords, rows padded by 16 bytes (see cix)
    uint16_t wq[NW][WPX];         // per-warp pixel queue (compacted in place)
    uint16_t glist[NW][RPW * NG]; // per-warp list of groups with a rejected pixel
};
// coords slot of tile pixel (rx, ry) / of unpadded pixel index p = ry*TW + rx: rows are padded
// by 4 words so that the 16-byte accesses of groups in different rows (the group passes) fall
// into different banks
constexpr int CROW = TW + 4;
__device__ __forceinline__ int cix(int p) { return p + (p >> 7) * 4; }
static_assert(TW == 128, "cix assumes 128-pixel rows");

static_assert(sizeof(Smem) % 16 == 0, "the cell tables after Smem need 16-byte alignment");

struct Cells {
    uint2* q;
    int2* d;
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

// NearestSeed keys (Alg. 2).  For a seed s and pixel p of a tile with origin
// (x0, y0), let S = 32 (s - origin), P = 32 (p - origin) = 32 (rx, ry).  A cell stores
//     S2 = |S|^2 + idx + KOFS,  X1 = -64 Sx,  Y1 = -64 Sy   (mod 2^32),
// idx = the cell's slot in the table, so that
//     key = S2 + rx X1 + ry Y1 = |S - P|^2 - |P|^2 + idx + KOFS = 1024 d + idx + KOFS - |P|^2.
// |P|^2 is the same for all 9 candidates of p, so the keys order p's candidates by d, then by
// idx.  The tables are column-major with cj < CS, so idx orders the 3 x 3 candidates like
// Alg. 2's loops (x outer, y inner): the minimum key is the first strict minimum (reading R7),
// and its low 10 bits (idx < 1024) address the winner.  Neighbouring pixels differ by one
// table word: key(rx + i, ry + r) = key(rx, ry) + i X1 + r Y1, one fused add-min (VIADDMNMX)
// per key.  KOFS = 1024 (132^2 + 32^2) > |P|^2 keeps every key >= 0, and
// 1024 d + idx + KOFS < 2^32 for d < 8 h^2, h <= 2^9 (tabled levels, see the launcher).
constexpr uint32_t KOFS = 1024u * (132u * 132u + 32u * 32u);
static_assert(MAXCELLS <= 1024, "cell index must fit the key's low 10 bits");

__device__ __forceinline__ void build_one(const Cells& T, const StylizeArgs& a, const uint32_t* __restrict__ gtf, int x0,
                                          int y0, int l, uint32_t c_l, const CellGrid& g, int c) {
    // c < ncx*ncy <= 1000, ncy <= 13: (c + 0.5) / ncy is >= 0.5/13 away from an integer, so the
    // floor is exact even with the approximate reciprocal (relative error ~2^-23; the IEEE
    // __frcp_rn carries a slow-path branch)
    float rcp;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rcp) : "f"((float)g.ncy));
    const int ci = (int)(((float)c + 0.5f) * rcp);
    const int cj = c - ci * g.ncy;
    int sx, sy;
    cell_seed(g.cx0 + ci, g.cy0 + cj, l, c_l, a.zero_jitter != 0, sx, sy);
    const int qx = min(max(sx, 0), a.wt - 1);
    const int qy = min(max(sy, 0), a.ht - 1);
    SB_CHECK(qx >= 0 && qx < a.wt && qy >= 0 && qy < a.ht, "table-build G_T[q]");
    const uint32_t u = __ldg(a.lut + (__ldg(gtf + (uint32_t)(qy * a.wt + qx)) & a.key_mask));
    // delta = u* - q packed as dy*65536 + dx: p_packed + delta is the packed candidate s
    const int dpack = ((int)(u >> 16) - qy) * 65536 + ((int)(u & 0xFFFFu) - qx);
    const int idx = g.off + ci * CS + cj;
    SB_CHECK(ci >= 0 && ci < g.ncx && cj >= 0 && cj < g.ncy && cj < CS && idx >= 0 && idx < 1024, "cell slot");
    const uint32_t Sx = (uint32_t)(32 * (sx - x0)), Sy = (uint32_t)(32 * (sy - y0));
    const uint32_t S2 = Sx * Sx + Sy * Sy + (uint32_t)idx + KOFS;
    const uint32_t X1 = 0u - 64u * Sx;
    T.q[idx] = make_uint2(S2, X1);
    T.d[idx] = make_int2((int)(0u - 64u * Sy), dpack);
}



// Exclusive warp prefix sum of v; *total receives the warp-wide sum.
__device__ __forceinline__ int warp_excl_scan(int v, int* total) {
    const int lane = threadIdx.x & 31;
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += t;
    }
    *total = __shfl_sync(0xFFFFFFFFu, incl, 31);
    return incl - v;
}

// Candidate test of Alg. 2 lines 384-385 on the packed candidate c = s.x | s.y<<16:
// s inside the source (R9; a negative component borrows into a field >= 0x8000 > 32767)
// and D = ||G_T[p] - G_S[s]||^2 < T2.  Branch-free: an outside candidate reads G_S[0].
// G_S gather for the packed candidate c = s.x | s.y<<16 (Alg. 2).  *in: s inside the
// source (R9; a negative component borrows into a field >= 0x8000 > 32767), tested with one
// packed 16-bit min against (ws-1 | (hs-1)<<16).  The index is y*ws + x = c + y*(ws - 65536)
// (mod 2^32), or, with the strided exemplar copy (PAD: rows of 2^16 pixels), c itself; an
// outside candidate reads pixel 0.  Branch-free.
template <bool PAD>
__device__ __forceinline__ uint32_t gather_gs(const StylizeArgs& a, const uint32_t* __restrict__ gs, uint32_t c,
                                              bool* in) {
    const uint32_t lim = ((uint32_t)(a.hs - 1) << 16) | (uint32_t)(a.ws - 1);
    uint32_t mn;
    asm("min.u16x2 %0, %1, %2;" : "=r"(mn) : "r"(c), "r"(lim));
    *in = mn == c;
    const uint32_t gi = *in ? (PAD ? c : c + (c >> 16) * (uint32_t)(a.ws - 65536)) : 0u;
    SB_CHECK(PAD ? ((gi & 0xFFFFu) < (uint32_t)a.ws && (gi >> 16) < (uint32_t)a.hs) : gi < (uint32_t)(a.ws * a.hs),
             "G_S gather");
    const uint32_t* p;
    asm("mad.wide.u32 %0, %1, 4, %2;" : "=l"(p) : "r"(gi), "l"(gs));
    return __ldg(p);
}

template <bool EXT, bool PAD>
__device__ __forceinline__ bool accept(const StylizeArgs& a, const uint32_t* __restrict__ gs, uint32_t gp,
                                       uint32_t c) {
    bool inb;
    const uint32_t g = gather_gs<PAD>(a, gs, c, &inb);
    if (EXT) return inb & guide_ok_ext(gp, g, a.cmask, a.w, a.lmask, a.T2);
    return inb & (guide_d2(gp, g, a.cmask) < a.T2);
}

// Slot of the home cell's (-1,-1) neighbour in a level table (column-major, stride CS).
__device__ __forceinline__ int home_slot(const CellGrid& g, int l, int px, int py) {
    return g.off + ((px >> l) - g.cx0 - 1) * CS + ((py >> l) - g.cy0 - 1);
}

// NearestSeed for the 4 pixels (x0+rx0+i, y0+ry) of a group, h >= 4: they share their home
// cell; per candidate A = key of pixel 0 (2 IMAD) and key_i = A + X_i (fused add-min).
__device__ __forceinline__ void group_ns(const Cells& T, const CellGrid& g, int l, int x0, int y0, int rx0, int ry,
                                         uint32_t key[4]) {
    const int h0 = home_slot(g, l, x0 + rx0, y0 + ry);
    SB_CHECK(h0 >= g.off && h0 + 2 * CS + 2 < g.off + g.ncx * CS, "group home slot");
#pragma unroll
    for (int c = 0; c < 9; ++c) {
        const int slot = h0 + (c / 3) * CS + (c % 3);  // x = c/3 - 1 outer, y = c%3 - 1 inner
        const uint2 s = T.q[slot];
        const uint32_t Y1 = (uint32_t)T.d[slot].x;
        const uint32_t A = s.x + (uint32_t)rx0 * s.y + (uint32_t)ry * Y1;
        const uint32_t X2 = s.y + s.y, X3 = X2 + s.y;
        const uint32_t kc[4] = {A, A + s.y, A + X2, A + X3};
#pragma unroll
        for (int i = 0; i < 4; ++i) key[i] = c == 0 ? kc[i] : min(key[i], kc[i]);
    }
}

// NearestSeed for the thread's whole 4 x 4 block (pixels x0+rx0+i, y0+ry0+r; 4-aligned, h >= 4):
// the 16 pixels share their home cell, so per candidate the seed load, A = key of pixel (0,0)
// and the row bases B_r = A + r Y1 are computed once, and each of the 16 keys costs one fused
// add-min.
__device__ __forceinline__ void block_ns(const Cells& T, const CellGrid& g, int l, int x0, int y0, int rx0, int ry0,
                                         uint32_t key[4][4]) {
    const int h0 = home_slot(g, l, x0 + rx0, y0 + ry0);
    SB_CHECK(h0 >= g.off && h0 + 2 * CS + 2 < g.off + g.ncx * CS, "block home slot");
#pragma unroll
    for (int c = 0; c < 9; ++c) {
        const int slot = h0 + (c / 3) * CS + (c % 3);
        const uint2 s = T.q[slot];
        const uint32_t Y1 = (uint32_t)T.d[slot].x;
        uint32_t B = s.x + (uint32_t)rx0 * s.y + (uint32_t)ry0 * Y1;
        const uint32_t X2 = s.y + s.y, X3 = X2 + s.y;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            if (r > 0) B += Y1;
            const uint32_t kc[4] = {B, B + s.y, B + X2, B + X3};
#pragma unroll
            for (int i = 0; i < 4; ++i) key[r][i] = c == 0 ? kc[i] : min(key[r][i], kc[i]);
        }
    }
}

// delta = u* - q of the winning cell
__device__ __forceinline__ uint32_t winner_delta(const Cells& T, uint32_t key) {
    SB_CHECK((key & 1023u) < (uint32_t)MAXCELLS, "winner slot");
    return (uint32_t)T.d[key & 1023u].y;
}

// Alg. 2 at level l (h >= 4) for the 4 pixels (px0..px0+3, py) that share one cell.  Writes the
// 4 packed candidates; returns the acceptance bits.
template <bool EXT, bool PAD>
__device__ __forceinline__ uint32_t group_eval(const Cells& T, const StylizeArgs& a, const uint32_t* __restrict__ gs,
                                               const CellGrid& g, int l, int x0, int y0, int rx0, int ry, uint4 gp4,
                                               uint32_t m, uint32_t cand[4]) {
    uint32_t keys[4];
    group_ns(T, g, l, x0, y0, rx0, ry, keys);
    const uint32_t gpv[4] = {gp4.x, gp4.y, gp4.z, gp4.w};
    const uint32_t p0 = ((uint32_t)(y0 + ry) << 16) | (uint32_t)(x0 + rx0);
    uint32_t acc = 0;
    // every pixel of the group looks up its winner and gathers (the caller keeps only the
    // still-rejected ones, m & acc): predicating the look-ups per pixel measured slower
    //
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        {
            const uint32_t c = p0 + (uint32_t)i + winner_delta(T, keys[i]);
            cand[i] = c;
            acc |= (uint32_t)accept<EXT, PAD>(a, gs, gpv[i], c) << i;
        }
    }
    return acc;
}

template <bool EXT>
__device__ __forceinline__ uint32_t group_test(const StylizeArgs& a, uint4 gp4, const uint32_t gv[4], uint32_t inb) {
    const uint32_t gpv[4] = {gp4.x, gp4.y, gp4.z, gp4.w};
    uint32_t acc = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const bool ok = EXT ? guide_ok_ext(gpv[i], gv[i], a.cmask, a.w, a.lmask, a.T2)
                            : guide_d2(gpv[i], gv[i], a.cmask) < a.T2;
        acc |= (uint32_t)ok << i;
    }
    return acc & inb;
}

// Alg. 2 at level l for one pixel, NearestSeed straight from the hash.
__device__ __forceinline__ uint32_t direct_candidate(const StylizeArgs& a, const uint32_t* __restrict__ gtf, int px,
                                                     int py, int l, uint32_t c_l) {
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
    const uint32_t u = __ldg(a.lut + (__ldg(gtf + (uint32_t)(qy * a.wt + qx)) & a.key_mask));
    const int sx = (int)(u & 0xFFFFu) + (px - qx);
    const int sy = (int)(u >> 16) + (py - qy);
    return (uint32_t)(sy * 65536 + sx);
}

}  // namespace

// LT > 0: the hierarchy depth as a compile-time constant (the common depths; all level geometry
// folds), LT = 0: a.L at run time.  PAD: the exemplar gathers index the strided copy
// a.exemplar (sb_prepare_exemplar) with the packed coordinate itself.
// RAG: a ragged width (wt % 4 != 0): rows are not 16-byte aligned and the last group of a row
// has 1..3 pixels, so G_T is read and the outputs are written pixel by pixel there (pixels past
// the row end are computed on G_T = 0 and never written).
template <bool EXT, bool LVL, int LT, bool PAD, bool NOCT = false, bool RAG = false>
__global__ void __launch_bounds__(NT, RAG ? 8 : 9) stylize_tiled_kernel(const __grid_constant__ StylizeArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
    const int L = LT > 0 ? LT : a.L;
    const int ncells = table_cells(L);
    Cells T;
    T.q = reinterpret_cast<uint2*>(smem_raw + sizeof(Smem));
    T.d = reinterpret_cast<int2*>(T.q + ncells);
    uint8_t* lvl = reinterpret_cast<uint8_t*>(T.d + ncells);  // result levels (only when a.level != nullptr)

    const int x0 = blockIdx.x * TW;
    // tiles start at row_begin rounded down to a multiple of 4, so a thread's 4 rows are one
    // 4-aligned block (block_ns); rows before row_begin are computed but never written
    const int y0 = (a.row_begin & ~3) + blockIdx.y * TH;
    const int frame = blockIdx.z;
    const int64_t fpx = (int64_t)a.wt * a.ht;
    const uint32_t* __restrict__ gtf = reinterpret_cast<const uint32_t*>(a.gt) + fpx * frame;
    const uint32_t* __restrict__ gs = reinterpret_cast<const uint32_t*>(PAD ? a.exemplar : a.gs);
    const uint32_t seed = a.frame_seed(frame);
    const uint32_t wt = (uint32_t)a.wt;

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned lt_mask = (1u << lane) - 1u;
    const int rx0 = lane * 4;               // this thread's 4-pixel group column
    const bool colok = x0 + rx0 < a.wt;     // the group has a pixel inside the row
    const int nin = min(4, a.wt - (x0 + rx0));  // its pixels inside the row (4 unless RAG)
    const int rows_here = min(TH, a.row_end - y0);
    const int row_lo = a.row_begin - y0;  // > 0 only in the first tile row of an unaligned range
    // tile row of this warp's j-th row, and whether its group exists
    auto row_of = [&](int j) { return RPW * warp + j; };  // the thread's 4 groups form a 4x4 block
    auto ok_of = [&](int j) { return colok && row_of(j) < rows_here && row_of(j) >= row_lo; };

    // The thread's 4 G_T rows (the HBM stream, consumed at level L) are issued first: their
    // latency overlaps the table build and its barrier.
    // G_T of the group in row j: one 16-byte load, or (RAG) up to 4 scalar loads
    auto load_gt = [&](int j) {
        const uint32_t* p = gtf + (uint32_t)((y0 + row_of(j)) * a.wt + x0 + rx0);
        if (!RAG) return *reinterpret_cast<const uint4*>(p);
        if (nin == 4) return ld_4w(p);  // widest load the row's alignment allows
        return make_uint4(__ldg(p), nin > 1 ? __ldg(p + 1) : 0u, nin > 2 ? __ldg(p + 2) : 0u, 0u);
    };
    uint4 gp[RPW];
#pragma unroll
    for (int j = 0; j < RPW; ++j) gp[j] = (L >= 2 && ok_of(j)) ? load_gt(j) : make_uint4(0u, 0u, 0u, 0u);

    // ---- tables of the levels among L, L-1, L-2 with h >= 4: the only CTA barrier ----
    const bool t0 = L >= 2, t1 = L - 1 >= 2, t2 = L - 2 >= 2;
    const CellGrid gL = cell_grid(x0, y0, L, 0);
    // valid cells per level (built) and slots per level (column stride CS)
    const int ncL = t0 ? gL.ncx * gL.ncy : 0;
    const CellGrid gL1 = cell_grid(x0, y0, L - 1, gL.ncx * CS);
    const int ncL1 = t1 ? gL1.ncx * gL1.ncy : 0;
    const CellGrid gL2 = cell_grid(x0, y0, L - 2, gL.ncx * CS + gL1.ncx * CS);
    const int ncL2 = t2 ? gL2.ncx * gL2.ncy : 0;
    for (int c = threadIdx.x; c < ncL + ncL1 + ncL2; c += NT) {
        const bool s0 = c < ncL, s1 = c < ncL + ncL1;
        const CellGrid& g = s0 ? gL : (s1 ? gL1 : gL2);
        const int l = s0 ? L : (s1 ? L - 1 : L - 2);
        build_one(T, a, gtf, x0, y0, l, level_salt(seed, l), g, c - (s0 ? 0 : (s1 ? ncL : ncL + ncL1)));
    }
    __syncthreads();
    // From here on a warp only touches its own rows: no further CTA barrier.

    uint16_t* q = sm.wq[warp];
    int n = 0;      // entries in the warp's pixel queue
    int l;          // level of the pixel queue
    const uint64_t pol = policy_evict_first();
    if (L >= 2) {
        // ---- level L: every pixel, in 4-pixel groups; G_T streamed once from HBM ----
        // Software-pipelined over the warp's rows: row j's NearestSeed and gathers are issued
        // before row j-1's threshold test, so the G_T load and the G_S gathers of a row are
        // in flight while the next row's NearestSeed runs.
        uint32_t rej = 0;  // 4 bits per row j
        // the block's G_T rows (the HBM stream) are issued before NearestSeed covers their latency
        uint32_t key[RPW][4];
        block_ns(T, gL, L, x0, y0, rx0, row_of(0), key);
        // rows pipelined: row j's candidates and G_S gathers are issued before row j-1's test
        uint32_t pcand[4] = {0u, 0u, 0u, 0u}, pgv[4] = {0u, 0u, 0u, 0u}, pinb = 0;
#pragma unroll
        for (int j = 0; j <= RPW; ++j) {
            uint32_t cand[4], gv[4], inb = 0;
            if (j < RPW && ok_of(j)) {
                const uint32_t p0 = ((uint32_t)(y0 + row_of(j)) << 16) | (uint32_t)(x0 + rx0);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    cand[i] = p0 + (uint32_t)i + winner_delta(T, key[j][i]);
                    bool in;
                    gv[i] = gather_gs<PAD>(a, gs, cand[i], &in);
                    inb |= (uint32_t)in << i;
                }
            }
            if (j >= 1 && ok_of(j - 1)) {
                const int ry = row_of(j - 1);
                const uint32_t acc = group_test<EXT>(a, gp[j - 1], pgv, pinb);
                // a rejected pixel's slot holds its G_T value until a finer level accepts it
                // (the group passes and the pixel queue read it from there, not from global)
                const uint4 g4 = gp[j - 1];
                *reinterpret_cast<uint4*>(&sm.coord[ry * CROW + rx0]) =
                    make_uint4((acc & 1u) ? pcand[0] : g4.x, (acc & 2u) ? pcand[1] : g4.y,
                               (acc & 4u) ? pcand[2] : g4.z, (acc & 8u) ? pcand[3] : g4.w);
                if (LVL) *reinterpret_cast<uint32_t*>(&lvl[ry * TW + rx0]) = 0x01010101u * (uint32_t)L;
                rej |= (~acc & 0xFu) << (4 * (j - 1));
            }
            if (j < RPW) {
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    pcand[i] = cand[i];
                    pgv[i] = gv[i];
                }
                pinb = inb;
            }
        }
        // ---- the warp's groups that still have a rejected pixel: lane | j<<5 | mask<<8
        uint16_t* gl = sm.glist[warp];
        int ng = 0;
#pragma unroll
        for (int j = 0; j < RPW; ++j) {
            const uint32_t m = (rej >> (4 * j)) & 0xFu;
            const unsigned b = __ballot_sync(0xFFFFFFFFu, m != 0);
            if (m) gl[ng + __popc(b & lt_mask)] = (uint16_t)(lane | (j << 5) | (m << 8));
            ng += __popc(b);
        }
        __syncwarp();
        // One tabled level (h >= 4) on the listed groups, densely; the list is compacted in
        // place to the groups that still have a rejected pixel (entry k is rewritten only at
        // an index <= k, after the ballot that follows every read of its batch).
        auto group_pass = [&](int lp, const CellGrid& g) {
            int nn = 0;
            for (int k0 = 0; k0 < ng; k0 += 32) {
                const int k = k0 + lane;
                uint32_t still = 0, e = 0;
                if (k < ng) {
                    e = gl[k];
                    SB_CHECK(k < RPW * NG, "group list");
                    const int grx0 = (int)(e & 31u) * 4;
                    const int ry = row_of((int)((e >> 5) & 7u));
                    const uint32_t m = e >> 8;
                    const int pbase = ry * TW + grx0;
                    // the group's slots: coords of its accepted pixels, G_T of the rejected (m)
                    uint4 cv = *reinterpret_cast<const uint4*>(&sm.coord[ry * CROW + grx0]);
                    uint32_t cand[4];
                    const uint32_t acc = group_eval<EXT, PAD>(T, a, gs, g, lp, x0, y0, grx0, ry, cv, m, cand);
                    // merge the newly accepted pixels: one 16-byte read-modify-write instead of
                    // four conflicting scalar stores
                    const uint32_t take = m & acc;
                    cv.x = (take & 1u) ? cand[0] : cv.x;
                    cv.y = (take & 2u) ? cand[1] : cv.y;
                    cv.z = (take & 4u) ? cand[2] : cv.z;
                    cv.w = (take & 8u) ? cand[3] : cv.w;
                    *reinterpret_cast<uint4*>(&sm.coord[ry * CROW + grx0]) = cv;
                    if (LVL) {
#pragma unroll
                        for (int i = 0; i < 4; ++i)
                            if ((take >> i) & 1u) lvl[pbase + i] = (uint8_t)lp;
                    }
                    still = m & ~acc;
                }
                const unsigned b = __ballot_sync(0xFFFFFFFFu, still != 0);
                // in place: entry k is rewritten only at an index <= k; the warp barrier orders
                // every lane's read of this batch before any lane's write (memory order, not
                // just convergence: __ballot_sync alone does not promise it)
                __syncwarp();
                if (still) gl[nn + __popc(b & lt_mask)] = (uint16_t)((e & 0xFFu) | (still << 8));
                nn += __popc(b);
            }
            __syncwarp();
            ng = nn;
        };
        l = L - 1;
        if (t1) {
            group_pass(L - 1, gL1);  // level L-1 on the groups with a rejected pixel
            l = L - 2;
            if (t2) {
                group_pass(L - 2, gL2);
                l = L - 3;
            }
        }
        // the pixels still rejected go to the per-pixel levels
        for (int k0 = 0; k0 < ng; k0 += 32) {
            const int k = k0 + lane;
            uint32_t still = 0;
            int pbase = 0;
            if (k < ng) {
                const uint32_t e = gl[k];
                pbase = row_of((int)((e >> 5) & 7u)) * TW + (int)(e & 31u) * 4;
                still = e >> 8;
            }
            int tot;
            int pos = n + warp_excl_scan(__popc(still), &tot);
#pragma unroll
            for (int i = 0; i < 4; ++i)
                if ((still >> i) & 1u) q[pos++] = (uint16_t)(pbase + i);
            n += tot;
        }
    } else {
        // L == 1: every valid pixel starts in the pixel queue
        int mine = 0;
        for (int j = 0; j < RPW; ++j) mine += ok_of(j) ? nin : 0;
        int tot;
        int pos = warp_excl_scan(mine, &tot);
        for (int j = 0; j < RPW; ++j) {
            if (!ok_of(j)) continue;
            for (int i = 0; i < nin; ++i) q[pos++] = (uint16_t)(row_of(j) * TW + rx0 + i);
            // the queue reads G_T from the pixel's slot
            *reinterpret_cast<uint4*>(&sm.coord[row_of(j) * CROW + rx0]) = load_gt(j);
        }
        n = tot;
        l = 1;
    }
    __syncwarp();

    // ---- finer levels over the warp's pixel queue, compacted in place: the levels without a
    //      table (every tabled level had its group pass), NearestSeed from the hash ----
    for (; l >= 1 && n > 0; --l) {
        const uint32_t c_l = level_salt(seed, l);
        int nn = 0;
        for (int k0 = 0; k0 < n; k0 += 32) {
            const int k = k0 + lane;
            bool rej = false;
            int idx = 0;
            if (k < n) {
                idx = q[k];
                SB_CHECK(k < WPX && idx < TP, "pixel queue");
                const int rx = idx & (TW - 1), ry = idx / TW;
                const uint32_t cand = direct_candidate(a, gtf, x0 + rx, y0 + ry, l, c_l);
                const uint32_t gp = sm.coord[cix(idx)];  // G_T while the pixel is rejected
                if (accept<EXT, PAD>(a, gs, gp, cand)) {
                    sm.coord[cix(idx)] = cand;
                    if (LVL) lvl[idx] = (uint8_t)l;
                } else {
                    rej = true;
                }
            }
            const unsigned m = __ballot_sync(0xFFFFFFFFu, rej);
            __syncwarp();  // every lane's reads of this round are ordered before the in-place writes
            if (rej) q[nn + __popc(m & lt_mask)] = (uint16_t)idx;  // nn + rank <= k: in place
            nn += __popc(m);
        }
        __syncwarp();
        n = nn;
    }

    // ---- level 0: the look-up fallback (reading R12) ----
    if (l == 0) {
        for (int k = lane; k < n; k += 32) {
            const int idx = q[k];
            sm.coord[cix(idx)] = __ldg(a.lut + (sm.coord[cix(idx)] & a.key_mask));  // the slot holds G_T
            if (LVL) lvl[idx] = 0;
        }
    }
    __syncwarp();

    // ---- outputs: coords, levels, blit colours ----
    const uint32_t* __restrict__ cs = reinterpret_cast<const uint32_t*>(
        PAD ? a.exemplar + (size_t)a.hs * ((size_t)1 << 18) : a.cs);
    const uint32_t ws = (uint32_t)a.ws;
#pragma unroll 2
    for (int j = 0; j < RPW; ++j) {
        if (!ok_of(j)) continue;
        const int ry = row_of(j);
        const int64_t o = fpx * frame + (int64_t)((y0 + ry) * wt + (uint32_t)(x0 + rx0));
        const uint4 cv = *reinterpret_cast<const uint4*>(&sm.coord[ry * CROW + rx0]);
        SB_CHECK(o + nin <= fpx * (frame + 1) && o >= fpx * frame, "output pixel");
        SB_CHECK((cv.x & 0xFFFFu) < (uint32_t)a.ws && (cv.x >> 16) < (uint32_t)a.hs, "final coordinate");
        if (RAG && nin == 4) {  // a whole group of an unaligned row: the widest stores its address allows
            if (a.coords) st_cs_4w(a.coords + o, cv);
            if (a.level) {
                for (int i = 0; i < 4; ++i) a.level[o + i] = lvl[ry * TW + rx0 + i];
            }
            if (!NOCT && a.ct) {
                auto idx = [&](uint32_t c) { return PAD ? c : (c >> 16) * ws + (c & 0xFFFFu); };
                st_cs_4w(reinterpret_cast<uint32_t*>(a.ct) + o,
                         make_uint4(__ldg(cs + idx(cv.x)), __ldg(cs + idx(cv.y)), __ldg(cs + idx(cv.z)),
                                    __ldg(cs + idx(cv.w))));
            }
            continue;
        }
        if (RAG) {  // the row's last, partial group: pixel by pixel, only those inside the row
            const uint32_t cvv[4] = {cv.x, cv.y, cv.z, cv.w};
            for (int i = 0; i < nin; ++i) {
                if (a.coords) st_cs_u32(a.coords + o + i, cvv[i]);
                if (a.level) a.level[o + i] = lvl[ry * TW + rx0 + i];
                if (!NOCT && a.ct) {
                    const uint32_t c = cvv[i];
                    st_cs_u32(a.ct + 4 * (o + i), __ldg(cs + (PAD ? c : (c >> 16) * ws + (c & 0xFFFFu))));
                }
            }
            continue;
        }
        if (a.coords) st_cs_u4(a.coords + o, cv);
        if (a.level) st_cs_u32(a.level + o, *reinterpret_cast<const uint32_t*>(&lvl[ry * TW + rx0]));
        if (!NOCT && a.ct) {
            uint4 col;
            // packed x | y<<16 -> pixel index y*ws + x (PAD: the packed value itself)
            auto idx = [&](uint32_t c) { return PAD ? c : (c >> 16) * ws + (c & 0xFFFFu); };
            col.x = __ldg(cs + idx(cv.x));
            col.y = __ldg(cs + idx(cv.y));
            col.z = __ldg(cs + idx(cv.z));
            col.w = __ldg(cs + idx(cv.w));
            st_cs_u4(a.ct + 4 * o, col);
        }
    }
}

cudaError_t launch_stylize_tiled(const StylizeArgs& a, int n_frames, cudaStream_t st, int* launches) {
    // tables sized for this L; the level map only when requested
    const size_t smem = sizeof(Smem) + (size_t)table_cells(a.L) * (sizeof(uint2) + sizeof(int2)) + (a.level ? TP : 0);
    void (*kern)(StylizeArgs);
    const bool pad = a.exemplar != nullptr;  // the strided exemplar copy: L in 3..5, no weights/labels
    if (a.wt % 4 != 0) {
        // ragged widths: run-time L, per-pixel row I/O
        kern = a.ext ? (a.level ? stylize_tiled_kernel<true, true, 0, false, false, true>
                                : stylize_tiled_kernel<true, false, 0, false, false, true>)
             : a.level ? (pad ? stylize_tiled_kernel<false, true, 0, true, false, true>
                              : stylize_tiled_kernel<false, true, 0, false, false, true>)
             : a.L == 5 && pad ? stylize_tiled_kernel<false, false, 5, true, false, true>
             : pad ? stylize_tiled_kernel<false, false, 0, true, false, true>
                   : stylize_tiled_kernel<false, false, 0, false, false, true>;
    } else if (a.ext) {
        kern = a.level ? stylize_tiled_kernel<true, true, 0, false> : stylize_tiled_kernel<true, false, 0, false>;
    } else if (a.level) {
        kern = a.L == 5 ? (pad ? stylize_tiled_kernel<false, true, 5, true> : stylize_tiled_kernel<false, true, 5, false>)
             : a.L == 4 ? (pad ? stylize_tiled_kernel<false, true, 4, true> : stylize_tiled_kernel<false, true, 4, false>)
             : a.L == 3 ? (pad ? stylize_tiled_kernel<false, true, 3, true> : stylize_tiled_kernel<false, true, 3, false>)
                        : stylize_tiled_kernel<false, true, 0, false>;
    } else {
        // NOCT: coordinates only (the blend path: the vote makes the colours)
        const bool noct = a.ct == nullptr;
        kern = a.L == 5 ? (pad ? (noct ? stylize_tiled_kernel<false, false, 5, true, true>
                                       : stylize_tiled_kernel<false, false, 5, true>)
                               : stylize_tiled_kernel<false, false, 5, false>)
             : a.L == 4 ? (pad ? stylize_tiled_kernel<false, false, 4, true> : stylize_tiled_kernel<false, false, 4, false>)
             : a.L == 3 ? (pad ? stylize_tiled_kernel<false, false, 3, true> : stylize_tiled_kernel<false, false, 3, false>)
                        : stylize_tiled_kernel<false, false, 0, false>;
    }
    cudaError_t e = ensure_smem(reinterpret_cast<const void*>(kern), (int)smem);
    if (e != cudaSuccess) return e;
    static const int carve = [] {
        const char* ev = getenv("SB_STYLIZE_CARVEOUT");
        return ev ? atoi(ev) : -1;
    }();
    if ((e = ensure_carveout(reinterpret_cast<const void*>(kern), carve)) != cudaSuccess) return e;
    dim3 grid((unsigned)((a.wt + TW - 1) / TW), (unsigned)((a.row_end - (a.row_begin & ~3) + TH - 1) / TH),
              (unsigned)n_frames);
    kern<<<grid, NT, smem, st>>>(a);
    *launches += 1;
    return cudaPeekAtLastError();
}

}  // namespace sb
