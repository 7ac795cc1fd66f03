// api.cu -- the C ABI of include/styleblit.h: argument validation, T2 conversion, launches,
// and the host-streaming batch pipeline.  No compute happens on the host: every step of the
// method runs in the kernels of lut_build.cu, stylize.cu / stylize_naive.cu and vote.cu.
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "../../include/styleblit.h"
#include "sb_kernels.cuh"

namespace {

thread_local char g_err[512] = "";
thread_local int g_launches = 0;

sb_status fail(sb_status s, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return s;
}

sb_status cuda_fail(cudaError_t e, const char* where) {
    return fail(SB_ECUDA, "%s: %s (%s)", where, cudaGetErrorString(e), cudaGetErrorName(e));
}

constexpr int kMaxDim = SB_MAX_DIM;

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

sb_status check_dims(const char* name, int32_t w, int32_t h) {
    if (w < 1 || w > kMaxDim || h < 1 || h > kMaxDim)
        return fail(SB_EINVAL, "%s: dimensions %dx%d outside [1,%d]", name, w, h, kMaxDim);
    return SB_OK;
}

// Which stylize kernel: the tiled kernel (any width; ragged widths take its per-pixel row I/O
// instantiation) needs L <= 9 (its tabled NearestSeed keys 1024 d + code fit 32 bits for
// h <= 2^9, stylize.cu) and every image side <= 32767 (packed candidate arithmetic); the
// one-thread-per-pixel kernel (signed coordinates, 64-bit distances) serves the rest.
// SB_KERNEL=naive selects it always (A/B).
bool use_naive(const sb::StylizeArgs& a) {
    static const int forced = [] {
        const char* e = getenv("SB_KERNEL");
        return (e && strcmp(e, "naive") == 0) ? 1 : 0;
    }();
    const int big = sb::kPackedMaxDim;
    return forced || a.L > 9 || a.wt > big || a.ht > big || a.ws > big || a.hs > big;
}

struct Prepared {
    sb::StylizeArgs s;
    sb::VoteArgs v;
    bool vote;
};

sb_status validate(const sb_params* prm, int32_t n_frames, const uint8_t* cs, const uint8_t* gs, int32_t ws,
                   int32_t hs, const uint32_t* lut, const uint8_t* gt, int32_t wt, int32_t ht, uint8_t* ct,
                   uint32_t* coords, bool device_outputs, Prepared* out) {
    if (!prm) return fail(SB_EINVAL, "prm is NULL");
    if (n_frames < 0) return fail(SB_EINVAL, "n_frames=%d < 0", n_frames);
    sb_status s;
    if ((s = check_dims("source (ws,hs)", ws, hs)) != SB_OK) return s;
    if ((s = check_dims("target (wt,ht)", wt, ht)) != SB_OK) return s;
    const float t = prm->threshold;
    if (!std::isfinite(t) || t < 0.f) return fail(SB_EINVAL, "threshold t=%g must be finite and >= 0", (double)t);
    if (prm->levels < 1 || prm->levels > SB_MAX_LEVELS)
        return fail(SB_EINVAL, "levels L=%d outside [1,%d]", prm->levels, SB_MAX_LEVELS);
    if (prm->blend_radius < 0 || prm->blend_radius > SB_MAX_RADIUS)
        return fail(SB_EINVAL, "blend_radius r=%d outside [0,%d]", prm->blend_radius, SB_MAX_RADIUS);
    if (prm->guide_channels < 2 || prm->guide_channels > 4)
        return fail(SB_EINVAL, "guide_channels C=%d not in {2,3,4}", prm->guide_channels);
    if (prm->flags & ~(SB_JITTER_ZERO | SB_NO_COLOR | SB_LABEL | SB_LUT_RGB | SB_HOST_RGB))
        return fail(SB_EINVAL, "flags 0x%x has unknown bits", prm->flags);
    if ((prm->flags & SB_LABEL) && (prm->label_channel < 0 || prm->label_channel > 3))
        return fail(SB_EINVAL, "label_channel=%d outside [0,3]", prm->label_channel);
    int rb = prm->row_begin, re = prm->row_end;
    if (rb == 0 && re == 0) re = ht;
    if (rb < 0 || re > ht || rb >= re)
        return fail(SB_EINVAL, "rows [row_begin=%d,row_end=%d) not a non-empty range inside [0,%d)", prm->row_begin,
                    prm->row_end, ht);
    if (!cs) return fail(SB_EINVAL, "cs (style exemplar C_S) is NULL");
    if (!gs) return fail(SB_EINVAL, "gs (source guide G_S) is NULL");
    if (!lut) return fail(SB_EINVAL, "lut is NULL");
    // per-frame buffers of an empty batch hold zero bytes: NULL is then valid for them
    const bool frames = n_frames > 0;
    if (!gt && frames) return fail(SB_EINVAL, "gt (target guide G_T) is NULL");
    const bool no_color = (prm->flags & SB_NO_COLOR) != 0;
    const int r = prm->blend_radius;
    if (!no_color && !ct && frames) return fail(SB_EINVAL, "ct is NULL (pass SB_NO_COLOR to skip colours)");
    if (r > 0 && !no_color && !coords && frames)
        return fail(SB_EINVAL, "coords is NULL but blend_radius=%d needs it", r);
    if (device_outputs) {
        if (!aligned16(cs) || !aligned16(gs) || !aligned16(gt) || (ct && !aligned16(ct)) ||
            (coords && !aligned16(coords)) || !aligned16(lut) || (prm->exemplar && !aligned16(prm->exemplar)))
            return fail(SB_EINVAL, "image/LUT/exemplar base pointers must be 16-byte aligned");
    }

    Prepared& p = *out;
    memset(&p, 0, sizeof(p));
    sb::StylizeArgs& a = p.s;
    a.cs = cs; a.gs = gs; a.ws = ws; a.hs = hs; a.lut = lut; a.gt = gt; a.wt = wt; a.ht = ht;
    a.exemplar = prm->exemplar;
    a.key_mask = (prm->flags & SB_LUT_RGB) ? 0xFFFFFFu : 0xFFFFu;
    a.L = prm->levels;
    const double t2 = std::ceil((double)t * (double)t);  // exact: t is a float (reading R2)
    a.T2 = t2 >= 4294967295.0 ? 0xFFFFFFFFu : (uint32_t)t2;
    a.cmask = prm->guide_channels == 4 ? 0xFFFFFFFFu : (prm->guide_channels == 3 ? 0x00FFFFFFu : 0x0000FFFFu);
    const bool unit = (prm->weights[0] | prm->weights[1] | prm->weights[2] | prm->weights[3]) == 0;
    bool ones = true;
    for (int c = 0; c < 4; ++c) {
        a.w[c] = unit ? 1u : prm->weights[c];
        if (c < prm->guide_channels && a.w[c] != 1u) ones = false;
    }
    a.lmask = 0;
    if (prm->flags & SB_LABEL) {
        a.lmask = 0xFFu << (8 * prm->label_channel);
        a.cmask &= ~a.lmask;  // the label byte does not enter e
    }
    a.ext = (!ones || a.lmask) ? 1 : 0;
    a.zero_jitter = (prm->flags & SB_JITTER_ZERO) ? 1 : 0;
    a.seed_base = prm->seed;
    a.coords = coords;
    p.vote = (r > 0) && !no_color;
    // rows computed by the stylize kernel: the output strip plus the vote's coords halo
    a.row_begin = p.vote ? (rb - r < 0 ? 0 : rb - r) : rb;
    a.row_end = p.vote ? (re + r > ht ? ht : re + r) : re;
    a.ct = (no_color || p.vote) ? nullptr : ct;
    if (p.vote) {
        sb::VoteArgs& v = p.v;
        v.coords = coords; v.cs = cs; v.ws = ws; v.hs = hs; v.wt = wt; v.ht = ht; v.r = r; v.ct = ct;
        v.cs_pad = prm->exemplar ? prm->exemplar + (size_t)hs * ((size_t)1 << 18) : nullptr;
        v.row_begin = rb; v.row_end = re;
    }
    return SB_OK;
}

// Launch stylize (+vote) for n frames starting at frame offset f0 of the given buffers.
sb_status launch_frames(Prepared& p, int n_frames, const uint32_t* frame_seeds, uint32_t seed_base_f0,
                        uint8_t* level, cudaStream_t st) {
    const int64_t fpx = (int64_t)p.s.wt * p.s.ht;
    // Seeds of the form s0 + i (the default, and the usual explicit choice) need no parameter
    // array: the kernel derives them, and one launch covers up to 65535 frames (grid.z), so small
    // frames fill many waves instead of a few tail-bound launches of kSeedsPerLaunch frames.
    if (frame_seeds) {
        bool ap = true;
        for (int i = 1; i < n_frames && ap; ++i) ap = frame_seeds[i] == frame_seeds[0] + (uint32_t)i;
        if (ap && n_frames > 0) {
            seed_base_f0 = frame_seeds[0];
            frame_seeds = nullptr;
        }
    }
    const int per = frame_seeds ? sb::kSeedsPerLaunch : 65535;
    for (int f0 = 0; f0 < n_frames; f0 += per) {
        const int nf = (n_frames - f0) < per ? (n_frames - f0) : per;
        sb::StylizeArgs a = p.s;
        a.gt = p.s.gt + 4 * fpx * f0;
        a.ct = p.s.ct ? p.s.ct + 4 * fpx * f0 : nullptr;
        a.coords = p.s.coords ? p.s.coords + fpx * f0 : nullptr;
        a.level = level ? level + fpx * f0 : nullptr;
        a.has_seeds = frame_seeds ? 1 : 0;
        a.seed_base = seed_base_f0 + (uint32_t)f0;
        if (frame_seeds) memcpy(a.seeds, frame_seeds + f0, sizeof(uint32_t) * nf);
        cudaError_t e = use_naive(a) ? sb::launch_stylize_naive(a, nf, st, &g_launches)
                                        : sb::launch_stylize_tiled(a, nf, st, &g_launches);
        if (e != cudaSuccess) return cuda_fail(e, "stylize launch");
        if (p.vote) {
            sb::VoteArgs v = p.v;
            v.coords = a.coords;
            v.ct = p.v.ct + 4 * fpx * f0;
            e = sb::launch_vote(v, nf, st, &g_launches);
            if (e != cudaSuccess) return cuda_fail(e, "vote launch");
        }
    }
    return SB_OK;
}

// The host pipeline's streams and events: created on first use per (thread, device) and
// reused by every later sb_stylize_batch_host call on that thread and device (one pipeline
// runs at a time per thread, and every call drains it before returning).
struct Pipeline {
    cudaStream_t h2d = nullptr, cmp = nullptr, d2h = nullptr;
    cudaEvent_t start = nullptr;
    cudaEvent_t in_ready[8] = {}, cmp_done[8] = {}, out_done[8] = {};
};

sb_status pipeline(Pipeline** out) {
    thread_local Pipeline cache[16];
    thread_local bool ready[16] = {};
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    if (dev < 0 || dev >= 16) return fail(SB_EUNSUPPORTED, "device index %d >= 16", dev);
    Pipeline& p = cache[dev];
    if (!ready[dev]) {
        Pipeline q;
        auto undo = [&](cudaError_t err, const char* what) {
            for (cudaStream_t s : {q.h2d, q.cmp, q.d2h})
                if (s) cudaStreamDestroy(s);
            for (int k = 0; k < 8; ++k)
                for (cudaEvent_t ev : {q.in_ready[k], q.cmp_done[k], q.out_done[k]})
                    if (ev) cudaEventDestroy(ev);
            if (q.start) cudaEventDestroy(q.start);
            return cuda_fail(err, what);
        };
        if ((e = cudaStreamCreateWithFlags(&q.h2d, cudaStreamNonBlocking)) != cudaSuccess ||
            (e = cudaStreamCreateWithFlags(&q.cmp, cudaStreamNonBlocking)) != cudaSuccess ||
            (e = cudaStreamCreateWithFlags(&q.d2h, cudaStreamNonBlocking)) != cudaSuccess)
            return undo(e, "pipeline stream creation");
        if ((e = cudaEventCreateWithFlags(&q.start, cudaEventDisableTiming)) != cudaSuccess)
            return undo(e, "pipeline event creation");
        for (int k = 0; k < 8; ++k)
            if ((e = cudaEventCreateWithFlags(&q.in_ready[k], cudaEventDisableTiming)) != cudaSuccess ||
                (e = cudaEventCreateWithFlags(&q.cmp_done[k], cudaEventDisableTiming)) != cudaSuccess ||
                (e = cudaEventCreateWithFlags(&q.out_done[k], cudaEventDisableTiming)) != cudaSuccess)
                return undo(e, "pipeline event creation");
        p = q;
        ready[dev] = true;
    }
    *out = &p;
    return SB_OK;
}

}  // namespace

extern "C" {

size_t sb_lut_workspace_bytes(void) { return 65536 * (sizeof(uint32_t) + 2 * sizeof(uint32_t)); }

sb_status sb_build_lut(const uint8_t* gs, int32_t ws, int32_t hs, uint32_t* lut, void* workspace, void* stream) {
    g_launches = 0;
    sb_status s;
    if (!gs) return fail(SB_EINVAL, "gs (source guide G_S) is NULL");
    if (!lut) return fail(SB_EINVAL, "lut is NULL");
    if (!workspace) return fail(SB_EINVAL, "workspace is NULL (need sb_lut_workspace_bytes() bytes)");
    if ((s = check_dims("source (ws,hs)", ws, hs)) != SB_OK) return s;
    if (!aligned16(gs) || !aligned16(workspace) || !aligned16(lut))
        return fail(SB_EINVAL, "gs/lut/workspace must be 16-byte aligned");
    cudaError_t e = sb::launch_build_lut(gs, ws, hs, lut, workspace, (cudaStream_t)stream, &g_launches);
    if (e != cudaSuccess) return cuda_fail(e, "sb_build_lut launch");
    return SB_OK;
}

size_t sb_exemplar_bytes(int32_t ws, int32_t hs) {
    if (ws < 1 || hs < 1 || ws > 32767 || hs > SB_EXEMPLAR_MAX_HS) return 0;
    return (size_t)2 * (size_t)hs * ((size_t)1 << 18);
}

sb_status sb_prepare_exemplar(const uint8_t* cs, const uint8_t* gs, int32_t ws, int32_t hs, uint8_t* exemplar,
                              void* stream) {
    g_launches = 0;
    sb_status s;
    if (!cs) return fail(SB_EINVAL, "cs (style exemplar C_S) is NULL");
    if (!gs) return fail(SB_EINVAL, "gs (source guide G_S) is NULL");
    if (!exemplar) return fail(SB_EINVAL, "exemplar is NULL (need sb_exemplar_bytes(ws, hs) bytes)");
    if ((s = check_dims("source (ws,hs)", ws, hs)) != SB_OK) return s;
    if (hs > SB_EXEMPLAR_MAX_HS)
        return fail(SB_EUNSUPPORTED, "hs=%d > SB_EXEMPLAR_MAX_HS=%d: the strided copy would need %zu MiB; pass "
                    "exemplar = NULL instead", hs, SB_EXEMPLAR_MAX_HS, ((size_t)hs << 19) >> 20);
    if (!aligned16(cs) || !aligned16(gs) || !aligned16(exemplar))
        return fail(SB_EINVAL, "cs/gs/exemplar must be 16-byte aligned");
    cudaError_t e = sb::launch_prepare_exemplar(cs, gs, ws, hs, exemplar, (cudaStream_t)stream, &g_launches);
    if (e != cudaSuccess) return cuda_fail(e, "sb_prepare_exemplar launch");
    return SB_OK;
}

size_t sb_lut3_workspace_bytes(void) { return ((size_t)1 << 24) * 2 * sizeof(uint32_t); }

sb_status sb_build_lut3(const uint8_t* gs, int32_t ws, int32_t hs, uint32_t* lut3, void* workspace, void* stream) {
    g_launches = 0;
    sb_status s;
    if (!gs) return fail(SB_EINVAL, "gs (source guide G_S) is NULL");
    if (!lut3) return fail(SB_EINVAL, "lut3 is NULL");
    if (!workspace) return fail(SB_EINVAL, "workspace is NULL (need sb_lut3_workspace_bytes() bytes)");
    if ((s = check_dims("source (ws,hs)", ws, hs)) != SB_OK) return s;
    if (!aligned16(gs) || !aligned16(workspace) || !aligned16(lut3))
        return fail(SB_EINVAL, "gs/lut3/workspace must be 16-byte aligned");
    cudaError_t e = sb::launch_build_lut3(gs, ws, hs, lut3, workspace, (cudaStream_t)stream, &g_launches);
    if (e != cudaSuccess) return cuda_fail(e, "sb_build_lut3 launch");
    return SB_OK;
}

sb_status sb_stylize(const sb_params* prm, const uint8_t* cs, const uint8_t* gs, int32_t ws, int32_t hs,
                     const uint32_t* lut, const uint8_t* gt, int32_t wt, int32_t ht, uint8_t* ct, uint32_t* coords,
                     uint8_t* level, void* stream) {
    return sb_stylize_batch(prm, 1, nullptr, cs, gs, ws, hs, lut, gt, wt, ht, ct, coords, level, stream);
}

sb_status sb_stylize_batch(const sb_params* prm, int32_t n_frames, const uint32_t* frame_seeds, const uint8_t* cs,
                           const uint8_t* gs, int32_t ws, int32_t hs, const uint32_t* lut, const uint8_t* gt,
                           int32_t wt, int32_t ht, uint8_t* ct, uint32_t* coords, uint8_t* level, void* stream) {
    g_launches = 0;
    if (prm && (prm->flags & SB_HOST_RGB))
        return fail(SB_EINVAL, "flags: SB_HOST_RGB applies to sb_stylize_batch_host only");
    Prepared p;
    sb_status s = validate(prm, n_frames, cs, gs, ws, hs, lut, gt, wt, ht, ct, coords, true, &p);
    if (s != SB_OK) return s;
    if (level && !aligned16(level)) return fail(SB_EINVAL, "level must be 16-byte aligned");
    if (n_frames == 0) return SB_OK;
    return launch_frames(p, n_frames, frame_seeds, prm->seed, level, (cudaStream_t)stream);
}

sb_status sb_vote(const uint32_t* coords, int32_t n_frames, int32_t wt, int32_t ht, const uint8_t* cs, int32_t ws,
                  int32_t hs, int32_t r, uint8_t* ct, int32_t row_begin, int32_t row_end, const uint8_t* exemplar,
                  void* stream) {
    g_launches = 0;
    sb_status s;
    if (n_frames < 0) return fail(SB_EINVAL, "n_frames=%d < 0", n_frames);
    if (!coords && n_frames > 0) return fail(SB_EINVAL, "coords is NULL");  // NULL is valid for 0 frames
    if (!cs) return fail(SB_EINVAL, "cs (style exemplar C_S) is NULL");
    if (!ct && n_frames > 0) return fail(SB_EINVAL, "ct is NULL");
    if ((s = check_dims("source (ws,hs)", ws, hs)) != SB_OK) return s;
    if ((s = check_dims("target (wt,ht)", wt, ht)) != SB_OK) return s;
    if (r < 0 || r > SB_MAX_RADIUS) return fail(SB_EINVAL, "r=%d outside [0,%d]", r, SB_MAX_RADIUS);
    if (row_begin == 0 && row_end == 0) row_end = ht;
    if (row_begin < 0 || row_end > ht || row_begin >= row_end)
        return fail(SB_EINVAL, "rows [row_begin=%d,row_end=%d) not a non-empty range inside [0,%d)", row_begin, row_end,
                    ht);
    if (!aligned16(coords) || !aligned16(cs) || !aligned16(ct) || (exemplar && !aligned16(exemplar)))
        return fail(SB_EINVAL, "coords/cs/ct/exemplar must be 16-byte aligned");
    const int64_t fpx = (int64_t)wt * ht;
    for (int f0 = 0; f0 < n_frames; f0 += 65535) {
        const int nf = (n_frames - f0) < 65535 ? (n_frames - f0) : 65535;
        sb::VoteArgs v{};
        v.coords = coords + fpx * f0; v.cs = cs; v.ws = ws; v.hs = hs; v.wt = wt; v.ht = ht; v.r = r;
        v.cs_pad = exemplar ? exemplar + (size_t)hs * ((size_t)1 << 18) : nullptr;
        v.ct = ct + 4 * fpx * f0; v.row_begin = row_begin; v.row_end = row_end;
        cudaError_t e = sb::launch_vote(v, nf, (cudaStream_t)stream, &g_launches);
        if (e != cudaSuccess) return cuda_fail(e, "vote launch");
    }
    return SB_OK;
}

// One slot of the host pipeline: G_T, C_T and coords of one frame, each 256-byte aligned.
static size_t host_seg_bytes(int32_t wt, int32_t ht) { return (((size_t)wt * (size_t)ht * 4) + 255) & ~(size_t)255; }

size_t sb_host_workspace_bytes(int32_t wt, int32_t ht, int32_t blend_radius, int32_t depth) {
    if (wt < 1 || ht < 1 || depth < 1) return 0;
    (void)blend_radius;
    // per slot: G_T, C_T, coords (RGBA / uint32) + packed-RGB staging in and out (SB_HOST_RGB)
    return 5 * host_seg_bytes(wt, ht) * (size_t)depth;
}

sb_status sb_stylize_batch_host(const sb_params* prm, int32_t n_frames, const uint32_t* frame_seeds,
                                const uint8_t* cs, const uint8_t* gs, int32_t ws, int32_t hs, const uint32_t* lut,
                                const uint8_t* gt_host, int32_t wt, int32_t ht, uint8_t* ct_host,
                                uint32_t* coords_host, void* workspace, size_t workspace_bytes, int32_t depth,
                                void* stream) {
    g_launches = 0;
    if (n_frames < 0) return fail(SB_EINVAL, "n_frames=%d < 0", n_frames);
    if (depth < 1 || depth > 8) return fail(SB_EINVAL, "depth=%d outside [1,8]", depth);
    if (!workspace) return fail(SB_EINVAL, "workspace is NULL");
    if (!gt_host && n_frames > 0) return fail(SB_EINVAL, "gt_host is NULL");  // NULL is valid for 0 frames
    if (!ct_host && n_frames > 0 && !(prm && (prm->flags & SB_NO_COLOR))) return fail(SB_EINVAL, "ct_host is NULL");
    if (workspace_bytes < sb_host_workspace_bytes(wt, ht, prm ? prm->blend_radius : 0, depth))
        return fail(SB_EINVAL, "workspace_bytes=%zu < sb_host_workspace_bytes()=%zu", workspace_bytes,
                    sb_host_workspace_bytes(wt, ht, prm ? prm->blend_radius : 0, depth));
    if (!aligned16(workspace)) return fail(SB_EINVAL, "workspace must be 16-byte aligned");
    // Validate against slot 0 (device pointers) so the per-frame launches cannot fail validation.
    if (wt < 1 || ht < 1) return fail(SB_EINVAL, "target (wt,ht): dimensions %dx%d", wt, ht);
    const size_t fpx = (size_t)wt * (size_t)ht;
    const size_t seg = host_seg_bytes(wt, ht);
    auto slot_ptr = [&](int k, int part) { return static_cast<uint8_t*>(workspace) + ((size_t)k * 5 + part) * seg; };
    const bool rgb = prm && (prm->flags & SB_HOST_RGB);
    if (rgb) {
        if (prm->guide_channels > 3) return fail(SB_EINVAL, "SB_HOST_RGB needs guide_channels <= 3");
        if ((prm->flags & SB_LABEL) && prm->label_channel == 3)
            return fail(SB_EINVAL, "SB_HOST_RGB: label_channel 3 is not carried by packed RGB frames");
        if (wt % 4 != 0) return fail(SB_EUNSUPPORTED, "SB_HOST_RGB needs wt %% 4 == 0 (got %d)", wt);
    }
    const size_t hb = rgb ? 3 : 4;  // host bytes per pixel
    Prepared p;
    sb_status s = validate(prm, n_frames, cs, gs, ws, hs, lut, slot_ptr(0, 0), wt, ht, slot_ptr(0, 1),
                           reinterpret_cast<uint32_t*>(slot_ptr(0, 2)), true, &p);
    if (s != SB_OK) return s;
    if (prm->row_begin != 0 || prm->row_end != 0) return fail(SB_EUNSUPPORTED, "host batches are whole frames");
    if (n_frames == 0) return SB_OK;

    cudaStream_t user = (cudaStream_t)stream;
    Pipeline* pl = nullptr;
    if ((s = pipeline(&pl)) != SB_OK) return s;
    cudaStream_t sH2D = pl->h2d, sCmp = pl->cmp, sD2H = pl->d2h;
    cudaEvent_t start = pl->start, *inReady = pl->in_ready, *cmpDone = pl->cmp_done, *outDone = pl->out_done;
    cudaError_t e;
    // everything is ordered after the work already queued on the caller's stream
    if ((e = cudaEventRecord(start, user)) != cudaSuccess || (e = cudaStreamWaitEvent(sH2D, start, 0)) != cudaSuccess ||
        (e = cudaStreamWaitEvent(sCmp, start, 0)) != cudaSuccess)
        return cuda_fail(e, "pipeline ordering");
    int total_launches = 0;
    sb_status st = SB_OK;
    for (int i = 0; i < n_frames && st == SB_OK; ++i) {
        const int k = i % depth;
        uint8_t* dgt = slot_ptr(k, 0);
        uint8_t* dct = slot_ptr(k, 1);
        uint32_t* dco = reinterpret_cast<uint32_t*>(slot_ptr(k, 2));
        if (i >= depth && (e = cudaStreamWaitEvent(sH2D, outDone[k], 0)) != cudaSuccess) {  // slot free again
            st = cuda_fail(e, "pipeline ordering");
            break;
        }
        uint8_t* stage_in = slot_ptr(k, 3);
        uint8_t* stage_out = slot_ptr(k, 4);
        e = cudaMemcpyAsync(rgb ? stage_in : dgt, gt_host + hb * fpx * (size_t)i, hb * fpx, cudaMemcpyHostToDevice,
                            sH2D);
        if (e != cudaSuccess) { st = cuda_fail(e, "H2D copy"); break; }
        if ((e = cudaEventRecord(inReady[k], sH2D)) != cudaSuccess ||
            (e = cudaStreamWaitEvent(sCmp, inReady[k], 0)) != cudaSuccess) {
            st = cuda_fail(e, "pipeline ordering");
            break;
        }
        if (rgb) {
            e = sb::launch_unpack_rgb(stage_in, dgt, fpx, sCmp, &total_launches);
            if (e != cudaSuccess) { st = cuda_fail(e, "unpack launch"); break; }
        }
        Prepared pf = p;
        pf.s.gt = dgt;
        pf.s.ct = pf.s.ct ? dct : nullptr;
        pf.s.coords = dco;
        if (pf.vote) { pf.v.coords = dco; pf.v.ct = dct; }
        const uint32_t seed_i = frame_seeds ? frame_seeds[i] : prm->seed + (uint32_t)i;
        st = launch_frames(pf, 1, nullptr, seed_i, nullptr, sCmp);
        total_launches += g_launches;
        g_launches = 0;
        if (st != SB_OK) break;
        if (rgb && ct_host) {
            e = sb::launch_pack_rgb(dct, stage_out, fpx, sCmp, &total_launches);
            if (e != cudaSuccess) { st = cuda_fail(e, "pack launch"); break; }
        }
        if ((e = cudaEventRecord(cmpDone[k], sCmp)) != cudaSuccess ||
            (e = cudaStreamWaitEvent(sD2H, cmpDone[k], 0)) != cudaSuccess) {
            st = cuda_fail(e, "pipeline ordering");
            break;
        }
        if (ct_host) {
            e = cudaMemcpyAsync(ct_host + hb * fpx * (size_t)i, rgb ? stage_out : dct, hb * fpx,
                                cudaMemcpyDeviceToHost, sD2H);
            if (e != cudaSuccess) { st = cuda_fail(e, "D2H copy"); break; }
        }
        if (coords_host) {
            e = cudaMemcpyAsync(coords_host + fpx * (size_t)i, dco, 4 * fpx, cudaMemcpyDeviceToHost, sD2H);
            if (e != cudaSuccess) { st = cuda_fail(e, "D2H copy"); break; }
        }
        if ((e = cudaEventRecord(outDone[k], sD2H)) != cudaSuccess) {
            st = cuda_fail(e, "pipeline ordering");
            break;
        }
    }
    // drain all three streams (also after an error, so the cached pipeline is idle again)
    e = cudaStreamSynchronize(sD2H);
    cudaError_t e2 = cudaStreamSynchronize(sCmp);
    cudaError_t e3 = cudaStreamSynchronize(sH2D);
    if (st == SB_OK && e != cudaSuccess) st = cuda_fail(e, "pipeline sync");
    if (st == SB_OK && e2 != cudaSuccess) st = cuda_fail(e2, "pipeline sync");
    if (st == SB_OK && e3 != cudaSuccess) st = cuda_fail(e3, "pipeline sync");
    g_launches = total_launches;
    return st;
}

int32_t sb_last_launch_count(void) { return g_launches; }
const char* sb_last_error(void) { return g_err; }
const char* sb_version(void) { return "styleblit-b200 0.1 (sm_100a)"; }

}  // extern "C"
