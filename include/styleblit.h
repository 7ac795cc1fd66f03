/*
 * styleblit.h -- C ABI of the B200-native StyleBlit hot path (arXiv 1807.03249).
 *
 * The boundary of SURVEY.md 8(b).  Three entry points carry the method:
 *
 *   sb_build_lut      the guide look-up table of PAPER.md:246-249 ("a simple look-up table
 *                     to retrieve ... the corresponding location in the source exemplar")
 *                     and Alg. 2 line 383 (u* = argmin_u ||G_T[q_l] - G_S[u]||, "found via
 *                     lookup").
 *   sb_stylize        Alg. 2 "ParallelStyleBlit" for every target pixel,
 *                     followed, when blend_radius > 0, by the voting step of PAPER.md:412-421.
 *   sb_stylize_batch  the same over n frames with per-frame jitter seeds -- the animation
 *                     extension of PAPER.md:423-433 ("randomization of seed points").
 *
 * plus sb_stylize_batch_host (the same batch with HOST frame buffers, streamed through
 * the device by a double-buffered copy/compute pipeline), sb_vote (the vote alone),
 * sb_build_lut3 (the exact three-channel guide search), sb_prepare_exemplar (an optional
 * strided exemplar copy that makes packed source coordinates their own gather index) and
 * status helpers.
 *
 * Conventions (all entry points)
 * ------------------------------
 *  - Images are row-major, contiguous, 4 bytes per pixel (uint8 x4; RGBA8 colours,
 *    up to 4 guide channels), pixel (x,y) at byte offset 4*(y*W + x).  Frames of a batch
 *    are contiguous: frame i starts at byte 4*W*H*i.  Base pointers must be 16-byte
 *    aligned.  1 <= W, H <= 65535 (SB_MAX_DIM).  Sides up to 32767 run on the tiled
 *    packed-coordinate kernels; larger ones on per-pixel kernels with signed coordinates
 *    (identical results, slower).
 *  - Source coordinates are packed x | y << 16 (uint32) in SOURCE space.
 *  - The LUT has 65536 uint32 entries indexed by key = G[0] | G[1] << 8 (the first two
 *    guide channels, the paper's "two values").
 *  - Unless a name says _host, every pointer is a DEVICE pointer.  The caller owns every
 *    buffer; the library allocates no device memory and keeps no state between calls except
 *    host-side caches that never change results: per device, the SM count and the kernels'
 *    shared-memory attributes; per thread and device, the 3 streams and 25 events of the
 *    sb_stylize_batch_host pipeline (created on its first call, drained before it returns).
 *  - Work is enqueued on `stream` (a cudaStream_t passed as void*; NULL = legacy default
 *    stream) and the call returns after launch (asynchronous), except
 *    sb_stylize_batch_host, which returns when its results are in host memory.
 *  - Errors are status codes, never exceptions.  SB_EINVAL: a null required pointer, a
 *    size or parameter out of range, misalignment; sb_last_error() names the argument.
 *    SB_ECUDA: a launch/runtime error reported by the CUDA runtime (the message carries
 *    cudaGetErrorString).  Errors that happen while a kernel executes surface at the
 *    caller's next synchronisation, as with any CUDA call.
 *  - Thread safety: calls are reentrant; sb_last_error() is thread-local.
 */
#ifndef STYLEBLIT_H
#define STYLEBLIT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    SB_OK = 0,
    SB_EINVAL = 1,        /* invalid argument (see sb_last_error)          */
    SB_EUNSUPPORTED = 2,  /* valid but not supported by this build         */
    SB_ECUDA = 3          /* CUDA runtime error                            */
} sb_status;

/* sb_params.flags */
#define SB_JITTER_ZERO 0x1u  /* RandomJitterTable == 0: seeds on the regular grid (tests)  */
#define SB_NO_COLOR    0x2u  /* compute coords/levels only; ct may be NULL                 */
#define SB_LABEL       0x4u  /* guide byte `label_channel` is a segmentation label (below)   */
#define SB_LUT_RGB     0x8u  /* `lut` is the exact 3-channel table of sb_build_lut3 (2^24
                                entries, key G[0] | G[1]<<8 | G[2]<<16) instead of the
                                2-channel table                                            */
#define SB_HOST_RGB   0x10u  /* sb_stylize_batch_host only: the HOST frames are packed 3 bytes
                                per pixel -- gt_host holds guide channels 0..2 (channel 3 is
                                taken as 0; needs guide_channels <= 3 and no label in byte 3)
                                and ct_host receives C_T channels 0..2 -- so 3/4 of the PCIe
                                bytes move; the device kernels unpack/pack them.  wt % 4 == 0. */

#define SB_MAX_DIM 65535      /* image sides W, H in [1, SB_MAX_DIM] (target and source)      */
#define SB_MAX_LEVELS 15      /* level l uses spacing h = 2^l, l in [1, SB_MAX_LEVELS]; L <= 9
                                 on the tiled kernel, L in 10..15 on the per-pixel kernel     */
#define SB_MAX_RADIUS 8       /* voting radius r in [0, SB_MAX_RADIUS]; the tiled SWAR vote sums
                                 16-bit lanes (r = 8: two lane pairs, dy < 0 and dy >= 0)     */

typedef struct {
    /* t: the threshold of Alg. 2 line 385 ("e < t"), in 8-bit guide units.  The error e is
     * the Euclidean norm over the first guide_channels bytes; the test is evaluated exactly
     * as D < ceil(t*t) on the integer squared error D.  0 <= t, finite.  t = 0 accepts
     * nothing (every pixel takes the level-0 look-up, the Lit Sphere transfer).           */
    float    threshold;
    /* L: number of hierarchy levels; level l uses seed spacing
     * h = 2^l, visited l = L..1 (coarse to fine).  1 <= L <= SB_MAX_LEVELS.               */
    int32_t  levels;
    /* r: voting radius; the patch of a target pixel q is the
     * (2r+1)x(2r+1) square around it.  0 = plain blit C_T[p] = C_S[s(p)].              */
    int32_t  blend_radius;
    /* C: guide channels entering e, 2..4.  The LUT key always uses channels 0 and 1.      */
    int32_t  guide_channels;
    /* Jitter seed of the RandomJitterTable; frame i of a batch uses
     * frame_seeds[i] (default seed + i).                                */
    uint32_t seed;
    uint32_t flags;       /* SB_JITTER_ZERO | SB_NO_COLOR | SB_LABEL | SB_LUT_RGB          */
    /* Output strip [row_begin, row_end) of the target (0,0 = all rows).  Only these rows
     * of ct are written; with r > 0 the coords/level rows [row_begin - r, row_end + r)
     * (clipped) are written because the vote reads them.  Results equal the whole-frame
     * results.                                                                           */
    int32_t  row_begin, row_end;
    /* Per-channel integer weights of the squared error: e^2 = sum_c w_c (G_T[p].c - G_S[s].c)^2
     * over the first guide_channels bytes (SPEC compose_guides).  All zero = unit
     * weights (the paper's plain norm).                                                   */
    uint8_t  weights[4];
    /* With SB_LABEL: guide byte label_channel (0..3) holds a segmentation label; a candidate
     * whose label differs from the target pixel's is rejected at every level -- the
     * "segmentation guide which prevents chunks to cross boundaries" of PAPER.md:514-517 --
     * and that byte does not enter e.  (The level-0 look-up ignores labels.)              */
    int32_t  label_channel;
    /* Optional device pointer (16-byte aligned): the strided exemplar copy written by
     * sb_prepare_exemplar(cs, gs) for THIS cs/gs.  NULL = read cs and gs directly.  With it,
     * the exemplar gathers of Alg. 2 line 384 (G_S[s]), of the blit (C_S[s], line 387) and of
     * the vote index the copy with the packed coordinate x | y<<16 itself; results are
     * identical, only the address arithmetic per gather is gone.  Used by the tiled stylize
     * kernel for L in 3..5 without weights/labels and by the vote; ignored elsewhere.      */
    const uint8_t* exemplar;
} sb_params;

/* Bytes of device workspace sb_build_lut needs (65536 x 12: sites, then per-column nearest sites). */
size_t sb_lut_workspace_bytes(void);

/* Guide LUT: lut[k] = x | y<<16 of the source pixel u minimising
 * (k0 - G_S[u].c0)^2 + (k1 - G_S[u].c1)^2, k = k0 | k1<<8, ties -> the smallest
 * row-major index y*ws + x (SURVEY.md 8(c) reading R10).
 *   gs         device, ws*hs*4 bytes, the source guide G_S (channels 2,3 ignored)
 *   lut        device, 65536 uint32, output
 *   workspace  device, sb_lut_workspace_bytes() bytes, scratch (contents undefined after) */
sb_status sb_build_lut(const uint8_t* gs, int32_t ws, int32_t hs, uint32_t* lut,
                       void* workspace, void* stream);

/* Bytes of device workspace sb_build_lut3 needs (2^24 x 8 = 128 MiB). */
size_t sb_lut3_workspace_bytes(void);

/* Exact three-channel guide search, tabulated (the look-up "or a tree
 * search"; reading R26): lut3[k] = x | y<<16 of the source
 * pixel u minimising sum_{c<3} (k_c - G_S[u].c)^2, k = k0 | k1<<8 | k2<<16, ties -> the
 * smallest row-major index (the rule of R10).  Used by sb_stylize* with SB_LUT_RGB.
 *   gs         device, ws*hs*4 bytes, the source guide G_S (channel 3 ignored)
 *   lut3       device, 2^24 uint32 (64 MiB), output
 *   workspace  device, sb_lut3_workspace_bytes() bytes, scratch (contents undefined after) */
sb_status sb_build_lut3(const uint8_t* gs, int32_t ws, int32_t hs, uint32_t* lut3,
                        void* workspace, void* stream);

/* Bytes of the strided exemplar copy for a ws x hs exemplar: G_S and C_S, each hs rows of
 * 2^16 pixels (row stride 256 KiB), i.e. 2 * hs * 2^18 bytes (256 MiB for hs = 512, 1 GiB
 * for hs = 2048).  Only ws pixels of a row are written and read (2 * ws * hs * 4 bytes, the
 * exemplar's own size, are ever touched), but the whole range must be allocated.  Capped at
 * hs <= SB_EXEMPLAR_MAX_HS (2 GiB): returns 0 above it (and for ws > 32767), and such
 * exemplars are used directly (sb_params.exemplar = NULL; identical results, a few percent
 * slower).                                                                                 */
#define SB_EXEMPLAR_MAX_HS 4096
size_t sb_exemplar_bytes(int32_t ws, int32_t hs);

/* The strided exemplar copy used through sb_params.exemplar: exemplar[0 .. hs*2^18) holds
 * G_S with pixel (x,y) at byte 4*(y*65536 + x), exemplar[hs*2^18 ..) holds C_S the same way,
 * so a packed source coordinate x | y<<16 is its own pixel index (the two
 * exemplar gathers of Alg. 2).  Rebuild it whenever cs or gs change (like the LUT).
 *   cs, gs     device, ws*hs*4: style exemplar C_S and source guide G_S
 *   exemplar   device, sb_exemplar_bytes(ws, hs) bytes, 16-byte aligned, output
 * SB_EUNSUPPORTED for hs > SB_EXEMPLAR_MAX_HS.                                            */
sb_status sb_prepare_exemplar(const uint8_t* cs, const uint8_t* gs, int32_t ws, int32_t hs,
                              uint8_t* exemplar, void* stream);

/* Alg. 2 for every target pixel, then the vote when prm->blend_radius > 0.
 *   cs, gs     device, ws*hs*4: style exemplar C_S and source guide G_S
 *   lut        device, 65536 uint32 from sb_build_lut(gs); with SB_LUT_RGB, 2^24 uint32
 *              from sb_build_lut3(gs)
 *   gt         device, wt*ht*4: target guide G_T
 *   ct         device, wt*ht*4, output C_T (may be NULL iff SB_NO_COLOR)
 *   coords     device, wt*ht uint32, output source coordinate per pixel (the NNF,
 *              PAPER.md:414-417); may be NULL iff blend_radius == 0
 *   level      device, wt*ht bytes, output accepting level (L..1; 0 = no level accepted,
 *              the look-up fallback); may be NULL                                         */
sb_status sb_stylize(const sb_params* prm,
                     const uint8_t* cs, const uint8_t* gs, int32_t ws, int32_t hs,
                     const uint32_t* lut,
                     const uint8_t* gt, int32_t wt, int32_t ht,
                     uint8_t* ct, uint32_t* coords, uint8_t* level, void* stream);

/* n_frames frames of wt x ht (contiguous), frame i jittered with frame_seeds[i]
 * (HOST array of n_frames; NULL => prm->seed + i mod 2^32).  Same buffers and rules as
 * sb_stylize, each with n_frames frames.  Seeds of the form s0 + i (mod 2^32) -- NULL, or an
 * explicit array of that form -- run as one launch per 65535 frames; other seed arrays as one
 * launch per 512 frames (they travel in the kernel parameters).  n_frames = 0 is a valid empty batch: SB_OK, no
 * launch, and the per-frame buffers (gt, ct, coords, level) may then be NULL (likewise for
 * sb_vote and sb_stylize_batch_host).                                                     */
sb_status sb_stylize_batch(const sb_params* prm, int32_t n_frames, const uint32_t* frame_seeds,
                           const uint8_t* cs, const uint8_t* gs, int32_t ws, int32_t hs,
                           const uint32_t* lut,
                           const uint8_t* gt, int32_t wt, int32_t ht,
                           uint8_t* ct, uint32_t* coords, uint8_t* level, void* stream);

/* The voting step alone (SPEC resolve_colors/vote): C_T from a given
 * coordinate field (the NNF of PAPER.md:414-417), for n_frames contiguous frames.
 *   coords     device, n_frames*wt*ht uint32 (x | y<<16 in source space, inside the source)
 *   cs         device, ws*hs*4, style exemplar C_S
 *   r          voting radius, 0..SB_MAX_RADIUS (0 = blit)
 *   ct         device, n_frames*wt*ht*4, output; only rows [row_begin, row_end) are written
 *              (0,0 = all rows); coords rows [row_begin - r, row_end + r) are read.
 *   exemplar   NULL, or the strided copy of sb_prepare_exemplar for this cs (speed only:
 *              the colour gathers then index it with packed coordinates; same results)     */
sb_status sb_vote(const uint32_t* coords, int32_t n_frames, int32_t wt, int32_t ht,
                  const uint8_t* cs, int32_t ws, int32_t hs, int32_t r,
                  uint8_t* ct, int32_t row_begin, int32_t row_end, const uint8_t* exemplar,
                  void* stream);

/* Bytes of device workspace sb_stylize_batch_host needs for frames of wt x ht with
 * `depth` frames in flight per stage (2 = double buffering). */
size_t sb_host_workspace_bytes(int32_t wt, int32_t ht, int32_t blend_radius, int32_t depth);

/* sb_stylize_batch with HOST frame buffers: gt_host (n_frames*wt*ht*4, input) and
 * ct_host (same size, output; 3 bytes per pixel each with SB_HOST_RGB) are host memory
 * (pinned for full copy bandwidth); cs, gs,
 * lut and workspace are device memory.  Frames stream through `depth` device slots:
 * host->device copy of frame i+1, compute of frame i and device->host copy of frame i-1
 * overlap on the library's own streams, ordered after `stream`.  Returns when ct_host
 * holds every frame.  coords_host may be NULL (coords are then kept on the device only).   */
sb_status sb_stylize_batch_host(const sb_params* prm, int32_t n_frames, const uint32_t* frame_seeds,
                                const uint8_t* cs, const uint8_t* gs, int32_t ws, int32_t hs,
                                const uint32_t* lut,
                                const uint8_t* gt_host, int32_t wt, int32_t ht,
                                uint8_t* ct_host, uint32_t* coords_host,
                                void* workspace, size_t workspace_bytes, int32_t depth,
                                void* stream);

/* Number of kernels the last successful call on this thread launched (for accounting). */
int32_t sb_last_launch_count(void);
const char* sb_last_error(void);   /* thread-local message naming the offending argument */
const char* sb_version(void);

#ifdef __cplusplus
}
#endif
#endif /* STYLEBLIT_H */
