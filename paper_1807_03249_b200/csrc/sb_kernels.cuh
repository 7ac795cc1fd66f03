// sb_kernels.cuh -- kernel argument blocks and launchers of libstyleblit (sm_100a).
#pragma once
#include "sb_device.cuh"

namespace sb {

constexpr int kSeedsPerLaunch = 512;  // frames per launch (per-frame seeds travel as params)
#define SB_MAX_LEVELS_DEV 15           // == SB_MAX_LEVELS of include/styleblit.h
constexpr int kPackedMaxDim = 32767;  // packed-arithmetic kernels: every image side <= this

struct StylizeArgs {
    const uint8_t* cs;
    const uint8_t* gs;
    int ws, hs;
    const uint32_t* lut;
    uint32_t key_mask;  // LUT key bits of a guide value: 0xFFFF (2-channel) or 0xFFFFFF (SB_LUT_RGB)
    const uint8_t* exemplar;  // strided G_S | C_S copy (sb_prepare_exemplar) or NULL
    const uint8_t* gt;  // frame 0 of this launch
    int wt, ht;
    uint8_t* ct;        // NULL: no colour output (SB_NO_COLOR or vote follows)
    uint32_t* coords;   // may be NULL
    uint8_t* level;     // may be NULL
    int L;
    uint32_t T2;        // accept iff D < T2 (= ceil(t*t), saturated)
    uint32_t cmask;     // guide channel byte mask for D
    int ext;            // weighted channels and/or segmentation label in use
    uint32_t w[4];      // per-channel weights (ext)
    uint32_t lmask;     // byte mask of the segmentation label (ext; 0 = none)
    int zero_jitter;
    int row_begin, row_end;  // rows computed
    uint32_t seed_base;
    int has_seeds;
    uint32_t seeds[kSeedsPerLaunch];
    __device__ __forceinline__ uint32_t frame_seed(int f) const {
        return has_seeds ? seeds[f] : seed_base + (uint32_t)f;
    }
};

struct VoteArgs {
    const uint32_t* coords;  // frame 0 of this launch
    const uint8_t* cs;
    const uint8_t* cs_pad;   // C_S in the strided exemplar copy (rows of 2^16 pixels) or NULL
    int ws, hs;
    int wt, ht;
    int r;
    uint8_t* ct;
    int row_begin, row_end;  // rows written
};

// launch_util.cu: per-device cached SM count and one-time kernel attributes
int sm_count();
cudaError_t ensure_smem(const void* kern, int bytes);
cudaError_t ensure_carveout(const void* kern, int pct);

cudaError_t launch_build_lut(const uint8_t* gs, int ws, int hs, uint32_t* lut, void* workspace,
                             cudaStream_t st, int* launches);
cudaError_t launch_build_lut3(const uint8_t* gs, int ws, int hs, uint32_t* lut3, void* workspace,
                              cudaStream_t st, int* launches);
cudaError_t launch_unpack_rgb(const uint8_t* rgb, uint8_t* rgba, size_t n_px, cudaStream_t st, int* launches);
cudaError_t launch_pack_rgb(const uint8_t* rgba, uint8_t* rgb, size_t n_px, cudaStream_t st, int* launches);
cudaError_t launch_prepare_exemplar(const uint8_t* cs, const uint8_t* gs, int ws, int hs, uint8_t* exemplar,
                                    cudaStream_t st, int* launches);
cudaError_t launch_stylize_naive(const StylizeArgs& a, int n_frames, cudaStream_t st, int* launches);
cudaError_t launch_stylize_tiled(const StylizeArgs& a, int n_frames, cudaStream_t st, int* launches);
cudaError_t launch_vote(const VoteArgs& a, int n_frames, cudaStream_t st, int* launches);
cudaError_t launch_vote_wide(const VoteArgs& a, int n_frames, cudaStream_t st, int* launches);
cudaError_t launch_vote_hist(const VoteArgs& a, int n_frames, cudaStream_t st, int* launches);
cudaError_t launch_vote_peel(const VoteArgs& a, int n_frames, cudaStream_t st, int* launches);

}  // namespace sb
