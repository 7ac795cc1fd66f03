// exemplar.cu -- the strided exemplar copy of sb_prepare_exemplar (include/styleblit.h).
//
// G_S and C_S are copied to rows of 2^16 pixels, so that a packed source coordinate
// s = x | y<<16 -- the candidate of Alg. 2 line 384 and the blit source of line 387
// -- is its own pixel index and the stylize kernel's exemplar gathers need no
// index arithmetic.  Once per exemplar (like the LUT): ws*hs*8 bytes read, ws*hs*8 written.
#include "sb_kernels.cuh"

namespace sb {

// one thread per 16 bytes (4 pixels) of a source row; grid.y = rows, grid.z = {G_S, C_S}
__global__ void __launch_bounds__(256) exemplar_pad_kernel(const uint8_t* __restrict__ cs,
                                                           const uint8_t* __restrict__ gs, int ws, int hs,
                                                           uint8_t* __restrict__ ex) {
    const int y = blockIdx.y;
    const uint8_t* src = blockIdx.z == 0 ? gs : cs;
    uint8_t* dst = ex + (size_t)blockIdx.z * (size_t)hs * ((size_t)1 << 18) + ((size_t)y << 18);
    const uint8_t* row = src + (size_t)y * ws * 4;
    const int x4 = blockIdx.x * blockDim.x + threadIdx.x;  // 4-pixel group
    const int x = 4 * x4;
    if (x >= ws) return;
    if (x + 3 < ws && (ws & 3) == 0) {
        *reinterpret_cast<uint4*>(dst + 4 * (size_t)x) = __ldg(reinterpret_cast<const uint4*>(row + 4 * (size_t)x));
    } else {
        for (int k = 0; k < 4 && x + k < ws; ++k)
            *reinterpret_cast<uint32_t*>(dst + 4 * (size_t)(x + k)) =
                __ldg(reinterpret_cast<const uint32_t*>(row + 4 * (size_t)(x + k)));
    }
}

cudaError_t launch_prepare_exemplar(const uint8_t* cs, const uint8_t* gs, int ws, int hs, uint8_t* exemplar,
                                    cudaStream_t st, int* launches) {
    const int groups = (ws + 3) / 4;
    dim3 grid((unsigned)((groups + 255) / 256), (unsigned)hs, 2u);
    exemplar_pad_kernel<<<grid, 256, 0, st>>>(cs, gs, ws, hs, exemplar);
    *launches += 1;
    return cudaPeekAtLastError();
}

}  // namespace sb
