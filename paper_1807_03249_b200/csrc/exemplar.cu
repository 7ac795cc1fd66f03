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

// Packed RGB <-> RGBA for the SB_HOST_RGB host frames (include/styleblit.h): one thread per 4
// pixels (12 packed bytes = 3 words).  n_px % 4 == 0.  Unpacking sets byte 3 to 0; packing
// drops it.
__global__ void __launch_bounds__(256) unpack_rgb_kernel(const uint32_t* __restrict__ rgb, uint4* __restrict__ rgba,
                                                         size_t n4) {
    const size_t g = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n4) return;
    const uint32_t a = __ldg(rgb + 3 * g), b = __ldg(rgb + 3 * g + 1), c = __ldg(rgb + 3 * g + 2);
    // bytes: a = r0 g0 b0 r1 | b = g1 b1 r2 g2 | c = b2 r3 g3 b3
    uint4 o;
    o.x = a & 0x00FFFFFFu;
    o.y = __byte_perm(a, b, 0x0543) & 0x00FFFFFFu;
    o.z = __byte_perm(b, c, 0x0432) & 0x00FFFFFFu;
    o.w = c >> 8;
    st_cs_u4(rgba + g, o);
}

__global__ void __launch_bounds__(256) pack_rgb_kernel(const uint4* __restrict__ rgba, uint32_t* __restrict__ rgb,
                                                       size_t n4) {
    const size_t g = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n4) return;
    const uint4 v = __ldg(rgba + g);
    rgb[3 * g] = __byte_perm(v.x, v.y, 0x4210);
    rgb[3 * g + 1] = __byte_perm(v.y, v.z, 0x5421);
    rgb[3 * g + 2] = __byte_perm(v.z, v.w, 0x6542);
}

cudaError_t launch_unpack_rgb(const uint8_t* rgb, uint8_t* rgba, size_t n_px, cudaStream_t st, int* launches) {
    const size_t n4 = n_px / 4;
    unpack_rgb_kernel<<<(unsigned)((n4 + 255) / 256), 256, 0, st>>>(reinterpret_cast<const uint32_t*>(rgb),
                                                                   reinterpret_cast<uint4*>(rgba), n4);
    *launches += 1;
    return cudaPeekAtLastError();
}

cudaError_t launch_pack_rgb(const uint8_t* rgba, uint8_t* rgb, size_t n_px, cudaStream_t st, int* launches) {
    const size_t n4 = n_px / 4;
    pack_rgb_kernel<<<(unsigned)((n4 + 255) / 256), 256, 0, st>>>(reinterpret_cast<const uint4*>(rgba),
                                                                 reinterpret_cast<uint32_t*>(rgb), n4);
    *launches += 1;
    return cudaPeekAtLastError();
}

}  // namespace sb
