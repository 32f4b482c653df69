// ft_lines.cu -- C entry points of the 3D line-decomposition curve kernel
// (kernel: ft_lines3d.cuh; per-type launchers: ft_lines_*.cu).
#include "ft_lines3d.cuh"

namespace ft {

__global__ void lines_sbase_probe(uint32_t* out)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    *out = (uint32_t)__cvta_generic_to_shared(smem_raw);
}

// The kernels address shared memory absolutely (LINES_SBASE): check once.
int lines_check_sbase()
{
    static int state = -1;  // -1 unchecked, FT_OK, or an error code
    if (state >= 0) return state;
    uint32_t *d = nullptr, v = 0;
    if (cudaMalloc(&d, 4) != cudaSuccess) return FT_ERR_CUDA_BASE + (int)cudaGetLastError();
    lines_sbase_probe<<<1, 1, 16>>>(d);
    const cudaError_t e = cudaMemcpy(&v, d, 4, cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (e != cudaSuccess) return FT_ERR_CUDA_BASE + (int)e;
    state = v == LINES_SBASE ? FT_OK : FT_ERR_INTERNAL;
    return state;
}

}  // namespace ft

using namespace ft;

extern "C" int ft_lines3d(const ft_window* win, int64_t H, int64_t W, int64_t D, int64_t v0, int64_t v1,
                          const ft_quant* q, int32_t M, uint64_t* hist, void* stream)
{
    if (!win || !hist || H < 1 || W < 1 || D < 1 || M < 0 || v0 < 0 || v1 > H + 1 || v0 > v1) return FT_ERR_ARG;
    if (W * D > INT32_MAX / 2 || !lines_ok(M)) return FT_ERR_ARG;
    if (v0 == v1) return FT_OK;
    if (!window_ok(win, H, v0, v1, 2)) return FT_ERR_ARG;
    const int qm = effective_qmode(q, true);
    if (qm != FT_Q_IDENTITY && !q->thresholds) return FT_ERR_ARG;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    switch (win->dtype) {
    case FT_I32:
    case FT_U8: return lines3d_u8i32(win, H, W, D, v0, v1, q, M, hist, st, win->dtype, qm);
    case FT_U16: return lines3d_u16(win, H, W, D, v0, v1, q, M, hist, st, qm);
    case FT_F32:
        if (qm == FT_Q_IDENTITY) return FT_ERR_ARG;
        if (qm == FT_Q_POW2) return lines3d_f32_pow2(win, H, W, D, v0, v1, q, M, hist, st);
        return lines3d_f32_table(win, H, W, D, v0, v1, q, M, hist, st, qm);
    }
    return FT_ERR_ARG;
}

extern "C" int ft_lines3d_ok(int32_t M) { return M >= 0 && lines_ok(M) ? 1 : 0; }
