// ft_lines.cu -- C entry points of the 3D line-decomposition curve kernel
// (kernel: ft_lines3d.cuh; per-type launchers: ft_lines_*.cu).
#include "ft_lines3d.cuh"

namespace ft {

// The three device quantizers of the fused kernels, run on a flat buffer
// (verification hook for the exhaustive quantizer tests): path 0 to_level
// (ft_quantize, hist/wide kernels), 1 to_level4 (march / lattice kernels,
// incl. the table-free FT_Q_POW2 one), 2 pack_pow2_sat (line kernels, f32
// pairs).  Each writes int32 levels.
template <int DT, int QM, int PATH>
__global__ void quant_probe_kernel(const typename Elem<DT>::T* __restrict__ x, int64_t n, QuantDev q, int M,
                                   int32_t* __restrict__ out)
{
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    if constexpr (PATH == 3) {
        using P2 = typename Pair<DT>::T;
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; 2 * i < n; i += stride) {
            const P2 v = reinterpret_cast<const P2*>(x)[i];
            const uint32_t w = pack_pair_umagic<DT>(v, q, 4u, 0u);
            out[2 * i] = (int32_t)((w & 0xFFFFu) >> 2);
            out[2 * i + 1] = (int32_t)(w >> 18);
        }
    } else if constexpr (PATH == 2) {
        using P2 = typename Pair<DT>::T;
        const float Mf = (float)M;
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; 2 * i < n; i += stride) {
            const P2 v = reinterpret_cast<const P2*>(x)[i];
            const uint32_t w = pack_pow2_sat<DT>(v, q.inv, Mf, 4u, 0u);
            out[2 * i] = (int32_t)((w & 0xFFFFu) >> 2);
            out[2 * i + 1] = (int32_t)(w >> 18);
        }
    } else {
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
            if constexpr (PATH == 0)
                out[i] = (int32_t)to_level<DT, QM>(x[i], q.tt, q.scale, q.bias, q.negate, M);
            else
                out[i] = (int32_t)(to_level4<DT, QM>(x[i], q.tt, q.scale, q.bias, q.negate, M) >> 2);
        }
    }
}

}  // namespace ft

using namespace ft;

extern "C" int ft_quantize_probe(const void* x, int32_t dtype, int64_t n, const ft_quant* q, int32_t M,
                                 int32_t path, int32_t* out, void* stream)
{
    if (!x || !q || !out || n < 0 || M < 1 || path < 0 || path > 3) return FT_ERR_ARG;
    if (q->mode == FT_Q_IDENTITY || !q->thresholds || (dtype != FT_F32 && dtype != FT_U16)) return FT_ERR_ARG;
    const int qm = effective_qmode(q, path != 0);
    if (path == 2 && (dtype != FT_F32 || qm != FT_Q_POW2 || n % 2)) return FT_ERR_ARG;
    if (n == 0) return FT_OK;
    QuantDev qd = qdev(q);
    if (path == 3) {
        // the line kernels' integer decoding of uint16 pairs (FT_Q_UMAGIC); FT_ERR_ARG
        // when the range does not qualify (they would take the table then)
        if (dtype != FT_U16 || n % 2 || !umagic_fill(q, M, 65536, qd)) return FT_ERR_ARG;
        const int g3 = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(n / 2, 256), 148 * 16));
        quant_probe_kernel<FT_U16, FT_Q_UMAGIC, 3><<<g3, 256, 0, static_cast<cudaStream_t>(stream)>>>(
            static_cast<const uint16_t*>(x), n, qd, M, out);
        FT_CUDA_TRY(cudaGetLastError());
        return FT_OK;
    }
    qd.mode = qm;
    if (qm == FT_Q_POW2) qd.inv = q->scale / (float)M;  // 1 / hi, as launch_lines3d sets it
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 256), 148 * 16));
#define FT_PROBE(DT, QM, P) \
    quant_probe_kernel<DT, QM, P><<<grid, 256, 0, st>>>(static_cast<const typename Elem<DT>::T*>(x), n, qd, M, out)
    if (path == 2) {
        FT_PROBE(FT_F32, FT_Q_POW2, 2);
    } else if (dtype == FT_F32) {
        if (path == 1 && qm == FT_Q_POW2) FT_PROBE(FT_F32, FT_Q_POW2, 1);
        else if (qm == FT_Q_TABLE || qm == FT_Q_POW2) {
            if (path == 0) FT_PROBE(FT_F32, FT_Q_TABLE, 0); else FT_PROBE(FT_F32, FT_Q_TABLE, 1);
        } else {
            if (path == 0) FT_PROBE(FT_F32, FT_Q_TABLE_ROBUST, 0); else FT_PROBE(FT_F32, FT_Q_TABLE_ROBUST, 1);
        }
    } else {
        if (path == 1 && qm == FT_Q_POW2) FT_PROBE(FT_U16, FT_Q_POW2, 1);
        else if (qm == FT_Q_TABLE || qm == FT_Q_POW2) {
            if (path == 0) FT_PROBE(FT_U16, FT_Q_TABLE, 0); else FT_PROBE(FT_U16, FT_Q_TABLE, 1);
        } else {
            if (path == 0) FT_PROBE(FT_U16, FT_Q_TABLE_ROBUST, 0); else FT_PROBE(FT_U16, FT_Q_TABLE_ROBUST, 1);
        }
    }
#undef FT_PROBE
    FT_CUDA_TRY(cudaGetLastError());
    return FT_OK;
}

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
