// ft_finalize.cu -- transition histograms -> contribution maps and curves,
// plus the standalone quantize and min/max kernels.
//
// finalize replaces the reference's host-side merge of worker maps
// (contrib2d.py:290-294, contrib3d.py:454-458) and curve assembly
// (counts_at_levels + descriptor_curve, descriptors.py:153-178):
//   q_in[t][l]  = sum over classes (a -> t) of hist[c][l]
//   q_out[t][l] = sum over classes (t -> b) of hist[c][l]
//   numerators[d][l] = prefix-sum over levels 0..l of sum_c w_d[c] hist[c][l]
// where w_d[c] = eighths[dst] - eighths[src] (ft_class_weights).  Curves never
// see the sentinel bin M+1, like counts_at_levels' [:M+1] slice.
#include <algorithm>

#include "ft_common.cuh"
#include "ft_tables.h"

namespace ft {

__global__ void qmap_kernel(const unsigned long long* __restrict__ hist, int C, int T, int M2, int64_t batch,
                            ClassMap cm, unsigned long long* __restrict__ q_in,
                            unsigned long long* __restrict__ q_out)
{
    const int64_t n = batch * T * M2;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = t / ((int64_t)T * M2);
        const int ty = (int)((t / M2) % T);
        const int l = (int)(t % M2);
        const unsigned long long* hb = hist + b * (int64_t)C * M2;
        unsigned long long si = 0, so = 0;
        for (int c = 0; c < C; ++c) {
            const unsigned long long v = hb[(int64_t)c * M2 + l];
            if (cm.dst[c] == ty) si += v;
            if (cm.src[c] == ty) so += v;
        }
        if (q_in) q_in[t] = si;
        if (q_out) q_out[t] = so;
    }
}

// One block per (image, descriptor): segmented inclusive scan over levels.
__global__ void __launch_bounds__(256) curve_kernel(const unsigned long long* __restrict__ hist, int C, int M,
                                                    int n_desc, const int64_t* __restrict__ class_w,
                                                    int64_t* __restrict__ numerators)
{
    __shared__ long long part[256];
    const int M1 = M + 1, M2 = M + 2;
    const int d = blockIdx.x % n_desc;
    const int64_t b = blockIdx.x / n_desc;
    const unsigned long long* hb = hist + b * (int64_t)C * M2;
    const int64_t* w = class_w + (int64_t)d * C;
    int64_t* out = numerators + (b * n_desc + d) * (int64_t)M1;
    const int seg = (M1 + blockDim.x - 1) / blockDim.x;
    const int l0 = threadIdx.x * seg, l1 = min(l0 + seg, M1);
    long long acc = 0;
    for (int l = l0; l < l1; ++l)
        for (int c = 0; c < C; ++c) acc += (long long)w[c] * (long long)hb[(int64_t)c * M2 + l];
    part[threadIdx.x] = acc;
    __syncthreads();
    for (int off = 1; off < blockDim.x; off <<= 1) {  // Hillis-Steele over 256 partials
        long long v = threadIdx.x >= off ? part[threadIdx.x - off] : 0;
        __syncthreads();
        part[threadIdx.x] += v;
        __syncthreads();
    }
    long long run = threadIdx.x ? part[threadIdx.x - 1] : 0;
    for (int l = l0; l < l1; ++l) {
        for (int c = 0; c < C; ++c) run += (long long)w[c] * (long long)hb[(int64_t)c * M2 + l];
        out[l] = run;
    }
}

template <int DT, int QM>
__global__ void quantize_kernel(const typename Elem<DT>::T* __restrict__ x, int64_t n, QuantDev q, int M,
                                int32_t* __restrict__ out)
{
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
        out[t] = (int32_t)to_level<DT, QM>(ld_stream(x + t), q.tt, q.scale, q.bias, q.negate, M);
}

template <int QM>
__global__ void quantize_f64_kernel(const double* __restrict__ x, int64_t n, QuantDev q, int M,
                                    int32_t* __restrict__ out)
{
    const double* tt = reinterpret_cast<const double*>(q.tt);
    const double scale = q.scale, bias = q.bias;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
        out[t] = (int32_t)to_level_f64<QM>(x[t], tt, scale, bias, q.negate, M);
}

__device__ __forceinline__ uint64_t order_key64(double f)
{
    uint64_t u = __double_as_longlong(f);
    return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

__global__ void minmax64_init(unsigned long long* out)
{
    out[0] = 0xFFFFFFFFFFFFFFFFull;
    out[1] = 0ull;
}

__global__ void __launch_bounds__(256) minmax_f64_kernel(const double* __restrict__ x, int64_t n,
                                                         unsigned long long* out)
{
    unsigned long long lo = 0xFFFFFFFFFFFFFFFFull, hi = 0ull;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long k = order_key64(x[t]);
        lo = min(lo, k);
        hi = max(hi, k);
    }
    for (int off = 16; off; off >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xFFFFFFFFu, lo, off));
        hi = max(hi, __shfl_xor_sync(0xFFFFFFFFu, hi, off));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(&out[0], lo);
        atomicMax(&out[1], hi);
    }
}

__device__ __forceinline__ uint32_t order_key(float f)
{
    uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
template <int DT>
__device__ __forceinline__ uint32_t elem_key(typename Elem<DT>::T v)
{
    if constexpr (DT == FT_F32) return order_key(v);
    else if constexpr (DT == FT_I32) return (uint32_t)v ^ 0x80000000u;
    else return (uint32_t)v;
}

__global__ void minmax_init(uint32_t* out)
{
    out[0] = 0xFFFFFFFFu;
    out[1] = 0u;
}

template <int DT>
__global__ void __launch_bounds__(256) minmax_kernel(const typename Elem<DT>::T* __restrict__ x, int64_t n,
                                                     uint32_t* out)
{
    uint32_t lo = 0xFFFFFFFFu, hi = 0u;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t k = elem_key<DT>(ld_stream(x + t));
        lo = min(lo, k);
        hi = max(hi, k);
    }
    for (int off = 16; off; off >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xFFFFFFFFu, lo, off));
        hi = max(hi, __shfl_xor_sync(0xFFFFFFFFu, hi, off));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(&out[0], lo);
        atomicMax(&out[1], hi);
    }
}

static int nsm()
{
    int dev = 0, n = kSMs;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
}

}  // namespace ft

using namespace ft;

extern "C" int ft_finalize(int32_t ndim, int32_t M, int64_t batch, const uint64_t* hist, uint64_t* q_in,
                           uint64_t* q_out, int32_t n_desc, const int64_t* class_w, int64_t* numerators,
                           void* stream)
{
    if ((ndim != 2 && ndim != 3) || M < 0 || batch < 1 || !hist || n_desc < 0) return FT_ERR_ARG;
    if (n_desc > 0 && (!class_w || !numerators)) return FT_ERR_ARG;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const Tables& t = tables(ndim);
    const int C = t.n_classes, T = ndim == 3 ? FT_NTYPE_3D : FT_NTYPE_2D, M2 = M + 2;
    auto* h = reinterpret_cast<const unsigned long long*>(hist);
    if (q_in || q_out) {
        ClassMap cm;
        for (int c = 0; c < 64; ++c) {
            cm.src[c] = c < C ? (int8_t)t.src[c] : (int8_t)-2;
            cm.dst[c] = c < C ? (int8_t)t.dst[c] : (int8_t)-2;
        }
        const int64_t n = batch * T * M2;
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 256), 8 * nsm()));
        qmap_kernel<<<grid, 256, 0, st>>>(h, C, T, M2, batch, cm, reinterpret_cast<unsigned long long*>(q_in),
                                          reinterpret_cast<unsigned long long*>(q_out));
        FT_CUDA_TRY(cudaGetLastError());
    }
    if (n_desc > 0) {
        curve_kernel<<<(unsigned)(batch * n_desc), 256, 0, st>>>(h, C, M, n_desc, class_w, numerators);
        FT_CUDA_TRY(cudaGetLastError());
    }
    return FT_OK;
}

extern "C" int ft_curves(const uint64_t* rows, int32_t n_rows, int32_t M, int64_t batch, int32_t n_desc,
                         const int64_t* row_w, int64_t* numerators, void* stream)
{
    if (!rows || n_rows < 1 || M < 0 || batch < 1 || n_desc < 1 || !row_w || !numerators) return FT_ERR_ARG;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    curve_kernel<<<(unsigned)(batch * n_desc), 256, 0, st>>>(reinterpret_cast<const unsigned long long*>(rows),
                                                             n_rows, M, n_desc, row_w, numerators);
    FT_CUDA_TRY(cudaGetLastError());
    return FT_OK;
}

extern "C" int ft_quantize(const void* x, int32_t dtype, int64_t n, const ft_quant* q, int32_t M, int32_t* out,
                           void* stream)
{
    if (!q || !out || n < 0 || M < 0) return FT_ERR_ARG;
    if (n == 0) return FT_OK;
    if (!x) return FT_ERR_ARG;
    if (q->mode != FT_Q_IDENTITY && !q->thresholds) return FT_ERR_ARG;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int qmode = effective_qmode(q);
    QuantDev qd{qmode, q->negate, q->scale, q->bias, q->thresholds};
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 256), 16 * nsm()));
#define FT_Q_LAUNCH(DT, QM) \
    quantize_kernel<DT, QM><<<grid, 256, 0, st>>>(static_cast<const typename Elem<DT>::T*>(x), n, qd, M, out)
    switch (dtype) {
    case FT_U8:
        if (qmode == FT_Q_IDENTITY) FT_Q_LAUNCH(FT_U8, FT_Q_IDENTITY);
        else if (qmode == FT_Q_TABLE) FT_Q_LAUNCH(FT_U8, FT_Q_TABLE);
        else FT_Q_LAUNCH(FT_U8, FT_Q_TABLE_ROBUST);
        break;
    case FT_U16:
        if (qmode == FT_Q_IDENTITY) FT_Q_LAUNCH(FT_U16, FT_Q_IDENTITY);
        else if (qmode == FT_Q_TABLE) FT_Q_LAUNCH(FT_U16, FT_Q_TABLE);
        else FT_Q_LAUNCH(FT_U16, FT_Q_TABLE_ROBUST);
        break;
    case FT_F32:
        if (qmode == FT_Q_IDENTITY) return FT_ERR_ARG;
        if (qmode == FT_Q_TABLE) FT_Q_LAUNCH(FT_F32, FT_Q_TABLE);
        else FT_Q_LAUNCH(FT_F32, FT_Q_TABLE_ROBUST);
        break;
    case FT_F64:
        // scale / bias travel as float in ft_quant; the double estimate only
        // needs to land within +-1 level (host-checked), the table decides.
        if (qmode == FT_Q_IDENTITY) return FT_ERR_ARG;
        if (qmode == FT_Q_TABLE)
            quantize_f64_kernel<FT_Q_TABLE><<<grid, 256, 0, st>>>(static_cast<const double*>(x), n, qd, M, out);
        else
            quantize_f64_kernel<FT_Q_TABLE_ROBUST><<<grid, 256, 0, st>>>(static_cast<const double*>(x), n, qd, M, out);
        break;
    default: return FT_ERR_ARG;
    }
#undef FT_Q_LAUNCH
    FT_CUDA_TRY(cudaGetLastError());
    return FT_OK;
}

extern "C" int ft_minmax(const void* x, int32_t dtype, int64_t n, uint32_t* out, void* stream)
{
    if (!x || !out || n < 1) return FT_ERR_ARG;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (dtype == FT_F64) {  // out is then uint64[2] (16 bytes, 8-aligned)
        auto* o = reinterpret_cast<unsigned long long*>(out);
        minmax64_init<<<1, 1, 0, st>>>(o);
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 256 * 8), 8 * nsm()));
        minmax_f64_kernel<<<grid, 256, 0, st>>>(static_cast<const double*>(x), n, o);
        FT_CUDA_TRY(cudaGetLastError());
        return FT_OK;
    }
    minmax_init<<<1, 1, 0, st>>>(out);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 256 * 8), 8 * nsm()));
    switch (dtype) {
    case FT_I32: minmax_kernel<FT_I32><<<grid, 256, 0, st>>>(static_cast<const int32_t*>(x), n, out); break;
    case FT_U8: minmax_kernel<FT_U8><<<grid, 256, 0, st>>>(static_cast<const uint8_t*>(x), n, out); break;
    case FT_U16: minmax_kernel<FT_U16><<<grid, 256, 0, st>>>(static_cast<const uint16_t*>(x), n, out); break;
    case FT_F32: minmax_kernel<FT_F32><<<grid, 256, 0, st>>>(static_cast<const float*>(x), n, out); break;
    default: return FT_ERR_ARG;
    }
    FT_CUDA_TRY(cudaGetLastError());
    return FT_OK;
}

extern "C" double ft_key64_to_double(uint64_t key)
{
    uint64_t u = (key >> 63) ? (key & 0x7FFFFFFFFFFFFFFFull) : ~key;
    double d;
    memcpy(&d, &u, 8);
    return d;
}

extern "C" double ft_key_to_double(int32_t dtype, uint32_t key)
{
    switch (dtype) {
    case FT_F32: {
        uint32_t u = (key & 0x80000000u) ? (key & 0x7FFFFFFFu) : ~key;
        float f;
        memcpy(&f, &u, 4);
        return (double)f;
    }
    case FT_I32: return (double)(int32_t)(key ^ 0x80000000u);
    default: return (double)key;
    }
}

// ------------------------------------------------------ BMP pixel decode
// 8-bit BMP pixel rows as stored (padded to 4 bytes, bottom-up when the
// header height is positive) -> compact top-first rows (reference read_bmp,
// sources.py:154-164, on the device).  One thread per output pixel quad.
__global__ void bmp_decode_kernel(const uint8_t* __restrict__ raw, int64_t H, int64_t W, int64_t stride,
                                  int bottom_up, uint8_t* __restrict__ out)
{
    const int64_t n = H * W;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / W, c = i - r * W;
        const int64_t src_row = bottom_up ? H - 1 - r : r;
        out[i] = raw[src_row * stride + c];
    }
}

extern "C" int ft_bmp_decode(const uint8_t* raw, int64_t H, int64_t W, int64_t row_stride, int32_t bottom_up,
                             uint8_t* out, void* stream)
{
    if (!raw || !out || H < 1 || W < 1 || row_stride < W) return FT_ERR_ARG;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(H * W, 256), 16 * nsm()));
    bmp_decode_kernel<<<grid, 256, 0, st>>>(raw, H, W, row_stride, bottom_up ? 1 : 0, out);
    FT_CUDA_TRY(cudaGetLastError());
    return FT_OK;
}
