// ft_stream.cu -- native runtime entry points around the kernels:
//
// * ft_stream_begin / push / end: out-of-core chunk streaming for callers of
//   the C ABI (the reference's low-memory mode, _stream_rows_2d /
//   _stream_slabs_3d, contrib2d.py:235-251, contrib3d.py:392-414, rebuilt as
//   double-buffered host -> HBM streaming).  The caller pushes consecutive
//   rows / planes from host memory in any batch sizes; they are copied on an
//   internal copy stream into two device buffers of `chunk_rows` rows, the
//   LOW_HALO rows a buffer shares with the next are carried device-to-device
//   (every row crosses PCIe once), and the kernel for every vertex row whose
//   planes have all arrived runs on the caller's stream while the next
//   buffer fills.  Same engine as gather.stream_hist (Python), in C++.
// * ft_multi_gather3d: one process driving several GPUs (the reference's
//   worker split, _parallel.py:8-33, across devices): every slab's histogram
//   on its own device, then ONE all-reduce of the histograms -- NCCL
//   (ncclAllReduce, sum, uint64; NVLink / NVSwitch) when every slab is on a
//   distinct device, a peer-copy reduction otherwise.  NCCL is resolved at
//   run time (dlopen), so the library has no link-time NCCL dependency and
//   reuses the NCCL torch has already loaded.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <vector>

#include "ft_common.cuh"

extern "C" {
int ft_hist2d(const ft_window* win, int64_t H, int64_t W, int64_t v0, int64_t v1, const ft_quant* q, int32_t M,
              uint64_t* hist, void* stream);
int ft_hist3d(const ft_window* win, int64_t H, int64_t W, int64_t D, int64_t v0, int64_t v1, const ft_quant* q,
              int32_t M, uint64_t* hist, void* stream);
int ft_lines3d(const ft_window* win, int64_t H, int64_t W, int64_t D, int64_t v0, int64_t v1, const ft_quant* q,
               int32_t M, uint64_t* hist, void* stream);
int ft_lines2d(const ft_window* win, int64_t H, int64_t W, int64_t v0, int64_t v1, const ft_quant* q, int32_t M,
               uint64_t* hist, void* stream);
}

namespace ft {

constexpr int64_t LOW_HALO = 2;  // planes below a slab's first vertex row a kernel reads (fused: signatures)

static int64_t elem_bytes(int dt)
{
    switch (dt) {
    case FT_I32: return 4;
    case FT_U8: return 1;
    case FT_U16: return 2;
    case FT_F32: return 4;
    default: return 0;
    }
}

static int launch_kind(int ndim, int kind, const ft_window& w, int64_t H, int64_t W, int64_t D, int64_t v0, int64_t v1,
                       const ft_quant* q, int32_t M, uint64_t* hist, cudaStream_t st)
{
    if (v1 <= v0) return FT_OK;
    if (ndim == 2)
        return kind == FT_KIND_MAP ? ft_hist2d(&w, H, W, v0, v1, q, M, hist, st) : ft_lines2d(&w, H, W, v0, v1, q, M, hist, st);
    return kind == FT_KIND_MAP ? ft_hist3d(&w, H, W, D, v0, v1, q, M, hist, st)
                               : ft_lines3d(&w, H, W, D, v0, v1, q, M, hist, st);
}

}  // namespace ft

using namespace ft;

struct ft_stream {
    int ndim, kind, dtype;
    int64_t H, W, D, row_bytes, cap;
    ft_quant q;
    int32_t M;
    uint64_t* hist;
    cudaStream_t user, copy;
    char* buf[2] = {nullptr, nullptr};
    cudaEvent_t copied[2] = {nullptr, nullptr}, done[2] = {nullptr, nullptr};
    bool used[2] = {false, false};
    int b = 0;          // buffer being filled
    int64_t base = 0;   // first row held by buf[b]
    int64_t fill = 0;   // rows held by buf[b]
    int64_t pushed = 0; // rows received from the caller
    int64_t vnext = 0;  // first vertex row not yet booked
};

static void stream_free(ft_stream* s)
{
    for (int i = 0; i < 2; ++i) {
        if (s->buf[i]) cudaFree(s->buf[i]);
        if (s->copied[i]) cudaEventDestroy(s->copied[i]);
        if (s->done[i]) cudaEventDestroy(s->done[i]);
    }
    if (s->copy) cudaStreamDestroy(s->copy);
    delete s;
}

// Book every vertex row whose planes are in buf[b]; switch buffers unless final.
static int stream_flush(ft_stream* s, bool final)
{
    const int b = s->b;
    FT_CUDA_TRY(cudaEventRecord(s->copied[b], s->copy));
    FT_CUDA_TRY(cudaStreamWaitEvent(s->user, s->copied[b], 0));
    const int64_t vend = final ? s->H + 1 : s->base + s->fill;  // vertex row v needs plane v (if v < H)
    const ft_window w{s->buf[b], s->dtype, s->base, s->fill, 1, 0};
    if (const int rc = launch_kind(s->ndim, s->kind, w, s->H, s->W, s->D, s->vnext, vend, &s->q, s->M, s->hist, s->user))
        return rc;
    FT_CUDA_TRY(cudaEventRecord(s->done[b], s->user));
    s->used[b] = true;
    s->vnext = std::max(s->vnext, vend);
    if (final) return FT_OK;
    const int nb = 1 - b;
    if (s->used[nb]) FT_CUDA_TRY(cudaStreamWaitEvent(s->copy, s->done[nb], 0));  // its kernel is done with it
    const int64_t carry = std::min(LOW_HALO, s->fill);
    FT_CUDA_TRY(cudaMemcpyAsync(s->buf[nb], s->buf[b] + (s->fill - carry) * s->row_bytes, carry * s->row_bytes,
                                cudaMemcpyDeviceToDevice, s->copy));
    s->base += s->fill - carry;
    s->fill = carry;
    s->b = nb;
    return FT_OK;
}

extern "C" int ft_stream_begin(int32_t ndim, int64_t H, int64_t W, int64_t D, int32_t dtype, const ft_quant* q,
                               int32_t M, int32_t kind, int64_t chunk_rows, uint64_t* hist, void* stream,
                               ft_stream** out)
{
    if (!out) return FT_ERR_ARG;
    *out = nullptr;
    if ((ndim != 2 && ndim != 3) || H < 1 || W < 1 || (ndim == 3 && D < 1) || M < 0 || !hist ||
        (kind != FT_KIND_MAP && kind != FT_KIND_FUSED) || chunk_rows < LOW_HALO + 1 || elem_bytes(dtype) == 0)
        return FT_ERR_ARG;
    auto* s = new ft_stream();
    s->ndim = ndim;
    s->kind = kind;
    s->dtype = dtype;
    s->H = H;
    s->W = W;
    s->D = ndim == 3 ? D : 1;
    s->row_bytes = W * s->D * elem_bytes(dtype);
    s->cap = std::min(chunk_rows, H + LOW_HALO);
    s->q = q ? *q : ft_quant{FT_Q_IDENTITY, 0, 0.f, 0.f, nullptr};
    s->M = M;
    s->hist = hist;
    s->user = static_cast<cudaStream_t>(stream);
    cudaError_t e = cudaStreamCreateWithFlags(&s->copy, cudaStreamNonBlocking);
    for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
        e = cudaMalloc(&s->buf[i], (size_t)(s->cap * s->row_bytes));
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s->copied[i], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s->done[i], cudaEventDisableTiming);
    }
    if (e != cudaSuccess) {
        stream_free(s);
        return FT_ERR_CUDA_BASE + (int)e;
    }
    // the copy stream starts after everything already queued on the caller's
    // stream (e.g. the zeroing of hist)
    cudaEvent_t start;
    if (cudaEventCreateWithFlags(&start, cudaEventDisableTiming) == cudaSuccess) {
        cudaEventRecord(start, s->user);
        cudaStreamWaitEvent(s->copy, start, 0);
        cudaEventDestroy(start);
    }
    *out = s;
    return FT_OK;
}

extern "C" int ft_stream_push(ft_stream* s, const void* rows, int64_t nrows)
{
    if (!s || nrows < 0 || (nrows && !rows) || s->pushed + nrows > s->H) return FT_ERR_ARG;
    const char* p = static_cast<const char*>(rows);
    while (nrows > 0) {
        const int64_t m = std::min(nrows, s->cap - s->fill);
        FT_CUDA_TRY(cudaMemcpyAsync(s->buf[s->b] + s->fill * s->row_bytes, p, m * s->row_bytes, cudaMemcpyDefault,
                                    s->copy));
        s->fill += m;
        s->pushed += m;
        p += m * s->row_bytes;
        nrows -= m;
        if (s->fill == s->cap && s->pushed < s->H)
            if (const int rc = stream_flush(s, false)) return rc;
    }
    return FT_OK;
}

extern "C" int ft_stream_end(ft_stream* s)
{
    if (!s) return FT_ERR_ARG;
    int rc = s->pushed == s->H ? stream_flush(s, true) : FT_ERR_ARG;
    const cudaError_t e = cudaStreamSynchronize(s->user);
    if (rc == FT_OK && e != cudaSuccess) rc = FT_ERR_CUDA_BASE + (int)e;
    stream_free(s);
    return rc;
}

// ------------------------------------------------------------ multi-GPU

namespace {

struct Nccl {
    decltype(&ncclCommInitAll) init_all = nullptr;
    decltype(&ncclAllReduce) all_reduce = nullptr;
    decltype(&ncclGroupStart) group_start = nullptr;
    decltype(&ncclGroupEnd) group_end = nullptr;
    decltype(&ncclCommDestroy) destroy = nullptr;
    bool ok = false;
};

const Nccl& nccl()
{
    static const Nccl n = [] {
        Nccl r;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the NCCL torch loaded, if any
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return r;
        r.init_all = reinterpret_cast<decltype(r.init_all)>(dlsym(h, "ncclCommInitAll"));
        r.all_reduce = reinterpret_cast<decltype(r.all_reduce)>(dlsym(h, "ncclAllReduce"));
        r.group_start = reinterpret_cast<decltype(r.group_start)>(dlsym(h, "ncclGroupStart"));
        r.group_end = reinterpret_cast<decltype(r.group_end)>(dlsym(h, "ncclGroupEnd"));
        r.destroy = reinterpret_cast<decltype(r.destroy)>(dlsym(h, "ncclCommDestroy"));
        r.ok = r.init_all && r.all_reduce && r.group_start && r.group_end && r.destroy;
        return r;
    }();
    return n;
}

__global__ void add_u64(unsigned long long* __restrict__ dst, const unsigned long long* __restrict__ src, int64_t n)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] += src[i];
}

struct DeviceGuard {
    int prev = 0;
    DeviceGuard() { cudaGetDevice(&prev); }
    ~DeviceGuard() { cudaSetDevice(prev); }
};

}  // namespace

extern "C" int ft_multi_gather3d(const ft_slab* slabs, int32_t nslab, int64_t H, int64_t W, int64_t D, int32_t M,
                                 int32_t kind, int32_t* used_nccl)
{
    if (!slabs || nslab < 1 || H < 1 || W < 1 || D < 1 || M < 0 || (kind != FT_KIND_MAP && kind != FT_KIND_FUSED))
        return FT_ERR_ARG;
    if (used_nccl) *used_nccl = 0;
    const int64_t rows = kind == FT_KIND_MAP ? FT_NCLASS_3D : 3;
    const int64_t count = rows * (M + 2);
    DeviceGuard guard;
    std::vector<cudaStream_t> st(nslab, nullptr);
    int rc = FT_OK;
    auto cleanup = [&] {
        for (int i = 0; i < nslab; ++i)
            if (st[i]) {
                cudaSetDevice(slabs[i].device);
                cudaStreamDestroy(st[i]);
            }
    };
    // 1. every slab's histogram on its own device
    for (int i = 0; i < nslab && rc == FT_OK; ++i) {
        const ft_slab& s = slabs[i];
        cudaError_t e = cudaSetDevice(s.device);
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&st[i], cudaStreamNonBlocking);
        if (e != cudaSuccess) {
            rc = FT_ERR_CUDA_BASE + (int)e;
            break;
        }
        if (!s.hist) {
            rc = FT_ERR_ARG;
            break;
        }
        rc = launch_kind(3, kind, s.win, H, W, D, s.v0, s.v1, &s.quant, M, s.hist, st[i]);
    }
    // 2. one all-reduce of the histograms
    std::vector<int> devs(nslab);
    for (int i = 0; i < nslab; ++i) devs[i] = slabs[i].device;
    std::vector<int> sorted = devs;
    std::sort(sorted.begin(), sorted.end());
    const bool distinct = std::adjacent_find(sorted.begin(), sorted.end()) == sorted.end();
    if (rc == FT_OK && nslab > 1 && distinct && nccl().ok) {
        std::vector<ncclComm_t> comms(nslab);
        if (nccl().init_all(comms.data(), nslab, devs.data()) == ncclSuccess) {
            nccl().group_start();
            for (int i = 0; i < nslab; ++i)
                nccl().all_reduce(slabs[i].hist, slabs[i].hist, (size_t)count, ncclUint64, ncclSum, comms[i], st[i]);
            const ncclResult_t r = nccl().group_end();
            for (int i = 0; i < nslab && rc == FT_OK; ++i) {
                cudaSetDevice(devs[i]);
                const cudaError_t e = cudaStreamSynchronize(st[i]);
                if (e != cudaSuccess) rc = FT_ERR_CUDA_BASE + (int)e;
            }
            for (auto c : comms) nccl().destroy(c);
            if (r != ncclSuccess && rc == FT_OK) rc = FT_ERR_INTERNAL;
            if (used_nccl && rc == FT_OK) *used_nccl = 1;
            cleanup();
            return rc;
        }
    }
    if (rc == FT_OK && nslab > 1) {
        // peer-copy reduction into slab 0's histogram, then copies back out
        unsigned long long* tmp = nullptr;
        cudaSetDevice(devs[0]);
        cudaError_t e = cudaMalloc(&tmp, count * sizeof(uint64_t));
        for (int i = 1; i < nslab && e == cudaSuccess; ++i) {
            cudaSetDevice(devs[i]);
            e = cudaStreamSynchronize(st[i]);
            cudaSetDevice(devs[0]);
            if (e == cudaSuccess) e = cudaMemcpyPeerAsync(tmp, devs[0], slabs[i].hist, devs[i], count * sizeof(uint64_t), st[0]);
            if (e == cudaSuccess) {
                add_u64<<<(unsigned)std::min<int64_t>(cdiv(count, 256), 1024), 256, 0, st[0]>>>(
                    reinterpret_cast<unsigned long long*>(slabs[0].hist), tmp, count);
                e = cudaGetLastError();
            }
        }
        if (e == cudaSuccess) e = cudaStreamSynchronize(st[0]);
        for (int i = 1; i < nslab && e == cudaSuccess; ++i)
            e = cudaMemcpyPeer(slabs[i].hist, devs[i], slabs[0].hist, devs[0], count * sizeof(uint64_t));
        if (tmp) {
            cudaSetDevice(devs[0]);
            cudaFree(tmp);
        }
        if (e != cudaSuccess) rc = FT_ERR_CUDA_BASE + (int)e;
    }
    for (int i = 0; i < nslab && rc == FT_OK; ++i) {
        cudaSetDevice(devs[i]);
        const cudaError_t e = cudaStreamSynchronize(st[i]);
        if (e != cudaSuccess) rc = FT_ERR_CUDA_BASE + (int)e;
    }
    cleanup();
    return rc;
}
