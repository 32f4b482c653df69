/*
 * fieldtopo_b200.h -- C ABI of the B200-native vertex-contribution engine.
 *
 * Drop-in boundary for the hot path of the reference package `fieldtopo`
 * (arXiv 2311.11740).  The reference's native layer is three Numba kernels
 * that accumulate birth/death histograms in place; each entry point below
 * replaces one of them (or the numpy pass after them) with a stream-ordered
 * CUDA launch on device memory.  Plain pointers and sizes only: no torch or
 * CUDA C++ types cross this boundary (`stream` is a cudaStream_t passed as
 * void*; NULL = legacy default stream).
 *
 * Conventions:
 *   return 0 = ok, 1 = bad argument (-> ValueError), 2 = classification
 *   failure (-> ClassificationError), >= 1000 = CUDA error 1000 + cudaError_t
 *   (-> RuntimeError).  The library never frees caller memory; histogram
 *   outputs are ACCUMULATED (+=) exactly like the reference kernels' q_in/q_out
 *   arguments, so callers zero them first.  Calls are asynchronous on
 *   `stream`; all arguments are read before the call returns.
 */
#ifndef FIELDTOPO_B200_H
#define FIELDTOPO_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FT_OK 0
#define FT_ERR_ARG 1
#define FT_ERR_CLASSIFY 2
#define FT_ERR_INTERNAL 3 /* unsupported device state (e.g. the shared-memory base the line kernels address absolutely) */
#define FT_ERR_CUDA_BASE 1000

/* element type of a field buffer */
#define FT_I32 0 /* int32 levels (Field2D/Field3D values, fields.py:17) */
#define FT_U8 1
#define FT_U16 2
#define FT_F32 3
#define FT_F64 4 /* ft_quantize / ft_minmax only (thresholds are then doubles) */

/* level decoding */
#define FT_Q_IDENTITY 0     /* the element IS the level */
#define FT_Q_TABLE 1        /* quantize_with_range via threshold table (fast) */
#define FT_Q_TABLE_ROBUST 2 /* same, for ill-conditioned ranges */
#define FT_Q_POW2 3         /* lo == 0, hi == 2^p: exact without a table (scale = M/hi);
                               kernels without a specialised path treat it as FT_Q_TABLE */

#define FT_NCLASS_2D 6  /* transition classes, 2D */
#define FT_NCLASS_3D 40 /* transition classes, 3D */
#define FT_NTYPE_2D 5   /* q1 q2 qd q3 q4            (contrib2d.py:36)    */
#define FT_NTYPE_3D 21  /* q10 .. q80                (contrib3d.py:35-44) */

/* Level decoding of a raw buffer.  For FT_Q_TABLE*: level(x) is the
 * reference quantize_with_range(x, lo, hi, M) (fields.py:20-33), decided by
 * `thresholds` (device, M+2 floats: [-inf, t_1 .. t_M, NaN], t_l = smallest
 * float32 whose reference level is >= l) after the estimate
 * est = clamp(floor(fmaf(x', scale, bias)), 0, M), x' = negate ? -x : x.
 * FT_Q_TABLE requires est in {L-1, L} (the caller checks the conditioning;
 * bias = -lo * scale) and negate == 0: level = est + (x >= t[est+1]).  FT_Q_TABLE_ROBUST
 * walks the table from any estimate. */
typedef struct ft_quant {
    int32_t mode;
    int32_t negate;
    float scale;
    float bias;
    const float *thresholds;
    /* the (lo, hi) of quantize_with_range the table was built from; 0, 0 when
     * unknown.  For uint8 / uint16 inputs and an integer range 0 <= lo < hi
     * the line kernels then decode levels in exact integer arithmetic
     * (floor((2 (x - lo) M + (hi - lo)) / (2 (hi - lo))) by a multiply-high,
     * checked against the float64 formula for every input value when a range
     * is first seen) instead of the table. */
    double lo, hi;
} ft_quant;

/* A device-resident run of consecutive rows (2D) or planes (3D) of a field
 * whose full extent is H rows/planes.  Rows/planes outside [0, H) are absent
 * cells (sentinel M+1, like the reference's padded border, sources.py:66-74);
 * rows/planes inside [0, H) that a launch needs must lie in
 * [first, first + count).  Element (r, ...) lives at
 * data + ((r - first) * row_elems + ...) + b * batch_stride. */
typedef struct ft_window {
    const void *data;
    int32_t dtype;
    int64_t first;
    int64_t count;
    int64_t batch;        /* 2D only: images sharing H x W; else 1 */
    int64_t batch_stride; /* elements between consecutive images */
} ft_window;

/* 2D transition histograms for vertex rows [v0, v1) (0 <= v0 <= v1 <= H+1)
 * of an H x W field (row-major, W contiguous).  hist: device uint64
 * [batch][6][M+2], accumulated.  Replaces _scan_rows_2d(padded, i0, i1, q_in,
 * q_out) (contrib2d.py:161-162) and its two-row streaming window
 * (_stream_rows_2d, contrib2d.py:235-251). */
int ft_hist2d(const ft_window *win, int64_t H, int64_t W, int64_t v0, int64_t v1,
              const ft_quant *q, int32_t M, uint64_t *hist, void *stream);

/* 3D transition histograms for vertex rows [v0, v1) of an H x W x D field
 * (index (i, j, k), k fastest; raw layout (i*W + j)*D + k, sources.py:379-386).
 * hist: device uint64 [40][M+2], accumulated.  Replaces _scan_slabs_3d
 * (contrib3d.py:351-352) and _scan_pencil_pair_3d / _stream_slabs_3d
 * (contrib3d.py:373-414). */
int ft_hist3d(const ft_window *win, int64_t H, int64_t W, int64_t D, int64_t v0, int64_t v1,
              const ft_quant *q, int32_t M, uint64_t *hist, void *stream);

/* Fused curve path (no maps): histograms, by level, of the cells of the
 * closed cubical complex -- an element appears at the MIN level of its
 * incident cells (MAX level for the "all incident cells active" counts).
 * Order-free, so no tie-breaking; every builtin descriptor_curve
 * (descriptors.py:83-97, 169-178) is an integer combination of the rows
 * (DESIGN.md §3b).  Lattice points cover [v0, v1) x [0, W] (x [0, D]).
 * 3D hist: device uint64 [4][M+2] rows (cells, face mins, edge mins,
 *   vertex mins); requires (M+1)*4 <= 65535 and, unlike ft_hist3d, the
 *   window must also hold plane v0-2 (when >= 0).
 * 2D hist: device uint64 [batch][4][M+2] rows (cells, edge mins, vertex
 *   mins, vertex maxes; the last only when maxes != 0).
 * Both accumulate, like ft_hist2d/3d. */
int ft_lattice3d(const ft_window *win, int64_t H, int64_t W, int64_t D, int64_t v0, int64_t v1,
                 const ft_quant *q, int32_t M, uint64_t *hist, void *stream);
int ft_lattice2d(const ft_window *win, int64_t H, int64_t W, int64_t v0, int64_t v1,
                 const ft_quant *q, int32_t M, int32_t maxes, uint64_t *hist, void *stream);

/* Fused curve path for 3D EC / surface-area / volume (ft_lines.cu): the same
 * counts as ft_lattice3d folded into three rows, with ~2.6 instead of 10
 * shared-memory events per lattice point (EC by 1D extremum events along i of
 * four min-derived line families, cubes and faces by per-cell signatures;
 * DESIGN.md §3e).  hist: device uint64 [3][M+2], accumulated: cells C,
 * faces F, and X = V - E (two's complement, may be negative), so
 * EC_26C = X + F - C, surface area = 2F - 6C, volume = C; tables outside
 * span{C, F, V - E} need ft_lattice3d.  Window as ft_lattice3d (planes
 * v0-2 .. v1-1).  Requires ft_lines3d_ok(M) (M <= ~2300). */
int ft_lines3d(const ft_window *win, int64_t H, int64_t W, int64_t D, int64_t v0, int64_t v1,
               const ft_quant *q, int32_t M, uint64_t *hist, void *stream);
int ft_lines3d_ok(int32_t M);

/* Fused curve path for 2D EC_8C / perimeter / area (ft_lines2d.cu), batched
 * like ft_lattice2d: the same rows 0..2 (cells, edge mins, vertex mins) of
 * hist [batch][4][M+2], accumulated, computed with the vertices from sparse
 * 1D extremum events (EC = sum over column lines of chi1(min over adjacent
 * columns) - chi1(column)); row 3 (vertex maxes, EC_4C) is not
 * touched -- use ft_lattice2d with maxes for it.  Replaces the same
 * reference path as ft_lattice2d (contrib2d.py:161-232 + descriptors.py:
 * 169-178).  Window: rows v0-2 .. v1-1.  Requires ft_lines2d_ok(M)
 * (M <= ~1000). */
int ft_lines2d(const ft_window *win, int64_t H, int64_t W, int64_t v0, int64_t v1,
               const ft_quant *q, int32_t M, uint64_t *hist, void *stream);
int ft_lines2d_ok(int32_t M);

/* Transition histograms -> contribution maps and descriptor curves.
 * hist [batch][C][M+2] (C = 6 or 40).  q_in / q_out (may be NULL): device
 * uint64 [batch][T][M+2], OVERWRITTEN with the reference maps
 * (ContributionMap2D/3D.q_in/q_out, contrib2d.py:45-105, contrib3d.py:138-200).
 * class_w: device int64 [n_desc][C] per-class curve deltas in eighths
 * (w[dst] - w[src], see ft_class_weights); numerators: device int64
 * [batch][n_desc][M+1] OVERWRITTEN with descriptor_curve(...).numerators
 * (counts_at_levels + eighths @ counts, descriptors.py:153-178) computed as a
 * device prefix scan over levels. */
int ft_finalize(int32_t ndim, int32_t M, int64_t batch, const uint64_t *hist, uint64_t *q_in,
                uint64_t *q_out, int32_t n_desc, const int64_t *class_w, int64_t *numerators,
                void *stream);

/* Generic weighted level prefix scan: numerators[b][d][l] =
 * sum_{l' <= l} sum_r row_w[d][r] * rows[b][r][l'] for l in [0, M]; rows:
 * device uint64 [batch][n_rows][M+2], row_w: device int64 [n_desc][n_rows].
 * With rows = (q_in; q_out) and row_w = (eighths; -eighths) this is
 * descriptor_curve(cmap, table).numerators (descriptors.py:169-178); with
 * one-hot weights it is counts_at_levels (descriptors.py:153-161). */
int ft_curves(const uint64_t *rows, int32_t n_rows, int32_t M, int64_t batch, int32_t n_desc,
              const int64_t *row_w, int64_t *numerators, void *stream);

/* Per-class curve deltas for a weight table in eighths (WeightTable.eighths,
 * descriptors.py:27-48): out[c] = eighths[dst(c)] - eighths[src(c)] (host). */
int ft_class_weights(int32_t ndim, const int64_t *eighths, int64_t *out);

/* The transition tables compiled into the library (host memory):
 * step[(1 << S) * S] (class booked when slot joins mask, -1 invalid),
 * src[C], dst[C] (type index; -1 = empty stage).  S = 4 (2D) or 8 (3D). */
int ft_tables(int32_t ndim, int32_t *step, int32_t *src, int32_t *dst);

/* quantize_with_range (fields.py:20-33) on device: out[i] = level(x[i]). */
int ft_quantize(const void *x, int32_t dtype, int64_t n, const ft_quant *q, int32_t M,
                int32_t *out, void *stream);

/* ------------------------------------------------------------ runtime */

#define FT_KIND_MAP 0   /* transition-class histograms (ft_hist2d / ft_hist3d layout) */
#define FT_KIND_FUSED 1 /* fused curve rows: 3D ft_lines3d [3][M+2], 2D ft_lines2d [4][M+2] (rows 0..2) */

/* Out-of-core chunk streaming (the reference's low-memory mode,
 * _stream_rows_2d / _stream_slabs_3d, contrib2d.py:235-251,
 * contrib3d.py:392-414).  begin: a field of H rows/planes (W [x D] elements
 * each, `dtype`, decoded by `q`; q->thresholds must stay valid until end)
 * whose histogram `hist` (device, zeroed, layout of `kind`) is accumulated on
 * `stream`; two device buffers of `chunk_rows` rows (>= 3).  push: the next
 * `nrows` consecutive rows from host (pinned or pageable) or device memory,
 * any batch size; copies run on an internal stream into the buffer being
 * filled, the 2 rows a full buffer shares with the next are carried
 * device-to-device, and the kernel for every vertex row whose planes have
 * arrived runs on `stream` while the next buffer fills.  end: after all H
 * rows were pushed, books the last vertex rows, waits for `stream` and frees
 * the state (also on error).  Replaces the Python-level window loops with
 * one native engine (gather.stream_hist is its Python twin). */
typedef struct ft_stream ft_stream;
int ft_stream_begin(int32_t ndim, int64_t H, int64_t W, int64_t D, int32_t dtype, const ft_quant *q, int32_t M,
                    int32_t kind, int64_t chunk_rows, uint64_t *hist, void *stream, ft_stream **out);
int ft_stream_push(ft_stream *s, const void *rows, int64_t nrows);
int ft_stream_end(ft_stream *s);

/* One slab of a field spread over several GPUs of this process: planes
 * `win` resident on `device` (with `quant`'s thresholds on that device) and
 * the vertex rows [v0, v1) it books into `hist` (device memory on `device`,
 * zeroed, layout of `kind`). */
typedef struct ft_slab {
    int32_t device;
    ft_window win;
    int64_t v0, v1;
    ft_quant quant;
    uint64_t *hist;
} ft_slab;

/* The reference's worker split (_parallel.py:8-33) across GPUs: every slab's
 * histogram on its own device, then ONE all-reduce so that every slab's
 * `hist` holds the whole-field histogram -- ncclAllReduce (sum, uint64) when
 * all devices are distinct and NCCL is loadable (*used_nccl = 1), else a
 * peer-copy reduction.  Synchronous: returns when every hist is final. */
int ft_multi_gather3d(const ft_slab *slabs, int32_t nslab, int64_t H, int64_t W, int64_t D, int32_t M, int32_t kind,
                      int32_t *used_nccl);

/* Classification status of the 3D map kernels since the last call (waits for
 * `stream`): FT_ERR_CLASSIFY when a vertex neighbourhood fell outside the
 * configuration table -- the reference's ValueError (contrib3d.py:304-305,
 * 330) / ClassificationError (contrib3d.py:425-426) -- else FT_OK.  The
 * tables are total over the 8! slot orders, so only a corrupted table can
 * trip it; ft_debug_trap_tables(1) (tests only) installs such a table on the
 * current device and ft_debug_trap_tables(0) restores the real one. */
int ft_classify_status(void *stream);
int ft_debug_trap_tables(int32_t on);

/* 8-bit BMP pixel data as stored in the file (H rows of row_stride bytes,
 * bottom-up when bottom_up != 0) -> compact top-first H x W uint8 levels on
 * the device (reference read_bmp, sources.py:154-164: row flip + unpadding). */
int ft_bmp_decode(const uint8_t *raw, int64_t H, int64_t W, int64_t row_stride, int32_t bottom_up, uint8_t *out,
                  void *stream);

/* Verification hook (tests only, not a reference interface): run one of the
 * device quantizers the fused kernels inline -- path 0 to_level (map / wide
 * kernels, ft_quantize), 1 to_level4 (march / lattice kernels, incl. the
 * table-free FT_Q_POW2 form), 2 pack_pow2_sat (line kernels, float32 pairs,
 * FT_Q_POW2 only, n even), 3 the line kernels' exact integer decoding of
 * uint16 pairs (integer ranges lo < hi <= 65535 with q->lo / q->hi set, n
 * even; FT_ERR_ARG for other ranges) -- over a flat float32 / uint16 buffer
 * into int32 levels, so every input value can be checked against
 * fields.py:20-33. */
int ft_quantize_probe(const void *x, int32_t dtype, int64_t n, const ft_quant *q, int32_t M, int32_t path,
                      int32_t *out, void *stream);

/* Device min / max of a buffer (quantize's data range, fields.py:44-45;
 * RawVolumeSource._scan_range, sources.py:335-347).  out: device uint32[2],
 * OVERWRITTEN with order-preserving keys of (min, max); decode with
 * ft_key_to_double (FT_F64: see below). */
int ft_minmax(const void *x, int32_t dtype, int64_t n, uint32_t *out, void *stream);
double ft_key_to_double(int32_t dtype, uint32_t key);
/* FT_F64 buffers: out is uint64[2]; decode with ft_key64_to_double. */
double ft_key64_to_double(uint64_t key);

/* Library version string. */
const char *ft_version(void);

#ifdef __cplusplus
}
#endif
#endif /* FIELDTOPO_B200_H */
