// ft_lines_f32p.cu -- ft_lines3d launcher for float32 fields on a power-of-two
// range (the benchmark path, C4a / C5); kernel in ft_lines3d.cuh.
#include "ft_lines3d.cuh"

namespace ft {
int lines3d_f32_pow2(FT_LINES3D_ARGS) { return launch_lines3d<FT_F32, FT_Q_POW2>(win, H, W, D, v0, v1, q, M, hist, st); }
}  // namespace ft
