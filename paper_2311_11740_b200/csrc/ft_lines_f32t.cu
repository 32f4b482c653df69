// ft_lines_f32t.cu -- ft_lines3d launchers for float32 fields quantized by
// threshold table (any range); kernel in ft_lines3d.cuh.
#include "ft_lines3d.cuh"

namespace ft {
int lines3d_f32_table(FT_LINES3D_ARGS, int qm)
{
    if (qm == FT_Q_TABLE) return launch_lines3d<FT_F32, FT_Q_TABLE>(win, H, W, D, v0, v1, q, M, hist, st);
    return launch_lines3d<FT_F32, FT_Q_TABLE_ROBUST>(win, H, W, D, v0, v1, q, M, hist, st);
}
}  // namespace ft
