// ft_lines_u8i32.cu -- ft_lines3d launchers for uint8 fields and int32 level
// fields; kernel in ft_lines3d.cuh.
#include "ft_lines3d.cuh"

namespace ft {
int lines3d_u8i32(FT_LINES3D_ARGS, int dtype, int qm)
{
    if (dtype == FT_I32) {
        if (qm != FT_Q_IDENTITY) return FT_ERR_ARG;
        return launch_lines3d<FT_I32, FT_Q_IDENTITY>(win, H, W, D, v0, v1, q, M, hist, st);
    }
    if (qm == FT_Q_IDENTITY) return launch_lines3d<FT_U8, FT_Q_IDENTITY>(win, H, W, D, v0, v1, q, M, hist, st);
    QuantDev probe{};
    if (umagic_fill(q, M, 256, probe)) return launch_lines3d<FT_U8, FT_Q_UMAGIC>(win, H, W, D, v0, v1, q, M, hist, st);
    if (qm == FT_Q_TABLE || qm == FT_Q_POW2) return launch_lines3d<FT_U8, FT_Q_TABLE>(win, H, W, D, v0, v1, q, M, hist, st);
    return launch_lines3d<FT_U8, FT_Q_TABLE_ROBUST>(win, H, W, D, v0, v1, q, M, hist, st);
}
}  // namespace ft
