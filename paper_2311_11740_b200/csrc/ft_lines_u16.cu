// ft_lines_u16.cu -- ft_lines3d launchers for uint16 fields (C4b); kernel in
// ft_lines3d.cuh.
#include "ft_lines3d.cuh"

namespace ft {
int lines3d_u16(FT_LINES3D_ARGS, int qm)
{
    if (qm == FT_Q_IDENTITY) return launch_lines3d<FT_U16, FT_Q_IDENTITY>(win, H, W, D, v0, v1, q, M, hist, st);
    // integer range (e.g. the data's min / max): exact integer decoding, no table
    QuantDev probe{};
    if (umagic_fill(q, M, 65536, probe)) return launch_lines3d<FT_U16, FT_Q_UMAGIC>(win, H, W, D, v0, v1, q, M, hist, st);
    if (qm == FT_Q_POW2) return launch_lines3d<FT_U16, FT_Q_POW2>(win, H, W, D, v0, v1, q, M, hist, st);
    if (qm == FT_Q_TABLE) return launch_lines3d<FT_U16, FT_Q_TABLE>(win, H, W, D, v0, v1, q, M, hist, st);
    return launch_lines3d<FT_U16, FT_Q_TABLE_ROBUST>(win, H, W, D, v0, v1, q, M, hist, st);
}
}  // namespace ft
