// Dev harness: instantiate ONE lines3d_kernel variant for fast ptxas / SASS checks.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -Xptxas -v -cubin tools/dev/lines_one.cu
#include "../../paper_2311_11740_b200/csrc/ft_lines3d.cuh"
#ifndef DEV_FOLD
#define DEV_FOLD true
#endif
#ifndef DEV_EDGE
#define DEV_EDGE 2
#endif
#ifndef DEV_DS
#define DEV_DS 2048
#endif
#ifndef DEV_GUARD
#define DEV_GUARD false
#endif
template __global__ void ft::lines3d_kernel<FT_F32, FT_Q_POW2, true, ft::LINES_R, DEV_FOLD, DEV_DS, DEV_EDGE>(const float*, ft::LGeo, ft::QuantDev,
                                                                                   unsigned long long*);
