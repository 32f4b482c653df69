// ft_tables.h -- transition-class tables shared by the kernels' launchers.
#pragma once
#include <stdint.h>

#include "../../include/fieldtopo_b200.h"

namespace ft {

struct Tables {
    int S;          // slots per neighbourhood (4 or 8)
    int n_classes;  // 6 or 40
    int step[256 * 8];
    int src[64];
    int dst[64];
};

const Tables& tables(int ndim);

// Kernel-parameter copies (passed by value: 2 KB fits the 32 KB parameter
// space of sm_70+ under CUDA 12.1+, so no per-device constant upload).
struct Step3 {
    uint8_t cls[256 * 8];  // 255 = invalid
};
struct ClassMap {
    int8_t src[64];
    int8_t dst[64];
};

}  // namespace ft
