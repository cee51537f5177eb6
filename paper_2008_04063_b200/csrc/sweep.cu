// K6 placeholder (filled in below in a later step).
#include "hb_kernels.cuh"
