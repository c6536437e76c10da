// Hot kernels (k_xmarch, k_xslab) of degree 1.
#define ST_HOT_P 1
#include "st_hot.cuh"
