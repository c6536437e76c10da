// Hot kernels (k_xmarch, k_xslab) of degree 3.
#define ST_HOT_P 3
#include "st_hot.cuh"
