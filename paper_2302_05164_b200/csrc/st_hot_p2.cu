// Hot kernels (k_xmarch, k_xslab) of degree 2.
#define ST_HOT_P 2
#include "st_hot.cuh"
