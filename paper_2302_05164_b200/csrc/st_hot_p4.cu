// Hot kernels (k_xmarch, k_xslab) of degree 4.
#define ST_HOT_P 4
#include "st_hot.cuh"
