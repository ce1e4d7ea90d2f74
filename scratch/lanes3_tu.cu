#include <cudaTypedefs.h>
#include "stmf_kernels.cuh"
#include "stmf_maxplus.cuh"
#include "../../scratch/lanes_v3.cuh"
template __global__ void stmf::k_maxplus_err_lanes<1>(int64_t, int64_t, const unsigned char*, const int64_t*, const float*, const float*, stmf::u64*, int*, int, double, int, int, int);
template __global__ void stmf::k_maxplus_err_lanes<4>(int64_t, int64_t, const unsigned char*, const int64_t*, const float*, const float*, stmf::u64*, int*, int, double, int, int, int);
