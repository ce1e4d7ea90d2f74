// scratch translation unit: compiles only the config-5 kernels (fast codegen iteration)
#include <cudaTypedefs.h>
#include "stmf_kernels.cuh"
#include "stmf_maxplus.cuh"
#include "stmf_maxplus_lanes.cuh"
template __global__ void stmf::k_maxplus_err_lanes<1, 2048>(int64_t, int64_t, const unsigned char*, const int64_t*, const float*, const float*, stmf::u64*, int*, int, double, int, int, int);
template __global__ void stmf::k_maxplus_err_lanes<4, 512>(int64_t, int64_t, const unsigned char*, const int64_t*, const float*, const float*, stmf::u64*, int*, int, double, int, int, int);
