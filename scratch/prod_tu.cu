#include <cudaTypedefs.h>
#include "stmf_kernels.cuh"
template __global__ void stmf::k_product2<float>(int64_t, const int32_t*, const int32_t*, int64_t, int64_t, int, const float*, const float*, const float*, const float*, int, int, float*, float*, uint8_t*, uint8_t*, const int*);
template __global__ void stmf::k_product2<double>(int64_t, const int32_t*, const int32_t*, int64_t, int64_t, int, const double*, const double*, const double*, const double*, int, int, double*, double*, uint8_t*, uint8_t*, const int*);
