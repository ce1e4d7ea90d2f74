// stmf_maxplus.cuh — config-5 kernel: dense masked max-plus product + error
// reduction (BASELINE.json configs[4]).  Included by stmf_api.cu.
//
//   err = sum over given (i, j) of |X_ij - max_k (U_ik + V_kj)|      (binary32,
//   exact-sum semantics as the fit's objective, tropical.py:214-222 in fp32)
//
// Layout: X dense m x n fp32 row-major, mask bit-packed (32 columns per word,
// row-major words), U stored k-major (r x m) and V (r x n) so a k-slice of either
// tile is one contiguous vector.
//
// Block tile 64 rows x 128 columns, 256 threads, each thread a 4 x 8 register
// micro-tile.  k-slices of U and V are staged in shared memory (double-buffered
// by k-chunks of 16); the inner loop per k-pair issues FADD2 (packed fp32 add,
// 2 sums per instruction) and a 3-input FMNMX (max of the accumulator and two
// sums), i.e. 1/32 warp-instruction per (entry, k).  The epilogue reads X with
// 128-bit loads and the mask word once per 32 columns, and accumulates the given
// residuals exactly (fp64 partials of values on the 2^-g grid -> 128-bit fixed
// point).  No tensor cores: max-plus is not a multiply-add contraction.
#pragma once

namespace stmf {

__device__ __forceinline__ float max3f(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
#if defined(__CUDA_ARCH__) && __CUDA_ARCH__ >= 1000
  return __fadd2_rn(a, b);
#else
  return make_float2(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y));
#endif
}

constexpr int kMpTR = 64, kMpTC = 128, kMpKC = 16;
constexpr int kMaxplusDynSmem = (kMpTR * kMpTC + kMpTR * kMpTC / 32) * 4;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }

// m % 64 == 0, n % 128 == 0 (k-slices beyond r are -inf); KC = k-chunk (even)
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

// TMA = true: the block's 64 x 128 X tile arrives by one bulk tensor copy
// (cp.async.bulk.tensor, tensor map xmap) completing on an mbarrier, instead of 2048
// 16-byte cp.async copies issued by all threads
template <int KC, bool TMA = false>
__global__ void __launch_bounds__(256, KC <= 4 ? 4 : 3)
k_maxplus_err(int64_t m, int64_t n, int r, const float* __restrict__ X, const uint32_t* __restrict__ mask,
              const float* __restrict__ Ut, const float* __restrict__ V, u64* __restrict__ acc,
              int* __restrict__ flags, int F, double exact_limit, const __grid_constant__ CUtensorMap xmap = {},
              const __grid_constant__ CUtensorMap umap = {}, const __grid_constant__ CUtensorMap vmap = {}) {
  __shared__ __align__(128) float Us[2][KC][kMpTR];
  __shared__ __align__(128) float Vs[2][KC][kMpTC];
  // dynamic shared memory (kMaxplusDynSmem): the block's 64 x 128 X tile (32 KB) and its mask words
  extern __shared__ __align__(128) unsigned char dyn_smem[];
  float (*Xs)[kMpTC] = reinterpret_cast<float (*)[kMpTC]>(dyn_smem);
  uint32_t (*Ms)[kMpTC / 32] = reinterpret_cast<uint32_t (*)[kMpTC / 32]>(dyn_smem + sizeof(float) * kMpTR * kMpTC);
  __shared__ double red[8];
  int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  int64_t row0 = (int64_t)blockIdx.y * kMpTR, col0 = (int64_t)blockIdx.x * kMpTC;
  // the epilogue's HBM traffic is issued first (async copies into shared memory),
  // so it streams while the k-loop computes
  __shared__ __align__(8) uint64_t xbar, fbar[2];
  // when r is a multiple of KC every k-chunk of the factor slices arrives by TMA too
  // (double-buffered, one mbarrier per buffer; the k >= r rows that staging fills
  // with -inf do not exist then)
  const bool tma_f = TMA && r % KC == 0;
  auto issue_f = [&](int buf, int k0) {  // thread 0: chunk k0.. into buffer buf
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&fbar[buf])),
                 "r"((unsigned)(sizeof(float) * KC * (kMpTR + kMpTC))));
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
        "[%4];" ::"r"(smem_u32(&Us[buf][0][0])),
        "l"(&umap), "r"((int)row0), "r"(k0), "r"(smem_u32(&fbar[buf]))
        : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
        "[%4];" ::"r"(smem_u32(&Vs[buf][0][0])),
        "l"(&vmap), "r"((int)col0), "r"(k0), "r"(smem_u32(&fbar[buf]))
        : "memory");
  };
  auto wait_f = [&](int buf, int parity) {
    asm volatile(
        "{\n .reg .pred p;\n FWAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra FWAIT_%=;\n}" ::"r"(smem_u32(&fbar[buf])),
        "r"(parity)
        : "memory");
  };
  if constexpr (TMA) {
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&xbar)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&fbar[0])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&fbar[1])));
      asm volatile("fence.proxy.async.shared::cta;");
      if (tma_f) issue_f(0, 0);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&xbar)),
                   "r"((unsigned)(sizeof(float) * kMpTR * kMpTC)));
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
          "[%4];" ::"r"(smem_u32(&Xs[0][0])),
          "l"(&xmap), "r"((int)col0), "r"((int)row0), "r"(smem_u32(&xbar))
          : "memory");
    }
  } else {
#pragma unroll
    for (int h = 0; h < 8; h++) {
      int e = threadIdx.x + 256 * h;  // 2048 16-byte chunks
      int rr = e >> 5, c4 = (e & 31) * 4;
      cp_async16(&Xs[rr][c4], X + (row0 + rr) * n + col0 + c4);
    }
  }
  if (threadIdx.x < kMpTR) {
    const uint32_t* mw = mask + ((row0 + threadIdx.x) * n + col0) / 32;
    cp_async16(&Ms[threadIdx.x][0], mw);
  }
  asm volatile("cp.async.commit_group;\n" ::);
  float a4[4][8];
#pragma unroll
  for (int i = 0; i < 4; i++)
#pragma unroll
    for (int j = 0; j < 8; j++) a4[i][j] = -CUDART_INF_F;

  // staging: a KC x 64 U slice (KC*16 float4) and a KC x 128 V slice (KC*32 float4)
  auto stage = [&](int buf, int k0) {
    for (int e = threadIdx.x; e < KC * 16; e += 256) {
      int kk = e >> 4, c4 = (e & 15) * 4;
      float4 v = make_float4(-CUDART_INF_F, -CUDART_INF_F, -CUDART_INF_F, -CUDART_INF_F);
      if (k0 + kk < r) v = *reinterpret_cast<const float4*>(Ut + (int64_t)(k0 + kk) * m + row0 + c4);
      *reinterpret_cast<float4*>(&Us[buf][kk][c4]) = v;
    }
    for (int e = threadIdx.x; e < KC * 32; e += 256) {
      int kk = e >> 5, c4 = (e & 31) * 4;
      float4 v = make_float4(-CUDART_INF_F, -CUDART_INF_F, -CUDART_INF_F, -CUDART_INF_F);
      if (k0 + kk < r) v = *reinterpret_cast<const float4*>(V + (int64_t)(k0 + kk) * n + col0 + c4);
      *reinterpret_cast<float4*>(&Vs[buf][kk][c4]) = v;
    }
  };

  int nchunks = (r + KC - 1) / KC;
  if (!tma_f) stage(0, 0);
  __syncthreads();
  for (int ch = 0; ch < nchunks; ch++) {
    int buf = ch & 1;
    if (tma_f) {
      // buffer buf^1 was last read in chunk ch-1, which ended with __syncthreads
      if (threadIdx.x == 0 && ch + 1 < nchunks) issue_f(buf ^ 1, (ch + 1) * KC);
      wait_f(buf, (ch >> 1) & 1);
    } else if (ch + 1 < nchunks) {
      stage(buf ^ 1, (ch + 1) * KC);
    }
#pragma unroll
    for (int kk = 0; kk < KC; kk += 2) {
      float4 ua = *reinterpret_cast<const float4*>(&Us[buf][kk][ty * 4]);
      float4 ub = *reinterpret_cast<const float4*>(&Us[buf][kk + 1][ty * 4]);
      float4 va0 = *reinterpret_cast<const float4*>(&Vs[buf][kk][tx * 8]);
      float4 va1 = *reinterpret_cast<const float4*>(&Vs[buf][kk][tx * 8 + 4]);
      float4 vb0 = *reinterpret_cast<const float4*>(&Vs[buf][kk + 1][tx * 8]);
      float4 vb1 = *reinterpret_cast<const float4*>(&Vs[buf][kk + 1][tx * 8 + 4]);
      float u0[4] = {ua.x, ua.y, ua.z, ua.w}, u1[4] = {ub.x, ub.y, ub.z, ub.w};
      float2 v0[4] = {make_float2(va0.x, va0.y), make_float2(va0.z, va0.w), make_float2(va1.x, va1.y),
                      make_float2(va1.z, va1.w)};
      float2 v1[4] = {make_float2(vb0.x, vb0.y), make_float2(vb0.z, vb0.w), make_float2(vb1.x, vb1.y),
                      make_float2(vb1.z, vb1.w)};
#pragma unroll
      for (int i = 0; i < 4; i++) {
        float2 s0 = make_float2(u0[i], u0[i]), s1 = make_float2(u1[i], u1[i]);
#pragma unroll
        for (int jj = 0; jj < 4; jj++) {
          float2 p = fadd2(s0, v0[jj]);
          float2 q = fadd2(s1, v1[jj]);
          a4[i][2 * jj] = max3f(a4[i][2 * jj], p.x, q.x);
          a4[i][2 * jj + 1] = max3f(a4[i][2 * jj + 1], p.y, q.y);
        }
      }
    }
    __syncthreads();
  }
  // epilogue: given residuals, exact accumulation
  cp_async_wait_all();
  if constexpr (TMA) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n"
        " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(&xbar))
        : "memory");
  }
  __syncthreads();
  double part = 0.0;
#pragma unroll
  for (int i = 0; i < 4; i++) {
    int rl = ty * 4 + i;
    float4 x0 = *reinterpret_cast<const float4*>(&Xs[rl][tx * 8]);
    float4 x1 = *reinterpret_cast<const float4*>(&Xs[rl][tx * 8 + 4]);
    float xs[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
    uint32_t word = Ms[rl][(tx * 8) >> 5];
    uint32_t bits = (word >> ((tx * 8) & 31)) & 0xffu;
#pragma unroll
    for (int j = 0; j < 8; j++)
      if (bits & (1u << j)) part = __dadd_rn(part, (double)fabsf(__fsub_rn(xs[j], a4[i][j])));
  }
  // block reduction (per-thread partials are exact; the sum of 256 of them too)
  for (int o = 16; o; o >>= 1) part = __dadd_rn(part, __shfl_xor_sync(0xffffffffu, part, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = part;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < 8; w++) s = __dadd_rn(s, red[w]);
    int fl = 0;
    if (!(s < exact_limit)) fl |= 4;
    u64 hi, lo;
    fx_from_double(s, F, hi, lo, fl);
    fx_atomic_add(acc, hi, lo);
    if (fl) atomicOr(flags, fl);
  }
}

// counter-based uniform floats on the 2^-24 grid in [lo, lo + 2): splitmix64
__device__ __forceinline__ u64 splitmix64(u64 x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

__global__ void k_gen_uniform(int64_t count, u64 seed, float* __restrict__ out) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; t < count; t += stride) {
    u64 h = splitmix64(seed ^ (u64)t * 0xD1B54A32D192ED03ull);
    out[t] = (float)(int)(h >> 40) * (1.0f / 16777216.0f) * 2.0f - 1.0f;  // U[-1, 1), multiples of 2^-23
  }
}

// bit-packed iid mask with P(given) = density
__global__ void k_gen_mask(int64_t words, u64 seed, uint32_t threshold24, uint32_t* __restrict__ mask) {
  int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; w < words; w += stride) {
    uint32_t bits = 0;
    for (int b = 0; b < 32; b++) {
      u64 h = splitmix64(seed ^ ((u64)w * 32 + b) * 0x9E3779B97F4A7C15ull);
      bits |= (uint32_t)((h >> 40) < threshold24) << b;
    }
    mask[w] = bits;
  }
}

}  // namespace stmf
