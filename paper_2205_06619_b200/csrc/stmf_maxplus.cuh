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

// ----------------------------------------------------------------------------
// Sampled (compacted) variant for low densities: only the given entries are read and
// computed.  The reference's objective ranges over the given entries only
// (tropical.py:214-222: b_norm of the residual at mask), so a layout that stores just
// the given values (plus the bit-packed mask that says where they are) is the
// algorithmic minimum: m*n/8 + 4*given bytes, versus m*n*(4 + 1/8) for the dense tile.
//
// Layout: tiles of 128 x 128 entries in row-major tile order; a tile's given values
// are packed contiguously, row-major within the tile (tile_off[t] = first value of
// tile t, an exclusive scan of the tile counts).  Factors row-major with a padded
// stride RS (U: m x RS, V: n x RS; padding = -inf, so it never wins a max).
//
// Per tile (one block of 256 threads, persistent over tiles): the factor rows of the
// tile are staged in shared memory, the tile's 128 x 4 mask words (prefetched into
// registers while the previous tile computed) are decoded into a list of (row, column)
// codes in exactly the packed-value order (warp scans of the row counts, popc ranks
// within words), and the threads walk that list: one coalesced value load + RQ float4
// loads of each factor row per given entry, FADD2 pairs and 3-input max.  Exact
// accumulation as the dense kernel.
constexpr int kSpT = 128;      // tile edge
__host__ __device__ constexpr int sp_stride(int rq) { return rq % 2 ? 4 * rq : 4 * rq + 4; }

template <int RQ, bool SEARCH = false>
__global__ void __launch_bounds__(256)
k_maxplus_err_sampled(int64_t m, int64_t n, const uint32_t* __restrict__ mask, const float* __restrict__ vals,
                      const int64_t* __restrict__ tile_off, const float* __restrict__ Urm,
                      const float* __restrict__ Vrm, u64* __restrict__ acc, int* __restrict__ flags, int F,
                      double exact_limit) {
  constexpr int RS = sp_stride(RQ);
  extern __shared__ __align__(16) unsigned char sp_smem[];
  float* Us = reinterpret_cast<float*>(sp_smem);
  float* Vs = Us + kSpT * RS;
  uint16_t* list = reinterpret_cast<uint16_t*>(Vs + kSpT * RS);
  __shared__ __align__(16) uint4 Mw[kSpT];
  __shared__ int rowoff[kSpT + 1], wsum[4];
  __shared__ double red[8];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  // tile indices fit in 32 bits (m, n < 2^31 and 128 x 128 tiles)
  const int ntx = (int)(n / kSpT), T = (int)((m / kSpT) * ntx);
  const int64_t wpr = n / 32;  // mask words per matrix row
  double part = 0.0;
  // the first tile's mask words (one 16-byte load per row); later tiles' are prefetched
  // into registers while the previous tile computes
  uint4 mw = make_uint4(0, 0, 0, 0);
  int t = blockIdx.x;
  if (t < T && tid < kSpT)
    mw = __ldg(reinterpret_cast<const uint4*>(mask + ((int64_t)(t / ntx) * kSpT + tid) * wpr + (t % ntx) * (kSpT / 32)));
  for (; t < T; t += gridDim.x) {
    const int64_t row0 = (int64_t)(t / ntx) * kSpT, col0 = (int64_t)(t % ntx) * kSpT;
    // 1. factor rows of the tile (L2-resident across tiles)
    for (int e = tid; e < kSpT * RQ; e += 256) {
      int rr = e / RQ, q = e - rr * RQ;
      *reinterpret_cast<float4*>(Us + rr * RS + 4 * q) =
          __ldg(reinterpret_cast<const float4*>(Urm + (row0 + rr) * RS) + q);
      *reinterpret_cast<float4*>(Vs + rr * RS + 4 * q) =
          __ldg(reinterpret_cast<const float4*>(Vrm + (col0 + rr) * RS) + q);
    }
    // 2. row counts, exclusive scan over the tile's 128 rows (warps 0..3)
    if (tid < kSpT) {
      Mw[tid] = mw;
      int c = __popc(mw.x) + __popc(mw.y) + __popc(mw.z) + __popc(mw.w), x = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      rowoff[tid] = x - c;  // within the warp; the warp prefixes are added below
      if (lane == 31) wsum[wid] = x;
    }
    __syncthreads();
    const int tn = t + gridDim.x;  // prefetch the next tile's mask words (consumed at its step 2)
    if (tn < T && tid < kSpT)
      mw = __ldg(reinterpret_cast<const uint4*>(mask + ((int64_t)(tn / ntx) * kSpT + tid) * wpr + (tn % ntx) * (kSpT / 32)));
    const int pre0 = wsum[0], pre1 = pre0 + wsum[1], pre2 = pre1 + wsum[2];
    const int total = pre2 + wsum[3];
    if (SEARCH) {
      // SEARCH: every thread locates its entries by binary search over the tile's row
      // offsets and a select within the row's words (no code list; lanes stay converged)
      int* rg = reinterpret_cast<int*>(list);  // the code-list space holds the global row offsets
      if (tid < kSpT) rg[tid] = rowoff[tid] + (tid >= 96 ? pre2 : tid >= 64 ? pre1 : tid >= 32 ? pre0 : 0);
      __syncthreads();
      const float* vc = vals + tile_off[t];
      for (int e = tid; e < total; e += 256) {
        int lo = 0;
#pragma unroll
        for (int step = 64; step; step >>= 1)
          if (rg[lo + step] <= e) lo += step;
        int kq = e - rg[lo];
        uint4 v4 = Mw[lo];
        int c0 = __popc(v4.x), c1 = __popc(v4.y), c2 = __popc(v4.z);
        uint32_t wd;
        int wi;
        if (kq < c0) { wd = v4.x; wi = 0; }
        else if (kq < c0 + c1) { wd = v4.y; wi = 1; kq -= c0; }
        else if (kq < c0 + c1 + c2) { wd = v4.z; wi = 2; kq -= c0 + c1; }
        else { wd = v4.w; wi = 3; kq -= c0 + c1 + c2; }
        int b = (int)__fns(wd, 0, kq + 1);
        float x = __ldg(vc + e);
        const float4* ur = reinterpret_cast<const float4*>(Us + lo * RS);
        const float4* vr = reinterpret_cast<const float4*>(Vs + (wi * 32 + b) * RS);
        float p0 = -CUDART_INF_F, p1 = -CUDART_INF_F;
#pragma unroll
        for (int q = 0; q < RQ; q++) {
          float4 u = ur[q], v = vr[q];
          float2 a = fadd2(make_float2(u.x, u.y), make_float2(v.x, v.y));
          float2 c = fadd2(make_float2(u.z, u.w), make_float2(v.z, v.w));
          p0 = max3f(p0, a.x, a.y);
          p1 = max3f(p1, c.x, c.y);
        }
        part = __dadd_rn(part, (double)fabsf(__fsub_rn(x, fmaxf(p0, p1))));
      }
      __syncthreads();
      continue;
    }
    // 3. decode into (row, column) codes in the packed-value order: 2 (row, word) pairs per thread
#pragma unroll
    for (int h = 0; h < 2; h++) {
      int pr = tid + 256 * h;
      int rl = pr >> 2, wi = pr & 3;
      uint4 v4 = Mw[rl];
      uint32_t wd = wi == 0 ? v4.x : wi == 1 ? v4.y : wi == 2 ? v4.z : v4.w;
      int pos = rowoff[rl] + (rl >= 96 ? pre2 : rl >= 64 ? pre1 : rl >= 32 ? pre0 : 0);
      if (wi > 0) pos += __popc(v4.x);
      if (wi > 1) pos += __popc(v4.y);
      if (wi > 2) pos += __popc(v4.z);
      while (wd) {
        int b = __ffs(wd) - 1;
        wd &= wd - 1;
        list[pos++] = (uint16_t)((rl << 7) | (wi * 32 + b));
      }
    }
    __syncthreads();
    // 4. the given entries: one coalesced value load, RQ float4 loads of each factor row
    const float* vc = vals + tile_off[t];
    for (int e = tid; e < total; e += 256) {
      float x = __ldg(vc + e);
      int code = list[e];
      const float4* ur = reinterpret_cast<const float4*>(Us + (code >> 7) * RS);
      const float4* vr = reinterpret_cast<const float4*>(Vs + (code & 127) * RS);
      float p0 = -CUDART_INF_F, p1 = -CUDART_INF_F;
#pragma unroll
      for (int q = 0; q < RQ; q++) {
        float4 u = ur[q], v = vr[q];
        float2 a = fadd2(make_float2(u.x, u.y), make_float2(v.x, v.y));
        float2 b = fadd2(make_float2(u.z, u.w), make_float2(v.z, v.w));
        p0 = max3f(p0, a.x, a.y);
        p1 = max3f(p1, b.x, b.y);
      }
      part = __dadd_rn(part, (double)fabsf(__fsub_rn(x, fmaxf(p0, p1))));
    }
    __syncthreads();
  }
  for (int o = 16; o; o >>= 1) part = __dadd_rn(part, __shfl_xor_sync(0xffffffffu, part, o));
  if (lane == 0) red[wid] = part;
  __syncthreads();
  if (tid == 0) {
    double sum = 0.0;
    for (int w = 0; w < 8; w++) sum = __dadd_rn(sum, red[w]);
    int fl = 0;
    if (!(sum < exact_limit)) fl |= 4;
    u64 hi, lo;
    fx_from_double(sum, F, hi, lo, fl);
    fx_atomic_add(acc, hi, lo);
    if (fl) atomicOr(flags, fl);
  }
}

template <int RQ>
constexpr size_t sp_smem_bytes() {
  return sizeof(float) * 2 * kSpT * sp_stride(RQ) + sizeof(uint16_t) * kSpT * kSpT;
}

// data preparation for the sampled layout (not timed): per-tile given counts, then the
// packed values in the kernel's order, and the padded row-major factor copies
__global__ void k_sp_tile_count(int64_t m, int64_t n, const uint32_t* __restrict__ mask, int64_t* __restrict__ cnt) {
  const int64_t ntx = n / kSpT, T = (m / kSpT) * ntx, wpr = n / 32;
  int lane = threadIdx.x & 31;
  for (int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; t < T;
       t += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const uint32_t* mt = mask + (t / ntx) * kSpT * wpr + (t % ntx) * (kSpT / 32);
    int c = 0;
    for (int e = lane; e < kSpT * 4; e += 32) c += __popc(mt[(e >> 2) * wpr + (e & 3)]);
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) cnt[t] = c;
  }
}

__global__ void k_sp_tile_fill(int64_t m, int64_t n, const uint32_t* __restrict__ mask, const float* __restrict__ X,
                               const int64_t* __restrict__ tile_off, float* __restrict__ vals) {
  const int64_t ntx = n / kSpT, T = (m / kSpT) * ntx, wpr = n / 32;
  int lane = threadIdx.x & 31;
  for (int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; t < T;
       t += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t row0 = (t / ntx) * kSpT, col0 = (t % ntx) * kSpT;
    int64_t pos = tile_off[t];
    for (int rl = 0; rl < kSpT; rl++)
      for (int wi = 0; wi < 4; wi++) {
        uint32_t w = mask[(row0 + rl) * wpr + col0 / 32 + wi];
        if ((w >> lane) & 1u) vals[pos + __popc(w & ((1u << lane) - 1u))] = X[(row0 + rl) * n + col0 + wi * 32 + lane];
        pos += __popc(w);
      }
  }
}

// factor k-major (r x len) -> row-major padded (len x RS), padding -inf
__global__ void k_sp_factor(int64_t len, int r, int RS, const float* __restrict__ src, float* __restrict__ dst) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= len * RS) return;
  int64_t i = t / RS;
  int k = (int)(t - i * RS);
  dst[t] = k < r ? src[(int64_t)k * len + i] : -CUDART_INF_F;
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
