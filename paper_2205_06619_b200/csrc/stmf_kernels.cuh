// stmf_kernels.cuh — sm_100a device code of the FastSTMF fitting engine.
//
// Data layout in HBM (work orientation, m <= n after orient):
//   CSR  row_ptr[m+1] (int64), col_idx[N] (int32), xr[N] (T)     given entries by row
//   CSC  col_ptr[n+1] (int64), row_idx[N] (int32), xc[N] (T)     given entries by column
//   Ut   rank x m  (column k of U contiguous: the F-ULF/F-URF update unit)
//   V    rank x n
//   per-state product caches, in both CSR and CSC order:
//        t1[N] = (U(x)V)_ij, t2[N] = max_{l != arg} (U_il + V_lj), ag[N] = argmax (uint8)
//   per-k residuation statistics (top-2 minima with argmin):
//        colstats of (X_ij - U_ik) over i  -> cm1/cm2/cmarg (rank x n)
//        rowstats of (X_ij - V_kj) over j  -> rm1/rm2/rmarg (rank x m)
//
// Every elementwise op is a single correctly rounded IEEE add/sub or an exact
// max/min/abs, so products, argmax, residuations and residuals are bit-identical
// to numpy (T = double) or to the binary32 restatement (T = float).
#pragma once
#include <cuda_runtime.h>
#include <cub/block/block_merge_sort.cuh>
#include <math_constants.h>
#include <stdint.h>

namespace stmf {

typedef unsigned long long u64;

// Checked build (STMF_CHECKS, _ext.build(checked=True) -> lib/libstmf_b200_checked.so):
// every gathered index is range-checked on the device and a violation traps with the
// kernel's file:line (a stand-in for compute-sanitizer, which this pool does not run).
#ifdef STMF_CHECKS
#include <cstdio>
#define STMF_IDX(i, n)                                                                              \
  do {                                                                                            \
    if ((unsigned long long)(long long)(i) >= (unsigned long long)(long long)(n)) {               \
      printf("stmf check failed %s:%d: index %lld not in [0, %lld)\n", __FILE__, __LINE__,         \
             (long long)(i), (long long)(n));                                                     \
      __trap();                                                                                   \
    }                                                                                             \
  } while (0)
#else
#define STMF_IDX(i, n) \
  do {                 \
  } while (0)
#endif

struct U64Less {
  __device__ __forceinline__ bool operator()(u64 a, u64 b) const { return a < b; }
};

// Control state of the device-resident sweep (stmf_graph.cuh): the kernels of a
// captured CUDA graph read their per-row / per-batch parameters from here.
struct DevCtl {
  int64_t i;             // row being visited
  int64_t nc;            // its candidates
  int64_t t0;            // first candidate of the current batch
  int E, next;           // batch size, next batch size
  int accepted;          // the row visit accepted an update
  int win_op, win_q, win_k, win_slot;
  int cache_k;           // factor index of the last commit
  double err;            // current objective
  // fp64 decision scan over the batch's 2E evals (reference order)
  int pos, nchunk;
  int ch_ev[8], ch_q[8], ch_op[8], ch_cert[8];
  int fb[8];             // slot needs the full-sort fallback
  // run bookkeeping
  long long attempts, accepts, visits, evaluated, escalations, traj_len, traj_cap;
  long long batches, esc_rounds;
  int direct;            // accept committed before its numpy replica (certain accept)
  long long start_row;   // first row of this graph launch (resumption after error 4)
  int direct_cap;        // changed-entry limit of a direct accept's delta replica
  double err_prev;       // err before a direct accept (its replica must be below)
  unsigned long long tb0, phaseB_ns;  // graph-mode phase-B timing (%globaltimer)
  unsigned long long te0, esc_ns, ta0, acc_ns, sweep_ns;  // escalation rounds, accept bodies, whole sweep
  double sweep;          // trajectory time stamp of this sweep
  int error;             // 1: decision bound violated, 2: trajectory capacity
  int stop;              // time budget reached
  unsigned long long deadline_ns;  // %globaltimer deadline (0: none)
  // schedule (Session::row_visit)
  double sched_scale, sched_growth;
  int sched_add, batch_floor, Emax, first0;
  int e_round;  // batch sizes are rounded up to a multiple of this (kEG: whole eval groups)
  int ema_first;         // rows without depth history: first batch from depth_ema
  double depth_ema;      // running mean of accepting depths (candidates)
};

// Phase B costs a whole group of kEG evals per side whether the group is full or not, so a
// batch of E candidates is rounded up to whole groups: the padding slots become speculative
// evals of the next candidates instead of duplicates (same decisions in the same order).
__host__ __device__ inline int round_batch(int e, int r, int emax) {
  if (r > 1) e = (e + r - 1) / r * r;
  return e < emax ? e : emax;
}

// ----------------------------------------------------------------------------
// scalar helpers (explicit _rn intrinsics: no contraction, no fast-math)
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
// fp64 min/max as compare-select: no NaN can occur on the path (given entries and
// factors are finite; +-inf only as identities), so IEEE fmin's NaN handling is
// dead weight (DSETP + 2 selects instead of DSETP.MIN + SEL + LOP3 + FSEL)
__device__ __forceinline__ double vmin(double a, double b) { return b < a ? b : a; }
__device__ __forceinline__ float vmin(float a, float b) { return fminf(a, b); }
__device__ __forceinline__ double vmax(double a, double b) { return b > a ? b : a; }
__device__ __forceinline__ float vmax(float a, float b) { return fmaxf(a, b); }
__device__ __forceinline__ double vabs(double a) { return fabs(a); }
__device__ __forceinline__ float vabs(float a) { return fabsf(a); }
template <typename T> __device__ __forceinline__ T tinf();
template <> __device__ __forceinline__ double tinf<double>() { return CUDART_INF; }
template <> __device__ __forceinline__ float tinf<float>() { return CUDART_INF_F; }
__device__ __forceinline__ double shfl_xor(double v, int o) { return __shfl_xor_sync(0xffffffffu, v, o); }
__device__ __forceinline__ float shfl_xor(float v, int o) { return __shfl_xor_sync(0xffffffffu, v, o); }

// ----------------------------------------------------------------------------
// 128-bit fixed point (LSB 2^-F) used for every cross-thread error reduction.
// fp32 mode: F = data grid g (all values are multiples of 2^-g), the
// per-line fp64 partials are exact and the conversion below is exact.
// fp64 mode: F = 60, conversion truncates (<= 2^-60 per line, in the bound).
// flag bit 1: inexact conversion, bit 2: overflow / non-finite.
__device__ __forceinline__ void fx_from_double(double x, int F, u64& hi, u64& lo, int& flag) {
  u64 b = (u64)__double_as_longlong(x);
  int e = (int)((b >> 52) & 0x7ff);
  u64 mant = b & 0xFFFFFFFFFFFFFull;
  hi = 0; lo = 0;
  if (e == 0x7ff || (b >> 63)) { flag |= 2; return; }
  if (e == 0) { if (mant == 0) return; e = 1; } else mant |= (1ull << 52);
  int s = e - 1075 + F;
  if (s >= 0) {
    if (s > 74) { flag |= 2; return; }
    if (s == 0) lo = mant;
    else if (s < 64) { lo = mant << s; hi = mant >> (64 - s); }
    else hi = mant << (s - 64);
  } else {
    int t = -s;
    if (t >= 64) { if (mant) flag |= 1; return; }
    lo = mant >> t;
    if (mant & ((1ull << t) - 1)) flag |= 1;
  }
}

__device__ __forceinline__ void fx_atomic_add(u64* acc, u64 hi, u64 lo) {
  if (lo) {
    u64 old = atomicAdd(acc, lo);
    if (old + lo < old) hi += 1;
  }
  if (hi) atomicAdd(acc + 1, hi);
}

// ----------------------------------------------------------------------------
// Build kernels: dense X + byte mask -> CSR / CSC (given entries, index order).

__global__ void k_count_rows(int64_t m, int64_t n, const uint8_t* __restrict__ mask,
                             int64_t* __restrict__ cnt) {
  int lane = threadIdx.x & 31;
  int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = w; r < m; r += nw) {
    int64_t c = 0;
    for (int64_t j = lane; j < n; j += 32) c += mask[r * n + j] != 0;
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) cnt[r] = c;
  }
}

__global__ void k_count_cols(int64_t m, int64_t n, const uint8_t* __restrict__ mask,
                             int64_t* __restrict__ cnt) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  int64_t c = 0;
  for (int64_t r = 0; r < m; r++) c += mask[r * n + j] != 0;
  cnt[j] = c;
}

// exclusive scan of cnt[0..len) into ptr[0..len] (single block, len small: m or n)
__global__ void k_scan_ptr(int64_t len, const int64_t* __restrict__ cnt, int64_t* __restrict__ ptr) {
  __shared__ int64_t part[1024];
  int t = threadIdx.x, nt = blockDim.x;
  int64_t per = (len + nt - 1) / nt;
  int64_t b = t * per, e = b + per < len ? b + per : len;
  int64_t s = 0;
  for (int64_t i = b; i < e; i++) s += cnt[i];
  part[t] = s;
  __syncthreads();
  if (t == 0) {
    int64_t run = 0;
    for (int i = 0; i < nt; i++) { int64_t v = part[i]; part[i] = run; run += v; }
    ptr[len] = run;
  }
  __syncthreads();
  int64_t run = part[t];
  for (int64_t i = b; i < e; i++) { ptr[i] = run; run += cnt[i]; }
}

template <typename T>
__global__ void k_fill_csr(int64_t m, int64_t n, const T* __restrict__ X, const uint8_t* __restrict__ mask,
                           const int64_t* __restrict__ ptr, int32_t* __restrict__ idx, T* __restrict__ xv) {
  int lane = threadIdx.x & 31;
  int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = w; r < m; r += nw) {
    int64_t pos = ptr[r];
    for (int64_t j0 = 0; j0 < n; j0 += 32) {
      int64_t j = j0 + lane;
      bool g = j < n && mask[r * n + j] != 0;
      unsigned bal = __ballot_sync(0xffffffffu, g);
      if (g) {
        int64_t p = pos + __popc(bal & ((1u << lane) - 1));
        idx[p] = (int32_t)j;
        xv[p] = X[r * n + j];
      }
      pos += __popc(bal);
    }
  }
}

template <typename T>
__global__ void k_fill_csc(int64_t m, int64_t n, const T* __restrict__ X, const uint8_t* __restrict__ mask,
                           const int64_t* __restrict__ ptr, int32_t* __restrict__ idx, T* __restrict__ xv) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  int64_t p = ptr[j];
  for (int64_t r = 0; r < m; r++)
    if (mask[r * n + j]) { idx[p] = (int32_t)r; xv[p] = X[r * n + j]; p++; }
}

// ----------------------------------------------------------------------------
// Product caches.  CSR pass: warp per row (U_r. is warp-uniform).

template <typename T>
__device__ __forceinline__ void top2_entry(const T* __restrict__ Ut, const T* __restrict__ V, int64_t m,
                                           int64_t n, int rank, int64_t r, int64_t c, T& b1, T& b2, int& a) {
  b1 = add_rn(Ut[r], V[c]);
  b2 = -tinf<T>();
  a = 0;
  for (int l = 1; l < rank; l++) {
    T s = add_rn(Ut[(int64_t)l * m + r], V[(int64_t)l * n + c]);
    if (s > b1) { b2 = b1; b1 = s; a = l; }
    else b2 = vmax(b2, s);
  }
}

template <typename T>
__global__ void k_product_csr(int64_t m, int64_t n, int rank, const int64_t* __restrict__ ptr,
                              const int32_t* __restrict__ idx, const T* __restrict__ Ut, const T* __restrict__ V,
                              T* __restrict__ t1, T* __restrict__ t2, uint8_t* __restrict__ ag) {
  int lane = threadIdx.x & 31;
  int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = w; r < m; r += nw) {
    for (int64_t p = ptr[r] + lane; p < ptr[r + 1]; p += 32) {
      T b1, b2; int a;
      top2_entry(Ut, V, m, n, rank, r, (int64_t)idx[p], b1, b2, a);
      t1[p] = b1; t2[p] = b2; ag[p] = (uint8_t)a;
    }
  }
}

// CSC pass, fp64 oracle-compat: thread per column, rows ascending, so the column
// score is summed exactly in numpy's td_grid(...).sum(axis=0) order
// (strategies.py:185: sequential over rows).  Also the TD_A column histogram.
template <typename T>
__global__ void k_product_csc_seq(int64_t m, int64_t n, int rank, const int64_t* __restrict__ ptr,
                                  const int32_t* __restrict__ idx, const T* __restrict__ xc,
                                  const T* __restrict__ Ut, const T* __restrict__ V, T* __restrict__ t1,
                                  T* __restrict__ t2, uint8_t* __restrict__ ag, double* __restrict__ score,
                                  int32_t* __restrict__ colhist) {
  int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= n) return;
  double s = 0.0;
  int32_t* h = colhist + c * rank;
  for (int l = 0; l < rank; l++) h[l] = 0;
  for (int64_t p = ptr[c]; p < ptr[c + 1]; p++) {
    T b1, b2; int a;
    top2_entry(Ut, V, m, n, rank, (int64_t)idx[p], c, b1, b2, a);
    t1[p] = b1; t2[p] = b2; ag[p] = (uint8_t)a;
    s = __dadd_rn(s, (double)vabs(sub_rn(xc[p], b1)));
    h[a] += 1;
  }
  score[c] = s;
}

// CSC pass, fp64 oracle-compat, warp per column: lanes compute 32 entries'
// products in parallel, then every lane folds the 32 td values in row order with
// shuffles — the same sequential summation order as k_product_csc_seq.  The TD_A
// histogram is counted in a per-warp shared-memory slice (rank <= 255).
template <typename T>
__global__ void __launch_bounds__(256)
k_product_csc_warpseq(int64_t m, int64_t n, int rank, const int64_t* __restrict__ ptr,
                      const int32_t* __restrict__ idx, const T* __restrict__ xc, const T* __restrict__ Ut,
                      const T* __restrict__ V, T* __restrict__ t1, T* __restrict__ t2, uint8_t* __restrict__ ag,
                      double* __restrict__ score, int32_t* __restrict__ colhist) {
  __shared__ int32_t hist[8][256];
  int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t c = w; c < n; c += nw) {
    for (int l = lane; l < rank; l += 32) hist[wib][l] = 0;
    __syncwarp();
    double s = 0.0;
    int64_t beg = ptr[c], end = ptr[c + 1];
    for (int64_t base = beg; base < end; base += 32) {
      int64_t p = base + lane;
      double td = 0.0;
      if (p < end) {
        T b1, b2; int a;
        top2_entry(Ut, V, m, n, rank, (int64_t)idx[p], c, b1, b2, a);
        t1[p] = b1; t2[p] = b2; ag[p] = (uint8_t)a;
        td = (double)vabs(sub_rn(xc[p], b1));
        atomicAdd(&hist[wib][a], 1);
      }
      int cnt = end - base < 32 ? (int)(end - base) : 32;
      for (int l = 0; l < cnt; l++) s = __dadd_rn(s, __shfl_sync(0xffffffffu, td, l));
    }
    __syncwarp();
    if (lane == 0) score[c] = s;
    for (int l = lane; l < rank; l += 32) colhist[c * rank + l] = hist[wib][l];
    __syncwarp();
  }
}

// CSC pass, exact mode: warp per column; the fp64 partials of binary32 terms on
// the 2^-g grid are exact below 2^(53-g) (checked: flag bit 4), so the warp sum
// is the exact column score, order independent.
template <typename T>
__global__ void k_product_csc_exact(int64_t m, int64_t n, int rank, const int64_t* __restrict__ ptr,
                                    const int32_t* __restrict__ idx, const T* __restrict__ xc,
                                    const T* __restrict__ Ut, const T* __restrict__ V, T* __restrict__ t1,
                                    T* __restrict__ t2, uint8_t* __restrict__ ag, double* __restrict__ score,
                                    int32_t* __restrict__ colhist, double exact_limit, int* __restrict__ flags) {
  int lane = threadIdx.x & 31;
  int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t c = w; c < n; c += nw) {
    double s = 0.0;
    for (int64_t p = ptr[c] + lane; p < ptr[c + 1]; p += 32) {
      T b1, b2; int a;
      top2_entry(Ut, V, m, n, rank, (int64_t)idx[p], c, b1, b2, a);
      t1[p] = b1; t2[p] = b2; ag[p] = (uint8_t)a;
      s = __dadd_rn(s, (double)vabs(sub_rn(xc[p], b1)));
      atomicAdd(&colhist[c * rank + a], 1);
    }
    for (int o = 16; o; o >>= 1) s = __dadd_rn(s, shfl_xor(s, o));
    if (lane == 0) {
      if (!(s < exact_limit)) atomicOr(flags, 4);
      score[c] = s;
    }
  }
}

// ----------------------------------------------------------------------------
// Product caches with the second argmax (a2 = an index attaining t2; 255 if
// rank == 1).  After an accepted update only factor index k changed, so an
// entry whose top-2 indices exclude k is updated exactly from the new k-term
// alone; entries with k among them are recomputed over all l.  Either order
// (lines = CSR rows or CSC columns).
template <typename T>
__device__ __forceinline__ void top2_full(const T* __restrict__ Ut, const T* __restrict__ V, int64_t m, int64_t n,
                                          int rank, int64_t r, int64_t c, T& b1, T& b2, int& a1, int& a2) {
  b1 = add_rn(Ut[r], V[c]);
  b2 = -tinf<T>();
  a1 = 0;
  a2 = 255;
  for (int l = 1; l < rank; l++) {
    T s = add_rn(Ut[(int64_t)l * m + r], V[(int64_t)l * n + c]);
    if (s > b1) { b2 = b1; a2 = a1; b1 = s; a1 = l; }
    else if (s > b2) { b2 = s; a2 = l; }
  }
}

// top-2 of U_r. + V_.c from the row-major copies Urm (m x rp) and Vcm (n x rp),
// rp = rank padded to 16 bytes: every load is a 16-byte vector of consecutive l
template <typename T>
__device__ __forceinline__ void top2_vec(const T* __restrict__ Ur, const T* __restrict__ Vc, int rank, T& b1, T& b2,
                                         int& a1, int& a2) {
  constexpr int W = 16 / sizeof(T);
  b1 = -tinf<T>();
  b2 = -tinf<T>();
  a1 = 0;
  a2 = 255;
  for (int l0 = 0; l0 < rank; l0 += W) {
    T u[W], v[W];
    if (sizeof(T) == 4) {
      float4 a = __ldg(reinterpret_cast<const float4*>(Ur + l0));
      float4 b = __ldg(reinterpret_cast<const float4*>(Vc + l0));
      u[0] = a.x; u[1] = a.y; u[2] = a.z; u[3] = a.w;
      v[0] = b.x; v[1] = b.y; v[2] = b.z; v[3] = b.w;
    } else {
      double2 a = __ldg(reinterpret_cast<const double2*>(Ur + l0));
      double2 b = __ldg(reinterpret_cast<const double2*>(Vc + l0));
      u[0] = a.x; u[1] = a.y;
      v[0] = b.x; v[1] = b.y;
    }
#pragma unroll
    for (int q = 0; q < W; q++) {
      int l = l0 + q;
      if (l >= rank) break;
      T s = add_rn(u[q], v[q]);
      if (l == 0) { b1 = s; a1 = 0; }
      else if (s > b1) { b2 = b1; a2 = a1; b1 = s; a1 = l; }
      else if (s > b2) { b2 = s; a2 = l; }
    }
  }
}

template <typename T> struct Vec16;  // 16-byte vector of T (defined with the eval layouts below)

// the same with all NV 16-byte vectors of both rows loaded before the first compare: the
// rows come from L2, and one round of latency instead of NV dependent ones is what the
// recompute path of k_product2 costs (97% of its warps have a lane on it at rank 20)
template <typename T, int NV>
__device__ __forceinline__ void top2_vec_n(const T* __restrict__ Ur, const T* __restrict__ Vc, int rank, T& b1, T& b2,
                                           int& a1, int& a2) {
  constexpr int W = 16 / sizeof(T);
  using V16 = typename Vec16<T>::type;
  V16 u[NV], v[NV];
#pragma unroll
  for (int i = 0; i < NV; i++) {
    u[i] = __ldg(reinterpret_cast<const V16*>(Ur) + i);
    v[i] = __ldg(reinterpret_cast<const V16*>(Vc) + i);
  }
  b1 = -tinf<T>();
  b2 = -tinf<T>();
  a1 = 0;
  a2 = 255;
#pragma unroll
  for (int i = 0; i < NV; i++) {
    T uu[W], vv[W];
    Vec16<T>::unpack(u[i], uu, 0);
    Vec16<T>::unpack(v[i], vv, 0);
#pragma unroll
    for (int q = 0; q < W; q++) {
      int l = i * W + q;
      if (l >= rank) break;
      T s = add_rn(uu[q], vv[q]);
      if (l == 0) { b1 = s; a1 = 0; }
      else if (s > b1) { b2 = b1; a2 = a1; b1 = s; a1 = l; }
      else if (s > b2) { b2 = s; a2 = l; }
    }
  }
}

// rp = the padded row length (a multiple of 16 bytes)
template <typename T>
__device__ __forceinline__ void top2_rows(const T* __restrict__ Ur, const T* __restrict__ Vc, int rank, int rp, T& b1,
                                          T& b2, int& a1, int& a2) {
  switch (rp / (16 / (int)sizeof(T))) {
    case 1: top2_vec_n<T, 1>(Ur, Vc, rank, b1, b2, a1, a2); break;
    case 2: top2_vec_n<T, 2>(Ur, Vc, rank, b1, b2, a1, a2); break;
    case 3: top2_vec_n<T, 3>(Ur, Vc, rank, b1, b2, a1, a2); break;
    case 4: top2_vec_n<T, 4>(Ur, Vc, rank, b1, b2, a1, a2); break;
    case 5: top2_vec_n<T, 5>(Ur, Vc, rank, b1, b2, a1, a2); break;
    case 6: top2_vec_n<T, 6>(Ur, Vc, rank, b1, b2, a1, a2); break;
    default: top2_vec(Ur, Vc, rank, b1, b2, a1, a2); break;
  }
}

// copy factor column k (contiguous in Ut / V rows) into the padded row-major copy
template <typename T>
__global__ void k_scatter_factor(int64_t len, int rp, int k, const T* __restrict__ src, T* __restrict__ dst) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < len) dst[t * rp + k] = src[t];
}

// flat over the N given entries of one order (rowof/colof: the entry's row and
// column) -> perfectly balanced whatever the line lengths.
//
// k < 0: every entry recomputed over all l.  k >= 0 (after an accepted update only factor
// index k changed): an entry whose top-2 indices exclude k takes the new k-term alone; an
// entry with k among them needs all l again.  Those are ~2 / rank of the entries, so nearly
// every warp has one, and recomputing them in place made the whole pass issue-bound on a
// divergent path that ran with 7-13 of 32 lanes active (ncu at config 4: 8.6-14.6 warp
// instructions per entry, 19% of HBM; profiles/r02_product2.md).  Instead every warp queues
// the entries that need the recompute in shared memory and recomputes them 32 at a time, one
// per lane, whenever its queue holds a full warp's worth (and the rest at the end).  No block
// barriers, no global atomics.  (Tried first: a global list + a second kernel — the
// single-address atomics and the scattered second pass made it slower than the divergent
// version; then a per-block list between two barriers — 34% of HBM, a quarter of the stalls
// at the barriers.)
// 1: every thread owns 4 consecutive entries and reads each stream with one 16-byte load (config 4:
// 2.23 -> 1.80 ms per cache refresh; profiles/r02_ab9_kpack_pvec.log); 0: 2 entries, a block apart
#ifndef STMF_PROD_VEC
#define STMF_PROD_VEC 1
#endif
#ifndef STMF_PROD_U
#define STMF_PROD_U (STMF_PROD_VEC ? 4 : 2)
#endif
// 4 consecutive values of a cache stream with 16-byte loads
__device__ __forceinline__ void load4(const float* p, float (&o)[4]) {
  const float4 v = *reinterpret_cast<const float4*>(p);
  o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
}
__device__ __forceinline__ void load4(const double* p, double (&o)[4]) {
  const double2 a = *reinterpret_cast<const double2*>(p), b = *reinterpret_cast<const double2*>(p + 2);
  o[0] = a.x; o[1] = a.y; o[2] = b.x; o[3] = b.y;
}
constexpr int kProdU = STMF_PROD_U;  // entries per thread and iteration, their loads issued together
// resident blocks per SM (binary32): the pass is bound by load latency.  Scalar loads: 6 blocks (40
// registers, no spills) measured 15% faster than 4 at config 4 (profiles/r02_prod_ab.log).  Vector loads:
// 5 blocks (48 registers, no spills; 6 would spill 96 B, 4 measured the same as 5).  binary64 keeps 4.
#ifndef STMF_PROD_MINB
#define STMF_PROD_MINB (STMF_PROD_VEC ? 5 : 6)
#endif
template <typename T>
__global__ void __launch_bounds__(256, sizeof(T) == 4 ? STMF_PROD_MINB : 4)
k_product2(int64_t N, const int32_t* __restrict__ rowof, const int32_t* __restrict__ colof,
           int64_t m, int64_t n, int rank, const T* __restrict__ Ut, const T* __restrict__ V,
           const T* __restrict__ Urm, const T* __restrict__ Vcm, int rp, int k, T* __restrict__ t1,
           T* __restrict__ t2, uint8_t* __restrict__ ag, uint8_t* __restrict__ ag2,
           const int* __restrict__ kdev = nullptr) {
  if (kdev) k = *kdev;
  if (k < 0) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < N; p += (int64_t)gridDim.x * blockDim.x) {
      int64_t r = rowof[p], c = colof[p];
      STMF_IDX(r, m);
      STMF_IDX(c, n);
      T b1, b2;
      int a1, a2;
      top2_rows(Urm + r * rp, Vcm + c * rp, rank, rp, b1, b2, a1, a2);
      t1[p] = b1; t2[p] = b2; ag[p] = (uint8_t)a1; ag2[p] = (uint8_t)a2;
    }
    return;
  }
  // per-warp queue of entries that need all l (entry numbers fit 32 bits: N < 2^31 per device)
  __shared__ int32_t s_q[8][32 * (kProdU + 1)];
  const T* __restrict__ Uk = Ut + (int64_t)k * m;
  const T* __restrict__ Vk = V + (int64_t)k * n;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  int32_t* __restrict__ myq = s_q[wib];
  int qn = 0;  // queue length (warp-uniform)
  auto recompute = [&](int64_t q) {
    const int64_t rr = rowof[q], cc = colof[q];
    T n1, n2;
    int x1, x2;
    top2_rows(Urm + rr * rp, Vcm + cc * rp, rank, rp, n1, n2, x1, x2);
    t1[q] = n1; t2[q] = n2; ag[q] = (uint8_t)x1; ag2[q] = (uint8_t)x2;
  };
  const int64_t tile = (int64_t)blockDim.x * kProdU;
  for (int64_t base = blockIdx.x * tile; base < N; base += (int64_t)gridDim.x * tile) {
    int64_t p[kProdU];
    int32_t r[kProdU], c[kProdU];
    int a1[kProdU], a2[kProdU];
    T b1[kProdU], b2[kProdU], s[kProdU];
    bool ok[kProdU];
#if STMF_PROD_VEC
    // each thread owns kProdU = 4 consecutive entries: one 16-byte load per stream (4 bytes for
    // the index bytes) instead of four scalar ones, a warp reads 512 contiguous bytes per stream
    static_assert(kProdU == 4, "the vector variant handles 4 consecutive entries per thread");
    const int64_t p0 = base + (int64_t)threadIdx.x * 4;
    if (p0 + 4 <= N) {
      const int4 rv = *reinterpret_cast<const int4*>(rowof + p0);
      const int4 cv = *reinterpret_cast<const int4*>(colof + p0);
      const uchar4 av = *reinterpret_cast<const uchar4*>(ag + p0);
      const uchar4 aw = *reinterpret_cast<const uchar4*>(ag2 + p0);
      r[0] = rv.x; r[1] = rv.y; r[2] = rv.z; r[3] = rv.w;
      c[0] = cv.x; c[1] = cv.y; c[2] = cv.z; c[3] = cv.w;
      a1[0] = av.x; a1[1] = av.y; a1[2] = av.z; a1[3] = av.w;
      a2[0] = aw.x; a2[1] = aw.y; a2[2] = aw.z; a2[3] = aw.w;
      load4(t1 + p0, b1);
      load4(t2 + p0, b2);
#pragma unroll
      for (int u = 0; u < 4; u++) { p[u] = p0 + u; ok[u] = true; }
    } else {
#pragma unroll
      for (int u = 0; u < 4; u++) {
        p[u] = p0 + u;
        ok[u] = p[u] < N;
        const int64_t q = ok[u] ? p[u] : 0;
        r[u] = rowof[q]; c[u] = colof[q]; a1[u] = ag[q]; a2[u] = ag2[q]; b1[u] = t1[q]; b2[u] = t2[q];
      }
    }
#else
#pragma unroll
    for (int u = 0; u < kProdU; u++) {
      p[u] = base + u * (int64_t)blockDim.x + threadIdx.x;
      ok[u] = p[u] < N;
      const int64_t q = ok[u] ? p[u] : 0;
      r[u] = rowof[q];
      c[u] = colof[q];
      a1[u] = ag[q];
      a2[u] = ag2[q];
      b1[u] = t1[q];
      b2[u] = t2[q];
    }
#endif
#pragma unroll
    for (int u = 0; u < kProdU; u++) {
      STMF_IDX(r[u], m);
      STMF_IDX(c[u], n);
      s[u] = add_rn(Uk[r[u]], Vk[c[u]]);
    }
#pragma unroll
    for (int u = 0; u < kProdU; u++) {
      // k held a top-2 slot: all l again, from the warp's queue
      const bool slow = ok[u] && (a1[u] == k || a2[u] == k);
      const unsigned bal = __ballot_sync(0xffffffffu, slow);
      if (slow) myq[qn + __popc(bal & lt)] = (int32_t)p[u];
      qn += __popc(bal);
      if (!ok[u] || slow) continue;
      // k held neither top-2 slot: insert its new value (lowest index on max ties);
      // most entries keep their caches and are not written back
      T n1 = b1[u], n2 = b2[u];
      int x1 = a1[u], x2 = a2[u];
      if (s[u] > n1 || (s[u] == n1 && k < x1)) { n2 = n1; x2 = x1; n1 = s[u]; x1 = k; }
      else if (s[u] > n2) { n2 = s[u]; x2 = k; }
      else continue;
      t1[p[u]] = n1; t2[p[u]] = n2; ag[p[u]] = (uint8_t)x1; ag2[p[u]] = (uint8_t)x2;
    }
    __syncwarp();
    while (qn >= 32) {  // a full warp of recomputes (the queue holds fewer than 32 on loop entry)
      qn -= 32;
      const int64_t q = myq[qn + lane];
      __syncwarp();
      recompute(q);
    }
  }
  __syncwarp();
  if (lane < qn) recompute(myq[lane]);
}

// line index of every entry of a compacted layout (CSR -> row of each entry)
__global__ void k_line_of(int64_t nlines, const int64_t* __restrict__ ptr, int32_t* __restrict__ out) {
  int lane = threadIdx.x & 31;
  int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t L = w; L < nlines; L += nw)
    for (int64_t p = ptr[L] + lane; p < ptr[L + 1]; p += 32) out[p] = (int32_t)L;
}

// column scores + TD_A histogram from the CSC caches.  fp64 (numpy order): every
// lane folds the column's td values in row order; exact: warp sum of exact partials.
template <typename T>
__global__ void __launch_bounds__(256)
k_scores(int64_t n, int rank, const int64_t* __restrict__ ptr, const T* __restrict__ xc, const T* __restrict__ t1,
         const uint8_t* __restrict__ ag, double* __restrict__ score, int32_t* __restrict__ colhist, bool seq,
         double exact_limit, int* __restrict__ flags) {
  __shared__ int32_t hist[8][256];
  int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t c = w; c < n; c += nw) {
    for (int l = lane; l < rank; l += 32) hist[wib][l] = 0;
    __syncwarp();
    double s = 0.0;
    int64_t beg = ptr[c], end = ptr[c + 1];
    for (int64_t base = beg; base < end; base += 32) {
      int64_t p = base + lane;
      double td = 0.0;
      int a = -1;
      if (p < end) {
        td = (double)vabs(sub_rn(xc[p], t1[p]));
        a = ag[p];
      }
      // warp-aggregated histogram: one lane per distinct argmax adds its peers' count
      // (leaders hold distinct bins, so plain shared-memory adds do not race)
      unsigned peers = __match_any_sync(0xffffffffu, a);
      if (a >= 0 && lane == __ffs(peers) - 1) hist[wib][a] += __popc(peers);
      __syncwarp();  // orders this iteration's bin updates before the next iteration's
      if (seq) {
        int cnt = end - base < 32 ? (int)(end - base) : 32;
        for (int l = 0; l < cnt; l++) s = __dadd_rn(s, __shfl_sync(0xffffffffu, td, l));
      } else {
        s = __dadd_rn(s, td);
      }
    }
    if (!seq)
      for (int o = 16; o; o >>= 1) s = __dadd_rn(s, shfl_xor(s, o));
    __syncwarp();
    if (lane == 0) {
      if (!seq && !(s < exact_limit)) atomicOr(flags, 4);
      score[c] = s;
    }
    for (int l = lane; l < rank; l += 32) colhist[c * rank + l] = hist[wib][l];
    __syncwarp();
  }
}

// ----------------------------------------------------------------------------
// Residuation statistics for factor index k (top-2 minima + argmin).
template <typename T>
struct Top2 { T m1, m2; int a1; };

template <typename T>
__device__ __forceinline__ void top2_push(Top2<T>& t, T d, int idx) {
  if (d < t.m1) { t.m2 = t.m1; t.m1 = d; t.a1 = idx; }
  else t.m2 = vmin(t.m2, d);
}

template <typename T>
__device__ __forceinline__ Top2<T> top2_merge(const Top2<T>& A, const Top2<T>& B) {
  bool aw = (A.m1 < B.m1) || (A.m1 == B.m1 && A.a1 < B.a1);
  Top2<T> R;
  R.m1 = aw ? A.m1 : B.m1;
  R.a1 = aw ? A.a1 : B.a1;
  R.m2 = aw ? vmin(A.m2, B.m1) : vmin(B.m2, A.m1);
  return R;
}

template <typename T>
__device__ __forceinline__ Top2<T> top2_warp(Top2<T> t) {
  for (int o = 16; o; o >>= 1) {
    Top2<T> u;
    u.m1 = shfl_xor(t.m1, o);
    u.m2 = shfl_xor(t.m2, o);
    u.a1 = __shfl_xor_sync(0xffffffffu, t.a1, o);
    t = top2_merge(t, u);
  }
  return t;
}

// lines = CSR rows (other = V row k)  or  CSC columns (other = Ut row k):
// stats over entries p of line L of (x_p - other[idx_p]).
template <typename T>
__global__ void k_line_stats(int64_t nlines, const int64_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                             const T* __restrict__ xv, const T* __restrict__ other, T* __restrict__ s1,
                             T* __restrict__ s2, int32_t* __restrict__ sarg, int idx_offset = 0,
                             const int* __restrict__ kdev = nullptr, int64_t kso = 0, int64_t kss = 0) {
  if (kdev) {  // graph mode: factor index from the control block (row/col strides kso / kss)
    int k = *kdev;
    other += k * kso;
    s1 += k * kss;
    s2 += k * kss;
    sarg += k * kss;
  }
  int lane = threadIdx.x & 31;
  int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t L = w; L < nlines; L += nw) {
    Top2<T> t;
    t.m1 = tinf<T>(); t.m2 = tinf<T>(); t.a1 = 0x7fffffff;
    for (int64_t p = ptr[L] + lane; p < ptr[L + 1]; p += 32) {
      int j = idx[p];
      top2_push(t, sub_rn(xv[p], other[j]), j + idx_offset);  // argmin as a global index
    }
    t = top2_warp(t);
    if (lane == 0) { s1[L] = t.m1; s2[L] = t.m2; sarg[L] = t.a1; }
  }
}

// plain residuation of an arbitrary vector: out[L] = min_p x_p - vec[idx_p]
template <typename T>
__global__ void k_line_min(int64_t nlines, const int64_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                           const T* __restrict__ xv, const T* __restrict__ vec, T* __restrict__ out) {
  int lane = threadIdx.x & 31;
  int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t L = w; L < nlines; L += nw) {
    T mn = tinf<T>();
    for (int64_t p = ptr[L] + lane; p < ptr[L + 1]; p += 32) mn = vmin(mn, sub_rn(xv[p], vec[idx[p]]));
    for (int o = 16; o; o >>= 1) mn = vmin(mn, shfl_xor(mn, o));
    if (lane == 0) out[L] = mn;
  }
}

// ----------------------------------------------------------------------------
// Candidate list of one row visit (_ranked_row_candidates + TD_A votes).

__global__ void k_cand_keys(int64_t nc, const int32_t* __restrict__ cols, const double* __restrict__ score,
                            u64* __restrict__ keys, int32_t* __restrict__ vals) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= nc) return;
  // scores are >= +0: their bit patterns are monotone; ~ gives descending order,
  // the stable radix sort keeps ascending column order among equal scores
  // (np.argsort(-scores[cols], kind="stable"), strategies.py:187).
  keys[t] = ~(u64)__double_as_longlong(score[cols[t]]);
  vals[t] = (int32_t)t;
}

template <typename T>
__global__ void k_cand_build(int64_t nc, int rank, const int32_t* __restrict__ cols, const T* __restrict__ xrow,
                             const uint8_t* __restrict__ agrow, const int32_t* __restrict__ perm,
                             const int32_t* __restrict__ colhist, int32_t* __restrict__ cj, int32_t* __restrict__ ck,
                             T* __restrict__ cx, int sel = 0) {
  extern __shared__ int32_t rowhist[];
  for (int l = threadIdx.x; l < rank; l += blockDim.x) rowhist[l] = 0;
  __syncthreads();
  for (int64_t p = threadIdx.x; p < nc; p += blockDim.x) atomicAdd(&rowhist[agrow[p]], 1);
  __syncthreads();
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nc; t += (int64_t)gridDim.x * blockDim.x) {
    int p = perm[t];
    int j = cols[p];
    const int32_t* h = colhist + (int64_t)j * rank;
    int k = 0, best = -1;
    for (int l = 0; l < rank; l++) {  // _vote: argmax of bincount, lowest index on ties
      int v = rowhist[l] + h[l];
      if (v > best) { best = v; k = l; }
    }
    if (sel == 1) k = agrow[p];  // TD: argmax_k at (i, j) (strategies.py:146-148)
    cj[t] = j; ck[t] = k; cx[t] = xrow[p];
  }
}

// _ranked_row_candidates + TD_A votes + the dense copy of row i in ONE block for
// rows with nc <= 4 * 1024 given entries: keys ~score bits (descending score) with
// the entry index as value, stable block merge sort (equal scores keep ascending
// column order, np.argsort(-scores[cols], kind="stable"), strategies.py:187).
constexpr int kCandThreads = 1024;
template <typename T, int ITEMS>
__global__ void __launch_bounds__(kCandThreads)
k_cand_row(int nc, int64_t n, int rank, const int32_t* __restrict__ cols, const T* __restrict__ xrow,
           const uint8_t* __restrict__ agrow, const double* __restrict__ score, const int32_t* __restrict__ colhist,
           int32_t* __restrict__ cj, int32_t* __restrict__ ck, T* __restrict__ cx, T* __restrict__ xrow_dense,
           int64_t irow, const T* __restrict__ cm1, const T* __restrict__ cm2, const int32_t* __restrict__ cmarg,
           T* __restrict__ cmi, const DevCtl* __restrict__ g = nullptr, const int64_t* __restrict__ row_ptr = nullptr,
           int sel = 0) {
  using Sort = cub::BlockMergeSort<u64, kCandThreads, ITEMS, int>;
  __shared__ typename Sort::TempStorage tmp;
  __shared__ int32_t rowhist[256];
  if (g) irow = g->i;  // graph mode: the row from the control block
  // CM^(-i) of every k for the visited row (k_cmi): blocks 1.. when the launch has
  // them (rank * n values), else block 0 itself
  if (gridDim.x > 1) {
    if (blockIdx.x > 0) {
      for (int64_t t = (blockIdx.x - 1) * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)rank * n;
           t += (int64_t)(gridDim.x - 1) * blockDim.x)
        cmi[t] = (cmarg[t] == (int32_t)irow) ? cm2[t] : cm1[t];
      return;
    }
  } else {
    for (int64_t t = threadIdx.x; t < (int64_t)rank * n; t += blockDim.x)
      cmi[t] = (cmarg[t] == (int32_t)irow) ? cm2[t] : cm1[t];
  }
  if (g) {
    int64_t beg = row_ptr[irow];
    nc = (int)(row_ptr[irow + 1] - beg);
    cols += beg;
    xrow += beg;
    agrow += beg;
  }
  for (int l = threadIdx.x; l < rank; l += blockDim.x) rowhist[l] = 0;
  for (int64_t c = threadIdx.x; c < n; c += blockDim.x) xrow_dense[c] = tinf<T>();
  __syncthreads();
  u64 key[ITEMS];
  int val[ITEMS];
#pragma unroll
  for (int i = 0; i < ITEMS; i++) {
    int p = threadIdx.x * ITEMS + i;
    if (p < nc) {
      int c = cols[p];
      key[i] = ~(u64)__double_as_longlong(score[c]);
      atomicAdd(&rowhist[agrow[p]], 1);
      xrow_dense[c] = xrow[p];
    } else {
      key[i] = ~0ull;
    }
    val[i] = p;
  }
  Sort(tmp).StableSort(key, val, U64Less(), nc, ~0ull);
  __syncthreads();
#pragma unroll
  for (int i = 0; i < ITEMS; i++) {
    int t = threadIdx.x * ITEMS + i;
    if (t >= nc) continue;
    int p = val[i];
    int j = cols[p];
    const int32_t* h = colhist + (int64_t)j * rank;
    int k = 0, best = -1;
    for (int l = 0; l < rank; l++) {  // _vote: argmax of bincount, lowest index on ties
      int v = rowhist[l] + h[l];
      if (v > best) { best = v; k = l; }
    }
    if (sel == 1) k = agrow[p];  // TD: argmax_k at (i, j) (strategies.py:146-148)
    cj[t] = j; ck[t] = k; cx[t] = xrow[p];
  }
}

template <typename T>
__global__ void k_fill(int64_t len, T* __restrict__ a, T v) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < len) a[t] = v;
}

template <typename T>
__global__ void k_scatter_row(int64_t nc, const int32_t* __restrict__ cols, const T* __restrict__ x,
                              T* __restrict__ dense) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < nc) dense[cols[t]] = x[t];
}

// ----------------------------------------------------------------------------
// Phase A writes each eval's first-residuation vector in an eval-interleaved layout
// I[g][line][kEG]  (g = group of kEG evals): the kEG values of one given entry are one
// contiguous, naturally aligned row of kEG * sizeof(T) bytes (32 at binary32, 64 at
// binary64), fetched by phase B with 256-bit loads (LDG.E.256 on sm_100a).  A lane's
// gather then touches ONE cache line per entry and group instead of one per 16-byte plane
// of the earlier planar layout I[g][p][line][EGP] -- phase B at config 3 is bound by L1
// wavefronts, and each wavefront serves one line (profiles/r02_phaseB_c3.md).
// binary64 keeps the planar layout (its rows would be 64 bytes = two 256-bit loads, measured
// 3% slower at config 2); binary32 measured 1.4% (config 3) to 8-11% (config 4) faster with
// rows (profiles/r02_ilv_ab.log).  STMF_ILV_PLANAR=0 / 1 forces rows / planar for both types.
constexpr int kEG = 8;
#ifndef STMF_ILV_PLANAR
#define STMF_ILV_PLANAR -1
#endif

template <typename T>
struct Ilv {
  static constexpr int EGP = 16 / (int)sizeof(T);  // evals per 16-byte vector
  static constexpr int P = kEG / EGP;              // 16-byte vectors per entry and group
  // element stride between consecutive lines of one eval
  static constexpr bool PLANAR = STMF_ILV_PLANAR < 0 ? sizeof(T) == 8 : STMF_ILV_PLANAR != 0;
  static constexpr int STRIDE = PLANAR ? EGP : kEG;
};

// one 16-byte slot of the interleaved layout
template <typename T> struct Vec16;
template <> struct Vec16<float> {
  typedef float4 type;
  template <int N>
  __device__ __forceinline__ static void unpack(float4 a, float (&v)[N], int o) {
    v[o] = a.x; v[o + 1] = a.y; v[o + 2] = a.z; v[o + 3] = a.w;
  }
};
template <> struct Vec16<double> {
  typedef double2 type;
  template <int N>
  __device__ __forceinline__ static void unpack(double2 a, double (&v)[N], int o) {
    v[o] = a.x; v[o + 1] = a.y;
  }
};

template <typename T>
__host__ __device__ __forceinline__ int64_t ilv_index(int q, int64_t a, int64_t len) {
  if constexpr (Ilv<T>::PLANAR) {
    constexpr int EGP = Ilv<T>::EGP, P = Ilv<T>::P;
    int g = q / kEG, p = (q % kEG) / EGP, e = q % EGP;
    return (((int64_t)g * P + p) * len + a) * EGP + e;
  } else {
    return ((int64_t)(q / kEG) * len + a) * kEG + (q % kEG);
  }
}

template <typename T>
__device__ __forceinline__ void ilv_decode(int64_t t, int64_t len, int& q, int64_t& a) {
  if constexpr (Ilv<T>::PLANAR) {
    constexpr int EGP = Ilv<T>::EGP, P = Ilv<T>::P;
    int e = (int)(t % EGP);
    int64_t rest = t / EGP;
    a = rest % len;
    int64_t gp = rest / len;
    q = (int)(gp / P) * kEG + (int)(gp % P) * EGP + e;
  } else {
    int e = (int)(t % kEG);
    int64_t rest = t / kEG;
    a = rest % len;
    q = (int)(rest / len) * kEG + e;
  }
}

// 32 bytes (256-bit load, read-only path); p must be 32-byte aligned
__device__ __forceinline__ void ldg256(const float* p, float (&v)[8], int o = 0) {
  asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(v[o]), "=f"(v[o + 1]), "=f"(v[o + 2]), "=f"(v[o + 3]), "=f"(v[o + 4]), "=f"(v[o + 5]),
                 "=f"(v[o + 6]), "=f"(v[o + 7])
               : "l"(p));
}
__device__ __forceinline__ void ldg256(const double* p, double (&v)[8], int o) {
  asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(v[o]), "=d"(v[o + 1]), "=d"(v[o + 2]), "=d"(v[o + 3])
               : "l"(p));
}

// the kEG first-residuation values of line c of group g (vin = the whole buffer)
template <typename T>
__device__ __forceinline__ void load_group_row(const T* __restrict__ vin, int g, int64_t len, int64_t c, T (&v)[kEG]) {
  if constexpr (Ilv<T>::PLANAR) {
    using V16 = typename Vec16<T>::type;
    const V16* b = reinterpret_cast<const V16*>(vin) + (int64_t)g * Ilv<T>::P * len + c;
#pragma unroll
    for (int p = 0; p < Ilv<T>::P; p++) Vec16<T>::unpack(__ldg(b + p * len), v, p * Ilv<T>::EGP);
  } else {
    const T* b = vin + ((int64_t)g * len + c) * kEG;
    if constexpr (sizeof(T) == 4) {
      ldg256(b, v);
    } else {
      ldg256(b, v, 0);
      ldg256(b + 4, v, 4);
    }
  }
}

// Phase A.  F-ULF evals q: v'_c = min(CM^(-i)_c, X_ic - s_q), s_q = X_ij - V_kj
// (engine.py:222-223: U_ik <- X_ij - V_kj; V_k. <- rr(U_.k), with only u_i changed).
template <typename T>
__global__ void k_phaseA_ulf(int64_t n, int E, int64_t i, const int32_t* __restrict__ cj,
                             const int32_t* __restrict__ ck, const T* __restrict__ cx, const T* __restrict__ V,
                             const T* __restrict__ cm1, const T* __restrict__ cm2, const int32_t* __restrict__ cmarg,
                             const T* __restrict__ xrow_dense, T* __restrict__ vI, int* __restrict__ chg,
                             T* __restrict__ s_out = nullptr) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int G = (E + kEG - 1) / kEG;
  if (t >= (int64_t)G * kEG * n) return;
  int q;
  int64_t c;
  ilv_decode<T>(t, n, q, c);
  if (q >= E) { vI[t] = tinf<T>(); return; }
  int k = ck[q];
  int64_t kn = (int64_t)k * n;
  T s = sub_rn(cx[q], V[kn + cj[q]]);
  T cmx = (cmarg[kn + c] == (int32_t)i) ? cm2[kn + c] : cm1[kn + c];
  T v = vmin(cmx, sub_rn(xrow_dense[c], s));
  vI[t] = v;
  if (s_out && c == 0) s_out[q] = s;
  if (v != V[kn + c]) chg[q] = 1;
}

// CM^(-i) for every k: the column minima of X - U.k without row i (top-2 statistics)
template <typename T>
__global__ void k_cmi(int64_t n, int rank, int64_t i, const T* __restrict__ cm1, const T* __restrict__ cm2,
                      const int32_t* __restrict__ cmarg, T* __restrict__ out) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < (int64_t)rank * n) out[t] = (cmarg[t] == (int32_t)i) ? cm2[t] : cm1[t];
}

// F-URF evals q: u'_r = min(RM^(-j)_r, X_rj - s'_q), s'_q = X_ij - U_ik
// (engine.py:234-235).  Fill from the row statistics, then the seed column.
template <typename T>
__global__ void k_phaseA_urf_fill(int64_t m, int E, const int32_t* __restrict__ cj, const int32_t* __restrict__ ck,
                                  const T* __restrict__ rm1, const T* __restrict__ rm2,
                                  const int32_t* __restrict__ rmarg, T* __restrict__ uI) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int G = (E + kEG - 1) / kEG;
  if (t >= (int64_t)G * kEG * m) return;
  int q;
  int64_t r;
  ilv_decode<T>(t, m, q, r);
  if (q >= E) { uI[t] = tinf<T>(); return; }
  int64_t km = (int64_t)ck[q] * m;
  uI[t] = (rmarg[km + r] == cj[q]) ? rm2[km + r] : rm1[km + r];
}

// what phase A needs to apply the F-URF seed column itself (small m)
template <typename T>
struct SeedCols {
  const int64_t* col_ptr;
  const int32_t* row_idx;
  const T* xc;
  const T* Ut;
};

// Both first residuations of a batch in one launch: blocks [0, nb_ulf) run the F-ULF
// values (k_phaseA_ulf), the rest the F-URF fill (k_phaseA_urf_fill); block 0 also
// copies the batch's factor indices next to the results the host reads back.
template <typename T>
__global__ void k_phaseA(int64_t m, int64_t n, int E, int64_t i, unsigned nb_ulf, const int32_t* __restrict__ cj,
                         const int32_t* __restrict__ ck, const T* __restrict__ cx, const T* __restrict__ V,
                         const T* __restrict__ cm1, const T* __restrict__ cm2, const int32_t* __restrict__ cmarg,
                         const T* __restrict__ xrow_dense, T* __restrict__ vI, int* __restrict__ chg_ulf,
                         T* __restrict__ s_out, const T* __restrict__ rm1, const T* __restrict__ rm2,
                         const int32_t* __restrict__ rmarg, T* __restrict__ uI, int* __restrict__ hk_out,
                         const DevCtl* __restrict__ g = nullptr, u64* bst = nullptr,
                         const SeedCols<T>* __restrict__ sc = nullptr) {
  unsigned nb_total = gridDim.x;
  int* chg_urf = nullptr;
  if (g) {  // graph mode: batch window from the control block, grid-stride over virtual blocks
    E = g->E;
    i = g->i;
    cj += g->t0;
    ck += g->t0;
    cx += g->t0;
    chg_ulf = reinterpret_cast<int*>(bst + 2 + 4 * (int64_t)E);
    chg_urf = chg_ulf + E;
    int64_t G8 = (int64_t)((E + kEG - 1) / kEG) * kEG;
    nb_ulf = (unsigned)((G8 * n + 255) / 256);
    nb_total = nb_ulf + (unsigned)((G8 * m + 255) / 256);
  }
  int G = (E + kEG - 1) / kEG;
  for (unsigned vb = blockIdx.x; vb < nb_total; vb += gridDim.x) {
    if (vb < nb_ulf) {
      int64_t t = vb * (int64_t)blockDim.x + threadIdx.x;
      if (vb == 0 && hk_out)
        for (int q = threadIdx.x; q < E; q += blockDim.x) hk_out[q] = ck[q];
      if (t >= (int64_t)G * kEG * n) continue;
      int q;
      int64_t c;
      ilv_decode<T>(t, n, q, c);
      if (q >= E) { vI[t] = tinf<T>(); continue; }
      int k = ck[q];
      int64_t kn = (int64_t)k * n;
      T s = sub_rn(cx[q], V[kn + cj[q]]);
      T cmx = (cmarg[kn + c] == (int32_t)i) ? cm2[kn + c] : cm1[kn + c];
      T v = vmin(cmx, sub_rn(xrow_dense[c], s));
      vI[t] = v;
      if (c == 0) s_out[q] = s;
      if (v != V[kn + c]) chg_ulf[q] = 1;
    } else {
      int64_t t = (vb - nb_ulf) * (int64_t)blockDim.x + threadIdx.x;
      if (t >= (int64_t)G * kEG * m) continue;
      int q;
      int64_t r;
      ilv_decode<T>(t, m, q, r);
      if (q >= E) { uI[t] = tinf<T>(); continue; }
      int64_t km = (int64_t)ck[q] * m;
      int j = cj[q];
      T u = (rmarg[km + r] == j) ? rm2[km + r] : rm1[km + r];
      if (sc) {
        // the F-URF seed (k_phaseA_urf_seed_chk) fused: X_rj from a binary search of
        // row r in column j, then the change flag against the current U.k
        if (!chg_urf) chg_urf = chg_ulf + E;  // batch layout: chg = [F-ULF E][F-URF E]
        int lo = (int)sc->col_ptr[j], hi = (int)sc->col_ptr[j + 1];
        while (lo < hi) {
          int mid = (lo + hi) >> 1;
          if (sc->row_idx[mid] < (int32_t)r) lo = mid + 1;
          else hi = mid;
        }
        if (lo < (int)sc->col_ptr[j + 1] && sc->row_idx[lo] == (int32_t)r)
          u = vmin(u, sub_rn(sc->xc[lo], sub_rn(cx[q], sc->Ut[km + i])));
        if (u != sc->Ut[km + r]) chg_urf[q] = 1;
      }
      uI[t] = u;
    }
  }
}

// F-URF seed column j of eval q = blockIdx.x (rows of column j), then the change
// flag of the eval's whole first-residuation vector against the current U.k
template <typename T>
__global__ void k_phaseA_urf_seed_chk(int64_t m, int E, int64_t i, const int32_t* __restrict__ cj,
                                      const int32_t* __restrict__ ck, const T* __restrict__ cx,
                                      const T* __restrict__ Ut, const int64_t* __restrict__ col_ptr,
                                      const int32_t* __restrict__ row_idx, const T* __restrict__ xc,
                                      T* __restrict__ uI, int* __restrict__ chg_urf,
                                      const DevCtl* __restrict__ g = nullptr, u64* bst = nullptr) {
  if (g) {
    E = g->E;
    i = g->i;
    cj += g->t0;
    ck += g->t0;
    cx += g->t0;
    chg_urf = reinterpret_cast<int*>(bst + 2 + 4 * (int64_t)E) + E;
  }
  int q = blockIdx.x;
  if (q >= E) return;
  int j = cj[q];
  int64_t km = (int64_t)ck[q] * m;
  T s = sub_rn(cx[q], Ut[km + i]);
  T* u = uI + ilv_index<T>(q, 0, m);
  constexpr int EGP = Ilv<T>::STRIDE;
  for (int64_t p = col_ptr[j] + threadIdx.x; p < col_ptr[j + 1]; p += blockDim.x) {
    int64_t r = row_idx[p] * EGP;
    u[r] = vmin(u[r], sub_rn(xc[p], s));
  }
  __syncthreads();
  int ch = 0;
  for (int64_t r = threadIdx.x; r < m; r += blockDim.x) ch |= u[r * EGP] != Ut[km + r];
  if (__syncthreads_or(ch) && threadIdx.x == 0) chg_urf[q] = 1;
}

template <typename T>
__global__ void k_phaseA_urf_seed(int64_t m, int E, int64_t i, const int32_t* __restrict__ cj,
                                  const int32_t* __restrict__ ck, const T* __restrict__ cx,
                                  const T* __restrict__ Ut, const int64_t* __restrict__ col_ptr,
                                  const int32_t* __restrict__ row_idx, const T* __restrict__ xc,
                                  T* __restrict__ uI) {
  int q = blockIdx.x;
  if (q >= E) return;
  int j = cj[q];
  int64_t km = (int64_t)ck[q] * m;
  T s = sub_rn(cx[q], Ut[km + i]);
  T* u = uI + ilv_index<T>(q, 0, m);
  for (int64_t p = col_ptr[j] + threadIdx.x; p < col_ptr[j + 1]; p += blockDim.x) {
    int64_t r = row_idx[p] * Ilv<T>::STRIDE;
    u[r] = vmin(u[r], sub_rn(xc[p], s));
  }
}

// change flag of an interleaved vector against the current factor row
template <typename T>
__global__ void k_chk_ilv(int64_t len, int E, const int32_t* __restrict__ ck, const T* __restrict__ I,
                          const T* __restrict__ cur, int* __restrict__ chg) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int G = (E + kEG - 1) / kEG;
  if (t >= (int64_t)G * kEG * len) return;
  int q;
  int64_t a;
  ilv_decode<T>(t, len, q, a);
  if (q < E && I[t] != cur[(int64_t)ck[q] * len + a]) chg[q] = 1;
}

// eval q of an interleaved buffer -> contiguous vector
template <typename T>
__global__ void k_deinterleave(int64_t len, int q, const T* __restrict__ I, T* __restrict__ out) {
  int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (a < len) out[a] = I[ilv_index<T>(q, a, len)];
}

// ----------------------------------------------------------------------------
// Phase B — the hot kernel.  Work item = (line L, group of kEG evals).  For each
// eval q: line value w_q = min_p (x_p - vin_q[idx_p])  (the second residuation:
// rc for F-ULF on CSR rows, rr for F-URF on CSC columns), then the eval's error
// over the line: sum_p |x_p - max(Q^k_p, w_q + vin_q[idx_p])| with
// Q^k_p = (ag_p == k) ? t2_p : t1_p  (U(x)V with column/row k replaced).
// The line partial (fp64) goes to a 128-bit fixed-point accumulator per eval.
template <typename T>
struct SideB {
  int64_t nlines;
  const int64_t* ptr;
  const int32_t* idx;
  const T* xv;
  const T* t1;
  const T* t2;
  const uint8_t* ag;
  const T* vin;      // eval-interleaved [g][len_other][kEG]: first-residuation vectors
  int64_t len_other;
  const T* cur;      // rank x nlines: current factor row for this side
  T* out;            // E x nlines: second residuation
  u64* acc;          // 2 per eval
  int* chg;          // 1 per eval
  int mode;          // 0: min + error; 1: min only (local partial); 2: error with line values from out
  int64_t long_thr;  // lines with more entries are processed block-per-line (k_phaseB_long)
  int group_major;   // item order: 1 = eval-group major (entry data L2-resident: vin block
                     // stays hot in L1), 0 = line major (entry data streamed once per batch)
  // F-ULF side only (else null): per-k base CM^(-i) (rank x len_other), the dense
  // seed row X_i. (len_other) and s_q per eval, to recompute vin inline
  const T* inl_base = nullptr;
  const T* inl_xr = nullptr;
  const T* inl_s = nullptr;
  // F-ULF hit partition of the visited row (k_hit_partition): xv/idx/t1/t2/ag then
  // hold each line's entries reordered [columns not given in row i | the others], and
  // split[L] is the boundary (null: no partition)
  const int32_t* split = nullptr;
};

// Per row visit: reorder each CSR row's entries into [columns not given in row i |
// columns given in row i] (order inside the segments is irrelevant: minima are exact
// and the error partials' bound holds for any summation order), with the product
// caches, so phase B's F-ULF evals share one value on the first segment.
template <typename T>
__global__ void k_hit_partition(int64_t m, const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx,
                                const T* __restrict__ xr, const T* __restrict__ t1, const T* __restrict__ t2,
                                const uint8_t* __restrict__ ag, const T* __restrict__ xrow_dense,
                                int32_t* __restrict__ pidx, T* __restrict__ px, T* __restrict__ pt1,
                                T* __restrict__ pt2, uint8_t* __restrict__ pag, int32_t* __restrict__ split) {
  int lane = threadIdx.x & 31;
  int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned lt = (1u << lane) - 1;
  for (int64_t a = w; a < m; a += nw) {
    int beg = (int)row_ptr[a], end = (int)row_ptr[a + 1];
    int lo = beg, hi = end;
    for (int p0 = beg; p0 < end; p0 += 32) {
      int p = p0 + lane;
      bool ok = p < end;
      int c = ok ? col_idx[p] : 0;
      bool hit = ok && xrow_dense[c] != tinf<T>();
      unsigned bh = __ballot_sync(0xffffffffu, hit), bn = __ballot_sync(0xffffffffu, ok && !hit);
      if (ok) {
        int d = hit ? hi - 1 - __popc(bh & lt) : lo + __popc(bn & lt);
        pidx[d] = c;
        px[d] = xr[p];
        pt1[d] = t1[p];
        pt2[d] = t2[p];
        pag[d] = ag[p];
      }
      lo += __popc(bn);
      hi -= __popc(bh);
    }
    if (lane == 0) split[a] = lo;
  }
}

template <int EG, typename V>
__device__ __forceinline__ V lane_pick(const V (&a)[EG], int q) {
  V v = a[0];
#pragma unroll
  for (int i = 1; i < EG; i++)
    if (q == i) v = a[i];
  return v;
}

// the rows of one eval group in the phase-A buffer
template <typename T>
struct GroupRows {
  const T* vin;
  int g;
  int64_t len;
};

// the kEG first-residuation values of entry column c for the evals of a group:
// VM 0/1 read the planar phase-A buffer (plane pointers pl[]); VM 2 (F-ULF, one k
// for the group) recomputes them from the shared per-k base and the dense seed row,
// exactly as phase A does: v'_q,c = min(CM^(-i)_kc, X_ic - s_q)
template <typename T, int VM>
__device__ __forceinline__ void eval_vals(const T* __restrict__ xr_row, const T* __restrict__ base,
                                          const GroupRows<T>& pl, const T (&s)[kEG],
                                          int c, T (&v)[kEG]) {
  if (VM == 2) {
    T b = base[c], xr = xr_row[c];
#pragma unroll
    for (int q = 0; q < kEG; q++) v[q] = vmin(b, sub_rn(xr, s[q]));
  } else {
    load_group_row<T>(pl.vin, pl.g, pl.len, c, v);
  }
}

// min / sum of kEG per-lane values over the warp with a transposed butterfly:
// 4 + 2 + 1 exchanges halve the values per lane, then 2 plain steps.  Lane l ends
// with the reduction of eval (l >> 2) & 7.
template <typename V, bool SUM>
__device__ __forceinline__ V warp_reduce8(const V (&v)[kEG], int lane) {
  static_assert(kEG == 8, "transposed reduction of 8 evals");
  auto op = [](V a, V b) -> V {
    if constexpr (SUM) return __dadd_rn(a, b);
    else return vmin(a, b);
  };
  bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
  V t4[4], t2[2];
#pragma unroll
  for (int j = 0; j < 4; j++) {
    V send = b4 ? v[j] : v[j + 4], keep = b4 ? v[j + 4] : v[j];
    t4[j] = op(keep, shfl_xor(send, 16));
  }
#pragma unroll
  for (int j = 0; j < 2; j++) {
    V send = b3 ? t4[j] : t4[j + 2], keep = b3 ? t4[j + 2] : t4[j];
    t2[j] = op(keep, shfl_xor(send, 8));
  }
  V r = op(b2 ? t2[1] : t2[0], shfl_xor(b2 ? t2[0] : t2[1], 4));
  r = op(r, shfl_xor(r, 2));
  return op(r, shfl_xor(r, 1));
}

// Pass 1 over entries [lo, hi) of a line: per-eval line minima of x - v'.  SHARED
// (F-ULF entries whose column is not given in row i, VM 2 only): v' is the group's
// base value for every eval, so one minimum mn0 serves all 8 evals.
template <typename T, int VM, bool SHARED>
__device__ __forceinline__ void pass1_seg(const SideB<T>& S, const GroupRows<T>& pl,
                                          const T* __restrict__ base, const T (&s)[kEG], int lo, int hi, int lane,
                                          T (&mn)[kEG], T& mn0) {
  constexpr int EG = kEG;
  // U entries per lane per iteration: their idx -> vin gathers are in flight
  // together (the loop is latency-bound otherwise); missing slots use x = +inf
  constexpr int U = sizeof(T) == 8 ? 2 : 4;
  const T* __restrict__ xv = S.xv;
  const int32_t* __restrict__ idx = S.idx;
  for (int p0 = lo + lane; p0 < hi; p0 += 32 * U) {
    T x[U];
    int c[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      int p = p0 + 32 * u;
      bool ok = p < hi;
      x[u] = ok ? xv[p] : tinf<T>();
      c[u] = ok ? idx[p] : 0;
      STMF_IDX(c[u], S.len_other);
    }
    if (SHARED) {
#pragma unroll
      for (int u = 0; u < U; u++) mn0 = vmin(mn0, sub_rn(x[u], base[c[u]]));
    } else {
      T v[U][EG];
#pragma unroll
      for (int u = 0; u < U; u++) eval_vals<T, VM>(S.inl_xr, base, pl, s, c[u], v[u]);
#pragma unroll
      for (int u = 0; u < U; u++)
#pragma unroll
        for (int q = 0; q < EG; q++) mn[q] = vmin(mn[q], sub_rn(x[u], v[u][q]));
    }
  }
}

// Pass 2 over entries [lo, hi): per-eval error partials with the new line values mn.
// |x - max(Q, w)| == |min(x - Q, x - w)| exactly (x - . is monotone under rounding).
template <typename T, int UNR, int VM, bool SHARED>
__device__ __forceinline__ void pass2_seg(const SideB<T>& S, const GroupRows<T>& pl,
                                          const T* __restrict__ base, const T (&s)[kEG], int k0, unsigned klo,
                                          unsigned khi, int lo, int hi, int lane, const T (&mn)[kEG],
                                          double (&part)[kEG]) {
  constexpr int EG = kEG, U2 = UNR;
  const T* __restrict__ xv = S.xv;
  const int32_t* __restrict__ idx = S.idx;
  for (int p0 = lo + lane; p0 < hi; p0 += 32 * U2) {
    T x[U2], a1[U2], a2[U2];
    int a[U2], c[U2];
#pragma unroll
    for (int u = 0; u < U2; u++) {
      int p = p0 + 32 * u;
      bool ok = p < hi;
      int pp = ok ? p : lo;
      x[u] = xv[pp];
      c[u] = idx[pp];
      STMF_IDX(c[u], S.len_other);
      a1[u] = S.t1[pp];
      a2[u] = S.t2[pp];
      a[u] = ok ? (int)S.ag[pp] : -1;  // -1: slot beyond the segment (contributes 0)
    }
    T v[U2][EG];
    if (SHARED) {
#pragma unroll
      for (int u = 0; u < U2; u++) {
        T b = base[c[u]];
#pragma unroll
        for (int q = 0; q < EG; q++) v[u][q] = b;
      }
    } else {
#pragma unroll
      for (int u = 0; u < U2; u++) eval_vals<T, VM>(S.inl_xr, base, pl, s, c[u], v[u]);
    }
#pragma unroll
    for (int u = 0; u < U2; u++) {
      if (a[u] < 0) continue;
      if (VM >= 1) {
        T r1 = sub_rn(x[u], (a[u] == k0) ? a2[u] : a1[u]);
#pragma unroll
        for (int q = 0; q < EG; q++)
          part[q] = __dadd_rn(part[q], (double)vabs(vmin(r1, sub_rn(x[u], add_rn(mn[q], v[u][q])))));
      } else {
        // per-eval k: the 8 factor indices live as bytes of klo / khi (8 registers of indices
        // spilled in this loop); a byte of the xor is zero where the entry's argmax is eval q's k
        const unsigned ar = (unsigned)a[u] * 0x01010101u;
        const unsigned xl = klo ^ ar, xh = khi ^ ar;
#pragma unroll
        for (int q = 0; q < EG; q++) {
          const bool eq = (((q < 4) ? xl : xh) & (0xffu << (8 * (q & 3)))) == 0u;
          T Q = eq ? a2[u] : a1[u];
          T pm = vmax(Q, add_rn(mn[q], v[u][q]));
          part[q] = __dadd_rn(part[q], (double)vabs(sub_rn(x[u], pm)));
        }
      }
    }
  }
}

// the second residuation of a line for the kEG evals of a group: per-eval minima of
// x - v' over the line's entries (pass 1), reduced over the warp; every lane ends with
// all kEG values
template <typename T, int VM>
__device__ __forceinline__ void line_min8(const SideB<T>& S, const GroupRows<T>& pl,
                                          const T* __restrict__ base, const T (&s)[kEG], int beg, int sp, int end,
                                          int lane, T (&mn)[kEG]) {
#pragma unroll
  for (int q = 0; q < kEG; q++) mn[q] = tinf<T>();
  T mn0 = tinf<T>();
  if (VM == 2 && sp > beg) pass1_seg<T, VM, true>(S, pl, base, s, beg, sp, lane, mn, mn0);
  pass1_seg<T, VM, false>(S, pl, base, s, sp, end, lane, mn, mn0);
#pragma unroll
  for (int q = 0; q < kEG; q++) mn[q] = vmin(mn[q], mn0);
  T r = warp_reduce8<T, false>(mn, lane);
#pragma unroll
  for (int q = 0; q < kEG; q++) mn[q] = __shfl_sync(0xffffffffu, r, q << 2);
}

// VM: 0 = planar, per-eval k; 1 = planar, one k for the group (Q shared per
// entry); 2 = one k, F-ULF values recomputed inline (no per-eval gathers), and with
// a hit partition (S.split) the entries whose column is not given in row i share
// one value for all evals.  Entry offsets are 32-bit (N < 2^31 per device).
template <typename T, int UNR, int VM>
__device__ __forceinline__ void phaseB_body(const SideB<T>& S, int64_t L, int g, int e0, int ne,
                                            const int (&kq)[kEG], int lane, int* __restrict__ flags, int F,
                                            double exact_limit) {
  constexpr int EG = kEG;
  int64_t nlines = S.nlines;
  const GroupRows<T> pl{S.vin, g, S.len_other};
  T s[EG];
  const T* base = nullptr;
  if (VM == 2) {
    base = S.inl_base + (int64_t)kq[0] * S.len_other;
#pragma unroll
    for (int q = 0; q < EG; q++) s[q] = S.inl_s[e0 + (q < ne ? q : ne - 1)];
  }
  const int beg = (int)S.ptr[L], end = (int)S.ptr[L + 1];
  const int sp = (VM == 2 && S.split) ? S.split[L] : beg;  // [beg, sp): shared values
  // factor indices (< 256) packed as bytes: all the loops below need of kq
  const int k0 = kq[0];
  unsigned klo = 0, khi = 0;
#pragma unroll
  for (int q = 0; q < 4; q++) {
    klo |= (unsigned)kq[q] << (8 * q);
    khi |= (unsigned)kq[q + 4] << (8 * q);
  }
  // opaque from here on: otherwise the partial ors stay live next to the packed words
  asm volatile("" : "+r"(klo), "+r"(khi));
  T mn[EG];
  if (S.mode == 2) {
    // line values computed before this pass: the sharded F-URF all-reduced minima, or
    // the statistics walk of k_pass1_fast
#pragma unroll
    for (int q = 0; q < EG; q++) mn[q] = S.out[(int64_t)(e0 + (q < ne ? q : ne - 1)) * nlines + L];
  } else {
    line_min8<T, VM>(S, pl, base, s, beg, sp, end, lane, mn);
  }
  if (lane < ne) {
    T w = lane_pick<EG>(mn, lane);
    int kl = VM == 0 ? (int)(((lane < 4 ? klo : khi) >> (8 * (lane & 3))) & 0xffu) : k0;
    if (S.mode != 2) S.out[(int64_t)(e0 + lane) * nlines + L] = w;
    if (S.mode != 1 && w != S.cur[(int64_t)kl * nlines + L]) S.chg[e0 + lane] = 1;
  }
  if (S.mode == 1) return;  // sharded F-URF first half: local minima only
  double part[EG];
#pragma unroll
  for (int q = 0; q < EG; q++) part[q] = 0.0;
  if (VM == 2 && sp > beg) pass2_seg<T, UNR, VM, true>(S, pl, base, s, k0, klo, khi, beg, sp, lane, mn, part);
  pass2_seg<T, UNR, VM, false>(S, pl, base, s, k0, klo, khi, sp, end, lane, mn, part);
  double pv = warp_reduce8<double, true>(part, lane);
  int q = (lane >> 2) & 7;
  if ((lane & 3) == 0 && q < ne) {
    int fl = 0;
    if (!(pv < exact_limit)) fl |= 4;
    u64 hi, lo;
    fx_from_double(pv, F, hi, lo, fl);
    fx_atomic_add(S.acc + 2 * (e0 + q), hi, lo);
    if (fl & 6) atomicOr(flags, fl);
  }
}

template <typename T, int UNR>
__device__ __forceinline__ void phaseB_item(const SideB<T>& S, int64_t it, int E, const int32_t* __restrict__ ek,
                                            int lane, int* __restrict__ flags, int F, double exact_limit) {
  constexpr int EG = kEG;
  int64_t nlines = S.nlines;
  int ngroups = (E + EG - 1) / EG;
  // line-major: the warps of one line (one per eval group) run together, so the
  // line's entries are read from DRAM once per batch; the small vin blocks stay in L2.
  // group-major: concurrent warps share one group's vin block (L1-resident).
  int64_t L;
  int g;
  if (S.group_major) {
    g = (int)(it / nlines);
    L = it - (int64_t)g * nlines;
  } else {
    L = it / ngroups;
    g = (int)(it - L * ngroups);
  }
  int e0 = g * EG;
  int ne = E - e0 < EG ? E - e0 : EG;
  if (S.ptr[L + 1] - S.ptr[L] > S.long_thr) return;  // a long line: k_phaseB_long
  int kq[EG];
  bool unif = true;
#pragma unroll
  for (int q = 0; q < EG; q++) {
    kq[q] = ek[e0 + (q < ne ? q : ne - 1)];
    unif &= kq[q] == kq[0];
  }
  if (!unif) phaseB_body<T, UNR, 0>(S, L, g, e0, ne, kq, lane, flags, F, exact_limit);
  else if (S.inl_base) phaseB_body<T, UNR, 2>(S, L, g, e0, ne, kq, lane, flags, F, exact_limit);
  else phaseB_body<T, UNR, 1>(S, L, g, e0, ne, kq, lane, flags, F, exact_limit);
}

#ifndef STMF_PHASEB_CTAS_F32
#define STMF_PHASEB_CTAS_F32 4
#endif
constexpr int kPhaseBCtasF32 = STMF_PHASEB_CTAS_F32;  // resident phase-B CTAs per SM (binary32)
#ifndef STMF_PHASEB_CTAS_F64
#define STMF_PHASEB_CTAS_F64 3
#endif
constexpr int kPhaseBCtasF64 = STMF_PHASEB_CTAS_F64;  // (binary64, one entry per lane per iteration)

// graph mode: the batch window and the result slots of bstate
// ([flags: 4 int][acc: 4E u64][chg: 2E int]) from the control block
template <typename T>
__device__ __forceinline__ void batch_from_ctl(const DevCtl* g, u64* bst, SideB<T>& A, SideB<T>& B, int& E) {
  E = g->E;
  A.acc = bst + 2;
  B.acc = bst + 2 + 2 * (int64_t)E;
  A.chg = reinterpret_cast<int*>(bst + 2 + 4 * (int64_t)E);
  B.chg = A.chg + E;
}

// Phase B of both update rules in one launch: items [0, A) are F-ULF evals on CSR
// rows (rc + error), items [A, A+B) F-URF evals on CSC columns (rr + error).
// UNR = entries per lane per loop iteration (memory-level parallelism vs registers)
template <typename T, int UNR>
__global__ void __launch_bounds__(256, UNR > 2 ? 2 : (sizeof(T) == 8 && UNR > 1 ? 2 : (sizeof(T) == 4 ? kPhaseBCtasF32 : kPhaseBCtasF64)))
k_phaseB(SideB<T> A, SideB<T> B, int E, const int32_t* __restrict__ ek, int* __restrict__ flags, int F,
         double exact_limit, const DevCtl* __restrict__ g = nullptr, u64* bst = nullptr,
         const int32_t* __restrict__ ck = nullptr) {
  if (g) {
    batch_from_ctl(g, bst, A, B, E);
    ek = ck + g->t0;
  }
  int lane = threadIdx.x & 31;
  int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int ngroups = (E + kEG - 1) / kEG;
  int64_t itemsA = A.nlines * ngroups, items = itemsA + B.nlines * ngroups;
  for (int64_t it = w; it < items; it += nw) {
    if (it < itemsA) phaseB_item<T, UNR>(A, it, E, ek, lane, flags, F, exact_limit);
    else phaseB_item<T, UNR>(B, it - itemsA, E, ek, lane, flags, F, exact_limit);
  }
}

// Long lines (more than long_thr entries: e.g. the densest rows of config 4's
// row-clustered mask) with a whole block per (line, eval group): 8 warps stride the
// line, the minima and error partials are combined through shared memory in a
// fixed order.  Same arithmetic per entry as phaseB_item.
template <typename T>
__global__ void __launch_bounds__(256)
k_phaseB_long(SideB<T> A, SideB<T> B, int E, const int32_t* __restrict__ ek, const int32_t* __restrict__ longA,
              int nA, const int32_t* __restrict__ longB, int nB, int* __restrict__ flags, int F, double exact_limit,
              const DevCtl* __restrict__ g = nullptr, u64* bst = nullptr, const int32_t* __restrict__ ck = nullptr) {
  if (g) {
    batch_from_ctl(g, bst, A, B, E);
    ek = ck + g->t0;
  }
  constexpr int EG = kEG;
  __shared__ T smn[8][EG];
  __shared__ double spart[8][EG];
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int ngroups = (E + EG - 1) / EG;
  int64_t items = (int64_t)(nA + nB) * ngroups;
  for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
    int64_t li = it / ngroups;
    int g = (int)(it - li * ngroups);
    const SideB<T>& S = li < nA ? A : B;
    int64_t L = li < nA ? longA[li] : longB[li - nA];
    int64_t nlines = S.nlines;
    int e0 = g * EG;
    int ne = E - e0 < EG ? E - e0 : EG;
    int kq[EG];
#pragma unroll
    for (int q = 0; q < EG; q++) kq[q] = ek[e0 + (q < ne ? q : ne - 1)];
    int64_t beg = S.ptr[L], end = S.ptr[L + 1];
    T mn[EG];
    if (S.mode == 2) {
#pragma unroll
      for (int q = 0; q < EG; q++) mn[q] = S.out[(int64_t)(e0 + (q < ne ? q : ne - 1)) * nlines + L];
    } else {
#pragma unroll
      for (int q = 0; q < EG; q++) mn[q] = tinf<T>();
      for (int64_t p = beg + threadIdx.x; p < end; p += 256) {
        T x = S.xv[p];
        T v[EG];
        load_group_row<T>(S.vin, g, S.len_other, (int64_t)S.idx[p], v);
#pragma unroll
        for (int q = 0; q < EG; q++) mn[q] = vmin(mn[q], sub_rn(x, v[q]));
      }
#pragma unroll
      for (int q = 0; q < EG; q++) {
        for (int o = 16; o; o >>= 1) mn[q] = vmin(mn[q], shfl_xor(mn[q], o));
        if (lane == 0) smn[wid][q] = mn[q];
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < EG; q++) {
        T v = smn[0][q];
        for (int w = 1; w < 8; w++) v = vmin(v, smn[w][q]);
        mn[q] = v;
      }
      __syncthreads();
    }
    if (threadIdx.x < ne) {
      int q = threadIdx.x;
      T w = lane_pick<EG>(mn, q);
      int kl = lane_pick<EG>(kq, q);
      if (S.mode != 2) S.out[(int64_t)(e0 + q) * nlines + L] = w;
      if (S.mode != 1 && w != S.cur[(int64_t)kl * nlines + L]) S.chg[e0 + q] = 1;
    }
    if (S.mode == 1) continue;
    double part[EG];
#pragma unroll
    for (int q = 0; q < EG; q++) part[q] = 0.0;
    for (int64_t p = beg + threadIdx.x; p < end; p += 256) {
      T x = S.xv[p];
      T a1 = S.t1[p], a2 = S.t2[p];
      int a = S.ag[p];
      T v[EG];
      load_group_row<T>(S.vin, g, S.len_other, (int64_t)S.idx[p], v);
#pragma unroll
      for (int q = 0; q < EG; q++) {
        T Q = (a == kq[q]) ? a2 : a1;
        T pm = vmax(Q, add_rn(mn[q], v[q]));
        part[q] = __dadd_rn(part[q], (double)vabs(sub_rn(x, pm)));
      }
    }
#pragma unroll
    for (int q = 0; q < EG; q++) {
      for (int o = 16; o; o >>= 1) part[q] = __dadd_rn(part[q], shfl_xor(part[q], o));
      if (lane == 0) spart[wid][q] = part[q];
    }
    __syncthreads();
    if (threadIdx.x < ne) {
      int q = threadIdx.x;
      double pv = spart[0][q];
      for (int w = 1; w < 8; w++) pv = __dadd_rn(pv, spart[w][q]);
      int fl = 0;
      if (!(pv < exact_limit)) fl |= 4;
      u64 hi, lo;
      fx_from_double(pv, F, hi, lo, fl);
      fx_atomic_add(S.acc + 2 * (e0 + q), hi, lo);
      if (fl & 6) atomicOr(flags, fl);
    }
    __syncthreads();
  }
}

// lines longer than the sides' long_thr are listed in longA / longB and handled by
// k_phaseB_long (a block per line) — call sites set long_thr consistently
template <typename T>
inline void launch_phaseB(int unroll, unsigned grid, cudaStream_t st, const SideB<T>& A, const SideB<T>& B, int E,
                          const int32_t* ek, int* flags, int F, double exact_limit, const int32_t* longA = nullptr,
                          int nA = 0, const int32_t* longB = nullptr, int nB = 0, int nsm = 148) {
  if (unroll >= 4) k_phaseB<T, 4><<<grid, 256, 0, st>>>(A, B, E, ek, flags, F, exact_limit);
  else if (unroll == 2) k_phaseB<T, 2><<<grid, 256, 0, st>>>(A, B, E, ek, flags, F, exact_limit);
  else k_phaseB<T, 1><<<grid, 256, 0, st>>>(A, B, E, ek, flags, F, exact_limit);
  if (nA + nB > 0) {
    int64_t items = (int64_t)(nA + nB) * ((E + kEG - 1) / kEG);
    unsigned g = (unsigned)std::min<int64_t>(items, (int64_t)nsm * 8);
    k_phaseB_long<T><<<g, 256, 0, st>>>(A, B, E, ek, longA, nA, longB, nB, flags, F, exact_limit);
  }
}

// Exact/bounded objective of an explicit state: entries' residual |x - max(Q^k, a_r + b_c)|
// over CSR rows.  With a = Ut row k and b = V row k this is the current state.
template <typename T>
__global__ void k_objective(int64_t m, const int64_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                            const T* __restrict__ xv, const T* __restrict__ t1, const T* __restrict__ t2,
                            const uint8_t* __restrict__ ag, int k, const T* __restrict__ a, const T* __restrict__ b,
                            u64* __restrict__ acc, int* __restrict__ flags, int F, double exact_limit) {
  int lane = threadIdx.x & 31;
  int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = w; r < m; r += nw) {
    double part = 0.0;
    T ar = a[r];
    for (int64_t p = ptr[r] + lane; p < ptr[r + 1]; p += 32) {
      T Q = (ag[p] == k) ? t2[p] : t1[p];
      T pm = vmax(Q, add_rn(ar, b[idx[p]]));
      part = __dadd_rn(part, (double)vabs(sub_rn(xv[p], pm)));
    }
    for (int o = 16; o; o >>= 1) part = __dadd_rn(part, shfl_xor(part, o));
    if (lane == 0) {
      int fl = 0;
      if (!(part < exact_limit)) fl |= 4;
      u64 hi, lo;
      fx_from_double(part, F, hi, lo, fl);
      fx_atomic_add(acc, hi, lo);
      if (fl) atomicOr(flags, fl);
    }
  }
}

// numpy replica, step 1: the residual multiset of an explicit state (fp64 bit patterns).
template <typename T>
__global__ void k_residuals(int64_t m, const int64_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                            const T* __restrict__ xv, const T* __restrict__ t1, const T* __restrict__ t2,
                            const uint8_t* __restrict__ ag, int k, const T* __restrict__ a, int as,
                            const T* __restrict__ b, int bs, u64* __restrict__ out) {
  int lane = threadIdx.x & 31;
  int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = w; r < m; r += nw) {
    T ar = a[r * as];
    for (int64_t p = ptr[r] + lane; p < ptr[r + 1]; p += 32) {
      T Q = (ag[p] == k) ? t2[p] : t1[p];
      T pm = vmax(Q, add_rn(ar, b[(int64_t)idx[p] * bs]));
      out[p] = (u64)__double_as_longlong((double)vabs(sub_rn(xv[p], pm)));
    }
  }
}

// numpy replica, step 3: pairwise-sum leaves (n <= 128) of the sorted residuals,
// exactly numpy's DOUBLE_pairwise_sum leaf (8 strided accumulators + tail).
__global__ void k_pw_leaves(int nleaves, const int64_t* __restrict__ loff, const int32_t* __restrict__ llen,
                            const int32_t* __restrict__ lnode, const u64* __restrict__ sorted,
                            double* __restrict__ val) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nleaves) return;
  const double* a = reinterpret_cast<const double*>(sorted) + loff[t];
  int n = llen[t];
  double res;
  if (n < 8) {
    res = 0.0;
    for (int i = 0; i < n; i++) res = __dadd_rn(res, a[i]);
  } else {
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; j++) r[j] = a[j];
    int i;
    for (i = 8; i < n - (n % 8); i += 8)
#pragma unroll
      for (int j = 0; j < 8; j++) r[j] = __dadd_rn(r[j], a[i + j]);
    res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                    __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; i++) res = __dadd_rn(res, a[i]);
  }
  val[lnode[t]] = res;
}

// Same leaves, 8 lanes per leaf (4 leaves per warp): lane j of a group owns
// numpy's accumulator r[j] (elements j, j+8, ...), so every add happens in the
// same order as numpy's; the 3-level combine and the tail run on lane 0.
__global__ void k_pw_leaves8(int nleaves, const int64_t* __restrict__ loff, const int32_t* __restrict__ llen,
                             const int32_t* __restrict__ lnode, const u64* __restrict__ sorted,
                             double* __restrict__ val) {
  int lane = threadIdx.x & 31;
  int j = lane & 7;
  int t = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 3);
  bool ok = t < nleaves;
  const double* a = reinterpret_cast<const double*>(sorted) + (ok ? loff[t] : 0);
  int n = ok ? llen[t] : 0;
  double r = 0.0;
  int body = n - (n % 8);
  if (n >= 8) {
    r = a[j];
    for (int i = 8 + j; i < body; i += 8) r = __dadd_rn(r, a[i]);
  }
  // gather the 8 accumulators of this group into lane j == 0
  double r1 = __shfl_down_sync(0xffffffffu, r, 1);
  double r2 = __shfl_down_sync(0xffffffffu, r, 2);
  double r3 = __shfl_down_sync(0xffffffffu, r, 3);
  double r4 = __shfl_down_sync(0xffffffffu, r, 4);
  double r5 = __shfl_down_sync(0xffffffffu, r, 5);
  double r6 = __shfl_down_sync(0xffffffffu, r, 6);
  double r7 = __shfl_down_sync(0xffffffffu, r, 7);
  if (ok && j == 0) {
    double res;
    if (n < 8) {
      res = 0.0;
      for (int i = 0; i < n; i++) res = __dadd_rn(res, a[i]);
    } else {
      res = __dadd_rn(__dadd_rn(__dadd_rn(r, r1), __dadd_rn(r2, r3)), __dadd_rn(__dadd_rn(r4, r5), __dadd_rn(r6, r7)));
      for (int i = body; i < n; i++) res = __dadd_rn(res, a[i]);
    }
    val[lnode[t]] = res;
  }
}

// numpy replica, step 4: combine internal nodes level by level (heights 1..H).
__global__ void k_pw_combine(int H, const int32_t* __restrict__ lvl_off, const int32_t* __restrict__ nodes,
                             const int32_t* __restrict__ left, const int32_t* __restrict__ right,
                             double* __restrict__ val) {
  for (int h = 0; h < H; h++) {
    for (int t = lvl_off[h] + threadIdx.x; t < lvl_off[h + 1]; t += blockDim.x) {
      int nd = nodes[t];
      val[nd] = __dadd_rn(val[left[nd]], val[right[nd]]);
    }
    __syncthreads();
  }
}

}  // namespace stmf

namespace stmf {
// Dense max-plus product over all entries (prediction path): block = 32 x 8 outputs
// per pass; V tile of 32 columns x rank staged in shared memory, U row values are
// warp-uniform broadcasts.
template <typename T>
__global__ void k_maxplus_dense(int64_t m, int rank, int64_t n, const T* __restrict__ U, const T* __restrict__ V,
                                T* __restrict__ P, int32_t* __restrict__ arg) {
  int64_t j = blockIdx.x * 32 + threadIdx.x;
  int64_t i = blockIdx.y * 8 + threadIdx.y;
  if (i >= m || j >= n) return;
  const T* u = U + i * rank;
  T best = add_rn(u[0], V[j]);
  int a = 0;
  for (int k = 1; k < rank; k++) {
    T s = add_rn(u[k], V[(int64_t)k * n + j]);
    if (s > best) { best = s; a = k; }
  }
  if (P) P[i * n + j] = best;
  if (arg) arg[i * n + j] = a;
}
}  // namespace stmf

namespace stmf {
// numpy DOUBLE_pairwise_sum, single thread (recursive; depth ~ log2(n/128))
__device__ double np_pairwise_dev(const double* a, int64_t n) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; i++) res = __dadd_rn(res, a[i]);
    return res;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; j++) r[j] = a[j];
    int64_t i;
    for (i = 8; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; j++) r[j] = __dadd_rn(r[j], a[i + j]);
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; i++) res = __dadd_rn(res, a[i]);
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(np_pairwise_dev(a, n2), np_pairwise_dev(a + n2, n - n2));
}

// Column score of a single-column matrix (n == 1): numpy coalesces the unit axis
// and reduces the whole td_grid column (zeros at missing rows) pairwise.
template <typename T>
__global__ void k_colscore_single(int64_t m, const int64_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                                  const T* __restrict__ xc, const T* __restrict__ t1c, double* __restrict__ col,
                                  double* __restrict__ score) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  for (int64_t i = 0; i < m; i++) col[i] = 0.0;
  for (int64_t p = ptr[0]; p < ptr[1]; p++) col[idx[p]] = (double)vabs(sub_rn(xc[p], t1c[p]));
  score[0] = np_pairwise_dev(col, m);
}
}  // namespace stmf

namespace stmf {
// ----------------------------------------------------------------------------
// Incremental numpy replica.  The current state's residuals (per given entry, CSR
// order) and their ascending order S_cur are kept on the device.  A candidate's
// sorted residual multiset = S_cur minus the old values of its changed entries
// plus their new values; positions follow from binary searches (equal values are
// interchangeable in the sum, so any tie order gives numpy's result).

constexpr int kDeltaCap = 4096;

// new residual bits of every entry; changed entries appended to (olds, news)
template <typename T>
__global__ void k_residuals_delta(int64_t m, const int64_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                                  const T* __restrict__ xv, const T* __restrict__ t1, const T* __restrict__ t2,
                                  const uint8_t* __restrict__ ag, int k, const T* __restrict__ a,
                                  const T* __restrict__ b, const u64* __restrict__ res_cur, u64* __restrict__ out,
                                  u64* __restrict__ olds, u64* __restrict__ news, int* __restrict__ dcount) {
  int lane = threadIdx.x & 31;
  int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = w; r < m; r += nw) {
    T ar = a[r];
    int64_t beg = ptr[r], end = ptr[r + 1];
    for (int64_t base = beg; base < end; base += 32) {
      int64_t p = base + lane;
      bool ch = false;
      u64 nb = 0, ob = 0;
      if (p < end) {
        T Q = (ag[p] == k) ? t2[p] : t1[p];
        T pm = vmax(Q, add_rn(ar, b[idx[p]]));
        nb = (u64)__double_as_longlong((double)vabs(sub_rn(xv[p], pm)));
        ob = res_cur[p];
        out[p] = nb;
        ch = nb != ob;
      }
      unsigned bal = __ballot_sync(0xffffffffu, ch);
      if (bal) {
        int slot = 0;
        if (lane == 0) slot = atomicAdd(dcount, __popc(bal));
        slot = __shfl_sync(0xffffffffu, slot, 0) + __popc(bal & ((1u << lane) - 1));
        if (ch && slot < kDeltaCap) { olds[slot] = ob; news[slot] = nb; }
      }
    }
  }
}

// bitonic sort (ascending u64) of the first D <= kDeltaCap keys; block 0 sorts
// olds, block 1 news, in shared memory
__global__ void __launch_bounds__(1024) k_sort_delta(u64* __restrict__ olds, u64* __restrict__ news,
                                                     const int* __restrict__ dcount) {
  __shared__ u64 sh[kDeltaCap];
  u64* a = blockIdx.x == 0 ? olds : news;
  int D = *dcount;
  if (D > kDeltaCap) return;  // full-sort fallback on the host side
  int P = 1;
  while (P < D) P <<= 1;
  for (int i = threadIdx.x; i < P; i += blockDim.x) sh[i] = i < D ? a[i] : ~0ull;
  __syncthreads();
  for (int k = 2; k <= P; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < P; i += blockDim.x) {
        int l = i ^ j;
        if (l > i) {
          u64 x = sh[i], y = sh[l];
          bool up = (i & k) == 0;
          if ((x > y) == up) { sh[i] = y; sh[l] = x; }
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < D; i += blockDim.x) a[i] = sh[i];
}

__device__ __forceinline__ int64_t lower_bound_u64(const u64* __restrict__ a, int64_t n, u64 x) {
  int64_t lo = 0, hi = n;
  while (lo < hi) { int64_t mid = (lo + hi) >> 1; if (a[mid] < x) lo = mid + 1; else hi = mid; }
  return lo;
}
__device__ __forceinline__ int64_t upper_bound_u64(const u64* __restrict__ a, int64_t n, u64 x) {
  int64_t lo = 0, hi = n;
  while (lo < hi) { int64_t mid = (lo + hi) >> 1; if (a[mid] <= x) lo = mid + 1; else hi = mid; }
  return lo;
}

// S_new = (S_cur - olds) U news, K elements before equal news
__global__ void k_merge_delta(int64_t N, const u64* __restrict__ S_cur, const u64* __restrict__ olds,
                              const u64* __restrict__ news, const int* __restrict__ dcount, u64* __restrict__ out) {
  int D = *dcount;
  if (D > kDeltaCap) return;  // full-sort fallback on the host side
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < N) {
    u64 x = S_cur[t];
    int64_t le_old = upper_bound_u64(olds, D, x);
    int64_t lt_old = lower_bound_u64(olds, D, x);
    bool kept = true;
    if (le_old > lt_old) kept = (t - lower_bound_u64(S_cur, N, x)) >= le_old - lt_old;
    if (kept) out[t - le_old + lower_bound_u64(news, D, x)] = x;
  } else if (t < N + D) {
    int64_t q = t - N;
    u64 y = news[q];
    out[q + upper_bound_u64(S_cur, N, y) - upper_bound_u64(olds, D, y)] = y;
  }
}

// ---- the same replica steps for a round of slots in one launch each (slot = blockIdx.y)
// A slot's factor vectors are read with a stride: 1 for a contiguous vector, EGP for
// one eval of a planar interleaved phase-A buffer (no de-interleave copy needed).
template <typename T>
struct RepSlot {
  int k;
  int as, bs;        // element strides of a / b
  const T* a;
  const T* b;
  u64* res;
  u64* sorted;
  u64* olds;
  u64* news;
  int* dcount;
  double* pw;
  double* out;       // [0] the replica's value (root of the pairwise tree), [1] bits: D
};

// one replica round's slots, passed by value (no descriptor upload per round)
constexpr int kRepSlots = 8;
template <typename T>
struct RepRound {
  RepSlot<T> s[kRepSlots];
  int count;
};
// a kernel's slot: from the by-value round (host-driven) or, in graph mode, from
// the round the device-side decision wrote (Rp); blocks past the round's count exit
#define REP_SLOT(S)                                                   \
  if ((int)blockIdx.y >= (Rp ? Rp->count : R.count)) return;          \
  const RepSlot<T> S = Rp ? Rp->s[blockIdx.y] : R.s[blockIdx.y]

// the round's outputs: value and change count, then the count is reset for the next round
__device__ __forceinline__ void rep_finish(const double* root, int* dcount, double* out) {
  out[0] = *root;
  reinterpret_cast<long long*>(out)[1] = *dcount;
  *dcount = 0;
}

// entry-parallel over the CSR entries (rowof = row of each entry); changed entries
// are appended (warp ballot + one atomic) to the slot's (olds, news)
template <typename T>
__global__ void k_residuals_delta_multi(int64_t N, const int32_t* __restrict__ rowof, const int32_t* __restrict__ idx,
                                        const T* __restrict__ xv, const T* __restrict__ t1, const T* __restrict__ t2,
                                        const uint8_t* __restrict__ ag, const u64* __restrict__ res_cur,
                                        const RepRound<T> R, const RepRound<T>* __restrict__ Rp = nullptr) {
  REP_SLOT(S);
  int lane = threadIdx.x & 31;
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  bool ch = false;
  u64 nb = 0, ob = 0;
  if (p < N) {
    T Q = (ag[p] == S.k) ? t2[p] : t1[p];
    T pm = vmax(Q, add_rn(S.a[(int64_t)rowof[p] * S.as], S.b[(int64_t)idx[p] * S.bs]));
    nb = (u64)__double_as_longlong((double)vabs(sub_rn(xv[p], pm)));
    ob = res_cur[p];
    S.res[p] = nb;
    ch = nb != ob;
  }
  unsigned bal = __ballot_sync(0xffffffffu, ch);
  if (bal) {
    int slot = 0;
    if (lane == 0) slot = atomicAdd(S.dcount, __popc(bal));
    slot = __shfl_sync(0xffffffffu, slot, 0) + __popc(bal & ((1u << lane) - 1));
    if (ch && slot < kDeltaCap) { S.olds[slot] = ob; S.news[slot] = nb; }
  }
}

// ascending block merge sort of the D <= kDeltaCap changed values (block 0: olds,
// block 1: news); the tile size follows D (block-uniform branch)
constexpr int kSortThreads = 1024;
template <int ITEMS>
__device__ __forceinline__ void block_sort_u64(u64* a, int D, void* tmp_raw) {
  using Sort = cub::BlockMergeSort<u64, kSortThreads, ITEMS>;
  auto& tmp = *reinterpret_cast<typename Sort::TempStorage*>(tmp_raw);
  u64 key[ITEMS];
#pragma unroll
  for (int i = 0; i < ITEMS; i++) {
    int e = threadIdx.x * ITEMS + i;
    key[i] = e < D ? a[e] : ~0ull;
  }
  Sort(tmp).Sort(key, U64Less(), D, ~0ull);
#pragma unroll
  for (int i = 0; i < ITEMS; i++) {
    int e = threadIdx.x * ITEMS + i;
    if (e < D) a[e] = key[i];
  }
}
template <typename T>
__global__ void __launch_bounds__(kSortThreads) k_sort_delta_multi(const RepRound<T> R, const RepRound<T>* __restrict__ Rp = nullptr) {
  static_assert(kDeltaCap == 4 * kSortThreads, "two sort configurations");
  __shared__ union {
    typename cub::BlockMergeSort<u64, kSortThreads, 1>::TempStorage t1;
    typename cub::BlockMergeSort<u64, kSortThreads, 4>::TempStorage t4;
  } tmp;
  REP_SLOT(S);
  u64* a = blockIdx.x == 0 ? S.olds : S.news;
  int D = *S.dcount;
  if (D > kDeltaCap || D < 2) return;
  if (D <= kSortThreads) block_sort_u64<1>(a, D, &tmp);
  else block_sort_u64<4>(a, D, &tmp);
}

// warp-cooperative 32-ary searches over a sorted u64 array (all lanes return the
// result): first index with a[i] >= x (lower) or a[i] > x (upper)
template <bool UPPER>
__device__ __forceinline__ int64_t warp_bound_u64(const u64* __restrict__ a, int64_t n, u64 x, int lane) {
  int64_t lo = 0, hi = n;  // the answer lies in [lo, hi]
  while (hi - lo > 32) {
    int64_t step = (hi - lo + 31) / 32;
    int64_t idx = lo + (int64_t)(lane + 1) * step - 1;
    bool v = idx < hi;
    bool below = v && (UPPER ? a[idx] <= x : a[idx] < x);
    int c = __popc(__ballot_sync(0xffffffffu, below));
    int nv = __popc(__ballot_sync(0xffffffffu, v));
    int64_t nlo = lo + (int64_t)c * step;
    if (c < nv) hi = lo + (int64_t)(c + 1) * step - 1;
    lo = nlo;
  }
  int64_t idx = lo + lane;
  bool below = idx < hi && (UPPER ? a[idx] <= x : a[idx] < x);
  return lo + __popc(__ballot_sync(0xffffffffu, below));
}

// count of a[0, n) below x (UPPER: <= x), fixed trip count for a block-uniform n
template <bool UPPER>
__device__ __forceinline__ int bsearch_count(const u64* a, int n, int top, u64 x) {
  int pos = 0;
  for (int st = top; st > 0; st >>= 1)
    if (pos + st <= n && (UPPER ? a[pos + st - 1] <= x : a[pos + st - 1] < x)) pos += st;
  return pos;
}

// S_new = (S_cur - olds) U news, one block per tile of S_cur.  Tile b covers the
// values [x0_b, x0_(b+1)): the olds / news of that range are located once per block
// (warp-parallel 32-ary searches) and staged in shared memory, so each element's
// searches are short shared-memory searches; the block also places the news of
// its range.
constexpr int kMergeTile = 1024, kMergeEpt = kMergeTile / 256, kMergeWin = 1024;
template <typename T>
__global__ void __launch_bounds__(256) k_merge_delta_multi(int64_t N, const u64* __restrict__ S_cur,
                                                           const RepRound<T> R, const RepRound<T>* __restrict__ Rp = nullptr) {
  REP_SLOT(S);
  int D = *S.dcount;
  if (D > kDeltaCap) return;
  const u64* __restrict__ olds = S.olds;
  const u64* __restrict__ news = S.news;
  int64_t ntiles = (N + kMergeTile - 1) / kMergeTile;
  bool last = (int64_t)blockIdx.x == ntiles - 1;
  int64_t t0 = (int64_t)blockIdx.x * kMergeTile;
  int64_t t1 = last ? N : t0 + kMergeTile;
  __shared__ int64_t win[5];
  __shared__ u64 so[kMergeWin], sn[kMergeWin];
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  u64 x0 = S_cur[t0];
  if (wid < 5) {
    u64 xn = last ? 0 : S_cur[t1];
    int64_t v = 0;
    switch (wid) {
      case 0: v = warp_bound_u64<false>(olds, D, x0, lane); break;
      case 1: v = last ? D : warp_bound_u64<true>(olds, D, xn, lane); break;
      case 2: v = blockIdx.x == 0 ? 0 : warp_bound_u64<false>(news, D, x0, lane); break;
      case 3: v = last ? D : warp_bound_u64<false>(news, D, xn, lane); break;
      default: v = warp_bound_u64<false>(S_cur, N, x0, lane);  // first copy of x0
    }
    if (lane == 0) win[wid] = v;
  }
  __syncthreads();
  int o0 = (int)win[0], on = (int)(win[1] - win[0]), n0 = (int)win[2], nn = (int)(win[3] - win[2]);
  const u64* wo = olds + o0;
  const u64* wn = news + n0;
  if (on <= kMergeWin && nn <= kMergeWin) {
    for (int i = threadIdx.x; i < on; i += blockDim.x) so[i] = wo[i];
    for (int i = threadIdx.x; i < nn; i += blockDim.x) sn[i] = wn[i];
    wo = so;
    wn = sn;
  }
  __syncthreads();
  int topo = on ? 1 << (31 - __clz(on)) : 0, topn = nn ? 1 << (31 - __clz(nn)) : 0;
  u64 x[kMergeEpt];
  int le[kMergeEpt], lt[kMergeEpt], ln[kMergeEpt];
#pragma unroll
  for (int i = 0; i < kMergeEpt; i++) {
    int64_t t = t0 + threadIdx.x + i * 256;
    x[i] = t < t1 ? S_cur[t] : ~0ull;
  }
#pragma unroll
  for (int i = 0; i < kMergeEpt; i++) {
    le[i] = bsearch_count<true>(wo, on, topo, x[i]);
    lt[i] = bsearch_count<false>(wo, on, topo, x[i]);
    ln[i] = bsearch_count<false>(wn, nn, topn, x[i]);
  }
#pragma unroll
  for (int i = 0; i < kMergeEpt; i++) {
    int64_t t = t0 + threadIdx.x + i * 256;
    if (t >= t1) continue;
    bool kept = true;
    // equal values: the first (le - lt) copies of x in S_cur are the removed ones
    if (le[i] > lt[i]) {
      int64_t first = x[i] == x0 ? win[4] : t0 + lower_bound_u64(S_cur + t0, t - t0, x[i]);
      kept = (t - first) >= le[i] - lt[i];
    }
    if (kept) S.sorted[t - (o0 + le[i]) + n0 + ln[i]] = x[i];
  }
  // the news y of this tile (x0 <= y < x0_next): upper_bound(S_cur, y) lies in [t0, t1]
  for (int q = threadIdx.x; q < nn; q += blockDim.x) {
    u64 y = wn[q];
    int64_t ub = t0 + upper_bound_u64(S_cur + t0, t1 - t0, y);
    S.sorted[n0 + q + ub - (o0 + bsearch_count<true>(wo, on, topo, y))] = y;
  }
}

template <typename T>
__global__ void k_pw_leaves8_multi(int nleaves, const int64_t* __restrict__ loff, const int32_t* __restrict__ llen,
                                   const int32_t* __restrict__ lnode, const RepRound<T> R, const RepRound<T>* __restrict__ Rp = nullptr) {
  REP_SLOT(S);
  int lane = threadIdx.x & 31;
  int j = lane & 7;
  int t = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 3);
  bool ok = t < nleaves;
  const double* a = reinterpret_cast<const double*>(S.sorted) + (ok ? loff[t] : 0);
  int n = ok ? llen[t] : 0;
  double r = 0.0;
  int body = n - (n % 8);
  if (n >= 8) {
    r = a[j];
    for (int i = 8 + j; i < body; i += 8) r = __dadd_rn(r, a[i]);
  }
  double r1 = __shfl_down_sync(0xffffffffu, r, 1);
  double r2 = __shfl_down_sync(0xffffffffu, r, 2);
  double r3 = __shfl_down_sync(0xffffffffu, r, 3);
  double r4 = __shfl_down_sync(0xffffffffu, r, 4);
  double r5 = __shfl_down_sync(0xffffffffu, r, 5);
  double r6 = __shfl_down_sync(0xffffffffu, r, 6);
  double r7 = __shfl_down_sync(0xffffffffu, r, 7);
  if (ok && j == 0) {
    double res;
    if (n < 8) {
      res = 0.0;
      for (int i = 0; i < n; i++) res = __dadd_rn(res, a[i]);
    } else {
      res = __dadd_rn(__dadd_rn(__dadd_rn(r, r1), __dadd_rn(r2, r3)), __dadd_rn(__dadd_rn(r4, r5), __dadd_rn(r6, r7)));
      for (int i = body; i < n; i++) res = __dadd_rn(res, a[i]);
    }
    S.pw[lnode[t]] = res;
    if (lnode[t] == 0) rep_finish(S.pw, S.dcount, S.out);  // a single-leaf tree
  }
}

template <typename T>
__global__ void k_pw_combine_multi(int H, const int32_t* __restrict__ lvl_off, const int32_t* __restrict__ nodes,
                                   const int32_t* __restrict__ left, const int32_t* __restrict__ right,
                                   const RepRound<T> R, const RepRound<T>* __restrict__ Rp = nullptr) {
  REP_SLOT(S);
  double* val = S.pw;
  for (int h = 0; h < H; h++) {
    for (int t = lvl_off[h] + threadIdx.x; t < lvl_off[h + 1]; t += blockDim.x) {
      int nd = nodes[t];
      val[nd] = __dadd_rn(val[left[nd]], val[right[nd]]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) rep_finish(val, S.dcount, S.out);
}

// the same with the whole tree staged in shared memory: node values (nnodes doubles)
// and the internal nodes in level order as {node, left, right} triples
template <typename T>
__global__ void __launch_bounds__(1024) k_pw_combine_multi_smem(int H, int nnodes, int nops,
                                                                const int32_t* __restrict__ lvl_off,
                                                                const int4* __restrict__ ops,
                                                                const RepRound<T> R, const RepRound<T>* __restrict__ Rp = nullptr) {
  extern __shared__ double sval[];
  int4* sops = reinterpret_cast<int4*>(sval + ((nnodes + 1) & ~1));
  int* slvl = reinterpret_cast<int*>(sops + nops);
  REP_SLOT(S);
  double* val = S.pw;
  for (int i = threadIdx.x; i < nnodes; i += blockDim.x) sval[i] = val[i];
  for (int i = threadIdx.x; i < nops; i += blockDim.x) sops[i] = ops[i];
  for (int i = threadIdx.x; i <= H; i += blockDim.x) slvl[i] = lvl_off[i];
  __syncthreads();
  for (int h = 0; h < H; h++) {
    for (int t = slvl[h] + threadIdx.x; t < slvl[h + 1]; t += blockDim.x) {
      int4 o = sops[t];
      sval[o.x] = __dadd_rn(sval[o.y], sval[o.z]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) rep_finish(sval, S.dcount, S.out);
}
}  // namespace stmf
