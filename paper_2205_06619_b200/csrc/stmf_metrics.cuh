// stmf_metrics.cuh — the evaluation step after a fit:
// rmse (metrics.py:87-95) and distance_correlation / masked_dc (metrics.py:98-139)
// on the device, bit-identical to numpy.  numpy's reductions used there are
//   * np.mean over a contiguous 1-d or n x n array: DOUBLE_pairwise_sum over all
//     elements (the iterator coalesces a contiguous array), then one division;
//   * mean(axis=0) of a C-contiguous n x n array: per column, a sequential sum over
//     rows 0..n-1;
//   * mean(axis=1): per row, the pairwise sum over the row's n elements;
// the pairwise trees come from the host PWTree of the length in question.
#pragma once

namespace stmf {

// (pred - truth)**2 over the masked entries of m x n row-major arrays, compacted in
// row-major order (the order of (pred - truth)[mask]); ptr = row offsets.
__global__ void k_masked_sqdiff(int64_t m, int64_t n, const double* __restrict__ pred, const double* __restrict__ truth,
                                const uint8_t* __restrict__ mask, const int64_t* __restrict__ ptr,
                                double* __restrict__ out) {
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
        double d = __dsub_rn(pred[r * n + j], truth[r * n + j]);
        out[pos + __popc(bal & ((1u << lane) - 1))] = __dmul_rn(d, d);
      }
      pos += __popc(bal);
    }
  }
}

// d[i, j] = |x_i - x_j| (metrics.py:121)
__global__ void k_absdiff(int64_t n, const double* __restrict__ x, double* __restrict__ d) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n * n) return;
  int64_t i = t / n, j = t - i * n;
  d[t] = fabs(__dsub_rn(x[i], x[j]));
}

// d.mean(axis=0): sequential over rows, per column
__global__ void k_colmean_seq(int64_t n, const double* __restrict__ d, double* __restrict__ out) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  double s = d[j];
  for (int64_t i = 1; i < n; i++) s = __dadd_rn(s, d[i * n + j]);
  out[j] = __ddiv_rn(s, (double)n);
}

// d.mean(axis=1): numpy's pairwise sum of each contiguous row (tree of length n),
// one block per row, node values in a per-block scratch slice
__global__ void __launch_bounds__(256)
k_rowmean_pw(int64_t m, int64_t n, const double* __restrict__ d, int nleaves, const int64_t* __restrict__ loff,
             const int32_t* __restrict__ llen, const int32_t* __restrict__ lnode, int H,
             const int32_t* __restrict__ lvl_off, const int32_t* __restrict__ lvl_nodes,
             const int32_t* __restrict__ left, const int32_t* __restrict__ right, int nnodes,
             double* __restrict__ scratch, double* __restrict__ out) {
  double* val = scratch + (size_t)blockIdx.x * (size_t)nnodes;
  for (int64_t i = blockIdx.x; i < m; i += gridDim.x) {
    const double* row = d + i * n;
    for (int t = threadIdx.x; t < nleaves; t += blockDim.x) {
      const double* a = row + loff[t];
      int len = llen[t];
      double res;
      if (len < 8) {
        res = 0.0;
        for (int q = 0; q < len; q++) res = __dadd_rn(res, a[q]);
      } else {
        double r[8];
#pragma unroll
        for (int j = 0; j < 8; j++) r[j] = a[j];
        int q;
        for (q = 8; q < len - (len % 8); q += 8)
#pragma unroll
          for (int j = 0; j < 8; j++) r[j] = __dadd_rn(r[j], a[q + j]);
        res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                        __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
        for (; q < len; q++) res = __dadd_rn(res, a[q]);
      }
      val[lnode[t]] = res;
    }
    __syncthreads();
    for (int h = 0; h < H; h++) {
      for (int t = lvl_off[h] + threadIdx.x; t < lvl_off[h + 1]; t += blockDim.x) {
        int nd = lvl_nodes[t];
        val[nd] = __dadd_rn(val[left[nd]], val[right[nd]]);
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) out[i] = __ddiv_rn(val[0], (double)n);
    __syncthreads();
  }
}

// A = d - cm[None, :] - rm[:, None] + tm, evaluated left to right (metrics.py:122)
__global__ void k_center(int64_t n, double* __restrict__ d, const double* __restrict__ cm,
                         const double* __restrict__ rm, double tm) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n * n) return;
  int64_t i = t / n, j = t - i * n;
  d[t] = __dadd_rn(__dsub_rn(__dsub_rn(d[t], cm[j]), rm[i]), tm);
}

__global__ void k_mul(int64_t len, const double* __restrict__ a, const double* __restrict__ b, double* __restrict__ o) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < len) o[t] = __dmul_rn(a[t], b[t]);
}

}  // namespace stmf
