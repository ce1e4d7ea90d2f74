// stmf_strategies.cuh — candidate builders and scores for the reference's other fit
// methods on the same evaluation kernels:
//   * ByRow selections TD (argmax_k, strategies.py:146-148) and TD_B
//     (select_k_td_b, strategies.py:164-178); SEQ (byrow_seq, strategies.py:227-249)
//     reuses the entry x k candidate layout of the baseline;
//   * ByElement (byelement_sweep, strategies.py:252-269);
//   * the STMF baseline (_BaselineStrategy.sweep, engine.py:365-380);
//   * ByMatrix entry scores (bymatrix_step, strategies.py:272-299).
// Everything that decides a candidate's order or its factor index is exact, so the
// candidate lists are identical to the reference's.
#pragma once

#include <cub/block/block_scan.cuh>

namespace stmf {

// td_grid(R, U, V).sum(axis=1) for binary64 (strategies.py:172, 283): numpy reduces
// a contiguous row with DOUBLE_pairwise_sum over all n entries, zeros under the mask
// included, so the tree depends on n only (host PWTree of length n).  One block per
// row: the dense td row and the node values live in a per-block scratch slice.
__global__ void __launch_bounds__(256)
k_row_scores_pw(int64_t m, int64_t n, const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx,
                const double* __restrict__ xr, const double* __restrict__ t1, int nleaves,
                const int64_t* __restrict__ loff, const int32_t* __restrict__ llen, const int32_t* __restrict__ lnode,
                int H, const int32_t* __restrict__ lvl_off, const int32_t* __restrict__ lvl_nodes,
                const int32_t* __restrict__ left, const int32_t* __restrict__ right, int nnodes,
                double* __restrict__ scratch, double* __restrict__ out) {
  double* dense = scratch + (size_t)blockIdx.x * (size_t)(n + nnodes);
  double* val = dense + n;
  for (int64_t i = blockIdx.x; i < m; i += gridDim.x) {
    for (int64_t c = threadIdx.x; c < n; c += blockDim.x) dense[c] = 0.0;
    __syncthreads();
    for (int64_t p = row_ptr[i] + threadIdx.x; p < row_ptr[i + 1]; p += blockDim.x)
      dense[col_idx[p]] = fabs(__dsub_rn(xr[p], t1[p]));
    __syncthreads();
    for (int t = threadIdx.x; t < nleaves; t += blockDim.x) {
      const double* a = dense + loff[t];
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
    if (threadIdx.x == 0) out[i] = val[0];
    __syncthreads();
  }
}

// Row scores in the binary32 semantics (exact sum of the binary32 terms, rounded
// once to binary64, like the column scores): a warp per row; the fp64 partial sums
// are exact below exact_limit (flag 4 otherwise).
template <typename T>
__global__ void __launch_bounds__(256)
k_row_scores_exact(int64_t m, const int64_t* __restrict__ row_ptr, const T* __restrict__ xr, const T* __restrict__ t1,
                   double* __restrict__ out, double exact_limit, int* __restrict__ flags) {
  int lane = threadIdx.x & 31;
  int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = w; i < m; i += nw) {
    double s = 0.0;
    for (int64_t p = row_ptr[i] + lane; p < row_ptr[i + 1]; p += 32) s = __dadd_rn(s, (double)vabs(sub_rn(xr[p], t1[p])));
    for (int o = 16; o; o >>= 1) s = __dadd_rn(s, shfl_xor(s, o));
    if (lane == 0) {
      if (!(s < exact_limit)) atomicOr(flags, 4);
      out[i] = s;
    }
  }
}

// first index of the maximum of a[0, len) over one block (np.argmax)
__device__ __forceinline__ int64_t block_argmax(const double* __restrict__ a, int64_t len, double* sv, int64_t* si) {
  double bv = -CUDART_INF;
  int64_t bi = len;
  for (int64_t t = threadIdx.x; t < len; t += blockDim.x)
    if (a[t] > bv) { bv = a[t]; bi = t; }  // increasing t: keeps the first max of this thread
  sv[threadIdx.x] = bv;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      double v2 = sv[threadIdx.x + s];
      int64_t i2 = si[threadIdx.x + s];
      if (v2 > sv[threadIdx.x] || (v2 == sv[threadIdx.x] && i2 < si[threadIdx.x])) {
        sv[threadIdx.x] = v2;
        si[threadIdx.x] = i2;
      }
    }
    __syncthreads();
  }
  int64_t r = si[0];
  __syncthreads();
  return r;
}

// max_k U[a, k] + V[k, b] and its lowest argmax (trop_matmul / argmax_k, tropical.py:169, 232-234)
template <typename T>
__device__ __forceinline__ T prod_at(int rank, int64_t m, int64_t n, const T* __restrict__ Ut, const T* __restrict__ V,
                                     int64_t a, int64_t b, int* karg) {
  T best = add_rn(Ut[a], V[b]);
  int kb = 0;
  for (int k = 1; k < rank; k++) {
    T v = add_rn(Ut[(int64_t)k * m + a], V[(int64_t)k * n + b]);
    if (v > best) { best = v; kb = k; }
  }
  if (karg) *karg = kb;
  return best;
}

// select_k_td_b for every candidate of row i (strategies.py:164-178): j0 = argmax of
// the column scores, i0 = argmax of the row scores; k = argmax_k at (i, j0) when
// prod[i, j0] >= prod[i0, j], else at (i0, j).  One block of 256 threads.
template <typename T>
__global__ void __launch_bounds__(256)
k_cand_tdb(int nc, int rank, int64_t m, int64_t n, int64_t i, const T* __restrict__ Ut, const T* __restrict__ V,
           const double* __restrict__ rscore, const double* __restrict__ cscore, const int32_t* __restrict__ cj,
           int32_t* __restrict__ ck) {
  __shared__ double sv[256];
  __shared__ int64_t si[256];
  int64_t j0 = block_argmax(cscore, n, sv, si);
  int64_t i0 = block_argmax(rscore, m, sv, si);
  int k_ij0;
  T p_ij0 = prod_at<T>(rank, m, n, Ut, V, i, j0, &k_ij0);
  for (int t = threadIdx.x; t < nc; t += blockDim.x) {
    int j = cj[t];
    int k_i0j;
    T p_i0j = prod_at<T>(rank, m, n, Ut, V, i0, j, &k_i0j);
    ck[t] = p_ij0 >= p_i0j ? k_ij0 : k_i0j;
  }
}

// ByElement candidates of row i from entry position p0 (byelement_sweep,
// strategies.py:260-269): the given entries in column order whose current error
// |x - P| is nonzero, k = the entry's argmax; at most cap of them.  One block of
// 1024 threads (block scan per chunk).  pos[t] = the entry's CSR position; *cnt.
template <typename T>
__global__ void __launch_bounds__(1024)
k_cand_elem(int64_t p0, int64_t end, int cap, const int32_t* __restrict__ col_idx, const T* __restrict__ xr,
            const T* __restrict__ t1, const uint8_t* __restrict__ ag, int32_t* __restrict__ cj, int32_t* __restrict__ ck,
            T* __restrict__ cx, int64_t* __restrict__ pos, int* __restrict__ cnt) {
  using Scan = cub::BlockScan<int, 1024>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int base;
  if (threadIdx.x == 0) base = 0;
  __syncthreads();
  for (int64_t c0 = p0; c0 < end; c0 += 1024) {
    int64_t p = c0 + threadIdx.x;
    int keep = (p < end && xr[p] != t1[p]) ? 1 : 0;
    int off, tot;
    Scan(tmp).ExclusiveSum(keep, off, tot);
    int b = base;
    if (keep && b + off < cap) {
      int t = b + off;
      cj[t] = col_idx[p]; ck[t] = ag[p]; cx[t] = xr[p]; pos[t] = p;
    }
    __syncthreads();
    if (threadIdx.x == 0) base = b + tot;
    __syncthreads();
    if (base >= cap) break;
  }
  if (threadIdx.x == 0) *cnt = base < cap ? base : cap;
}

// Entry x factor-index candidates (STMF baseline / ByRow SEQ): entry e of
// [p0, p0 + ne) with k = 0..rank-1 at t = e * rank + k.
template <typename T>
__global__ void k_cand_entries(int64_t p0, int ne, int rank, const int32_t* __restrict__ col_idx,
                               const T* __restrict__ xr, int32_t* __restrict__ cj, int32_t* __restrict__ ck,
                               T* __restrict__ cx) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)ne * rank) return;
  int64_t e = t / rank;
  cj[t] = col_idx[p0 + e];
  ck[t] = (int32_t)(t - e * rank);
  cx[t] = xr[p0 + e];
}

// ByMatrix entry scores (strategies.py:281-286): row_sums[i] + col_sums[j] - grid[i, j]
// over the given entries in row-major order; keys ~bits (scores >= +0) so a stable
// ascending radix sort is np.argsort(-scores, kind="stable").
template <typename T>
__global__ void k_matrix_keys(int64_t N, const int32_t* __restrict__ rowof, const int32_t* __restrict__ col_idx,
                              const T* __restrict__ xr, const T* __restrict__ t1, const double* __restrict__ rs,
                              const double* __restrict__ cs, u64* __restrict__ keys, int32_t* __restrict__ vals,
                              double* __restrict__ sc) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= N) return;
  double g = (double)vabs(sub_rn(xr[p], t1[p]));
  double s = __dsub_rn(__dadd_rn(rs[rowof[p]], cs[col_idx[p]]), g);
  keys[p] = ~(u64)__double_as_longlong(s);
  vals[p] = (int32_t)p;
  sc[p] = s;
}

template <typename T>
__global__ void k_matrix_gather(int64_t N, const int32_t* __restrict__ perm, const int32_t* __restrict__ rowof,
                                const int32_t* __restrict__ col_idx, const uint8_t* __restrict__ ag,
                                const double* __restrict__ sc, int32_t* __restrict__ orow, int32_t* __restrict__ ocol,
                                int32_t* __restrict__ ok, double* __restrict__ osc) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= N) return;
  int p = perm[t];
  orow[t] = rowof[p];
  ocol[t] = col_idx[p];
  ok[t] = ag[p];
  osc[t] = sc[p];
}

}  // namespace stmf
