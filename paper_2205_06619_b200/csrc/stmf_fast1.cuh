// stmf_fast1.cuh — phase B's first half (the second residuation of every evaluation)
// from per-line order statistics instead of a pass over the given entries.
//
// An eval's second residuation of line L is  w_q(L) = min_p (x_p - v'_q[o_p])  over the
// line's entries p (o_p = the entry's index on the other side), i.e. _residuate_col /
// _residuate_row (engine.py:198-207) after the first one.  The first-residuation vector
// v'_q equals a BASE vector shared by every eval of the same factor index k except on a
// few indices:
//   F-ULF (lines = rows):    v'_q,c = min(CM^(-i)_k,c, X_ic - s_q)  <= CM^(-i)_k,c = base
//   F-URF (lines = columns): u'_q,r = min(RM^(-j)_k,r, X_rj - s'_q), RM^(-j) = RM except on
//                            the rows whose row minimum sits in column j (rmarg == j_q)
// Where v' <= base the entry's term x - v' can only grow.  So with the kTop smallest
// base terms of every line (value, other index, x; ascending), the line minimum is
// exact from a walk over them: exceptional entries (v' != base) contribute their new
// term, and the first unexceptional entry's base term bounds every entry outside the
// walked prefix.  The F-URF rows with rmarg == j_q (their u' may exceed the base, so
// their terms may shrink) are added by a scatter (k_pass1_dscatter) of their entries.
// Walks that meet kTop exceptional entries, and evals whose k has no statistics, fall
// back to the full pass over the line (line_min8).  min / sub are exact IEEE ops, so the
// result is the full pass's bit for bit.
//
// Statistics: F-ULF per row visit (the base CM^(-i)_k depends on the visited row i, k =
// the first candidate's factor index); F-URF per factor index k, valid until row k of V
// changes (a commit with index k invalidates it).
#pragma once

#include "stmf_kernels.cuh"

namespace stmf {

constexpr int kTop = 4;

// per line: the kTop smallest base terms (ascending), [kTop][nlines] each
template <typename T>
struct TopK {
  T* val;
  int32_t* oth;  // -1: empty slot (a line with fewer entries)
  T* xv;
};

// (nv, no) before slot t?  Empty slots come after every entry, ties keep insertion order.
template <typename T>
__device__ __forceinline__ bool top_lt(T nv, T v, int o) { return nv < v || (nv == v && o < 0); }

template <typename T>
__device__ __forceinline__ void top_insert(T (&v)[kTop], int (&o)[kTop], T (&x)[kTop], T nv, int no, T nx) {
  static_assert(kTop == 4, "unrolled insertion");
  if (!top_lt(nv, v[3], o[3])) return;
  bool c0 = top_lt(nv, v[0], o[0]), c1 = top_lt(nv, v[1], o[1]), c2 = top_lt(nv, v[2], o[2]);
  // slot 3
  v[3] = c2 ? v[2] : nv; o[3] = c2 ? o[2] : no; x[3] = c2 ? x[2] : nx;
  // slot 2
  T v2 = c1 ? v[1] : (c2 ? nv : v[2]);
  int o2 = c1 ? o[1] : (c2 ? no : o[2]);
  T x2 = c1 ? x[1] : (c2 ? nx : x[2]);
  v[2] = v2; o[2] = o2; x[2] = x2;
  T v1 = c0 ? v[0] : (c1 ? nv : v[1]);
  int o1 = c0 ? o[0] : (c1 ? no : o[1]);
  T x1 = c0 ? x[0] : (c1 ? nx : x[1]);
  v[1] = v1; o[1] = o1; x[1] = x1;
  if (c0) { v[0] = nv; o[0] = no; x[0] = nx; }
}

// top-kTop of the base terms x_p - base[o_p] of every line, one warp per line.
// kptr: the factor index (device; the F-ULF row k, or the F-URF k of the visit's first
// candidate); base = base0 + k * base_stride; out = out0 shifted by k * out_stride.
// skip (may be null): per-k validity flags -- nothing to do when skip[k] is set.
template <typename T>
__global__ void k_top_lines(int64_t nlines, const int64_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                            const T* __restrict__ xv, const T* __restrict__ base0, int64_t base_stride,
                            const int32_t* __restrict__ kptr, const int* __restrict__ skip, TopK<T> out0,
                            int64_t out_stride) {
  const int k = *kptr;
  if (skip && skip[k]) return;
  const T* __restrict__ base = base0 + (int64_t)k * base_stride;
  T* oval = out0.val + (int64_t)k * out_stride;
  int32_t* ooth = out0.oth + (int64_t)k * out_stride;
  T* oxv = out0.xv + (int64_t)k * out_stride;
  int lane = threadIdx.x & 31;
  int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t L = w; L < nlines; L += nw) {
    T v[kTop], x[kTop];
    int o[kTop];
#pragma unroll
    for (int t = 0; t < kTop; t++) { v[t] = tinf<T>(); o[t] = -1; x[t] = T(0); }
    for (int64_t p = ptr[L] + lane; p < ptr[L + 1]; p += 32) {
      int c = idx[p];
      STMF_IDX(c, base_stride);
      T xx = xv[p];
      top_insert(v, o, x, sub_rn(xx, base[c]), c, xx);
    }
#pragma unroll
    for (int m = 16; m; m >>= 1) {
      T pv[kTop], px[kTop];
      int po[kTop];
#pragma unroll
      for (int t = 0; t < kTop; t++) {
        pv[t] = __shfl_xor_sync(0xffffffffu, v[t], m);
        po[t] = __shfl_xor_sync(0xffffffffu, o[t], m);
        px[t] = __shfl_xor_sync(0xffffffffu, x[t], m);
      }
#pragma unroll
      for (int t = 0; t < kTop; t++)
        if (po[t] >= 0) top_insert(v, o, x, pv[t], po[t], px[t]);
    }
    // every lane holds the same multiset, but tied values may sit in different slots on
    // different lanes (the residuations make exact ties at the line minimum common):
    // one lane writes the whole list
    if (lane == 0) {
#pragma unroll
      for (int t = 0; t < kTop; t++) {
        oval[t * nlines + L] = v[t];
        ooth[t * nlines + L] = o[t];
        oxv[t * nlines + L] = x[t];
      }
    }
  }
}

// after k_top_lines: record what the statistics are valid for
__global__ void k_top_mark(const int32_t* __restrict__ kptr, int* __restrict__ valid, int* __restrict__ kout) {
  if (valid) valid[*kptr] = 1;
  if (kout) *kout = *kptr;
}

// what k_pass1_fast needs besides the two sides of phase B
template <typename T>
struct Fast1 {
  TopK<T> ulf;          // per row of the visit (base CM^(-i)_k, k = *ulf_k)
  const int* ulf_k;
  TopK<T> urf;          // per column per k ([k][kTop][n]), base RM_k = rm1 + k m
  const int* urf_valid; // per k
  const T* rm1;
  const int32_t* rmarg;
  const int32_t* cj;    // candidate columns (batch-relative after the graph offset)
  unsigned long long* stats = nullptr;  // diagnostics: {ULF items, ULF fallbacks, URF items, URF fallbacks}
};

// line values of every (line, eval group) item of both sides into S.out (eval-major)
template <typename T>
__device__ __forceinline__ void fast1_item(const SideB<T>& S, bool ulf, int64_t it, int E,
                                           const int32_t* __restrict__ ek, const Fast1<T>& FS, int lane) {
  constexpr int EG = kEG;
  const int64_t nlines = S.nlines;
  const int ngroups = (E + EG - 1) / EG;
  const int g = (int)(it / nlines);
  const int64_t L = it - (int64_t)g * nlines;
  const int e0 = g * EG;
  const int ne = E - e0 < EG ? E - e0 : EG;
  (void)ngroups;
  T w = tinf<T>();
  bool fb = false;
  int kq = ek[e0 + (lane < ne ? lane : ne - 1)];
  if (lane < ne) {
    bool done = false;
    if (ulf) {
      if (!S.inl_base || kq != *FS.ulf_k) {
        fb = true;
      } else {
        const T* __restrict__ base = S.inl_base + (int64_t)kq * S.len_other;
        const T sq = S.inl_s[e0 + lane];
#pragma unroll
        for (int t = 0; t < kTop && !done; t++) {
          int c = FS.ulf.oth[t * nlines + L];
          if (c < 0) { done = true; break; }
          STMF_IDX(c, S.len_other);
          T b = base[c];
          T vn = vmin(b, sub_rn(S.inl_xr[c], sq));
          if (vn == b) {
            w = vmin(w, FS.ulf.val[t * nlines + L]);
            done = true;
          } else {
            w = vmin(w, sub_rn(FS.ulf.xv[t * nlines + L], vn));
          }
        }
        fb = !done;
      }
    } else {
      if (!FS.urf_valid[kq]) {
        fb = true;
      } else {
        const int64_t ko = (int64_t)kq * kTop * nlines;
        const T* __restrict__ rm = FS.rm1 + (int64_t)kq * S.len_other;
#pragma unroll
        for (int t = 0; t < kTop && !done; t++) {
          int r = FS.urf.oth[ko + t * nlines + L];
          if (r < 0) { done = true; break; }
          STMF_IDX(r, S.len_other);
          T u = S.vin[ilv_index<T>(e0 + lane, r, S.len_other)];
          if (u == rm[r]) {
            w = vmin(w, FS.urf.val[ko + t * nlines + L]);
            done = true;
          } else {
            w = vmin(w, sub_rn(FS.urf.xv[ko + t * nlines + L], u));
          }
        }
        fb = !done;
      }
    }
  }
  if (FS.stats && lane < ne) {
    atomicAdd(FS.stats + (ulf ? 0 : 2), 1ull);
    if (fb) atomicAdd(FS.stats + (ulf ? 1 : 3), 1ull);
  }
  if (__ballot_sync(0xffffffffu, fb)) {
    // full pass over the line for the group (exact for all its evals)
    int kk[EG];
    bool unif = true;
#pragma unroll
    for (int q = 0; q < EG; q++) {
      kk[q] = ek[e0 + (q < ne ? q : ne - 1)];
      unif &= kk[q] == kk[0];
    }
    const GroupRows<T> pl{S.vin, g, S.len_other};
    const int beg = (int)S.ptr[L], end = (int)S.ptr[L + 1];
    T mn[EG], s[EG];
    if (ulf && unif && S.inl_base) {
#pragma unroll
      for (int q = 0; q < EG; q++) s[q] = S.inl_s[e0 + (q < ne ? q : ne - 1)];
      line_min8<T, 2>(S, pl, S.inl_base + (int64_t)kk[0] * S.len_other, s, beg, beg, end, lane, mn);
    } else {
#pragma unroll
      for (int q = 0; q < EG; q++) s[q] = T(0);
      line_min8<T, 0>(S, pl, nullptr, s, beg, beg, end, lane, mn);
    }
    T full = lane_pick<EG>(mn, lane < EG ? lane : 0);
    if (fb) w = full;
  }
  if (lane < ne) S.out[(int64_t)(e0 + lane) * nlines + L] = w;
}

template <typename T>
__global__ void __launch_bounds__(256) k_pass1_fast(SideB<T> A, SideB<T> B, int E, const int32_t* __restrict__ ek,
                                                    Fast1<T> FS, const DevCtl* __restrict__ g = nullptr,
                                                    const int32_t* __restrict__ ck = nullptr) {
  if (g) {
    E = g->E;
    ek = ck + g->t0;
  }
  int lane = threadIdx.x & 31;
  int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int ngroups = (E + kEG - 1) / kEG;
  int64_t itemsA = A.nlines * ngroups, items = itemsA + B.nlines * ngroups;
  for (int64_t it = w; it < items; it += nw) {
    if (it < itemsA) fast1_item<T>(A, true, it, E, ek, FS, lane);
    else fast1_item<T>(B, false, it - itemsA, E, ek, FS, lane);
  }
}

// float / double atomic minimum through compare-and-swap of the bit pattern
__device__ __forceinline__ void atomic_min_val(float* a, float v) {
  int* ai = reinterpret_cast<int*>(a);
  int old = *ai;
  while (v < __int_as_float(old)) {
    int prev = atomicCAS(ai, old, __float_as_int(v));
    if (prev == old) break;
    old = prev;
  }
}
__device__ __forceinline__ void atomic_min_val(double* a, double v) {
  unsigned long long* ai = reinterpret_cast<unsigned long long*>(a);
  unsigned long long old = *ai;
  while (v < __longlong_as_double((long long)old)) {
    unsigned long long prev = atomicCAS(ai, old, (unsigned long long)__double_as_longlong(v));
    if (prev == old) break;
    old = prev;
  }
}

// F-URF rows whose row minimum sits in the eval's column j_q (u' may exceed the base
// there): every entry of such a row offers x - u' to its column's line value.  One warp
// per (eval, 32 rows); the matches are rare (about m / n rows per eval).
template <typename T>
__global__ void k_pass1_dscatter(int64_t m, int64_t n, const int64_t* __restrict__ row_ptr,
                                 const int32_t* __restrict__ col_idx, const T* __restrict__ xr, int E,
                                 const int32_t* __restrict__ ek, const int32_t* __restrict__ ej,
                                 const int32_t* __restrict__ rmarg, const int* __restrict__ urf_valid,
                                 const T* __restrict__ vin, T* __restrict__ out, const DevCtl* __restrict__ g = nullptr,
                                 const int32_t* __restrict__ ck = nullptr, const int32_t* __restrict__ cjall = nullptr) {
  if (g) {
    E = g->E;
    ek = ck + g->t0;
    ej = cjall + g->t0;
  }
  int lane = threadIdx.x & 31;
  int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int64_t chunks = (m + 31) / 32;
  for (int64_t it = w; it < (int64_t)E * chunks; it += nw) {
    int q = (int)(it / chunks);
    int64_t r = (it - (int64_t)q * chunks) * 32 + lane;
    int k = ek[q], j = ej[q];
    if (!urf_valid[k]) continue;  // warp-uniform: the eval took the full pass
    bool match = r < m && rmarg[(int64_t)k * m + r] == j;
    unsigned bm = __ballot_sync(0xffffffffu, match);
    while (bm) {
      int l = __ffs(bm) - 1;
      bm &= bm - 1;
      int64_t rr = (it - (int64_t)q * chunks) * 32 + l;
      T u = vin[ilv_index<T>(q, rr, m)];
      for (int64_t p = row_ptr[rr] + lane; p < row_ptr[rr + 1]; p += 32) {
        STMF_IDX(col_idx[p], n);
        atomic_min_val(out + (int64_t)q * n + col_idx[p], sub_rn(xr[p], u));
      }
    }
  }
}

}  // namespace stmf
