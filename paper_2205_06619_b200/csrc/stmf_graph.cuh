// stmf_graph.cuh — device-resident sweep driver.
//
// Session::run with a sweep budget executes each sweep as ONE CUDA graph launch:
// nested conditional nodes replace the host loop of Session::row_visit /
// decide_batch (strategies.py:191-224 ByRow with TD_A, engine.py:278-295 attempt):
//
//   WHILE row < m                                     (h_row)
//     row_begin, candidates of row i (k_cand_row)
//     WHILE batch                                     (h_batch)
//       phase A, phase B of the batch, decide
//       WHILE escalation  [fp64]                      (h_esc)
//         numpy replicas of the pending evals, full-sort fallback (IF h_fb), decide_esc
//     IF accepted                                     (h_acc)
//       commit, product caches, scores, residuation statistics of k
//     row_end
//
// The decisions are the host loop's, made by one device thread from the same
// batch results, so the trajectory is identical; the host reads the control block
// and the trajectory once per sweep.
#pragma once
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "stmf_kernels.cuh"

namespace stmf {

// (hi:lo) * 2^-F rounded to nearest even binary64 (device twin of fx_to_double)
__device__ __forceinline__ double fx_to_double_dev(u64 hi, u64 lo, int F) {
  if (hi == 0) return scalbn(__ull2double_rn(lo), -F);
  int top = 64 + 63 - __clzll((long long)hi);
  int sh = top - 52;  // >= 12
  u64 q = sh >= 64 ? hi >> (sh - 64) : (hi << (64 - sh)) | (lo >> sh);
  q &= (1ull << 53) - 1;
  q |= 1ull << 52;
  int gp = sh - 1;  // guard bit position (>= 11); sticky = any bit below it
  int guard = (int)(gp >= 64 ? (hi >> (gp - 64)) & 1u : (lo >> gp) & 1u);
  bool sticky = gp >= 64 ? (lo != 0 || (gp > 64 && (hi & ((1ull << (gp - 64)) - 1)) != 0))
                         : (lo & ((1ull << gp) - 1)) != 0;
  if (guard && (sticky || (q & 1u))) q++;
  return scalbn((double)q, sh - F);
}

// buffers and constants of the device-side decisions
template <typename T>
struct GBufs {
  u64* bst;                  // batch results [flags][acc 4E][chg 2E]
  const int32_t* ck;         // factor index of every candidate of the row
  T* ubufB; T* vbuf; T* ubufA; T* vbufB;  // eval buffers (phase B outputs, planar phase A)
  int64_t m, n;
  long long* row_depth;
  double* traj_t; double* traj_e;
  RepRound<T>* rr;           // the pending replica round
  u64* res[kRepSlots]; u64* sorted[kRepSlots]; u64* olds[kRepSlots]; u64* news[kRepSlots];
  int* dcount; double* pw[kRepSlots]; double* out;  // out: value, count per slot
  int F;
  int exact;
  double dr[2], da[2], beta;  // fp64 decision bound (Session::margin_of)
  double* aval;               // the batch's eval objectives (fixed point -> binary64), 2 Emax
  int* urf_valid;             // per-k validity of the F-URF line statistics (stmf_fast1.cuh); may be null
};

__device__ __forceinline__ int grow_next(const DevCtl* c, int next) {
  int g = (int)(next * c->sched_growth);
  int v = next + 1 > g ? next + 1 : g;
  return round_batch(v, c->e_round, c->Emax);
}

__global__ void k_g_sweep_begin(DevCtl* c, int64_t m, cudaGraphConditionalHandle h_row) {
  c->i = c->start_row;
  cudaGraphSetConditional(h_row, (m > 0 && !c->error && !c->stop) ? 1 : 0);
}

// Session::row_visit prologue: batch window from the row's depth history
__global__ void k_g_row_begin(DevCtl* c, const int64_t* __restrict__ row_ptr, const long long* __restrict__ row_depth,
                              cudaGraphConditionalHandle h_batch, cudaGraphConditionalHandle h_acc) {
  int64_t i = c->i;
  int64_t nc = row_ptr[i + 1] - row_ptr[i];
  c->nc = nc;
  c->t0 = 0;
  c->accepted = 0;
  c->visits++;
  int first = c->first0;
  long long d = row_depth[i];
  double dd = d > 0 ? (double)d : (c->ema_first ? c->depth_ema : 0.0);
  if (dd > 0) {
    long long f = (long long)(c->sched_scale * dd) + c->sched_add;
    if (f > c->Emax) f = c->Emax;
    if (f < c->batch_floor) f = c->batch_floor;
    first = (int)f;
  }
  first = round_batch(first, c->e_round, c->Emax);
  c->E = (int)(nc < first ? nc : first);
  c->next = grow_next(c, first);
  cudaGraphSetConditional(h_batch, 1);
  cudaGraphSetConditional(h_acc, 0);
}

// zero the batch results ([flags][acc 4E][chg 2E])
__global__ void k_g_zero(const DevCtl* __restrict__ c, u64* bst) {
  int64_t words = 2 + 4 * (int64_t)c->E + c->E;  // chg: 2E int = E u64
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < words; t += (int64_t)gridDim.x * blockDim.x)
    bst[t] = 0;
}

template <typename T>
__device__ void g_accept(DevCtl* c, const GBufs<T>& B, int w, int q, int op, double value, int slot,
                         cudaGraphConditionalHandle h_batch, cudaGraphConditionalHandle h_acc) {
  c->attempts += w + 1;
  B.row_depth[c->i] = c->t0 + w / 2 + 1;
  {
    double dep = (double)(c->t0 + w / 2 + 1);
    c->depth_ema = c->depth_ema > 0 ? 0.9 * c->depth_ema + 0.1 * dep : dep;
  }
  c->err = value;
  c->accepted = 1;
  c->win_op = op;
  c->win_q = q;
  c->win_k = B.ck[c->t0 + q];
  c->win_slot = slot;
  c->direct = 0;
  if (c->traj_len >= c->traj_cap) {
    c->error = 2;
  } else {
    B.traj_t[c->traj_len] = c->sweep;
    B.traj_e[c->traj_len] = value;
    c->traj_len++;
  }
  cudaGraphSetConditional(h_batch, 0);
  cudaGraphSetConditional(h_acc, c->error ? 0 : 1);
}

// no accept in this batch: next batch of the row, or the row is exhausted
__device__ __forceinline__ void g_advance(DevCtl* c, long long* row_depth, cudaGraphConditionalHandle h_batch) {
  c->attempts += 2 * (long long)c->E;
  c->t0 += c->E;
  if (c->t0 >= c->nc) {
    row_depth[c->i] = c->nc;
    cudaGraphSetConditional(h_batch, 0);
  } else {
    int64_t rem = c->nc - c->t0;
    c->E = (int)(rem < c->next ? rem : c->next);
    c->next = grow_next(c, c->next);
    cudaGraphSetConditional(h_batch, 1);
  }
}

__device__ __forceinline__ bool g_flags_bad(const u64* bst, int exact) {
  int fl = reinterpret_cast<const int*>(bst)[0];
  return (fl & ~1 & 7) || (exact && (fl & 1));
}

// The batch's 2E evals in reference order (scan = 2q + op) are classified in
// parallel, one thread per eval (2E <= 1024): 0 = skip (state reproduced bit for
// bit, or certainly not below err), 1 = bound straddles err (fp64: replicate),
// 2 = below err (fp32: exact; fp64: certainly below, still replicated for its numpy
// value).  Block scans then pick what the host's sequential scan would pick.
constexpr int kDecideThreads = 1024;

template <typename T>
__device__ __forceinline__ int g_class(const DevCtl* c, const GBufs<T>& B, int scan, bool compute, double& A) {
  int E = c->E;
  int q = scan >> 1, op = scan & 1;
  if (compute) {
    const u64* acc = B.bst + 2;
    const int* chg = reinterpret_cast<const int*>(B.bst + 2 + 4 * (int64_t)E);
    A = chg[op * E + q] ? fx_to_double_dev(acc[2 * (int64_t)op * E + 2 * q + 1], acc[2 * (int64_t)op * E + 2 * q], B.F)
                        : -1.0;  // -1: unchanged (f == err exactly)
    B.aval[scan] = A;
  } else {
    A = B.aval[scan];
  }
  if (A < 0) return 0;
  if (B.exact) return A < c->err ? 2 : 0;
  double mg = 2.0 * ((B.dr[op] + B.beta) * fmax(A, c->err) + B.da[op]);
  if (A - mg >= c->err) return 0;
  return A + mg < c->err ? 2 : 1;
}

// fp64: the chunk from c->pos: selected evals (class >= 1) in order, up to 8 and up
// to the first certain one inclusive; writes the replica round.  Returns nchunk.
template <typename T>
__device__ int g_chunk(DevCtl* c, const GBufs<T>& B, int cls, int scan) {
  typedef cub::BlockScan<int, kDecideThreads> Scan;
  typedef cub::BlockReduce<int, kDecideThreads> Red;
  __shared__ typename Scan::TempStorage ts;
  __shared__ typename Red::TempStorage tr;
  __shared__ int s_fc, s_nsel_fc, s_total;
  int E = c->E, pos = c->pos;
  bool sel = scan < 2 * E && scan >= pos && cls >= 1;
  int cert_idx = (sel && cls == 2) ? scan : 1 << 30;
  int fc = Red(tr).Reduce(cert_idx, cub::Min());
  if (threadIdx.x == 0) s_fc = fc;
  __syncthreads();
  fc = s_fc;
  int rank, total;
  Scan(ts).ExclusiveSum(sel ? 1 : 0, rank, total);
  if (sel && scan == fc) s_nsel_fc = rank + 1;  // selected evals up to the first certain
  if (threadIdx.x == 0) s_total = total;
  __syncthreads();
  int lim = fc < (1 << 30) ? s_nsel_fc : s_total;
  int nch = lim < kRepSlots ? lim : kRepSlots;
  if (sel && rank < nch) {
    int q = scan >> 1, op = scan & 1;
    c->ch_ev[rank] = scan; c->ch_q[rank] = q; c->ch_op[rank] = op; c->ch_cert[rank] = cls == 2;
    RepSlot<T> S;
    constexpr int EGP = Ilv<T>::STRIDE;
    S.k = B.ck[c->t0 + q];
    if (op == 0) {
      S.a = B.ubufB + (int64_t)q * B.m; S.as = 1;
      S.b = B.vbuf + ilv_index<T>(q, 0, B.n); S.bs = EGP;
    } else {
      S.a = B.ubufA + ilv_index<T>(q, 0, B.m); S.as = EGP;
      S.b = B.vbufB + (int64_t)q * B.n; S.bs = 1;
    }
    S.res = B.res[rank]; S.sorted = B.sorted[rank]; S.olds = B.olds[rank]; S.news = B.news[rank];
    S.dcount = B.dcount + rank; S.pw = B.pw[rank]; S.out = B.out + 2 * rank;
    B.rr->s[rank] = S;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // host scan: stops after the 8th selected (scan = its index + 1), after the first
    // certain (its index + 1), or at the end of the batch
    int newpos = 2 * E;
    if (nch > 0 && (c->ch_cert[nch - 1] || nch == kRepSlots)) newpos = c->ch_ev[nch - 1] + 1;
    c->pos = newpos;
    c->nchunk = nch;
    B.rr->count = nch;
    c->escalations += nch;
  }
  return nch;
}

// fp64: a chunk that is exactly one certain accept is committed at once; its numpy
// value is replicated from the committed state inside the accept body, overlapped
// with the cache updates (k_res_from_product .. k_g_adopt)
template <typename T>
__device__ bool g_try_direct(DevCtl* c, const GBufs<T>& B, cudaGraphConditionalHandle h_batch,
                             cudaGraphConditionalHandle h_acc, cudaGraphConditionalHandle h_esc) {
  if (c->nchunk != 1 || !c->ch_cert[0]) return false;
  double err0 = c->err;
  double A = B.aval[c->ch_ev[0]];
  cudaGraphSetConditional(h_esc, 0);
  g_accept(c, B, c->ch_ev[0], c->ch_q[0], c->ch_op[0], A, -1, h_batch, h_acc);
  c->direct = 1;
  c->err_prev = err0;
  return true;
}

// after phase B: fp32 takes the first eval below err; fp64 opens an escalation
template <typename T>
__global__ void __launch_bounds__(kDecideThreads)
k_g_decide(DevCtl* c, GBufs<T> B, cudaGraphConditionalHandle h_batch, cudaGraphConditionalHandle h_acc,
           cudaGraphConditionalHandle h_esc) {
  __shared__ int s_bad, s_win;
  int E = c->E;
  if (threadIdx.x == 0) {
    c->evaluated += 2 * (long long)E;
    c->batches++;
    if (c->tb0) {
      unsigned long long now;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      c->phaseB_ns += now - c->tb0;
    }
    s_bad = g_flags_bad(B.bst, B.exact);
    s_win = 1 << 30;
    c->pos = 0;
  }
  __syncthreads();
  if (s_bad) {
    if (threadIdx.x == 0) {
      c->error = 3;
      cudaGraphSetConditional(h_batch, 0);
      if (!B.exact) cudaGraphSetConditional(h_esc, 0);
    }
    return;
  }
  int scan = threadIdx.x;
  double A = 0;
  int cls = scan < 2 * E ? g_class(c, B, scan, true, A) : 0;
  if (B.exact) {
    if (cls == 2) atomicMin(&s_win, scan);
    __syncthreads();
    if (threadIdx.x == 0) {
      if (s_win < (1 << 30)) g_accept(c, B, s_win, s_win >> 1, s_win & 1, B.aval[s_win], -1, h_batch, h_acc);
      else g_advance(c, B.row_depth, h_batch);
    }
    return;
  }
  int nch = g_chunk(c, B, cls, scan);
  if (threadIdx.x == 0) {
    if (nch) {
      if (!g_try_direct(c, B, h_batch, h_acc, h_esc)) cudaGraphSetConditional(h_esc, 1);
    } else {
      cudaGraphSetConditional(h_esc, 0);
      g_advance(c, B.row_depth, h_batch);
    }
  }
}

// fp64, after a replica round: does any slot need the full-sort fallback?
__global__ void k_g_fb_check(DevCtl* c, const double* __restrict__ out, cudaGraphConditionalHandle h_fb) {
  int any = 0;
  for (int s = 0; s < c->nchunk; s++) {
    long long D = reinterpret_cast<const long long*>(out)[2 * s + 1];
    c->fb[s] = D > kDeltaCap;
    any |= c->fb[s];
  }
  cudaGraphSetConditional(h_fb, any);
}

// fallback results: the root of the slot's pairwise tree over the CUB-sorted residuals
__global__ void k_g_fb_fix(const DevCtl* __restrict__ c, double* const* __restrict__ pw, double* out) {
  int s = threadIdx.x;
  if (s < c->nchunk && c->fb[s]) out[2 * s] = pw[s][0];
}

// fp64, after a replica round: the first replicated eval below err wins; otherwise
// scan on (next chunk) or finish the batch
template <typename T>
__global__ void __launch_bounds__(kDecideThreads)
k_g_decide_esc(DevCtl* c, GBufs<T> B, cudaGraphConditionalHandle h_batch, cudaGraphConditionalHandle h_acc,
               cudaGraphConditionalHandle h_esc) {
  __shared__ int s_done;
  if (threadIdx.x == 0) {
    c->esc_rounds++;
    s_done = 0;
    for (int s = 0; s < c->nchunk; s++) {
      double fr = B.out[2 * s];
      if (fr < c->err) {
        cudaGraphSetConditional(h_esc, 0);
        g_accept(c, B, c->ch_ev[s], c->ch_q[s], c->ch_op[s], fr, s, h_batch, h_acc);
        s_done = 1;
        break;
      }
      if (c->ch_cert[s]) {  // the decision bound failed its self-check
        c->error = 1;
        cudaGraphSetConditional(h_esc, 0);
        cudaGraphSetConditional(h_batch, 0);
        s_done = 1;
        break;
      }
    }
  }
  __syncthreads();
  if (s_done) return;
  int scan = threadIdx.x;
  double A = 0;
  int cls = scan < 2 * c->E ? g_class(c, B, scan, false, A) : 0;
  int nch = g_chunk(c, B, cls, scan);
  if (threadIdx.x == 0) {
    if (nch) {
      if (!g_try_direct(c, B, h_batch, h_acc, h_esc)) cudaGraphSetConditional(h_esc, 1);
    } else {
      cudaGraphSetConditional(h_esc, 0);
      g_advance(c, B.row_depth, h_batch);
    }
  }
}

// accept: column k of U and row k of V (and their row-major copies) := the eval's
// vectors; fp64 also adopts the winner's replica residuals as the current state
template <typename T>
__global__ void k_g_commit(DevCtl* c, GBufs<T> B, T* __restrict__ Ut, T* __restrict__ V, T* __restrict__ Urm,
                           T* __restrict__ Vcm, int rp, int64_t N, u64* __restrict__ res_cur, u64* __restrict__ S_cur) {
  int k = c->win_k, op = c->win_op, q = c->win_q;
  int64_t m = B.m, n = B.n;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m + n; t += stride) {
    if (t < m) {
      T a = op == 0 ? B.ubufB[(int64_t)q * m + t] : B.ubufA[ilv_index<T>(q, t, m)];
      Ut[(int64_t)k * m + t] = a;
      Urm[t * rp + k] = a;
    } else {
      int64_t cc = t - m;
      T b = op == 1 ? B.vbufB[(int64_t)q * n + cc] : B.vbuf[ilv_index<T>(q, cc, n)];
      V[(int64_t)k * n + cc] = b;
      Vcm[cc * rp + k] = b;
    }
  }
  int s = c->win_slot;
  if (s >= 0 && res_cur) {
    const u64* rs = B.res[s];
    const u64* ss = B.sorted[s];
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < N; p += stride) {
      res_cur[p] = rs[p];
      S_cur[p] = ss[p];
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    c->cache_k = k;
    c->accepts++;
    if (B.urf_valid) B.urf_valid[k] = 0;  // row k of V changes: its F-URF statistics too
  }
}

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long now;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
  return now;
}

// graph-mode profiling ticks: which = 0 phase-B start, 1 escalation round start,
// 2 escalation round end, 3 accept body start, 4 accept body end, 5 sweep start, 6 sweep end
__global__ void k_g_tick(DevCtl* c, int which) {
  unsigned long long now = gtime();
  switch (which) {
    case 0: c->tb0 = now; break;
    case 1: c->te0 = now; break;
    case 2: c->esc_ns += now - c->te0; break;
    case 3: c->ta0 = now; break;
    case 4: c->acc_ns += now - c->ta0; break;
    case 5: c->sweep_ns = now; break;
    default: c->sweep_ns = now - c->sweep_ns;
  }
}

// direct accept, replica of the committed state: residual bits |x - t1| (t1 = the
// new product, CSR order) into slot 0 with the changed entries appended; count 0
// (no direct accept) makes this and the following replica kernels no-ops
template <typename T>
__global__ void k_res_from_product(const DevCtl* __restrict__ c, int64_t N, const T* __restrict__ xv,
                                   const T* __restrict__ t1, const u64* __restrict__ res_cur,
                                   RepRound<T>* __restrict__ R) {
  if (!c->direct) {
    if (blockIdx.x == 0 && threadIdx.x == 0) R->count = 0;
    return;
  }
  RepSlot<T> S = R->s[0];
  int lane = threadIdx.x & 31;
  for (int64_t b0 = blockIdx.x * (int64_t)blockDim.x; b0 < N; b0 += (int64_t)gridDim.x * blockDim.x) {
    int64_t p = b0 + threadIdx.x;
    bool ch = false;
    u64 nb = 0, ob = 0;
    if (p < N) {
      nb = (u64)__double_as_longlong((double)vabs(sub_rn(xv[p], t1[p])));
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
}

// direct accept with more changed entries than the delta merge takes: full sort
// (IF h_fb1 body: CUB radix sort of slot 0, pairwise tree, k_g_fb1_fix)
__global__ void k_g_fb1_check(const DevCtl* __restrict__ c, const double* __restrict__ out,
                              cudaGraphConditionalHandle h_fb1) {
  int fb = c->direct && reinterpret_cast<const long long*>(out)[1] > c->direct_cap;
  cudaGraphSetConditional(h_fb1, fb);
}
__global__ void k_g_fb1_fix(const double* __restrict__ pw0, double* out) {
  out[0] = pw0[0];
  reinterpret_cast<long long*>(out)[1] = 0;
}

// direct accept: the replica's value becomes err (self-check: below the previous err)
// and its arrays the current state
template <typename T>
__global__ void k_g_adopt(DevCtl* c, GBufs<T> B, int64_t N, u64* __restrict__ res_cur, u64* __restrict__ S_cur) {
  if (!c->direct) return;
  const u64* rs = B.res[0];
  const u64* ss = B.sorted[0];
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < N; p += (int64_t)gridDim.x * blockDim.x) {
    res_cur[p] = rs[p];
    S_cur[p] = ss[p];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    double fr = B.out[0];
    if (!(fr < c->err_prev)) c->error = 1;  // the decision bound failed its self-check
    c->err = fr;
    if (c->traj_len > 0) B.traj_e[c->traj_len - 1] = fr;
  }
}

__global__ void k_g_row_end(DevCtl* c, const u64* __restrict__ bst, int exact, int64_t m,
                            cudaGraphConditionalHandle h_row) {
  if (g_flags_bad(bst, exact)) c->error = 3;
  c->i++;
  if (c->deadline_ns) {
    unsigned long long now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    if (now >= c->deadline_ns) c->stop = 1;
  }
  cudaGraphSetConditional(h_row, (c->i < m && !c->error && !c->stop) ? 1 : 0);
}

}  // namespace stmf
