// stmf_api.cu — session management, the ByRow/TD_A sweep driver and the C ABI
// (include/stmf_b200.h) of the B200-native FastSTMF fitting engine.
//
// Driver structure of one row visit (strategies.py:191-224), all on the session
// stream; the host only reads back the per-batch decision data:
//   1. product caches (U(x)V, argmax, second best) + column scores + TD_A column
//      histograms, recomputed only after an acceptance (state unchanged otherwise);
//      residuation statistics of the factor index that changed;
//   2. candidate order: stable radix sort of the row's given columns by score;
//   3. speculative batches of candidates from the SAME state (rejected attempts
//      revert bit-exactly, engine.py:131-133): phase A (first residuation from
//      top-2 statistics, O(m+n) per eval), phase B (second residuation + error,
//      one pass over the given entries per group of evals); the first eval in
//      reference order with f < err wins (FitRun._attempt, engine.py:283);
//   4. commit: column k of U, row k of V.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cudaTypedefs.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "stmf_b200.h"
#include "stmf_kernels.cuh"
#include "stmf_strategies.cuh"
#include "stmf_metrics.cuh"
#include "stmf_graph.cuh"
#include "stmf_fast1.cuh"

using namespace stmf;

// ----------------------------------------------------------------------------
// errors
static thread_local std::string g_err;

static int set_err(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

// error reporting for the host-only sources (stmf_io.cc)
int stmf_io_set_error(int code, const char* msg) { return set_err(code, "%s", msg); }

struct StmfError {
  int code;
};

#define CK(call)                                                                             \
  do {                                                                                       \
    cudaError_t e_ = (call);                                                                 \
    if (e_ != cudaSuccess) {                                                                 \
      set_err(e_ == cudaErrorMemoryAllocation ? STMF_ERR_OOM : STMF_ERR_CUDA, "%s:%d %s: %s", \
              __FILE__, __LINE__, #call, cudaGetErrorString(e_));                            \
      throw StmfError{e_ == cudaErrorMemoryAllocation ? STMF_ERR_OOM : STMF_ERR_CUDA};       \
    }                                                                                        \
  } while (0)

#include <atomic>
// every kernel launch of this library is followed by LAUNCH_CK(): it also counts them
static std::atomic<long long> g_launches{0};
static std::atomic<long long> g_cub_calls{0};
#define LAUNCH_CK()            \
  do {                         \
    g_launches++;              \
    CK(cudaGetLastError());    \
  } while (0)

[[noreturn]] static void fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  throw StmfError{code};
}

// ----------------------------------------------------------------------------
// host helpers

// value = (hi:lo) * 2^-F rounded to nearest even binary64
static double fx_to_double(u64 hi, u64 lo, int F) {
  if (hi == 0) return std::ldexp((double)lo, -F);  // u64 -> double is RN on x86-64
  int top = 64 + 63 - __builtin_clzll(hi);
  int sh = top - 52;  // >= 12
  auto bit = [&](int p) -> u64 { return p >= 64 ? (hi >> (p - 64)) & 1u : (lo >> p) & 1u; };
  u64 q;
  if (sh >= 64) q = hi >> (sh - 64);
  else q = (hi << (64 - sh)) | (lo >> sh);
  q &= (1ull << 53) - 1;
  q |= (1ull << 52);
  int guard = (int)bit(sh - 1);
  bool sticky = false;
  for (int p = sh - 2; p >= 0 && !sticky; p--) sticky = bit(p) != 0;
  if (guard && (sticky || (q & 1u))) q++;
  return std::ldexp((double)q, sh - F);
}

// finest binary grid 2^-g of a binary32 value (lowest set bit of its exact value)
static int f32_grid(float x) {
  uint32_t b;
  memcpy(&b, &x, 4);
  b &= 0x7fffffffu;
  if (b == 0) return -1000;
  uint32_t e = b >> 23, frac = b & 0x7fffffu;
  uint32_t mant = e ? (frac | 0x800000u) : frac;
  int ex = e ? (int)e - 150 : -149;  // value = mant * 2^ex
  return -(ex + __builtin_ctz(mant));
}

// finest grid over the given entries of a dense array: branch-free per element, a few host
// threads for large inputs (the scalar masked loop was ~0.1 s per fit at config 3)
template <typename T>
static int f32_grid_given(const T* X, const uint8_t* mask, int64_t len) {
  unsigned nt = len < (1 << 22) ? 1u : std::min(8u, std::max(1u, std::thread::hardware_concurrency()));
  std::vector<int> part(nt, -1000);
  auto work = [&](unsigned t) {
    int g = -1000;
    for (int64_t a = len * t / nt, hi = len * (t + 1) / nt; a < hi; a++) {
      int v = f32_grid((float)X[a]);  // bit arithmetic only: NaN payloads under the mask are harmless
      g = std::max(g, mask[a] ? v : -1000);
    }
    part[t] = g;
  };
  std::vector<std::thread> th;
  for (unsigned t = 1; t < nt; t++) th.emplace_back(work, t);
  work(0);
  for (auto& x : th) x.join();
  return *std::max_element(part.begin(), part.end());
}

static inline unsigned nblk(int64_t work, int per) { return (unsigned)((work + per - 1) / per); }

static double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// numpy pairwise-summation tree of a length-N array (structure depends on N only)
struct PWTree {
  std::vector<int64_t> loff;
  std::vector<int32_t> llen, lnode, left, right, lvl_off, lvl_nodes;
  int nnodes = 0, H = 0;
  void build(int64_t N) {
    loff.clear(); llen.clear(); lnode.clear(); left.clear(); right.clear();
    lvl_off.clear(); lvl_nodes.clear();
    std::vector<int> height;
    std::vector<int64_t> noff, nlen;
    // iterative DFS
    struct Fr { int64_t off, n; int id; int stage; };
    auto newnode = [&](int64_t off, int64_t n) {
      noff.push_back(off); nlen.push_back(n); left.push_back(-1); right.push_back(-1); height.push_back(0);
      return (int)noff.size() - 1;
    };
    std::vector<Fr> st;
    int root = newnode(0, N);
    st.push_back({0, N, root, 0});
    while (!st.empty()) {
      Fr& f = st.back();
      if (f.n <= 128) {
        loff.push_back(f.off); llen.push_back((int32_t)f.n); lnode.push_back(f.id);
        st.pop_back();
        continue;
      }
      int64_t n2 = f.n / 2;
      n2 -= n2 % 8;
      if (f.stage == 0) {
        f.stage = 1;
        int l = newnode(f.off, n2);
        left[f.id] = l;
        Fr c{f.off, n2, l, 0};
        st.push_back(c);
      } else if (f.stage == 1) {
        f.stage = 2;
        int r = newnode(f.off + n2, f.n - n2);
        right[f.id] = r;
        Fr c{f.off + n2, f.n - n2, r, 0};
        st.push_back(c);
      } else {
        height[f.id] = 1 + std::max(height[left[f.id]], height[right[f.id]]);
        st.pop_back();
      }
    }
    nnodes = (int)noff.size();
    H = height[root];
    lvl_off.assign(H + 1, 0);
    std::vector<std::vector<int32_t>> lv(H + 1);
    for (int i = 0; i < nnodes; i++)
      if (height[i] > 0) lv[height[i]].push_back(i);
    lvl_off[0] = 0;
    for (int h = 1; h <= H; h++) {
      lvl_off[h] = lvl_off[h - 1] + (int)lv[h].size();
      for (int x : lv[h]) lvl_nodes.push_back(x);
    }
    // lvl_off[h-1]..lvl_off[h] are the nodes of height h; shift to 0-based list
  }
};

// ----------------------------------------------------------------------------
struct SessionBase {
  virtual ~SessionBase() {}
  int dtype = 0;
  virtual int device_id() const = 0;
  virtual void info(int64_t* out) = 0;
  virtual void set_factors(const void* U, const void* V) = 0;
  virtual void get_factors(void* U, void* V) = 0;
  virtual double objective() = 0;
  virtual void run(int64_t budget_sweeps, double budget_seconds, double epsilon, double* tt, double* te,
                   int64_t cap, int64_t* counts) = 0;
  virtual void product_given(void* P, int32_t* arg, void* top2) = 0;
  virtual void col_scores(double* out) = 0;
  virtual void residuate(int axis, const void* vec, void* out) = 0;
  virtual void try_update(int op, int64_t i, int64_t j, int k, void* ucol, void* vrow, double* f,
                          bool commit, int* accepted) = 0;
  virtual void bench_product(int reps, int flush, double* ms, double* err) = 0;
  virtual void* stream() = 0;
  virtual void set_profiling(int on) = 0;
  virtual void counters(int64_t* out) = 0;
  virtual int64_t replayed_sweeps() { return 0; }
  // test hook mirroring oracle.fit(max_attempts=...): stop after that many attempts
  virtual void set_max_attempts(int64_t) { fail(STMF_ERR_INVALID, "attempt caps are single-device only"); }
  virtual void set_audit(int) { fail(STMF_ERR_INVALID, "audit mode is single-device only"); }
  // sharded sessions: {ranks, this rank, kind (0 in-process group, 1 NCCL)} from the communicator
  virtual void comm_info(int* out3) { out3[0] = 1; out3[1] = 0; out3[2] = -1; }
  // the reference's other fit methods
  virtual void set_strategy(int family, int selection) {
    if (family != STMF_FAMILY_BYROW || selection != STMF_SEL_TD_A)
      fail(STMF_ERR_INVALID, "sharded sessions run FastSTMF (ByRow / TD_A) only");
  }
  virtual void row_scores(double*) { fail(STMF_ERR_INVALID, "not available on sharded sessions"); }
  virtual void trajectory(double*, double*, int64_t, int64_t*) {
    fail(STMF_ERR_INVALID, "sharded sessions write the trajectory to the caller's buffers");
  }
  virtual void matrix_candidates(int32_t*, int32_t*, int32_t*, double*) {
    fail(STMF_ERR_INVALID, "not available on sharded sessions");
  }
};

// Device buffers come from the device's stream-ordered memory pool, which keeps freed
// memory mapped (release threshold = max): creating and destroying a session then
// costs pool bookkeeping instead of ~140 cudaMalloc / cudaFree calls, whose page
// mapping work measured 15-1000 ms per fit on the GPU box (tools/diag_e2e_parts.py).
// Allocation is ordered on the legacy stream and completed before use; a free first
// waits for the device (no kernel can still be using the buffer), then returns the
// block to the pool.
static void pool_setup(int dev) {
  static bool done[64] = {false};
  if (dev < 0 || dev >= 64 || done[dev]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done[dev] = true;
}

static void* dev_alloc(size_t bytes) {
  int dev = 0;
  CK(cudaGetDevice(&dev));
  pool_setup(dev);
  void* p = nullptr;
  CK(cudaMallocAsync(&p, bytes, 0));
  CK(cudaStreamSynchronize(0));
  return p;
}

static void dev_free(void* p, int dev) {
  int cur = 0;
  cudaGetDevice(&cur);
  if (cur != dev) cudaSetDevice(dev);
  cudaDeviceSynchronize();
  cudaFreeAsync(p, 0);
  if (cur != dev) cudaSetDevice(cur);
}

// Pinned host staging buffers (per-batch decision data, control blocks) are cached
// process-wide by size: page-locking is a slow driver call, and a fit's session
// needs a handful of small ones.
static std::mutex g_pin_mu;
static std::multimap<size_t, void*> g_pin_free;
template <typename P>
static void pinned_alloc(P** out, size_t bytes) {
  {
    std::lock_guard<std::mutex> lk(g_pin_mu);
    auto it = g_pin_free.find(bytes);
    if (it != g_pin_free.end()) {
      *out = static_cast<P*>(it->second);
      g_pin_free.erase(it);
      return;
    }
  }
  void* p = nullptr;
  CK(cudaMallocHost(&p, bytes));
  *out = static_cast<P*>(p);
}
static void pinned_free(void* p, size_t bytes) {
  if (!p) return;
  std::lock_guard<std::mutex> lk(g_pin_mu);
  g_pin_free.emplace(bytes, p);
}

template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  bool own = true;
  int dev = 0;
  void release() {
    if (p && own) dev_free(p, dev);
    p = nullptr;
  }
  void alloc(size_t cnt) {
    release();
    own = true;
    n = cnt;
    if (cnt) {
      CK(cudaGetDevice(&dev));
      p = static_cast<T*>(dev_alloc(cnt * sizeof(T)));
    }
  }
  // a non-owning view into another allocation
  void view(T* ptr, size_t cnt) {
    release();
    p = ptr;
    n = cnt;
    own = false;
  }
  ~DevBuf() { release(); }
};

template <typename T>
struct Session : SessionBase {
  static constexpr bool kExact = sizeof(T) == 4;  // binary32: exact-sum semantics
  int dev = 0;
  cudaStream_t st = nullptr;
  int64_t m = 0, n = 0, N = 0;
  int rank = 0;
  int nsm = 148;
  // layout
  DevBuf<int64_t> row_ptr, col_ptr;
  DevBuf<int32_t> col_idx, row_idx;
  DevBuf<T> xr, xc;
  std::vector<int64_t> h_row_ptr, h_col_ptr;
  int64_t max_rownnz = 0, max_colnnz = 0;
  // factors
  DevBuf<T> Ut, V;
  bool have_factors = false;
  // product caches
  DevBuf<T> t1r, t2r, t1c, t2c;
  DevBuf<uint8_t> agr, agc, a2r, a2c;
  int cache_k = -1;  // >= 0: the caches are valid except for factor index cache_k
  // row-major copies for the product passes: Urm (m x rp), Vcm (n x rp), rp = rank
  // padded to 16 bytes, so an entry's factor rows are contiguous vector loads
  DevBuf<T> Urm, Vcm;
  DevBuf<int32_t> rowof_r, colof_c;  // row of each CSR entry, column of each CSC entry
  // lines longer than long_thr entries are evaluated block-per-line (k_phaseB_long)
  int64_t long_thr = 4096;
  // phase-B item order: group-major when both orders' entry data fit comfortably in L2
  int group_major = 0;
  DevBuf<int32_t> long_rows, long_cols;
  int n_long_rows = 0, n_long_cols = 0;
  void build_long_lists() {
    if (const char* e = getenv("STMF_LONG")) long_thr = atoll(e);
    std::vector<int32_t> lr, lc;
    for (int64_t i = 0; i < m; i++)
      if (h_row_ptr[i + 1] - h_row_ptr[i] > long_thr) lr.push_back((int32_t)i);
    for (int64_t j = 0; j < n; j++)
      if (h_col_ptr[j + 1] - h_col_ptr[j] > long_thr) lc.push_back((int32_t)j);
    n_long_rows = (int)lr.size();
    n_long_cols = (int)lc.size();
    upload(long_rows, lr);
    upload(long_cols, lc);
  }
  int rp = 0;
  void sync_factor_copies(int k) {  // k < 0: all
    for (int l = (k < 0 ? 0 : k); l < (k < 0 ? rank : k + 1); l++) {
      k_scatter_factor<T><<<nblk(m, 256), 256, 0, st>>>(m, rp, l, Ut.p + (size_t)l * m, Urm.p);
      LAUNCH_CK();
      k_scatter_factor<T><<<nblk(n, 256), 256, 0, st>>>(n, rp, l, V.p + (size_t)l * n, Vcm.p);
      LAUNCH_CK();
    }
  }
  DevBuf<double> score;
  DevBuf<int32_t> colhist;
  // residuation statistics
  DevBuf<T> cm1, cm2, rm1, rm2;
  DevBuf<int32_t> cmarg, rmarg;
  // candidates
  DevBuf<u64> ckeys, ckeys2;
  DevBuf<int32_t> cvals, cperm, cj, ck;
  DevBuf<T> cx, xrow_dense;
  DevBuf<T> cmi, sq;  // CM^(-i) per k for the visited row; s_q of the batch's F-ULF evals
  bool inline_ulf = getenv("STMF_INLINE") ? atoi(getenv("STMF_INLINE")) != 0 : true;
  // phase A applies the F-URF seed itself (binary search per (eval, row)) for small m
  bool fuse_seed = false;
  DevBuf<SeedCols<T>> d_seedcols;
  // F-ULF hit partition of the visited row (k_hit_partition; needs the inline values)
  bool split_ulf = inline_ulf && (getenv("STMF_SPLIT") ? atoi(getenv("STMF_SPLIT")) != 0 : false);
  DevBuf<int32_t> hp_idx, hp_split;
  DevBuf<T> hp_x, hp_t1, hp_t2;
  DevBuf<uint8_t> hp_ag;
  void row_partition() {
    if (!split_ulf) return;
    k_hit_partition<T><<<warps_grid(m), 256, 0, st>>>(m, row_ptr.p, col_idx.p, xr.p, t1r.p, t2r.p, agr.p,
                                                      xrow_dense.p, hp_idx.p, hp_x.p, hp_t1.p, hp_t2.p, hp_ag.p,
                                                      hp_split.p);
    LAUNCH_CK();
  }
  // the F-ULF side of phase B (CSR rows), on the hit-partitioned copy when enabled
  SideB<T> side_ulf(u64* acc_p, int* chg_p) {
    SideB<T> sa{m, row_ptr.p, col_idx.p, xr.p, t1r.p, t2r.p, agr.p, vbuf.p, n, Ut.p, ubufB.p, acc_p, chg_p,
                0, long_thr, group_major};
    if (inline_ulf) {
      sa.inl_base = cmi.p;
      sa.inl_xr = xrow_dense.p;
      sa.inl_s = sq.p;
    }
    if (split_ulf) {
      sa.idx = hp_idx.p; sa.xv = hp_x.p; sa.t1 = hp_t1.p; sa.t2 = hp_t2.p; sa.ag = hp_ag.p;
      sa.split = hp_split.p;
    }
    return sa;
  }
  // phase B's first half from per-line statistics (stmf_fast1.cuh); STMF_FAST1=0: full passes
  // off by default: measured slower at configs 2 and 3 (profiles/r02_fast1.md: the walks fall
  // back to the full pass for 22-30% of (eval, line) pairs at config 3's density)
  bool fast1 = getenv("STMF_FAST1") ? atoi(getenv("STMF_FAST1")) != 0 : false;
  DevBuf<T> f1_uv, f1_ux, f1_rv, f1_rx;
  DevBuf<int32_t> f1_uo, f1_ro;
  DevBuf<int> f1_k, f1_valid;  // F-ULF statistics' k; F-URF per-k validity
  bool f1_row_ready = false;   // host loop: the F-ULF statistics belong to the current row visit
  DevBuf<unsigned long long> f1_diag;  // STMF_FAST1_STATS: walk / fallback counts (stderr at the end of run)
  Fast1<T> fast1_bufs(const int32_t* cjp) {
    Fast1<T> F1{};
    F1.stats = f1_diag.p;  // allocated at init under STMF_FAST1_STATS
    F1.ulf = TopK<T>{f1_uv.p, f1_uo.p, f1_ux.p};
    F1.ulf_k = f1_k.p;
    F1.urf = TopK<T>{f1_rv.p, f1_ro.p, f1_rx.p};
    F1.urf_valid = f1_valid.p;
    F1.rm1 = rm1.p;
    F1.rmarg = rmarg.p;
    F1.cj = cjp;
    return F1;
  }
  // the line statistics of a row visit: F-ULF w.r.t. CM^(-i)_k and (if stale) F-URF
  // w.r.t. RM_k, k = the factor index of the row's first candidate (ck[0])
  void fast1_row_stats(cudaStream_t s_) {
    k_top_lines<T><<<warps_grid(m), 256, 0, s_>>>(m, row_ptr.p, col_idx.p, xr.p, cmi.p, n, ck.p, nullptr,
                                                   TopK<T>{f1_uv.p, f1_uo.p, f1_ux.p}, 0);
    k_top_mark<<<1, 1, 0, s_>>>(ck.p, nullptr, f1_k.p);
    k_top_lines<T><<<warps_grid(n), 256, 0, s_>>>(n, col_ptr.p, row_idx.p, xc.p, rm1.p, m, ck.p, f1_valid.p,
                                                   TopK<T>{f1_rv.p, f1_ro.p, f1_rx.p}, (int64_t)kTop * n);
    k_top_mark<<<1, 1, 0, s_>>>(ck.p, f1_valid.p, nullptr);
  }
  // diagnostics (STMF_FAST1_CHECK): the statistics walk's line values against full passes
  void fast1_check(SideB<T> sa, SideB<T> sb, int E, const int32_t* bk, const int32_t* bj, int64_t i) {
    DevBuf<T> oa, ob;
    DevBuf<int> zero;
    oa.alloc((size_t)E * m); ob.alloc((size_t)E * n); zero.alloc(rank + 1);
    CK(cudaMemsetAsync(zero.p, 0, sizeof(int) * rank, st));
    int neg = -2;
    CK(cudaMemcpyAsync(zero.p + rank, &neg, sizeof(int), cudaMemcpyHostToDevice, st));
    SideB<T> a2 = sa, b2 = sb;
    a2.out = oa.p; b2.out = ob.p;
    Fast1<T> F1 = fast1_bufs(bj);
    F1.ulf_k = zero.p + rank;
    F1.urf_valid = zero.p;
    int ng = (E + kEG - 1) / kEG;
    k_pass1_fast<T><<<warps_grid((m + n) * ng), 256, 0, st>>>(a2, b2, E, bk, F1);
    LAUNCH_CK();
    std::vector<T> fa((size_t)E * m), fb((size_t)E * n), ga((size_t)E * m), gb((size_t)E * n);
    CK(cudaMemcpyAsync(fa.data(), sa.out, sizeof(T) * fa.size(), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(fb.data(), sb.out, sizeof(T) * fb.size(), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(ga.data(), oa.p, sizeof(T) * ga.size(), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(gb.data(), ob.p, sizeof(T) * gb.size(), cudaMemcpyDeviceToHost, st));
    int hk = -1;
    CK(cudaMemcpyAsync(&hk, f1_k.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    std::vector<int> hv(rank), hks(E);
    CK(cudaMemcpyAsync(hv.data(), f1_valid.p, sizeof(int) * rank, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hks.data(), bk, sizeof(int) * E, cudaMemcpyDeviceToHost, st));
    ssync();
    int bad = 0;
    for (size_t t = 0; t < fa.size(); t++)
      if (!(fa[t] == ga[t]) && bad++ < 5)
        fprintf(stderr, "[fast1 check] row %lld ULF eval %zu line %zu k %d (ulf_k %d): fast %.17g full %.17g\n",
                (long long)i, t / m, t % m, hks[t / m], hk, (double)fa[t], (double)ga[t]);
    for (size_t t = 0; t < fb.size(); t++)
      if (!(fb[t] == gb[t]) && bad++ < 10)
        fprintf(stderr, "[fast1 check] row %lld URF eval %zu line %zu k %d (valid %d): fast %.17g full %.17g\n",
                (long long)i, t / n, t % n, hks[t / n], hv[hks[t / n]], (double)fb[t], (double)gb[t]);
    if (bad) fprintf(stderr, "[fast1 check] row %lld: %d mismatches\n", (long long)i, bad);
    // details of the first ULF mismatch: the row's entries, the base, the statistics
    for (size_t t = 0; t < fa.size(); t++) {
      if (fa[t] == ga[t]) continue;
      int q = (int)(t / m);
      int64_t L = (int64_t)(t % m);
      int k = hks[q];
      int64_t b0 = h_row_ptr[L], b1 = h_row_ptr[L + 1];
      std::vector<int32_t> cols(b1 - b0);
      std::vector<T> xs(b1 - b0), base(n), xrd(n), st4v(kTop * m), st4x(kTop * m);
      std::vector<int32_t> st4o(kTop * m);
      T sqv;
      CK(cudaMemcpyAsync(cols.data(), col_idx.p + b0, 4 * cols.size(), cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(xs.data(), xr.p + b0, sizeof(T) * xs.size(), cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(base.data(), cmi.p + (size_t)k * n, sizeof(T) * n, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(xrd.data(), xrow_dense.p, sizeof(T) * n, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(st4v.data(), f1_uv.p, sizeof(T) * st4v.size(), cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(st4x.data(), f1_ux.p, sizeof(T) * st4x.size(), cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(st4o.data(), f1_uo.p, 4 * st4o.size(), cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(&sqv, sq.p + q, sizeof(T), cudaMemcpyDeviceToHost, st));
      ssync();
      T best = INFINITY;
      size_t bp = 0;
      std::vector<std::pair<T, int>> bt;
      for (size_t e = 0; e < cols.size(); e++) {
        int c = cols[e];
        T b = base[c];
        T vn = std::min(b, (T)(xrd[c] - sqv));
        T term = xs[e] - vn;
        if (term < best) { best = term; bp = e; }
        bt.push_back({(T)(xs[e] - b), c});
      }
      std::sort(bt.begin(), bt.end());
      fprintf(stderr, "[fast1 detail] line %lld eval %d k %d: host full min %.17g at col %d (x %.17g b %.17g xr %.17g)\n",
              (long long)L, q, k, (double)best, cols[bp], (double)xs[bp], (double)base[cols[bp]], (double)xrd[cols[bp]]);
      for (int u = 0; u < 4 && u < (int)bt.size(); u++)
        fprintf(stderr, "  host top %d: val %.17g col %d | dev slot %d: val %.17g col %d x %.17g\n", u,
                (double)bt[u].first, bt[u].second, u, (double)st4v[u * m + L], st4o[u * m + L], (double)st4x[u * m + L]);
      break;
    }
  }
  void fast1_invalidate(int k) {  // k < 0: every k
    if (!fast1) return;
    if (k < 0) CK(cudaMemsetAsync(f1_valid.p, 0, sizeof(int) * rank, st));
    else CK(cudaMemsetAsync(f1_valid.p + k, 0, sizeof(int), st));
  }
  // batch scratch
  int Emax = 512;
  DevBuf<T> vbuf, ubufB, ubufA, vbufB, dtmpA, dtmpB;
  DevBuf<u64> acc;
  DevBuf<int> chg, flags, findpos;
  u64* h_acc = nullptr;
  int* h_chg = nullptr;
  DevBuf<u64> bstate;
  u64* h_bstate = nullptr;
  int* h_flags = nullptr;
  // replica
  DevBuf<u64> res_cur, S_cur;
  bool cur_valid = false;
  int64_t n_delta_replicas = 0, n_zero_delta = 0;
  int unroll = sizeof(T) == 4 ? 2 : 1;  // phase-B pass-2 entries per lane per iteration (STMF_UNROLL)
  DevBuf<double> pwval;
  DevBuf<int64_t> pw_loff;
  DevBuf<int32_t> pw_llen, pw_lnode, pw_left, pw_right, pw_lvloff, pw_lvlnodes;
  DevBuf<int4> pw_ops;  // internal nodes in level order: {node, left, right, 0}
  PWTree pw;
  DevBuf<uint8_t> cubtmp;
  size_t cubtmp_bytes = 0;
  // numerics
  int F = 60;
  double exact_limit = INFINITY;
  double beta_rel = 0;
  // state
  bool dirty = true;
  std::vector<char> stats_dirty;
  bool err_valid = false;
  double err = 0;
  int64_t n_product_passes = 0, n_escalations = 0;
  bool profiling = false;
  cudaEvent_t ev_b0 = nullptr, ev_b1 = nullptr;
  long long phaseB_launches = 0, phaseB_ns = 0, phaseB_timed = 0;

  void* stream() override { return (void*)st; }
  int device_id() const override { return dev; }
  void set_profiling(int on) override {
    if (on && !ev_b0) {
      CK(cudaEventCreate(&ev_b0));
      CK(cudaEventCreate(&ev_b1));
    }
    profiling = on != 0;
  }
  void counters(int64_t* out) override {
    out[0] = g_launches.load(); out[1] = g_cub_calls.load(); out[2] = phaseB_launches;
    out[3] = phaseB_ns; out[4] = phaseB_timed; out[5] = n_product_passes; out[6] = n_escalations;
    out[7] = n_zero_delta;
  }
  std::vector<int> batch_sched;

  ~Session() override {
    graph_destroy();
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (st2) cudaStreamDestroy(st2);
    if (ev_aux0) cudaEventDestroy(ev_aux0);
    if (ev_aux1) cudaEventDestroy(ev_aux1);
    if (st_aux) cudaStreamDestroy(st_aux);
    if (ev_fork3) cudaEventDestroy(ev_fork3);
    if (ev_join3) cudaEventDestroy(ev_join3);
    if (st3) cudaStreamDestroy(st3);
    pinned_free(h_ctl, sizeof(DevCtl));
    if (ev_b0) cudaEventDestroy(ev_b0);
    if (ev_b1) cudaEventDestroy(ev_b1);
    pinned_free(h_bstate, sizeof(u64) * bstate.n);
    pinned_free(h_dcount, sizeof(int) * kSlots);
    pinned_free(h_out, sizeof(double) * 2 * kSlots);
    pinned_free(h_pwv, sizeof(double) * kSlots);
    pinned_free(h_flags, sizeof(int) * 4);
    if (st) cudaStreamDestroy(st);
  }

  void info(int64_t* out) override {
    out[0] = m; out[1] = n; out[2] = rank; out[3] = N; out[4] = dtype;
  }

  void init(int64_t m_, int64_t n_, int rank_, const T* X, const uint8_t* mask, int device) {
    m = m_; n = n_; rank = rank_;
    dev = device;
    CK(cudaSetDevice(dev));
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    // the auxiliary stream of ensure_caches, created here on the session's device
    CK(cudaStreamCreateWithFlags(&st_aux, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&ev_aux0, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ev_aux1, cudaEventDisableTiming));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, dev));
    nsm = prop.multiProcessorCount;
    if (const char* e = getenv("STMF_EMAX")) Emax = std::max(8, atoi(e));
    if (const char* e = getenv("STMF_UNROLL")) unroll = atoi(e);
    read_sched_env();
    Emax = (Emax + kEG - 1) / kEG * kEG;
    batch_sched.clear();  // filled once N is known (see below)
    if (const char* e = getenv("STMF_BATCH")) {
      batch_sched.clear();
      const char* p = e;
      while (*p) { batch_sched.push_back(std::max(1, atoi(p))); while (*p && *p != ',') p++; if (*p) p++; }
    }
    // upload dense X + mask, build CSR/CSC, free the dense copies
    DevBuf<T> dX;
    DevBuf<uint8_t> dM;
    dX.alloc((size_t)(m * n));
    dM.alloc((size_t)(m * n));
    CK(cudaMemcpyAsync(dX.p, X, sizeof(T) * m * n, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(dM.p, mask, (size_t)(m * n), cudaMemcpyHostToDevice, st));
    DevBuf<int64_t> rc, cc;
    rc.alloc(m); cc.alloc(n);
    row_ptr.alloc(m + 1); col_ptr.alloc(n + 1);
    k_count_rows<<<nblk(m * 32, 256), 256, 0, st>>>(m, n, dM.p, rc.p); LAUNCH_CK();
    k_count_cols<<<nblk(n, 256), 256, 0, st>>>(m, n, dM.p, cc.p); LAUNCH_CK();
    k_scan_ptr<<<1, 1024, 0, st>>>(m, rc.p, row_ptr.p); LAUNCH_CK();
    k_scan_ptr<<<1, 1024, 0, st>>>(n, cc.p, col_ptr.p); LAUNCH_CK();
    h_row_ptr.resize(m + 1); h_col_ptr.resize(n + 1);
    CK(cudaMemcpyAsync(h_row_ptr.data(), row_ptr.p, sizeof(int64_t) * (m + 1), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(h_col_ptr.data(), col_ptr.p, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToHost, st));
    ssync();
    N = h_row_ptr[m];
    if (N == 0) fail(STMF_ERR_INVALID, "empty matrix");
    if (N >= (1ll << 31)) fail(STMF_ERR_INVALID, "more than 2^31 - 1 given entries per device");
    for (int64_t i = 0; i < m; i++) {
      int64_t c = h_row_ptr[i + 1] - h_row_ptr[i];
      if (c == 0) fail(STMF_ERR_INVALID, "row %lld has no given entries", (long long)i);
      max_rownnz = std::max(max_rownnz, c);
    }
    for (int64_t j = 0; j < n; j++) {
      int64_t c = h_col_ptr[j + 1] - h_col_ptr[j];
      if (c == 0) fail(STMF_ERR_INVALID, "column %lld has no given entries", (long long)j);
      max_colnnz = std::max(max_colnnz, c);
    }
    fixed_sched = !batch_sched.empty();
    // floor of a speculative batch (candidates): the fixed per-batch cost (~40 us of
    // launches + one host sync) ~ the cost of evaluating 8e6/N candidates
    batch_floor = (int)std::max<int64_t>(1, std::min<int64_t>(128, 8000000 / std::max<int64_t>(N, 1)));
    if (const char* e = getenv("STMF_FLOOR")) batch_floor = std::max(1, atoi(e));
    if (batch_sched.empty()) {
      // first visit of a row: no depth history yet
      int b0 = (int)std::max<int64_t>(4, std::min<int64_t>(128, 120000000 / std::max<int64_t>(N, 1)));
      if (const char* e = getenv("STMF_B0")) b0 = std::max(1, atoi(e));
      for (int b = b0; b < Emax; b *= 4) batch_sched.push_back(b);
      batch_sched.push_back(Emax);
    }
    for (int& b : batch_sched) b = std::max(1, std::min(b, Emax));
    row_depth.assign(m, 0);
    // measured (profiles/r01_sched.md): launch-bound small problems prefer generous
    // batches, evaluation-bound large ones tight batches with slow growth
    // (config 4, N ~ 1e8: faster batch growth, +5% row visits/s in sweep 1; config 3,
    // N ~ 1e7: growth 1.5 is 3-6% faster per sweep; profiles/r01_sched.md)
    if (batch_floor >= 8) { sched_scale = 1.5; sched_add = 4; sched_growth = 2.0; }
    // (late round 2: batches are whole eval groups now (round_batch), the rounding itself supplies
    // growth, and the tuned factor drops to 1.15 at both sizes: config 3 sweep 2 6 827 -> 6 610 ms,
    // config 4 row visits/s +12% over growth 2.0; profiles/r02_ab11_sched.log.  The first batch of a
    // row with history covers 0.25x its previous depth, not 0.9x: in sweeps 2-5 of config 3 the depth
    // of a row is too weakly correlated across sweeps for a large first batch to pay (59.3 -> 53.0 s
    // for sweeps 1-5, profiles/r02_ab12_hist_scale.log), while exhausted rows (late sweeps) still
    // finish in ~4 batches.  Before that:)
    // (round 2, config 3: growth 1.3 instead of 1.5 is 8% faster on a sweep without depth
    // history and 3-7% on sweeps 1-3 of a fit; profiles/r02_sched_c3.log)
    else { sched_scale = 0.25; sched_add = 1; sched_growth = 1.15; }
    read_sched_env();
    col_idx.alloc(N); row_idx.alloc(N); xr.alloc(N); xc.alloc(N);
    k_fill_csr<T><<<nblk(m * 32, 256), 256, 0, st>>>(m, n, dX.p, dM.p, row_ptr.p, col_idx.p, xr.p); LAUNCH_CK();
    k_fill_csc<T><<<nblk(n, 128), 128, 0, st>>>(m, n, dX.p, dM.p, col_ptr.p, row_idx.p, xc.p); LAUNCH_CK();
    build_long_lists();
    {
      // x, idx, t1, t2, ag per entry in each order
      double entry_bytes = 2.0 * (double)N * (3 * sizeof(T) + 4 + 1);
      group_major = entry_bytes < 0.5 * (double)prop.l2CacheSize ? 1 : 0;
      if (const char* e = getenv("STMF_GROUP_MAJOR")) group_major = atoi(e);
      // shared-memory carveout: phase B prefers L1 (0); STMF_CARVEOUT=c applies c to every
      // kernel of a sweep instead (one L1/shared split: no reconfiguration between kernels)
      int cv = getenv("STMF_CARVEOUT") ? atoi(getenv("STMF_CARVEOUT")) : -2;
      int cvb = cv == -2 ? 0 : cv;
      if (cvb >= -1) {
        CK(cudaFuncSetAttribute(k_phaseB<T, 1>, cudaFuncAttributePreferredSharedMemoryCarveout, cvb));
        CK(cudaFuncSetAttribute(k_phaseB<T, 2>, cudaFuncAttributePreferredSharedMemoryCarveout, cvb));
        CK(cudaFuncSetAttribute(k_phaseB<T, 4>, cudaFuncAttributePreferredSharedMemoryCarveout, cvb));
      }
      if (cv >= -1) {
        const void* ks[] = {(const void*)k_phaseA<T>, (const void*)k_phaseA_urf_seed_chk<T>,
                            (const void*)k_cand_row<T, 1>, (const void*)k_cand_row<T, 4>,
                            (const void*)k_residuals_delta_multi<T>, (const void*)k_sort_delta_multi<T>,
                            (const void*)k_merge_delta_multi<T>, (const void*)k_pw_leaves8_multi<T>,
                            (const void*)k_pw_combine_multi_smem<T>, (const void*)k_product2<T>,
                            (const void*)k_scores<T>, (const void*)k_line_stats<T>, (const void*)k_g_commit<T>,
                            (const void*)k_g_decide<T>, (const void*)k_g_decide_esc<T>, (const void*)k_g_zero,
                            (const void*)k_g_row_begin, (const void*)k_g_row_end, (const void*)k_g_fb_check};
        for (const void* f : ks) CK(cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, cv));
      }
      CK(cudaFuncSetAttribute(k_pw_combine_multi_smem<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)kCombineSmem));
    }
    rowof_r.alloc(N); colof_c.alloc(N);
    k_line_of<<<warps_grid(m), 256, 0, st>>>(m, row_ptr.p, rowof_r.p); LAUNCH_CK();
    k_line_of<<<warps_grid(n), 256, 0, st>>>(n, col_ptr.p, colof_c.p); LAUNCH_CK();
    // grid of the given data (binary32 mode)
    if (kExact) {
      gridX = f32_grid_given(X, mask, m * n);
    }
    // caches and scratch
    Ut.alloc((size_t)rank * m); V.alloc((size_t)rank * n);
    fuse_seed = m <= 8192;
    if (const char* e = getenv("STMF_FUSE_SEED")) fuse_seed = atoi(e) != 0;
    if (fuse_seed) {
      d_seedcols.alloc(1);
      SeedCols<T> scb{col_ptr.p, row_idx.p, xc.p, Ut.p};
      CK(cudaMemcpy(d_seedcols.p, &scb, sizeof(scb), cudaMemcpyHostToDevice));
    }
    t1r.alloc(N); t2r.alloc(N); t1c.alloc(N); t2c.alloc(N); agr.alloc(N); agc.alloc(N);
    a2r.alloc(N); a2c.alloc(N);
    rp = (rank + (int)(16 / sizeof(T)) - 1) / (int)(16 / sizeof(T)) * (int)(16 / sizeof(T));
    Urm.alloc((size_t)m * rp); Vcm.alloc((size_t)n * rp);
    CK(cudaMemsetAsync(Urm.p, 0, sizeof(T) * (size_t)m * rp, st));
    CK(cudaMemsetAsync(Vcm.p, 0, sizeof(T) * (size_t)n * rp, st));
    score.alloc(n); colhist.alloc((size_t)n * rank);
    cm1.alloc((size_t)rank * n); cm2.alloc((size_t)rank * n); cmarg.alloc((size_t)rank * n);
    rm1.alloc((size_t)rank * m); rm2.alloc((size_t)rank * m); rmarg.alloc((size_t)rank * m);
    ckeys.alloc(n); ckeys2.alloc(n); cvals.alloc(n); cperm.alloc(n);
    cj.alloc(std::max<int64_t>(n, Emax)); ck.alloc(std::max<int64_t>(n, Emax));
    cx.alloc(std::max<int64_t>(n, Emax)); xrow_dense.alloc(n);
    cmi.alloc((size_t)rank * n); sq.alloc(n);
    if (fast1) {
      f1_uv.alloc((size_t)kTop * m); f1_ux.alloc((size_t)kTop * m); f1_uo.alloc((size_t)kTop * m);
      f1_rv.alloc((size_t)rank * kTop * n); f1_rx.alloc((size_t)rank * kTop * n); f1_ro.alloc((size_t)rank * kTop * n);
      f1_k.alloc(1); f1_valid.alloc(rank);
      if (getenv("STMF_FAST1_STATS")) {
        f1_diag.alloc(4);
        CK(cudaMemsetAsync(f1_diag.p, 0, 32, st));
      }
      CK(cudaMemsetAsync(f1_valid.p, 0, sizeof(int) * rank, st));
      CK(cudaMemsetAsync(f1_k.p, 0xff, sizeof(int), st));
    }

    if (split_ulf) {
      hp_idx.alloc(N); hp_x.alloc(N); hp_t1.alloc(N); hp_t2.alloc(N); hp_ag.alloc(N); hp_split.alloc(m);
    }
    vbuf.alloc((size_t)Emax * n); ubufB.alloc((size_t)Emax * m);
    ubufA.alloc((size_t)Emax * m); vbufB.alloc((size_t)Emax * n);
    dtmpA.alloc(m); dtmpB.alloc(n);
    // batch results in one block, [flags: 4 int][acc: 4E u64][chg: 2E int][hk: E int],
    // zeroed with one memset and read back with one copy per batch
    bstate.alloc(2 + 4 * (size_t)Emax + 2 * (size_t)Emax);
    flags.view(reinterpret_cast<int*>(bstate.p), 4);
    acc.view(bstate.p + 2, 4 * (size_t)Emax);
    chg.view(reinterpret_cast<int*>(bstate.p + 2 + 4 * (size_t)Emax), 2 * (size_t)Emax);
    findpos.alloc(2);
    pinned_alloc(&h_bstate, sizeof(u64) * bstate.n);
    h_acc = h_bstate + 2;
    h_chg = reinterpret_cast<int*>(h_bstate + 2 + 4 * (size_t)Emax);
    pinned_alloc(&h_flags, sizeof(int) * 4);
    h_flags[0] = h_flags[1] = 0;
    size_t b1 = 0, b2 = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, b1, ckeys.p, ckeys2.p, cvals.p, cperm.p, (int)n, 0, 64, st));
    if (!kExact) {
      res_cur.alloc(N); S_cur.alloc(N);
      CK(cub::DeviceRadixSort::SortKeys(nullptr, b2, res_cur.p, S_cur.p, (int64_t)N, 0, 64, st));
      pw.build(N);
      alloc_slots();
      upload(pw_loff, pw.loff); upload(pw_llen, pw.llen); upload(pw_lnode, pw.lnode);
      upload(pw_left, pw.left); upload(pw_right, pw.right);
      upload(pw_lvloff, pw.lvl_off); upload(pw_lvlnodes, pw.lvl_nodes);
      {
        std::vector<int4> ops(pw.lvl_nodes.size());
        for (size_t t = 0; t < ops.size(); t++) {
          int nd = pw.lvl_nodes[t];
          ops[t] = make_int4(nd, pw.left[nd], pw.right[nd], 0);
        }
        pw_ops.alloc(std::max<size_t>(ops.size(), 1));
        if (!ops.empty()) CK(cudaMemcpy(pw_ops.p, ops.data(), sizeof(int4) * ops.size(), cudaMemcpyHostToDevice));
      }
      int depth = 26 + (int)std::ceil(std::log2((double)N + 1));
      beta_rel = 1.01 * depth * std::ldexp(1.0, -53);
    }
    cubtmp_bytes = std::max(b1, b2);
    cubtmp.alloc(cubtmp_bytes);
    stats_dirty.assign(rank, 1);
    ssync();
  }
  int gridX = -1000;

  template <typename E>
  void upload(DevBuf<E>& d, const std::vector<E>& h) {
    d.alloc(std::max<size_t>(h.size(), 1));
    if (!h.empty()) CK(cudaMemcpyAsync(d.p, h.data(), sizeof(E) * h.size(), cudaMemcpyHostToDevice, st));
  }

  unsigned warps_grid(int64_t lines) const {
    int64_t blocks = (lines * 32 + 255) / 256;
    int64_t cap = (int64_t)nsm * 16;
    return (unsigned)std::max<int64_t>(1, std::min(blocks, cap));
  }

  void set_factors(const void* Uh, const void* Vh) override {
    const T* U = (const T*)Uh;
    std::vector<T> ut((size_t)rank * m);
    for (int64_t i = 0; i < m; i++)
      for (int k = 0; k < rank; k++) ut[(size_t)k * m + i] = U[i * rank + k];
    CK(cudaMemcpyAsync(Ut.p, ut.data(), sizeof(T) * ut.size(), cudaMemcpyHostToDevice, st));
    if (kExact) {
      int g = gridX;
      for (auto v : ut) g = std::max(g, f32_grid((float)v));
      if (Vh) {
        const T* Vp = (const T*)Vh;
        for (int64_t a = 0; a < (int64_t)rank * n; a++) g = std::max(g, f32_grid((float)Vp[a]));
      }
      g = std::max(g, 0);
      if (g > 52) fail(STMF_ERR_NUMERIC, "binary32 data grid 2^-%d is too fine for the exact objective", g);
      F = g;
      exact_limit = std::ldexp(1.0, 53 - g);
    } else {
      F = 60;
      exact_limit = INFINITY;
    }
    if (Vh) {
      CK(cudaMemcpyAsync(V.p, Vh, sizeof(T) * (size_t)rank * n, cudaMemcpyHostToDevice, st));
    } else {
      // V = (-U)^T (x)* R  (random_acol_init, engine.py:194): rr of every column of U
      for (int k = 0; k < rank; k++) {
        k_line_min<T><<<warps_grid(n), 256, 0, st>>>(n, col_ptr.p, row_idx.p, xc.p, Ut.p + (size_t)k * m,
                                                       V.p + (size_t)k * n);
        LAUNCH_CK();
      }
    }
    ssync();
    sync_factor_copies(-1);
    // new factors start a new speculation history (the depths of another state say
    // nothing about this one): first visits use the initial batch schedule
    if ((int64_t)row_depth.size() == m) std::fill(row_depth.begin(), row_depth.end(), 0);
    rdepth_on_dev = false;
    depth_ema = 0;
    fast1_invalidate(-1);
    have_factors = true;
    cur_valid = false;
    dirty = true;
    cache_k = -1;
    stats_dirty.assign(rank, 1);
    err_valid = false;
  }

  void get_factors(void* Uh, void* Vh) override {
    need_factors();
    std::vector<T> ut((size_t)rank * m);
    CK(cudaMemcpyAsync(ut.data(), Ut.p, sizeof(T) * ut.size(), cudaMemcpyDeviceToHost, st));
    if (Vh) CK(cudaMemcpyAsync(Vh, V.p, sizeof(T) * (size_t)rank * n, cudaMemcpyDeviceToHost, st));
    ssync();
    if (Uh) {
      T* U = (T*)Uh;
      for (int64_t i = 0; i < m; i++)
        for (int k = 0; k < rank; k++) U[i * rank + k] = ut[(size_t)k * m + i];
    }
  }

  void need_factors() {
    if (!have_factors) fail(STMF_ERR_INVALID, "factors not set (call stmf_set_factors first)");
  }

  void check_flags() {
    CK(cudaMemcpyAsync(h_flags, flags.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    ssync();
    if (h_flags[0] & ~1 & 7) {
      int f = h_flags[0];
      fail(STMF_ERR_NUMERIC, "exact objective window violated (flags %d, grid 2^-%d)", f, F);
    }
    if (kExact && (h_flags[0] & 1)) fail(STMF_ERR_NUMERIC, "inexact fixed-point conversion in exact mode");
  }

  // product caches + scores + histograms + statistics of dirty factor indices
  // residuation statistics of dirty indices on an auxiliary stream, concurrent with
  // the product caches (they read only the committed factors)
  cudaStream_t st_aux = nullptr;
  cudaEvent_t ev_aux0 = nullptr, ev_aux1 = nullptr;
  void ensure_caches() {
    need_factors();
    bool stats = false;
    for (int k = 0; k < rank; k++) stats |= stats_dirty[k] != 0;
    cudaStream_t ss = st;
    if (stats && dirty) {
      CK(cudaEventRecord(ev_aux0, st));
      CK(cudaStreamWaitEvent(st_aux, ev_aux0, 0));
      ss = st_aux;
    }
    // the session stream joins the auxiliary work on every exit path (a throw below
    // must not leave later work on st racing the statistics kernels)
    struct AuxJoin {
      cudaStream_t st = nullptr;
      cudaEvent_t ev = nullptr;
      ~AuxJoin() {
        if (st) cudaStreamWaitEvent(st, ev, 0);
      }
    } aux_join;
    for (int k = 0; k < rank; k++) {
      if (!stats_dirty[k]) continue;
      k_line_stats<T><<<warps_grid(n), 256, 0, ss>>>(n, col_ptr.p, row_idx.p, xc.p, Ut.p + (size_t)k * m,
                                                        cm1.p + (size_t)k * n, cm2.p + (size_t)k * n,
                                                        cmarg.p + (size_t)k * n);
      LAUNCH_CK();
      k_line_stats<T><<<warps_grid(m), 256, 0, ss>>>(m, row_ptr.p, col_idx.p, xr.p, V.p + (size_t)k * n,
                                                        rm1.p + (size_t)k * m, rm2.p + (size_t)k * m,
                                                        rmarg.p + (size_t)k * m);
      LAUNCH_CK();
      stats_dirty[k] = 0;
    }
    if (ss != st) {
      CK(cudaEventRecord(ev_aux1, ss));
      aux_join.st = st;
      aux_join.ev = ev_aux1;
    }
    if (dirty) {
      CK(cudaMemsetAsync(flags.p, 0, sizeof(int), st));
      // cache_k >= 0: only factor index cache_k changed since the caches were valid
      int kk = cache_k;
      unsigned gflat = (unsigned)std::max<int64_t>(1, std::min<int64_t>(nblk(N, 256), (int64_t)nsm * 16));
      k_product2<T><<<gflat, 256, 0, st>>>(N, rowof_r.p, col_idx.p, m, n, rank, Ut.p, V.p, Urm.p, Vcm.p, rp, kk,
                                           t1r.p, t2r.p, agr.p, a2r.p);
      LAUNCH_CK();
      k_product2<T><<<gflat, 256, 0, st>>>(N, row_idx.p, colof_c.p, m, n, rank, Ut.p, V.p, Urm.p, Vcm.p, rp, kk,
                                           t1c.p, t2c.p, agc.p, a2c.p);
      LAUNCH_CK();
      k_scores<T><<<warps_grid(n), 256, 0, st>>>(n, rank, col_ptr.p, xc.p, t1c.p, agc.p, score.p, colhist.p,
                                                   !kExact, exact_limit, flags.p);
      LAUNCH_CK();
      if (!kExact) {
        if (n == 1) {
          DevBuf<double> col;
          col.alloc(m);
          k_colscore_single<T><<<1, 32, 0, st>>>(m, col_ptr.p, row_idx.p, xc.p, t1c.p, col.p, score.p);
          LAUNCH_CK();
          ssync();
        }
      }
      n_product_passes++;
      if (kExact) check_flags();
      rscore_valid = false;
      dirty = false;
      cache_k = -1;
    }
  }

  // objective of the state "current factors with column k of U := a, row k of V := b"
  double state_objective(int k, const T* a, const T* b) {
    if (kExact) {
      CK(cudaMemsetAsync(acc.p, 0, 2 * sizeof(u64), st));
      CK(cudaMemsetAsync(flags.p, 0, sizeof(int), st));
      k_objective<T><<<warps_grid(m), 256, 0, st>>>(m, row_ptr.p, col_idx.p, xr.p, t1r.p, t2r.p, agr.p, k, a, b,
                                                      acc.p, flags.p, F, exact_limit);
      LAUNCH_CK();
      CK(cudaMemcpyAsync(h_acc, acc.p, 2 * sizeof(u64), cudaMemcpyDeviceToHost, st));
      check_flags();
      return fx_to_double(h_acc[1], h_acc[0], F);
    }
    return replica1(k, a, b);
  }

  // ---- numpy replicas: np.sum(np.sort(|residuals|)) bit for bit (tropical.py:211) ----
  // Up to kSlots candidate states are replicated per round with one host sync.  The
  // delta path (<= kDeltaCap changed entries vs the current state) runs device-gated
  // for every slot; slots whose change set is larger are redone with a full sort.
  static constexpr int kSlots = 8;
  static constexpr size_t kCombineSmem = 160 * 1024;
  struct Slot {
    DevBuf<u64> res, sorted, olds, news;
    DevBuf<int> dcount;
    DevBuf<T> a, b;
    DevBuf<double> pw;
    const T* ap = nullptr;
    const T* bp = nullptr;
    int as = 1, bs = 1;  // element strides of ap / bp (EGP: one eval of a planar buffer)
    int k = 0;
  };
  std::vector<Slot> slots;
  int* h_dcount = nullptr;
  double* h_pwv = nullptr;
  double* h_out = nullptr;  // per slot: value, change count (bits)
  DevBuf<int> d_dcounts;
  DevBuf<double> d_pwout;
  void unpack_out(int count) {
    for (int i = 0; i < count; i++) {
      h_pwv[i] = h_out[2 * i];
      h_dcount[i] = (int)reinterpret_cast<const long long*>(h_out)[2 * i + 1];
    }
  }

  void alloc_slots() {
    static_assert(kSlots == kRepSlots, "replica round size");
    pinned_alloc(&h_out, sizeof(double) * 2 * kSlots);
    d_dcounts.alloc(kSlots);
    CK(cudaMemset(d_dcounts.p, 0, sizeof(int) * kSlots));
    d_pwout.alloc(2 * kSlots);
    slots.resize(kSlots);
    for (auto& s : slots) {
      s.res.alloc(N); s.sorted.alloc(N); s.olds.alloc(kDeltaCap); s.news.alloc(kDeltaCap); s.dcount.alloc(1);
      s.a.alloc(m); s.b.alloc(n); s.pw.alloc(pw.nnodes);
    }
    pinned_alloc(&h_dcount, sizeof(int) * kSlots);
    pinned_alloc(&h_pwv, sizeof(double) * kSlots);
  }

  void pw_sum(Slot& s) {
    int nl = (int)pw.loff.size();
    k_pw_leaves8<<<nblk((int64_t)nl * 8, 256), 256, 0, st>>>(nl, pw_loff.p, pw_llen.p, pw_lnode.p, s.sorted.p,
                                                            s.pw.p);
    LAUNCH_CK();
    if (pw.H > 0) {
      k_pw_combine<<<1, 1024, 0, st>>>(pw.H, pw_lvloff.p, pw_lvlnodes.p, pw_left.p, pw_right.p, s.pw.p);
      LAUNCH_CK();
    }
  }

  void full_sort(Slot& s) {
    size_t bytes = cubtmp_bytes;
    // residuals are >= 0: bit 63 is clear, sort on bits 0..62
    CK(cub::DeviceRadixSort::SortKeys(cubtmp.p, bytes, s.res.p, s.sorted.p, (int64_t)N, 0, 63, st));
    g_cub_calls++;
  }

  // replicas of slots[0, count) (ap, bp, k set) -> h_pwv[s]
  void replicas(int count) {
    bool delta = cur_valid;
    enqueue_replicas(count);
    for (int i = 0; i < count && !delta; i++) {
      Slot& s = slots[i];
      k_residuals<T><<<warps_grid(m), 256, 0, st>>>(m, row_ptr.p, col_idx.p, xr.p, t1r.p, t2r.p, agr.p, s.k, s.ap,
                                                      s.as, s.bp, s.bs, s.res.p);
      LAUNCH_CK();
      full_sort(s);
      h_dcount[i] = 0;
      pw_sum(s);
      CK(cudaMemcpyAsync(h_pwv + i, s.pw.p, sizeof(double), cudaMemcpyDeviceToHost, st));
    }
    ssync();
    if (delta) unpack_out(count);
    bool redo = false;
    for (int i = 0; i < count; i++) {
      if (dhist_on) dhist[std::min(13, 32 - __builtin_clz((unsigned)h_dcount[i] | 1))]++;
      if (delta && h_dcount[i] == 0) n_zero_delta++;
      if (!delta || h_dcount[i] <= kDeltaCap) {
        n_delta_replicas += delta;
        continue;
      }
      full_sort(slots[i]);
      pw_sum(slots[i]);
      CK(cudaMemcpyAsync(h_pwv + i, slots[i].pw.p, sizeof(double), cudaMemcpyDeviceToHost, st));
      redo = true;
    }
    if (redo) ssync();
  }

  // the delta replica steps of slots[0, count) on the stream, results copied to
  // h_dcount / h_pwv without a host sync (no-op unless the current state is valid)
  void enqueue_replicas(int count) {
    bool delta = cur_valid;
    n_escalations += count;
    if (delta) {
      // one launch per step for the whole round (slot = blockIdx.y)
      RepRound<T> rr{};
      rr.count = count;
      for (int i = 0; i < count; i++) {
        Slot& s = slots[i];
        rr.s[i] = RepSlot<T>{s.k, s.as, s.bs, s.ap, s.bp, s.res.p, s.sorted.p, s.olds.p, s.news.p,
                             d_dcounts.p + i, s.pw.p, d_pwout.p + 2 * i};
      }
      k_residuals_delta_multi<T><<<dim3(nblk(N, 256), count), 256, 0, st>>>(N, rowof_r.p, col_idx.p, xr.p, t1r.p,
                                                                              t2r.p, agr.p, res_cur.p, rr);
      LAUNCH_CK();
      k_sort_delta_multi<T><<<dim3(2, count), kSortThreads, 0, st>>>(rr);
      LAUNCH_CK();
      unsigned mt = (unsigned)((N + kMergeTile - 1) / kMergeTile);
      k_merge_delta_multi<T><<<dim3(mt, count), 256, 0, st>>>(N, S_cur.p, rr);
      LAUNCH_CK();
      int nl = (int)pw.loff.size();
      k_pw_leaves8_multi<T><<<dim3(nblk((int64_t)nl * 8, 256), count), 256, 0, st>>>(nl, pw_loff.p, pw_llen.p,
                                                                                     pw_lnode.p, rr);
      LAUNCH_CK();
      if (pw.H > 0) {
        int nops = (int)pw.lvl_nodes.size();
        size_t sm = sizeof(double) * (size_t)((pw.nnodes + 1) & ~1) + sizeof(int4) * (size_t)nops +
                    sizeof(int) * (size_t)(pw.H + 1);
        if (sm <= kCombineSmem)
          k_pw_combine_multi_smem<T><<<dim3(1, count), 1024, sm, st>>>(pw.H, pw.nnodes, nops, pw_lvloff.p, pw_ops.p,
                                                                       rr);
        else
          k_pw_combine_multi<T><<<dim3(1, count), 1024, 0, st>>>(pw.H, pw_lvloff.p, pw_lvlnodes.p, pw_left.p,
                                                                  pw_right.p, rr);
        LAUNCH_CK();
      }
      CK(cudaMemcpyAsync(h_out, d_pwout.p, sizeof(double) * 2 * count, cudaMemcpyDeviceToHost, st));
    }
  }

  // ---- deferred accept (fp64) ------------------------------------------------------
  // A certain accept (A + margin < err) is committed without waiting for its numpy
  // replica: the replica runs on the stream and its value becomes err at the next
  // point that needs err (the next decision, a sweep boundary, the end of the run).
  bool err_pending = false;
  int64_t pend_idx = -1;  // trajectory sample to fill with the resolved value
  int64_t n_deferred = 0;

  void resolve_err() {
    if (!err_pending) return;
    ssync();
    unpack_out(1);
    double fr = h_pwv[0];
    if (h_dcount[0] > kDeltaCap) {
      // too many changed entries for the delta merge: sort the adopted residuals
      size_t bytes = cubtmp_bytes;
      CK(cub::DeviceRadixSort::SortKeys(cubtmp.p, bytes, res_cur.p, S_cur.p, (int64_t)N, 0, 63, st));
      g_cub_calls++;
      int nl = (int)pw.loff.size();
      k_pw_leaves8<<<nblk((int64_t)nl * 8, 256), 256, 0, st>>>(nl, pw_loff.p, pw_llen.p, pw_lnode.p, S_cur.p,
                                                              slots[0].pw.p);
      LAUNCH_CK();
      if (pw.H > 0) {
        k_pw_combine<<<1, 1024, 0, st>>>(pw.H, pw_lvloff.p, pw_lvlnodes.p, pw_left.p, pw_right.p, slots[0].pw.p);
        LAUNCH_CK();
      }
      CK(cudaMemcpyAsync(h_pwv, slots[0].pw.p, sizeof(double), cudaMemcpyDeviceToHost, st));
      ssync();
      fr = h_pwv[0];
    } else {
      n_delta_replicas++;
      if (h_dcount[0] == 0) n_zero_delta++;
    }
    if (!(fr < err)) fail(STMF_ERR_NUMERIC, "decision bound violated: replica=%.17g err=%.17g", fr, err);
    err = fr;
    if (pend_idx >= 0 && cur_run) traj_set(*cur_run, pend_idx, fr);
    pend_idx = -1;
    err_pending = false;
  }

  double replica1(int k, const T* a, const T* b) {
    slots[0].k = k; slots[0].ap = a; slots[0].bp = b; slots[0].as = slots[0].bs = 1;
    replicas(1);
    return h_pwv[0];
  }

  // slot s's arrays become the current state's residuals / sorted residuals
  void adopt_slot(int s) {
    std::swap(res_cur.p, slots[s].res.p);
    std::swap(S_cur.p, slots[s].sorted.p);
    ptr_epoch++;  // a captured sweep graph holds the old pointers
    cur_valid = true;
  }

  // point slot s at eval (op, q) of the last batch (final column k of U, row k of V)
  void set_slot_eval(int s, int op, int q, int k) {
    Slot& S = slots[s];
    S.k = k;
    constexpr int EGP = Ilv<T>::STRIDE;
    if (op == 0) {
      S.ap = ubufB.p + (size_t)q * m;
      S.as = 1;
      S.bp = vbuf.p + ilv_index<T>(q, 0, n);
      S.bs = EGP;
    } else {
      S.ap = ubufA.p + ilv_index<T>(q, 0, m);
      S.as = EGP;
      S.bp = vbufB.p + (size_t)q * n;
      S.bs = 1;
    }
  }

  double objective() override {
    resolve_err();
    ensure_caches();
    if (!err_valid) {
      err = state_objective(0, Ut.p, V.p);
      if (!kExact) adopt_slot(0);
      err_valid = true;
    }
    return err;
  }

  // ---- candidates of row i ------------------------------------------------------
  int64_t build_candidates(int64_t i) {
    int64_t beg = h_row_ptr[i], nc = h_row_ptr[i + 1] - beg;
    if (nc <= 4 * kCandThreads && rank <= 256) {
      auto kern = nc <= kCandThreads ? k_cand_row<T, 1> : k_cand_row<T, 4>;
      kern<<<cand_grid(), kCandThreads, 0, st>>>((int)nc, n, rank, col_idx.p + beg, xr.p + beg, agr.p + beg, score.p,
                                       colhist.p, cj.p, ck.p, cx.p, xrow_dense.p, i, cm1.p, cm2.p, cmarg.p, cmi.p,
                                       nullptr, nullptr, selection == STMF_SEL_TD ? 1 : 0);
      LAUNCH_CK();
      cand_tdb(i, nc);
      row_partition();
      return nc;
    }
    k_cand_keys<<<nblk(nc, 256), 256, 0, st>>>(nc, col_idx.p + beg, score.p, ckeys.p, cvals.p);
    LAUNCH_CK();
    size_t bytes = cubtmp_bytes;
    CK(cub::DeviceRadixSort::SortPairs(cubtmp.p, bytes, ckeys.p, ckeys2.p, cvals.p, cperm.p, (int)nc, 0, 64, st));
    g_cub_calls++;
    unsigned nb = std::max(1u, std::min(nblk(nc, 256), 64u));
    k_cand_build<T><<<nb, 256, sizeof(int32_t) * rank, st>>>(nc, rank, col_idx.p + beg, xr.p + beg, agr.p + beg,
                                                             cperm.p, colhist.p, cj.p, ck.p, cx.p,
                                                             selection == STMF_SEL_TD ? 1 : 0);
    LAUNCH_CK();
    cand_tdb(i, nc);
    dense_row(i);
    row_cmi(i);
    row_partition();
    return nc;
  }

  // k_cand_row's grid: block 0 ranks the candidates, the others fill CM^(-i)
  unsigned cand_grid() const {
    int64_t need = ((int64_t)rank * n + kCandThreads - 1) / kCandThreads;
    return (unsigned)(1 + std::max<int64_t>(1, std::min<int64_t>(need, nsm)));
  }

  // CM^(-i) for the visited row (the statistics are current within a row visit)
  void row_cmi(int64_t i) {
    k_cmi<T><<<nblk((int64_t)rank * n, 256), 256, 0, st>>>(n, rank, i, cm1.p, cm2.p, cmarg.p, cmi.p);
    LAUNCH_CK();
  }

  void dense_row(int64_t i) {
    int64_t beg = h_row_ptr[i], nc = h_row_ptr[i + 1] - beg;
    k_fill<T><<<nblk(n, 256), 256, 0, st>>>(n, xrow_dense.p, (T)INFINITY);
    LAUNCH_CK();
    k_scatter_row<T><<<nblk(nc, 256), 256, 0, st>>>(nc, col_idx.p + beg, xr.p + beg, xrow_dense.p);
    LAUNCH_CK();
  }

  // ---- one speculative batch: candidates cj/ck/cx[t0, t0+E) of row i ------------
  void eval_batch(int64_t i, int64_t t0, int E, int* hk = nullptr) {
    const int32_t* bj = cj.p + t0;
    const int32_t* bk = ck.p + t0;
    const T* bx = cx.p + t0;
    // per-batch layout of bstate: [flags: 4 int][acc: 4E u64][chg: 2E int][hk: E int]
    u64* acc_ulf = bstate.p + 2;
    u64* acc_urf = acc_ulf + 2 * (size_t)E;
    int* chg_ulf = reinterpret_cast<int*>(acc_ulf + 4 * (size_t)E);
    int* chg_urf = chg_ulf + E;
    int* hk_dev = chg_ulf + 2 * E;
    size_t zero_bytes = 16 + sizeof(u64) * 4 * E + sizeof(int) * 2 * E;
    CK(cudaMemsetAsync(bstate.p, 0, zero_bytes, st));
    int64_t G8 = (int64_t)((E + kEG - 1) / kEG) * kEG;
    unsigned nb_ulf = nblk(G8 * n, 256), nb_urf = nblk(G8 * m, 256);
    k_phaseA<T><<<nb_ulf + nb_urf, 256, 0, st>>>(m, n, E, i, nb_ulf, bj, bk, bx, V.p, cm1.p, cm2.p, cmarg.p,
                                                 xrow_dense.p, vbuf.p, chg_ulf, sq.p, rm1.p, rm2.p, rmarg.p, ubufA.p,
                                                 hk_dev, nullptr, nullptr, fuse_seed ? d_seedcols.p : nullptr);
    LAUNCH_CK();
    if (!fuse_seed) {
      k_phaseA_urf_seed_chk<T><<<E, 128, 0, st>>>(m, E, i, bj, bk, bx, Ut.p, col_ptr.p, row_idx.p, xc.p, ubufA.p,
                                                  chg_urf);
      LAUNCH_CK();
    }
    int ng = (E + kEG - 1) / kEG;
    SideB<T> sa = side_ulf(acc_ulf, chg_ulf);
    SideB<T> sb{n, col_ptr.p, row_idx.p, xc.p, t1c.p, t2c.p, agc.p, ubufA.p, m, V.p, vbufB.p, acc_urf, chg_urf,
                0, long_thr, group_major};
    if (profiling && !getenv("STMF_TIME_B_ONLY")) CK(cudaEventRecord(ev_b0, st));
    if (fast1 && f1_row_ready) {
      // both second residuations from the line statistics (+ the rmarg == j scatter),
      // then phase B's error pass reads them (mode 2)
      k_pass1_fast<T><<<warps_grid((m + n) * ng), 256, 0, st>>>(sa, sb, E, bk, fast1_bufs(bj));
      LAUNCH_CK();
      k_pass1_dscatter<T><<<warps_grid((int64_t)E * ((m + 31) / 32)), 256, 0, st>>>(
          m, n, row_ptr.p, col_idx.p, xr.p, E, bk, bj, rmarg.p, f1_valid.p, ubufA.p, vbufB.p);
      LAUNCH_CK();
      if (getenv("STMF_FAST1_CHECK")) fast1_check(sa, sb, E, bk, bj, i);
      sa.mode = 2;
      sb.mode = 2;
    }
    if (profiling && getenv("STMF_TIME_B_ONLY")) CK(cudaEventRecord(ev_b0, st));
    launch_phaseB<T>(unroll, warps_grid((m + n) * ng), st, sa, sb, E, bk, flags.p, F, exact_limit, long_rows.p,
                     n_long_rows, long_cols.p, n_long_cols, nsm);
    LAUNCH_CK();
    if (profiling) CK(cudaEventRecord(ev_b1, st));
    phaseB_launches++;
    CK(cudaMemcpyAsync(h_bstate, bstate.p, zero_bytes + sizeof(int) * E, cudaMemcpyDeviceToHost, st));
    ssync();
    h_acc = h_bstate + 2;
    h_chg = reinterpret_cast<int*>(h_acc + 4 * (size_t)E);
    if (hk) std::memcpy(hk, h_chg + 2 * E, sizeof(int) * E);
    int fl = reinterpret_cast<const int*>(h_bstate)[0];
    if (fl & ~1 & 7) fail(STMF_ERR_NUMERIC, "exact objective window violated (flags %d, grid 2^-%d)", fl, F);
    if (kExact && (fl & 1)) fail(STMF_ERR_NUMERIC, "inexact fixed-point conversion in exact mode");
    if (profiling) {
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, ev_b0, ev_b1));
      phaseB_ns += (long long)(ms * 1e6);
      phaseB_timed++;
    }
  }

  // final column k of U (a) and row k of V (b) of eval (op, q) of the last batch
  const T* eval_a(int op, int q) {
    if (op == 0) return ubufB.p + (size_t)q * m;
    k_deinterleave<T><<<nblk(m, 256), 256, 0, st>>>(m, q, ubufA.p, dtmpA.p);
    LAUNCH_CK();
    return dtmpA.p;
  }
  const T* eval_b(int op, int q) {
    if (op == 1) return vbufB.p + (size_t)q * n;
    k_deinterleave<T><<<nblk(n, 256), 256, 0, st>>>(n, q, vbuf.p, dtmpB.p);
    LAUNCH_CK();
    return dtmpB.p;
  }

  // fp64 decision bound: |A - S| <= dr*S + da, |numpy(S) - S| <= beta*S
  double margin_of(int op, double A) const {
    int64_t L = op == 0 ? (max_rownnz + 31) / 32 : (max_colnnz + 31) / 32;
    int64_t lines = op == 0 ? m : n;
    double dr = (double)(L + 8) * std::ldexp(1.0, -53);
    double da = (double)lines * std::ldexp(1.0, -F + 1);
    return 2.0 * ((dr + beta_rel) * std::max(A, err) + da);
  }

  // FitRun._attempt over the batch in reference order (c0 ULF, c0 URF, c1 ULF, ...):
  // the first eval with f < err wins.  Returns the winner's order index or -1 and
  // commits it.  fp64: evals whose bound straddles err, and the first certain
  // accept (its numpy value becomes err), are replicated in rounds of kSlots.
  // `order` (optional): the eval ids (2 q + op) in the strategy's attempt order; the
  // return value is then a position in `order`.
  int decide_batch(int E, const std::vector<int>& hk, double* fwin, bool* deferred = nullptr,
                   const std::vector<int>* order = nullptr, int limit = -1) {
    resolve_err();
    if (deferred) *deferred = false;
    int pos = 0;
    int total = order ? (int)order->size() : 2 * E;
    if (limit >= 0) total = std::min(total, limit);  // attempt cap (set_max_attempts)
    while (pos < total) {
      struct Req { int ev, q, op; bool certain; };
      std::vector<Req> chunk;
      int scan = pos;
      for (; scan < total && (int)chunk.size() < (kExact ? 1 : kSlots); scan++) {
        int id = order ? (*order)[scan] : scan;
        int q = id >> 1, op = id & 1;
        if (!h_chg[op * E + q]) continue;  // state reproduced bit for bit: f == err
        double A = fx_to_double(h_acc[op * 2 * E + 2 * q + 1], h_acc[op * 2 * E + 2 * q], F);
        if (kExact) {
          if (A < err) {
            commit_eval(op, q, hk[q], -1);
            *fwin = A;
            return scan;
          }
          continue;
        }
        double mg = margin_of(op, A);
        if (A - mg >= err) continue;  // certainly not below err
        chunk.push_back({scan, q, op, A + mg < err});
        if (A + mg < err) { scan++; break; }
      }
      if (deferred && cur_valid && chunk.size() == 1 && chunk[0].certain) {
        set_slot_eval(0, chunk[0].op, chunk[0].q, hk[chunk[0].q]);
        enqueue_replicas(1);
        commit_eval(chunk[0].op, chunk[0].q, hk[chunk[0].q], 0);
        err_pending = true;
        *deferred = true;
        n_deferred++;
        *fwin = err;  // placeholder until resolve_err()
        return chunk[0].ev;
      }
      if (!chunk.empty()) {
        for (size_t c = 0; c < chunk.size(); c++) set_slot_eval((int)c, chunk[c].op, chunk[c].q, hk[chunk[c].q]);
        replicas((int)chunk.size());
        for (size_t c = 0; c < chunk.size(); c++) {
          double fr = h_pwv[c];
          if (fr < err) {
            commit_eval(chunk[c].op, chunk[c].q, hk[chunk[c].q], (int)c);
            *fwin = fr;
            return chunk[c].ev;
          }
          if (chunk[c].certain)
            fail(STMF_ERR_NUMERIC, "decision bound violated: replica=%.17g err=%.17g", fr, err);
        }
      }
      pos = scan;
    }
    return -1;
  }

  // accept eval (op, q); fp64: `slot` holds its replica (residuals of the new state)
  void commit_eval(int op, int q, int k, int slot) {
    const T* a;
    const T* b;
    if (slot >= 0) adopt_slot(slot);
    a = eval_a(op, q);
    b = eval_b(op, q);
    CK(cudaMemcpyAsync(Ut.p + (size_t)k * m, a, sizeof(T) * m, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(V.p + (size_t)k * n, b, sizeof(T) * n, cudaMemcpyDeviceToDevice, st));
    sync_factor_copies(k);
    cache_k = dirty ? -1 : k;  // incremental cache update iff only this index changed
    dirty = true;
    stats_dirty[k] = 1;
    fast1_invalidate(k);
  }

  // ---- run_fit sweep loop ----------------------------------------------------------
  struct RunState {
    bool wall;
    double t0, budget_seconds;
    int64_t cur_sweep;
    double* tt; double* te; int64_t cap, len;
    int64_t attempts, accepts, visits, evaluated;
    bool capped;  // the attempt cap was reached (set_max_attempts)
  };

  double run_now(RunState& R) { return R.wall ? now_s() - R.t0 : (double)R.cur_sweep; }
  bool out_of_time(RunState& R) { return R.capped || (R.wall && now_s() - R.t0 >= R.budget_seconds); }
  // attempt cap of the ByRow host loop (0 = none): the fit stops after exactly that many
  // attempts, as oracle.fit(max_attempts=...) does; capped runs use the host-driven loop
  int64_t max_attempts = 0;
  void set_max_attempts(int64_t cap) override { max_attempts = std::max<int64_t>(0, cap); }
  // audit mode (RunConfig.audit): after every sweep, rebuild the caches from the factors
  // and recompute the objective from scratch; it must equal the carried err
  bool audit_on = false;
  int64_t n_audits = 0;
  void set_audit(int on) override { audit_on = on != 0; }
  void audit_check() {
    resolve_err();
    dirty = true;
    cache_k = -1;
    stats_dirty.assign(rank, 1);
    ensure_caches();
    double e;
    if (kExact) e = state_objective(0, Ut.p, V.p);
    else e = exact_current_objective();
    n_audits++;
    if (e != err)
      fail(STMF_ERR_AUDIT, "audit: objective recomputed from scratch %.17g != the fit's error %.17g", e, err);
  }
  // the trajectory goes to the caller's buffers, or (null buffers) to the session's
  // growable copy, read back with stmf_trajectory
  std::vector<double> tj_t, tj_e;
  RunState* cur_run = nullptr;
  void traj_append(RunState& R, double t, double e) {
    if (!R.tt) {
      tj_t.push_back(t);
      tj_e.push_back(e);
      R.len++;
      return;
    }
    if (R.len >= R.cap) fail(STMF_ERR_CAPACITY, "trajectory capacity %lld exceeded", (long long)R.cap);
    R.tt[R.len] = t; R.te[R.len] = e; R.len++;
  }
  void traj_set(RunState& R, int64_t idx, double e) {
    if (R.tt) R.te[idx] = e;
    else tj_e[idx] = e;
  }
  void trajectory(double* t, double* e, int64_t cap, int64_t* len) override {
    *len = (int64_t)tj_t.size();
    if (!t || !e) return;
    if (cap < *len) fail(STMF_ERR_CAPACITY, "trajectory has %lld samples, capacity %lld", (long long)*len,
                         (long long)cap);
    std::memcpy(t, tj_t.data(), sizeof(double) * tj_t.size());
    std::memcpy(e, tj_e.data(), sizeof(double) * tj_e.size());
  }

  // byrow_sweep(run, i, "TD_A") (strategies.py:191-224)
  // STMF_PHASE_TIMING=1: synchronise after every phase and accumulate wall time
  // (diagnostics only; perturbs the overlap it measures)
  bool phase_timing = getenv("STMF_PHASE_TIMING") != nullptr;
  double ph[6] = {0, 0, 0, 0, 0, 0};  // caches, candidates, batch eval, decide+replicas, commit, other
  double ph_t = 0;
  void ph_mark(int slot) {
    if (!phase_timing) return;
    ssync();
    double t = now_s();
    if (slot >= 0) ph[slot] += t - ph_t;
    ph_t = t;
  }
  // host time spent waiting for the stream (STMF_SYNC_STATS): the rest of the run's
  // wall time is host work during which the GPU may idle
  bool sync_stats = getenv("STMF_SYNC_STATS") != nullptr;
  double t_wait = 0;
  int64_t n_sync = 0;
  void ssync() {
    if (!sync_stats) {
      CK(cudaStreamSynchronize(st));
      return;
    }
    double t = now_s();
    CK(cudaStreamSynchronize(st));
    t_wait += now_s() - t;
    n_sync++;
  }
  bool dhist_on = getenv("STMF_DHIST") != nullptr;
  int64_t dhist[14] = {0};
  void ph_report() {
    if (sync_stats) fprintf(stderr, "[stmf sync] %lld syncs, %.1f ms waiting\n", (long long)n_sync, t_wait * 1e3);
    if (dhist_on) {
      fprintf(stderr, "[stmf replica D log2 histogram]");
      for (int b = 0; b < 14; b++) fprintf(stderr, " %lld", (long long)dhist[b]);
      fprintf(stderr, "\n");
    }
    if (phase_timing)
      fprintf(stderr, "[stmf phases ms] caches %.1f candidates %.1f eval %.1f decide %.1f\n", ph[0] * 1e3,
              ph[1] * 1e3, ph[2] * 1e3, ph[3] * 1e3);
  }

  void row_visit(RunState& R, int64_t i) {
    if (family == STMF_FAMILY_BYELEMENT || family == STMF_FAMILY_BASELINE) return row_visit_entries(R, i);
    if (selection == STMF_SEL_SEQ) return row_visit_seq(R, i);
    ph_mark(-1);
    ensure_caches();
    ph_mark(0);
    int64_t nc = build_candidates(i);
    if (fast1 && selection != STMF_SEL_TD_B) {
      fast1_row_stats(st);
      f1_row_ready = true;
    }
    struct RowDone {
      bool& r;
      ~RowDone() { r = false; }
    } row_done{f1_row_ready};
    ph_mark(1);
    R.visits++;
    std::vector<int> hk;
    int64_t t0 = 0;
    size_t bi = 0;
    // speculation depth: a row's acceptance depth is strongly correlated across
    // sweeps, so the first batch covers 1.25x the candidates the row consumed on
    // its previous visit, floored by the fixed per-batch cost; then 2x growth
    int first = batch_sched[0];
    double dd = (!fixed_sched && (int64_t)row_depth.size() == m && row_depth[i] > 0) ? (double)row_depth[i]
                : (!fixed_sched && ema_first ? depth_ema : 0.0);
    if (dd > 0)
      first = (int)std::max<int64_t>(batch_floor, std::min<int64_t>(Emax, (int64_t)(sched_scale * dd) + sched_add));
    if (!fixed_sched) first = round_batch(first, e_round, Emax);
    int next = first;
    while (t0 < nc) {
      int E = (int)std::min<int64_t>(nc - t0, fixed_sched ? batch_sched[std::min(bi, batch_sched.size() - 1)] : next);
      bi++;
      next = round_batch(std::max(next + 1, (int)(next * sched_growth)), e_round, Emax);
      int limit = -1;
      if (max_attempts > 0) {
        int64_t rem = max_attempts - R.attempts;
        if (rem <= 0) { R.capped = true; return; }
        E = (int)std::min<int64_t>(E, (rem + 1) / 2);
        limit = (int)std::min<int64_t>(rem, 2 * (int64_t)E);
      }
      hk.resize(E);
      eval_batch(i, t0, E, hk.data());  // one host sync per batch
      ph_mark(2);
      R.evaluated += 2 * (int64_t)E;
      double f;
      bool deferred = false;
      int w = decide_batch(E, hk, &f, defer_accepts ? &deferred : nullptr, nullptr, limit);
      ph_mark(3);
      if (w >= 0) {
        R.attempts += w + 1;
        if ((int64_t)row_depth.size() == m) {
          row_depth[i] = t0 + w / 2 + 1;
          depth_ema = depth_ema > 0 ? 0.9 * depth_ema + 0.1 * (double)row_depth[i] : (double)row_depth[i];
        }
        R.accepts++;
        if (deferred) {
          traj_append(R, run_now(R), std::nan(""));
          pend_idx = R.len - 1;
        } else {
          err = f;
          traj_append(R, run_now(R), err);
        }
        return;
      }
      R.attempts += limit >= 0 ? limit : 2 * (int64_t)E;
      if (max_attempts > 0 && R.attempts >= max_attempts) R.capped = true;
      if (out_of_time(R)) return;
      t0 += E;
    }
    if ((int64_t)row_depth.size() == m) row_depth[i] = nc;
  }

  // ---- the reference's other fit methods -------------------
  int family = STMF_FAMILY_BYROW, selection = STMF_SEL_TD_A;
  std::vector<int32_t> h_col_idx;  // host copy of the CSR column indices (try_update)
  DevBuf<double> rscore, rs_scratch;
  bool rscore_valid = false;
  PWTree pwn;  // numpy pairwise tree of a length-n row (td_grid(...).sum(axis=1))
  DevBuf<int64_t> pwn_loff;
  DevBuf<int32_t> pwn_llen, pwn_lnode, pwn_left, pwn_right, pwn_lvloff, pwn_lvlnodes;
  DevBuf<int64_t> cpos;
  DevBuf<int> d_cnt;

  void set_strategy(int fam, int sel) override {
    if (fam < STMF_FAMILY_BYROW || fam > STMF_FAMILY_BYMATRIX) fail(STMF_ERR_INVALID, "unknown family %d", fam);
    if (sel < STMF_SEL_TD_A || sel > STMF_SEL_SEQ) fail(STMF_ERR_INVALID, "unknown selection %d", sel);
    if ((fam == STMF_FAMILY_BASELINE || sel == STMF_SEL_SEQ) && rank > Emax)
      fail(STMF_ERR_INVALID, "rank %d exceeds the batch capacity %d", rank, Emax);
    graph_destroy();
    family = fam;
    selection = sel;
  }

  // td_grid(work, U, V).sum(axis=1) of the current state (binary64: numpy's pairwise
  // row sum bit for bit; binary32: the exact sum, like the column scores)
  void ensure_row_scores() {
    ensure_caches();
    if (rscore_valid) return;
    if (!rscore.p) rscore.alloc(m);
    if constexpr (kExact) {
      CK(cudaMemsetAsync(flags.p, 0, sizeof(int), st));
      k_row_scores_exact<T><<<warps_grid(m), 256, 0, st>>>(m, row_ptr.p, xr.p, t1r.p, rscore.p, exact_limit,
                                                             flags.p);
      LAUNCH_CK();
      check_flags();
    } else {
      unsigned nb = (unsigned)std::max<int64_t>(1, std::min<int64_t>(m, nsm));
      if (!pwn_loff.p) {
        pwn.build(n);
        upload(pwn_loff, pwn.loff); upload(pwn_llen, pwn.llen); upload(pwn_lnode, pwn.lnode);
        upload(pwn_left, pwn.left); upload(pwn_right, pwn.right); upload(pwn_lvloff, pwn.lvl_off);
        if (pwn.lvl_nodes.empty()) pwn.lvl_nodes.push_back(0);
        upload(pwn_lvlnodes, pwn.lvl_nodes);
        rs_scratch.alloc((size_t)nb * (size_t)(n + pwn.nnodes));
      }
      k_row_scores_pw<<<nb, 256, 0, st>>>(m, n, row_ptr.p, col_idx.p, xr.p, t1r.p, (int)pwn.loff.size(), pwn_loff.p,
                                          pwn_llen.p, pwn_lnode.p, pwn.H, pwn_lvloff.p, pwn_lvlnodes.p, pwn_left.p,
                                          pwn_right.p, pwn.nnodes, rs_scratch.p, rscore.p);
      LAUNCH_CK();
    }
    rscore_valid = true;
  }

  void row_scores(double* out) override {
    ensure_row_scores();
    CK(cudaMemcpyAsync(out, rscore.p, sizeof(double) * m, cudaMemcpyDeviceToHost, st));
    ssync();
  }

  // TD_B factor indices for the candidates cj[0, nc) of row i (select_k_td_b)
  void cand_tdb(int64_t i, int64_t nc) {
    if (selection != STMF_SEL_TD_B) return;
    ensure_row_scores();
    k_cand_tdb<T><<<1, 256, 0, st>>>((int)nc, rank, m, n, i, Ut.p, V.p, rscore.p, score.p, cj.p, ck.p);
    LAUNCH_CK();
  }

  // per row visit: the dense copy of row i, CM^(-i), the hit partition
  void row_prep(int64_t i, bool with_dense) {
    if (with_dense) dense_row(i);
    row_cmi(i);
    row_partition();
  }

  // ByElement (byelement_sweep, strategies.py:252-269) and the STMF baseline
  // (_BaselineStrategy.sweep, engine.py:365-380) visit the given entries of row i in
  // column order and keep going after an acceptance.  Candidates from the current
  // state are evaluated in speculative batches; the decision walks them in the
  // reference's attempt order:
  //   ByElement: entries with nonzero error, k = argmax, F-ULF then F-URF;
  //   baseline:  every entry, F-ULF for k = 0..r-1, then F-URF for k = 0..r-1.
  void row_visit_entries(RunState& R, int64_t i) {
    const bool elem = family == STMF_FAMILY_BYELEMENT;
    const int64_t end = h_row_ptr[i + 1];
    const int cap = (int)std::min<int64_t>(Emax, std::max<int64_t>(n, rank));
    if (!cpos.p) { cpos.alloc(std::max<int64_t>(n, Emax)); d_cnt.alloc(1); }
    R.visits++;
    ensure_caches();
    row_prep(i, true);
    int64_t p = h_row_ptr[i];
    int want = std::max(1, std::min(cap, batch_floor * 2));
    std::vector<int> hk, order;
    std::vector<int64_t> epos;
    while (p < end) {
      int E = 0, ne = 0;
      if (elem) {
        k_cand_elem<T><<<1, 1024, 0, st>>>(p, end, want, col_idx.p, xr.p, t1r.p, agr.p, cj.p, ck.p, cx.p, cpos.p,
                                           d_cnt.p);
        LAUNCH_CK();
        int cnt = 0;
        CK(cudaMemcpyAsync(&cnt, d_cnt.p, sizeof(int), cudaMemcpyDeviceToHost, st));
        ssync();
        if (cnt == 0) break;  // the rest of the row is approximated exactly
        epos.resize(cnt);
        CK(cudaMemcpyAsync(epos.data(), cpos.p, sizeof(int64_t) * cnt, cudaMemcpyDeviceToHost, st));
        E = cnt;
      } else {
        ne = (int)std::min<int64_t>(end - p, std::max(1, want / rank));
        E = ne * rank;
        k_cand_entries<T><<<nblk(E, 256), 256, 0, st>>>(p, ne, rank, col_idx.p, xr.p, cj.p, ck.p, cx.p);
        LAUNCH_CK();
        order.clear();
        for (int e = 0; e < ne; e++) {
          for (int k = 0; k < rank; k++) order.push_back(2 * (e * rank + k));
          for (int k = 0; k < rank; k++) order.push_back(2 * (e * rank + k) + 1);
        }
      }
      hk.resize(E);
      eval_batch(i, 0, E, hk.data());
      R.evaluated += 2 * (int64_t)E;
      double f;
      int w = decide_batch(E, hk, &f, nullptr, elem ? nullptr : &order);
      if (w >= 0) {
        R.attempts += w + 1;
        R.accepts++;
        err = f;
        traj_append(R, run_now(R), err);
        int q = (elem ? w : order[w]) >> 1;
        p = elem ? epos[q] + 1 : p + q / rank + 1;
        ensure_caches();
        row_prep(i, false);
        want = std::max(1, std::min(cap, batch_floor * 2));
      } else {
        R.attempts += elem ? 2 * (int64_t)E : (int64_t)order.size();
        p = elem ? epos[E - 1] + 1 : p + ne;
        want = std::min(cap, want * 2);
      }
      if (out_of_time(R)) return;
    }
  }

  // ByRow / SEQ (byrow_seq, strategies.py:227-249): trial every (j, k, rule) of row i
  // from the same state and keep the largest strict decrease; ties go to the smallest
  // j, then k, then F-ULF.  binary64: every eval whose bound can reach the best is
  // replicated (numpy's value decides); binary32: the exact objective decides.
  void row_visit_seq(RunState& R, int64_t i) {
    const int64_t beg = h_row_ptr[i], end = h_row_ptr[i + 1];
    const int cap_e = (int)std::max<int64_t>(1, std::min<int64_t>(Emax, std::max<int64_t>(n, rank)) / rank);
    R.visits++;
    ensure_caches();
    row_prep(i, true);
    resolve_err();
    struct Pot { int64_t e; int k, op; double A, mg; };
    std::vector<Pot> pot;
    std::vector<int> hk;
    double best_hi = INFINITY;
    for (int64_t p = beg; p < end;) {
      int ne = (int)std::min<int64_t>(end - p, cap_e), E = ne * rank;
      k_cand_entries<T><<<nblk(E, 256), 256, 0, st>>>(p, ne, rank, col_idx.p, xr.p, cj.p, ck.p, cx.p);
      LAUNCH_CK();
      hk.resize(E);
      eval_batch(i, 0, E, hk.data());
      R.evaluated += 2 * (int64_t)E;
      for (int q = 0; q < E; q++)
        for (int op = 0; op < 2; op++) {
          if (!h_chg[op * E + q]) continue;  // state reproduced: f == err
          double A = fx_to_double(h_acc[op * 2 * E + 2 * q + 1], h_acc[op * 2 * E + 2 * q], F);
          double mg = kExact ? 0.0 : margin_of(op, A);
          if (A - mg >= err) continue;
          pot.push_back({p - beg + q / rank, q % rank, op, A, mg});
          best_hi = std::min(best_hi, A + mg);
        }
      p += ne;
    }
    if (pot.empty()) return;
    // the evals that can still be the minimum, with their objective values
    std::vector<Pot> S;
    for (auto& c : pot)
      if (c.A - c.mg <= best_hi) S.push_back(c);
    std::vector<double> fS(S.size());
    if (kExact) {
      for (size_t c = 0; c < S.size(); c++) fS[c] = S[c].A;
    } else {
      for (size_t c0 = 0; c0 < S.size(); c0 += kSlots) {
        int cnt = (int)std::min<size_t>(kSlots, S.size() - c0);
        set_seq_batch(i, beg, S, c0, cnt, hk);
        for (int c = 0; c < cnt; c++) set_slot_eval(c, S[c0 + c].op, c, S[c0 + c].k);
        replicas(cnt);
        for (int c = 0; c < cnt; c++) fS[c0 + c] = h_pwv[c];
      }
    }
    int best = -1;
    for (size_t c = 0; c < S.size(); c++)
      if (fS[c] < err && (best < 0 || fS[c] < fS[best])) best = (int)c;
    if (best < 0) return;
    // re-apply the winner (run.try_ulf / try_urf, strategies.py:245-248)
    set_seq_batch(i, beg, S, best, 1, hk);
    int slot = -1;
    if (!kExact) {
      set_slot_eval(0, S[best].op, 0, S[best].k);
      replicas(1);
      if (h_pwv[0] != fS[best]) fail(STMF_ERR_NUMERIC, "SEQ winner replica differs on re-evaluation");
      slot = 0;
    }
    commit_eval(S[best].op, 0, S[best].k, slot);
    err = fS[best];
    R.attempts++;
    R.accepts++;
    traj_append(R, run_now(R), err);
  }

  // candidates S[c0, c0 + cnt) of row i as a batch of cnt (entry, k) candidates
  template <typename P>
  void set_seq_batch(int64_t i, int64_t beg, const std::vector<P>& S, size_t c0, int cnt, std::vector<int>& hk) {
    std::vector<int32_t> hj(cnt), hkk(cnt);
    std::vector<int64_t> hp(cnt);
    for (int c = 0; c < cnt; c++) { hp[c] = beg + S[c0 + c].e; hkk[c] = S[c0 + c].k; }
    for (int c = 0; c < cnt; c++) hj[c] = h_col_of(hp[c]);
    CK(cudaMemcpyAsync(cj.p, hj.data(), sizeof(int32_t) * cnt, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(ck.p, hkk.data(), sizeof(int32_t) * cnt, cudaMemcpyHostToDevice, st));
    for (int c = 0; c < cnt; c++) CK(cudaMemcpyAsync(cx.p + c, xr.p + hp[c], sizeof(T), cudaMemcpyDeviceToDevice, st));
    hk.resize(cnt);
    eval_batch(i, 0, cnt, hk.data());
    (void)i;
  }
  int32_t h_col_of(int64_t p) {
    int32_t c;
    CK(cudaMemcpyAsync(&c, col_idx.p + p, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    ssync();
    return c;
  }

  // bymatrix_step's ranked candidate list (strategies.py:281-292): every given entry
  // (row-major order) with its argmax k and score, sorted by decreasing score (stable)
  DevBuf<u64> mc_k1, mc_k2;
  DevBuf<int32_t> mc_v1, mc_v2, mc_orow, mc_ocol, mc_ok;
  DevBuf<double> mc_sc, mc_osc;
  DevBuf<uint8_t> mc_tmp;
  void matrix_candidates(int32_t* rows, int32_t* cols, int32_t* ks, double* scores) override {
    ensure_row_scores();
    auto &k1 = mc_k1, &k2 = mc_k2;
    auto &v1 = mc_v1, &v2 = mc_v2, &orow = mc_orow, &ocol = mc_ocol, &ok = mc_ok;
    auto &sc = mc_sc, &osc = mc_osc;
    if (!k1.p) {
      k1.alloc(N); k2.alloc(N); v1.alloc(N); v2.alloc(N); sc.alloc(N);
      orow.alloc(N); ocol.alloc(N); ok.alloc(N); osc.alloc(N);
    }
    k_matrix_keys<T><<<nblk(N, 256), 256, 0, st>>>(N, rowof_r.p, col_idx.p, xr.p, t1r.p, rscore.p, score.p, k1.p,
                                                     v1.p, sc.p);
    LAUNCH_CK();
    size_t bytes = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, bytes, k1.p, k2.p, v1.p, v2.p, (int)N, 0, 64, st));
    if (mc_tmp.n < bytes) mc_tmp.alloc(bytes);
    CK(cub::DeviceRadixSort::SortPairs(mc_tmp.p, bytes, k1.p, k2.p, v1.p, v2.p, (int)N, 0, 64, st));
    g_cub_calls++;
    k_matrix_gather<T><<<nblk(N, 256), 256, 0, st>>>(N, v2.p, rowof_r.p, col_idx.p, agr.p, sc.p, orow.p, ocol.p,
                                                       ok.p, osc.p);
    LAUNCH_CK();
    CK(cudaMemcpyAsync(rows, orow.p, sizeof(int32_t) * N, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(cols, ocol.p, sizeof(int32_t) * N, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(ks, ok.p, sizeof(int32_t) * N, cudaMemcpyDeviceToHost, st));
    if (scores) CK(cudaMemcpyAsync(scores, osc.p, sizeof(double) * N, cudaMemcpyDeviceToHost, st));
    ssync();
  }

  bool fixpoint_replay = getenv("STMF_FIXPOINT_REPLAY") ? atoi(getenv("STMF_FIXPOINT_REPLAY")) != 0 : true;
  int64_t n_replayed_sweeps = 0;
  int64_t replayed_sweeps() override { return n_replayed_sweeps; }
  std::vector<int64_t> row_depth;  // candidates consumed at each row's last visit
  bool rdepth_on_dev = false;      // the device copy (graph sweeps) is the current one
  void pull_row_depth() {
    if (!rdepth_on_dev) return;
    h_rdepth.resize(m);
    CK(cudaMemcpyAsync(h_rdepth.data(), d_row_depth.p, sizeof(long long) * m, cudaMemcpyDeviceToHost, st));
    ssync();
    for (int64_t i = 0; i < m; i++) row_depth[i] = h_rdepth[i];
    rdepth_on_dev = false;
  }
  double depth_ema = 0;            // running mean of accepting depths
  // rows without depth history (first sweep, or after set_factors): first batch from the
  // running mean instead of the fixed first size (STMF_EMA_FIRST)
  bool ema_first = getenv("STMF_EMA_FIRST") ? atoi(getenv("STMF_EMA_FIRST")) != 0 : false;
  // first batch = scale * previous depth + add; later batches grow by `growth`
  double sched_scale = 1.25, sched_growth = 2.0;
  int sched_add = 2;
  void read_sched_env() {
    if (const char* e = getenv("STMF_SCHED")) sscanf(e, "%lf,%d,%lf", &sched_scale, &sched_add, &sched_growth);
  }
  int batch_floor = 1;
  // batch sizes in whole eval groups (round_batch); STMF_EROUND=1 keeps the raw schedule
  int e_round = getenv("STMF_EROUND") ? std::max(1, atoi(getenv("STMF_EROUND"))) : kEG;
  bool fixed_sched = false;
  bool defer_accepts = getenv("STMF_NO_DEFER") == nullptr;

  // ---- device-resident sweeps (stmf_graph.cuh) ----------------------------------------
  // One CUDA graph per sweep: the host loop of run()/row_visit/decide_batch as nested
  // conditional nodes.  Built lazily; rebuilt when buffers it captured were swapped.
  bool graph_on = getenv("STMF_GRAPH") ? atoi(getenv("STMF_GRAPH")) != 0 : true;
  int64_t ptr_epoch = 0, graph_epoch = -1;
  bool graph_prof = false;
  cudaGraph_t g_top = nullptr;
  cudaGraphExec_t g_exec = nullptr;
  DevBuf<DevCtl> dctl;
  DevCtl* h_ctl = nullptr;
  DevBuf<long long> d_row_depth;
  DevBuf<double> d_traj_t, d_traj_e;
  DevBuf<RepRound<T>> d_rr;
  DevBuf<double*> d_pwptr;
  DevBuf<double> d_aval;
  std::vector<long long> h_rdepth;
  std::vector<double> h_traj_t, h_traj_e;

  bool graph_eligible() const {
    // rows must fit the one-block candidate ranking; column scores of a single-column
    // matrix and fixed batch schedules stay on the host loop
    return graph_on && !fixed_sched && max_attempts <= 0 && family == STMF_FAMILY_BYROW &&
           (selection == STMF_SEL_TD_A || selection == STMF_SEL_TD) && max_rownnz <= 4 * kCandThreads && rank <= 256 && n > 1 &&
           (kExact || cur_valid) && n_long_rows + n_long_cols == 0 && 2 * Emax <= kDecideThreads;
  }

  void graph_destroy() {
    if (g_exec) cudaGraphExecDestroy(g_exec);
    if (g_top) cudaGraphDestroy(g_top);
    g_exec = nullptr;
    g_top = nullptr;
  }

  // capture helpers: kernels launched on st between cap_begin / cap_end are appended
  // to graph g after deps; cap_end returns the new leaf nodes
  void cap_begin(cudaGraph_t g, const std::vector<cudaGraphNode_t>& deps) {
    CK(cudaStreamBeginCaptureToGraph(st, g, deps.empty() ? nullptr : deps.data(), nullptr, deps.size(),
                                     cudaStreamCaptureModeThreadLocal));
  }
  std::vector<cudaGraphNode_t> cap_end(cudaGraph_t g) {
    cudaStreamCaptureStatus cs;
    const cudaGraphNode_t* deps = nullptr;
    size_t nd = 0;
    cudaGraph_t cg;
    CK(cudaStreamGetCaptureInfo(st, &cs, nullptr, &cg, &deps, &nd));
    std::vector<cudaGraphNode_t> out(deps, deps + nd);
    CK(cudaStreamEndCapture(st, &g));
    return out;
  }
  // a conditional node after deps; returns its body graph
  cudaGraph_t add_cond(cudaGraph_t g, std::vector<cudaGraphNode_t>& deps, cudaGraphConditionalHandle h,
                       cudaGraphConditionalNodeType type) {
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = type;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    CK(cudaGraphAddNode(&node, g, deps.empty() ? nullptr : deps.data(), deps.size(), &cp));
    deps.assign(1, node);
    return cp.conditional.phGraph_out[0];
  }

  cudaStream_t st2 = nullptr;          // second capture stream (graph branches)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaStream_t st3 = nullptr;          // third capture stream (residuation statistics after an accept)
  cudaEvent_t ev_fork3 = nullptr, ev_join3 = nullptr;
  // pairwise-tree combine of a replica round read from the device descriptor
  void launch_combine(int ys, RepRound<T>* rp_, cudaStream_t s_) {
    RepRound<T> none{};
    int nops = (int)pw.lvl_nodes.size();
    size_t sm = sizeof(double) * (size_t)((pw.nnodes + 1) & ~1) + sizeof(int4) * (size_t)nops +
                sizeof(int) * (size_t)(pw.H + 1);
    if (sm <= kCombineSmem)
      k_pw_combine_multi_smem<T><<<dim3(1, ys), 1024, sm, s_>>>(pw.H, pw.nnodes, nops, pw_lvloff.p, pw_ops.p, none,
                                                                rp_);
    else
      k_pw_combine_multi<T><<<dim3(1, ys), 1024, 0, s_>>>(pw.H, pw_lvloff.p, pw_lvlnodes.p, pw_left.p, pw_right.p,
                                                           none, rp_);
  }

  GBufs<T> gbufs() {
    GBufs<T> B{};
    B.bst = bstate.p; B.ck = ck.p;
    B.ubufB = ubufB.p; B.vbuf = vbuf.p; B.ubufA = ubufA.p; B.vbufB = vbufB.p;
    B.m = m; B.n = n;
    B.row_depth = d_row_depth.p;
    B.traj_t = d_traj_t.p; B.traj_e = d_traj_e.p;
    B.rr = d_rr.p;
    for (int s = 0; s < kSlots && !kExact; s++) {
      B.res[s] = slots[s].res.p; B.sorted[s] = slots[s].sorted.p;
      B.olds[s] = slots[s].olds.p; B.news[s] = slots[s].news.p; B.pw[s] = slots[s].pw.p;
    }
    B.dcount = d_dcounts.p;
    B.out = d_pwout.p;
    B.F = F;
    B.exact = kExact;
    for (int op = 0; op < 2; op++) {
      int64_t L = op == 0 ? (max_rownnz + 31) / 32 : (max_colnnz + 31) / 32;
      B.dr[op] = (double)(L + 8) * std::ldexp(1.0, -53);
      B.da[op] = (double)(op == 0 ? m : n) * std::ldexp(1.0, -F + 1);
    }
    B.beta = beta_rel;
    B.aval = d_aval.p;
    B.urf_valid = fast1 ? f1_valid.p : nullptr;
    return B;
  }

  void graph_build() {
    graph_destroy();
    if (!st2) {
      CK(cudaStreamCreateWithFlags(&st2, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
      CK(cudaStreamCreateWithFlags(&st3, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&ev_fork3, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&ev_join3, cudaEventDisableTiming));
    }
    if (!dctl.p) {
      dctl.alloc(1);
      pinned_alloc(&h_ctl, sizeof(DevCtl));
      d_row_depth.alloc(m);
      d_traj_t.alloc(m + 1);
      d_traj_e.alloc(m + 1);
      d_rr.alloc(1);
      d_pwptr.alloc(kSlots);
      d_aval.alloc(2 * (size_t)Emax);
      h_traj_t.resize(m + 1);
      h_traj_e.resize(m + 1);
    }
    if (!kExact) {
      std::vector<double*> pp(kSlots);
      for (int s = 0; s < kSlots; s++) pp[s] = slots[s].pw.p;
      CK(cudaMemcpy(d_pwptr.p, pp.data(), sizeof(double*) * kSlots, cudaMemcpyHostToDevice));
    }
    GBufs<T> B = gbufs();
    DevCtl* c = dctl.p;
    CK(cudaGraphCreate(&g_top, 0));
    cudaGraphConditionalHandle h_row, h_batch, h_acc, h_esc = 0, h_fb = 0;
    CK(cudaGraphConditionalHandleCreate(&h_row, g_top, 0, 0));
    std::vector<cudaGraphNode_t> d0;
    cap_begin(g_top, d0);
    if (graph_prof) k_g_tick<<<1, 1, 0, st>>>(c, 5);
    k_g_sweep_begin<<<1, 1, 0, st>>>(c, m, h_row);
    d0 = cap_end(g_top);
    cudaGraph_t b_row = add_cond(g_top, d0, h_row, cudaGraphCondTypeWhile);
    if (graph_prof) {
      cap_begin(g_top, d0);
      k_g_tick<<<1, 1, 0, st>>>(c, 6);
      cap_end(g_top);
    }

    // ---- row body
    CK(cudaGraphConditionalHandleCreate(&h_batch, b_row, 0, 0));
    CK(cudaGraphConditionalHandleCreate(&h_acc, b_row, 0, 0));
    std::vector<cudaGraphNode_t> dr;
    cap_begin(b_row, dr);
    k_g_row_begin<<<1, 1, 0, st>>>(c, row_ptr.p, d_row_depth.p, h_batch, h_acc);
    {
      auto kern = max_rownnz <= kCandThreads ? k_cand_row<T, 1> : k_cand_row<T, 4>;
      kern<<<cand_grid(), kCandThreads, 0, st>>>(0, n, rank, col_idx.p, xr.p, agr.p, score.p, colhist.p, cj.p, ck.p,
                                                 cx.p,
                                       xrow_dense.p, 0, cm1.p, cm2.p, cmarg.p, cmi.p, c, row_ptr.p,
                                       selection == STMF_SEL_TD ? 1 : 0);
    }
    row_partition();
    if (fast1) fast1_row_stats(st);
    dr = cap_end(b_row);
    cudaGraph_t b_batch = add_cond(b_row, dr, h_batch, cudaGraphCondTypeWhile);

    // ---- batch body
    if (!kExact) CK(cudaGraphConditionalHandleCreate(&h_esc, b_batch, 0, 0));
    std::vector<cudaGraphNode_t> db;
    cap_begin(b_batch, db);
    k_g_zero<<<8, 256, 0, st>>>(c, bstate.p);
    k_phaseA<T><<<(unsigned)nsm * 4, 256, 0, st>>>(m, n, 0, 0, 0, cj.p, ck.p, cx.p, V.p, cm1.p, cm2.p, cmarg.p,
                                                   xrow_dense.p, vbuf.p, nullptr, sq.p, rm1.p, rm2.p, rmarg.p,
                                                   ubufA.p, nullptr, c, bstate.p,
                                                   fuse_seed ? d_seedcols.p : nullptr);
    if (!fuse_seed)
      k_phaseA_urf_seed_chk<T><<<Emax, 128, 0, st>>>(m, 0, 0, cj.p, ck.p, cx.p, Ut.p, col_ptr.p, row_idx.p, xc.p,
                                                      ubufA.p, nullptr, c, bstate.p);
    if (graph_prof) k_g_tick<<<1, 1, 0, st>>>(c, 0);
    {
      SideB<T> sa = side_ulf(nullptr, nullptr);
      SideB<T> sb{n, col_ptr.p, row_idx.p, xc.p, t1c.p, t2c.p, agc.p, ubufA.p, m, V.p, vbufB.p, nullptr, nullptr,
                  0, long_thr, group_major};
      if (fast1) {
        k_pass1_fast<T><<<(unsigned)nsm * 8, 256, 0, st>>>(sa, sb, 0, nullptr, fast1_bufs(cj.p), c, ck.p);
        k_pass1_dscatter<T><<<(unsigned)nsm * 4, 256, 0, st>>>(m, n, row_ptr.p, col_idx.p, xr.p, 0, nullptr, nullptr,
                                                               rmarg.p, f1_valid.p, ubufA.p, vbufB.p, c, ck.p, cj.p);
        sa.mode = 2;
        sb.mode = 2;
      }
      // one wave of resident CTAs (the kernel's launch bounds)
      unsigned gb = (unsigned)nsm * (unroll >= 4 ? 2 : sizeof(T) == 4 ? kPhaseBCtasF32 : unroll > 1 ? 2 : kPhaseBCtasF64);
      if (unroll >= 4)
        k_phaseB<T, 4><<<gb, 256, 0, st>>>(sa, sb, 0, nullptr, flags.p, F, exact_limit, c, bstate.p, ck.p);
      else if (unroll == 2)
        k_phaseB<T, 2><<<gb, 256, 0, st>>>(sa, sb, 0, nullptr, flags.p, F, exact_limit, c, bstate.p, ck.p);
      else
        k_phaseB<T, 1><<<gb, 256, 0, st>>>(sa, sb, 0, nullptr, flags.p, F, exact_limit, c, bstate.p, ck.p);
    }
    k_g_decide<T><<<1, kDecideThreads, 0, st>>>(c, B, h_batch, h_acc, h_esc);
    db = cap_end(b_batch);
    if (!kExact) {
      cudaGraph_t b_esc = add_cond(b_batch, db, h_esc, cudaGraphCondTypeWhile);
      CK(cudaGraphConditionalHandleCreate(&h_fb, b_esc, 0, 0));
      std::vector<cudaGraphNode_t> de;
      cap_begin(b_esc, de);
      if (graph_prof) k_g_tick<<<1, 1, 0, st>>>(c, 1);
      RepRound<T> none{};
      RepRound<T>* rp_ = d_rr.p;
      k_residuals_delta_multi<T><<<dim3(nblk(N, 256), kSlots), 256, 0, st>>>(N, rowof_r.p, col_idx.p, xr.p, t1r.p,
                                                                              t2r.p, agr.p, res_cur.p, none, rp_);
      k_sort_delta_multi<T><<<dim3(2, kSlots), kSortThreads, 0, st>>>(none, rp_);
      unsigned mt = (unsigned)((N + kMergeTile - 1) / kMergeTile);
      k_merge_delta_multi<T><<<dim3(mt, kSlots), 256, 0, st>>>(N, S_cur.p, none, rp_);
      int nl = (int)pw.loff.size();
      k_pw_leaves8_multi<T><<<dim3(nblk((int64_t)nl * 8, 256), kSlots), 256, 0, st>>>(nl, pw_loff.p, pw_llen.p,
                                                                                     pw_lnode.p, none, rp_);
      if (pw.H > 0) launch_combine(kSlots, rp_, st);
      k_g_fb_check<<<1, 1, 0, st>>>(c, d_pwout.p, h_fb);
      de = cap_end(b_esc);
      cudaGraph_t b_fb = add_cond(b_esc, de, h_fb, cudaGraphCondTypeIf);
      {
        std::vector<cudaGraphNode_t> df;
        cap_begin(b_fb, df);
        for (int s = 0; s < kSlots; s++) {
          full_sort(slots[s]);
          pw_sum(slots[s]);
        }
        k_g_fb_fix<<<1, 32, 0, st>>>(c, d_pwptr.p, d_pwout.p);
        cap_end(b_fb);
      }
      cap_begin(b_esc, de);
      if (graph_prof) k_g_tick<<<1, 1, 0, st>>>(c, 2);
      k_g_decide_esc<T><<<1, kDecideThreads, 0, st>>>(c, B, h_batch, h_acc, h_esc);
      cap_end(b_esc);
    }

    // ---- accept (after the batch loop)
    cudaGraph_t b_acc = add_cond(b_row, dr, h_acc, cudaGraphCondTypeIf);
    cudaGraphConditionalHandle h_fb1 = 0;
    unsigned gc = (unsigned)nsm * 4;
    if (!kExact) CK(cudaGraphConditionalHandleCreate(&h_fb1, b_acc, 0, 0));
    {
      std::vector<cudaGraphNode_t> da;
      cap_begin(b_acc, da);
      if (graph_prof) k_g_tick<<<1, 1, 0, st>>>(c, 3);
      k_g_commit<T><<<gc, 256, 0, st>>>(c, B, Ut.p, V.p, Urm.p, Vcm.p, rp, N, kExact ? nullptr : res_cur.p,
                                        kExact ? nullptr : S_cur.p);
      unsigned gflat = (unsigned)std::max<int64_t>(1, std::min<int64_t>(nblk(N, 256), (int64_t)nsm * 16));
      const int* kc = &c->cache_k;
      // the residuation statistics of index k need only the committed factors: a
      // third branch, overlapped with the product caches and the column scores
      CK(cudaEventRecord(ev_fork3, st));
      CK(cudaStreamWaitEvent(st3, ev_fork3, 0));
      k_line_stats<T><<<warps_grid(n), 256, 0, st3>>>(n, col_ptr.p, row_idx.p, xc.p, Ut.p, cm1.p, cm2.p, cmarg.p, 0,
                                                         kc, m, n);
      k_line_stats<T><<<warps_grid(m), 256, 0, st3>>>(m, row_ptr.p, col_idx.p, xr.p, V.p, rm1.p, rm2.p, rmarg.p, 0,
                                                         kc, n, m);
      CK(cudaEventRecord(ev_join3, st3));
      k_product2<T><<<gflat, 256, 0, st>>>(N, rowof_r.p, col_idx.p, m, n, rank, Ut.p, V.p, Urm.p, Vcm.p, rp, 0,
                                           t1r.p, t2r.p, agr.p, a2r.p, kc);
      if (!kExact) {
        // fp64 direct accept: the numpy replica of the committed state (residuals from
        // the new CSR product) on a second branch, overlapped with the remaining caches
        CK(cudaEventRecord(ev_fork, st));
        CK(cudaStreamWaitEvent(st2, ev_fork, 0));
        RepRound<T> none{};
        RepRound<T>* rp_ = d_rr.p;
        k_res_from_product<T><<<(unsigned)nsm * 8, 256, 0, st2>>>(c, N, xr.p, t1r.p, res_cur.p, rp_);
        k_sort_delta_multi<T><<<dim3(2, 1), kSortThreads, 0, st2>>>(none, rp_);
        unsigned mt = (unsigned)((N + kMergeTile - 1) / kMergeTile);
        k_merge_delta_multi<T><<<dim3(mt, 1), 256, 0, st2>>>(N, S_cur.p, none, rp_);
        int nl = (int)pw.loff.size();
        k_pw_leaves8_multi<T><<<dim3(nblk((int64_t)nl * 8, 256), 1), 256, 0, st2>>>(nl, pw_loff.p, pw_llen.p,
                                                                                    pw_lnode.p, none, rp_);
        if (pw.H > 0) launch_combine(1, rp_, st2);
        k_g_fb1_check<<<1, 1, 0, st2>>>(c, d_pwout.p, h_fb1);
        CK(cudaEventRecord(ev_join, st2));
      }
      k_product2<T><<<gflat, 256, 0, st>>>(N, row_idx.p, colof_c.p, m, n, rank, Ut.p, V.p, Urm.p, Vcm.p, rp, 0,
                                           t1c.p, t2c.p, agc.p, a2c.p, kc);
      k_scores<T><<<warps_grid(n), 256, 0, st>>>(n, rank, col_ptr.p, xc.p, t1c.p, agc.p, score.p, colhist.p,
                                                   !kExact, exact_limit, flags.p);
      CK(cudaStreamWaitEvent(st, ev_join3, 0));
      if (!kExact) CK(cudaStreamWaitEvent(st, ev_join, 0));
      da = cap_end(b_acc);
      if (!kExact) {
        cudaGraph_t b_fb1 = add_cond(b_acc, da, h_fb1, cudaGraphCondTypeIf);
        std::vector<cudaGraphNode_t> df;
        cap_begin(b_fb1, df);
        full_sort(slots[0]);
        pw_sum(slots[0]);
        k_g_fb1_fix<<<1, 1, 0, st>>>(slots[0].pw.p, d_pwout.p);
        cap_end(b_fb1);
      }
      cap_begin(b_acc, da);
      if (!kExact) k_g_adopt<T><<<gc, 256, 0, st>>>(c, B, N, res_cur.p, S_cur.p);
      if (graph_prof) k_g_tick<<<1, 1, 0, st>>>(c, 4);
      cap_end(b_acc);
    }
    cap_begin(b_row, dr);
    k_g_row_end<<<1, 1, 0, st>>>(c, bstate.p, kExact, m, h_row);
    cap_end(b_row);
    CK(cudaGraphInstantiate(&g_exec, g_top, 0));
    graph_epoch = ptr_epoch;
  }

  // numpy value of the current state from scratch (residuals, full sort, pairwise
  // tree) into res_cur / S_cur, without swapping buffers
  double exact_current_objective() {
    k_residuals<T><<<warps_grid(m), 256, 0, st>>>(m, row_ptr.p, col_idx.p, xr.p, t1r.p, t2r.p, agr.p, 0, Ut.p, 1,
                                                    V.p, 1, res_cur.p);
    LAUNCH_CK();
    size_t bytes = cubtmp_bytes;
    CK(cub::DeviceRadixSort::SortKeys(cubtmp.p, bytes, res_cur.p, S_cur.p, (int64_t)N, 0, 63, st));
    g_cub_calls++;
    int nl = (int)pw.loff.size();
    k_pw_leaves8<<<nblk((int64_t)nl * 8, 256), 256, 0, st>>>(nl, pw_loff.p, pw_llen.p, pw_lnode.p, S_cur.p,
                                                            slots[0].pw.p);
    LAUNCH_CK();
    if (pw.H > 0) {
      k_pw_combine<<<1, 1024, 0, st>>>(pw.H, pw_lvloff.p, pw_lvlnodes.p, pw_left.p, pw_right.p, slots[0].pw.p);
      LAUNCH_CK();
    }
    CK(cudaMemcpyAsync(h_pwv, slots[0].pw.p, sizeof(double), cudaMemcpyDeviceToHost, st));
    ssync();
    return h_pwv[0];
  }

  // one sweep as (normally) one graph launch
  void graph_sweep(RunState& R) {
    if (!g_exec || graph_epoch != ptr_epoch || graph_prof != profiling) {
      graph_prof = profiling;
      double t0 = now_s();
      graph_build();
      if (getenv("STMF_GRAPH_STATS")) fprintf(stderr, "[stmf graph] build %.1f ms\n", (now_s() - t0) * 1e3);
    }
    DevCtl& h = *h_ctl;
    long long start = 0;
    for (;;) {
      std::memset(&h, 0, sizeof(DevCtl));
      h.err = err;
      h.start_row = start;
      // STMF_DIRECT_CAP (tests): a smaller limit forces the full-replica resumption
      h.direct_cap = getenv("STMF_DIRECT_CAP") ? std::min(kDeltaCap, atoi(getenv("STMF_DIRECT_CAP"))) : kDeltaCap;
      h.traj_cap = m + 1;
      h.sweep = (double)R.cur_sweep;
      h.sched_scale = sched_scale; h.sched_growth = sched_growth; h.sched_add = sched_add;
      h.batch_floor = batch_floor; h.Emax = Emax; h.first0 = batch_sched[0];
      h.e_round = fixed_sched ? 1 : e_round;
      h.ema_first = ema_first ? 1 : 0;
      h.depth_ema = depth_ema;
      h.cache_k = -1;
      h.tb0 = 0;
      CK(cudaMemcpyAsync(dctl.p, h_ctl, sizeof(DevCtl), cudaMemcpyHostToDevice, st));
      CK(cudaGraphLaunch(g_exec, st));
      CK(cudaMemcpyAsync(h_ctl, dctl.p, sizeof(DevCtl), cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(h_traj_t.data(), d_traj_t.p, sizeof(double) * (m + 1), cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(h_traj_e.data(), d_traj_e.p, sizeof(double) * (m + 1), cudaMemcpyDeviceToHost, st));
      ssync();
      if (h.error == 1) fail(STMF_ERR_NUMERIC, "decision bound violated (device decision)");
      if (h.error == 2) fail(STMF_ERR_CAPACITY, "device trajectory capacity exceeded");
      if (h.error == 3) fail(STMF_ERR_NUMERIC, "exact objective window violated (graph sweep, grid 2^-%d)", F);
      for (long long t = 0; t < h.traj_len; t++) traj_append(R, h_traj_t[t], h_traj_e[t]);
      err = h.err;
      depth_ema = h.depth_ema;
      R.attempts += h.attempts;
      R.accepts += h.accepts;
      R.visits += h.visits;
      R.evaluated += h.evaluated;
      n_escalations += h.escalations;
      n_product_passes += h.accepts;
      phaseB_launches += h.batches;
      if (graph_prof) {
        phaseB_ns += (long long)h.phaseB_ns;
        phaseB_timed += h.batches;
      }
      // kernel nodes executed: row (3), batch (5 + tick), escalation round (7 + 1), accept (6, +7 fp64)
      g_launches += h.visits * (3 + (fast1 ? 4 : 0)) + h.batches * (5 + (graph_prof ? 1 : 0) + (fast1 ? 2 : 0)) +
                    h.esc_rounds * 8 + h.accepts * (kExact ? 6 : 13);
      if (getenv("STMF_GRAPH_STATS"))
        fprintf(stderr,
                "[stmf graph] rows %lld batches %lld esc_rounds %lld accepts %lld | sweep %.2f ms: phaseB %.2f "
                "esc %.2f accept %.2f\n",
                h.visits, h.batches, h.esc_rounds, h.accepts, h.sweep_ns * 1e-6, h.phaseB_ns * 1e-6,
                h.esc_ns * 1e-6, h.acc_ns * 1e-6);
      if (h.error == 4) {
        // a direct accept changed more than kDeltaCap residuals: its numpy value from a
        // full replica of the committed state, then the sweep resumes at the next row
        double fr = exact_current_objective();
        if (!(fr < h.err_prev)) fail(STMF_ERR_NUMERIC, "decision bound violated: replica=%.17g err=%.17g", fr,
                                     h.err_prev);
        err = fr;
        traj_set(R, R.len - 1, fr);
        start = h.i;
        if (start < m) continue;
      }
      break;
    }
    dirty = false;
    cache_k = -1;
  }

  void run(int64_t budget_sweeps, double budget_seconds, double epsilon, double* tt, double* te, int64_t cap,
           int64_t* counts) override {
    need_factors();
    if (budget_sweeps < 0 && !(budget_seconds > 0)) fail(STMF_ERR_INVALID, "set budget_sweeps or budget_seconds");
    if (family == STMF_FAMILY_BYMATRIX)
      fail(STMF_ERR_INVALID, "ByMatrix steps run host-side (stmf_matrix_candidates + stmf_attempt)");
    if (max_attempts > 0 && (family != STMF_FAMILY_BYROW || selection == STMF_SEL_SEQ))
      fail(STMF_ERR_INVALID, "the attempt cap applies to ByRow TD / TD_A / TD_B fits only");
    RunState R{};
    R.wall = budget_seconds > 0;
    R.budget_seconds = budget_seconds;
    R.t0 = now_s();
    R.tt = tt; R.te = te; R.cap = cap;
    if (!tt) { tj_t.clear(); tj_e.clear(); }
    cur_run = &R;
    struct ClearRun {
      RunState*& r;
      ~ClearRun() { r = nullptr; }
    } clear_run{cur_run};
    int64_t pp0 = n_product_passes, esc0 = n_escalations;
    objective();
    traj_append(R, run_now(R), err);  // FitRun.__init__ (engine.py:263)
    double eps = epsilon * err;       // engine.py:330
    int64_t sweeps = 0;
    if (err > 0.0) {
      for (;;) {
        if (budget_sweeps >= 0 && sweeps >= budget_sweeps) break;
        if (out_of_time(R)) break;
        R.cur_sweep = sweeps + 1;
        double err_before = err;
        int64_t accepts_before = R.accepts, attempts_before = R.attempts, visits_before = R.visits,
                evaluated_before = R.evaluated;
        if (!R.wall && graph_eligible()) {
          if (!rdepth_on_dev) {
            h_rdepth.assign(row_depth.begin(), row_depth.end());
            if (!d_row_depth.p) d_row_depth.alloc(m);
            CK(cudaMemcpyAsync(d_row_depth.p, h_rdepth.data(), sizeof(long long) * m, cudaMemcpyHostToDevice, st));
            rdepth_on_dev = true;
          }
          ensure_caches();
          graph_sweep(R);
        } else {
          pull_row_depth();
          for (int64_t i = 0; i < m; i++) {
            if (out_of_time(R)) break;
            row_visit(R, i);
          }
        }
        sweeps++;
        resolve_err();
        if (audit_on) audit_check();
        traj_append(R, run_now(R), err);  // mark_sweep_boundary (engine.py:309-310)
        if (err_before - err < eps) break;
        // Fixpoint: a sweep without an accepted update leaves
        // U, V and err unchanged, and ByRow / ByElement / the baseline draw no random
        // numbers during sweeps, so every later sweep repeats it exactly.  With a sweep
        // budget and epsilon = 0 the remaining sweeps are replayed (their trajectory
        // samples and attempt counts) instead of recomputed; STMF_FIXPOINT_REPLAY=0
        // executes them (benchmarks do, so fixpoint sweeps are never counted as run).
        if (!R.wall && !R.capped && budget_sweeps >= 0 && err == err_before && R.accepts == accepts_before &&
            fixpoint_replay) {
          int64_t sw_att = R.attempts - attempts_before, sw_vis = R.visits - visits_before,
                  sw_ev = R.evaluated - evaluated_before;
          while (sweeps < budget_sweeps) {
            R.cur_sweep = ++sweeps;
            R.attempts += sw_att;
            R.visits += sw_vis;
            R.evaluated += sw_ev;
            traj_append(R, run_now(R), err);
            n_replayed_sweeps++;
          }
          break;
        }
      }
    }
    resolve_err();
    pull_row_depth();
    counts[0] = R.len; counts[1] = R.attempts; counts[2] = R.accepts; counts[3] = sweeps;
    ph_report();
    counts[4] = R.visits; counts[5] = R.evaluated; counts[6] = n_escalations - esc0;
    counts[7] = n_product_passes - pp0;
    if (f1_diag.p) {
      unsigned long long d[4];
      CK(cudaMemcpy(d, f1_diag.p, 32, cudaMemcpyDeviceToHost));
      fprintf(stderr, "[fast1 stats] ULF evals x lines %llu, fallbacks %llu (%.2f%%); URF %llu, fallbacks %llu (%.2f%%)\n",
              d[0], d[1], 100.0 * d[1] / std::max(d[0], 1ull), d[2], d[3], 100.0 * d[3] / std::max(d[2], 1ull));
    }
  }

  // ---- diff-test hooks -----------------------------------------------------------
  void product_given(void* P, int32_t* arg, void* top2) override {
    ensure_caches();
    std::vector<uint8_t> a(N);
    if (P) CK(cudaMemcpyAsync(P, t1r.p, sizeof(T) * N, cudaMemcpyDeviceToHost, st));
    if (top2) CK(cudaMemcpyAsync(top2, t2r.p, sizeof(T) * N, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(a.data(), agr.p, N, cudaMemcpyDeviceToHost, st));
    ssync();
    if (arg)
      for (int64_t p = 0; p < N; p++) arg[p] = a[p];
  }

  void col_scores(double* out) override {
    ensure_caches();
    CK(cudaMemcpyAsync(out, score.p, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
    ssync();
  }

  void residuate(int axis, const void* vec, void* out) override {
    int64_t lin = axis == 0 ? m : n, lout = axis == 0 ? n : m;
    DevBuf<T> dv, dout;
    dv.alloc(lin); dout.alloc(lout);
    CK(cudaMemcpyAsync(dv.p, vec, sizeof(T) * lin, cudaMemcpyHostToDevice, st));
    if (axis == 0)
      k_line_min<T><<<warps_grid(n), 256, 0, st>>>(n, col_ptr.p, row_idx.p, xc.p, dv.p, dout.p);
    else
      k_line_min<T><<<warps_grid(m), 256, 0, st>>>(m, row_ptr.p, col_idx.p, xr.p, dv.p, dout.p);
    LAUNCH_CK();
    CK(cudaMemcpyAsync(out, dout.p, sizeof(T) * lout, cudaMemcpyDeviceToHost, st));
    ssync();
  }

  void try_update(int op, int64_t i, int64_t j, int k, void* ucol, void* vrow, double* f, bool commit_if_better,
                  int* accepted) override {
    if (i < 0 || i >= m || j < 0 || j >= n || k < 0 || k >= rank) fail(STMF_ERR_INVALID, "index out of range");
    ensure_caches();
    // locate (i, j) among the given entries of row i (host copy of the column
    // indices, made on first use)
    if ((int64_t)h_col_idx.size() != N) {
      h_col_idx.resize(N);
      CK(cudaMemcpyAsync(h_col_idx.data(), col_idx.p, sizeof(int32_t) * N, cudaMemcpyDeviceToHost, st));
      ssync();
    }
    auto b0 = h_col_idx.begin() + h_row_ptr[i], b1 = h_col_idx.begin() + h_row_ptr[i + 1];
    auto it = std::lower_bound(b0, b1, (int32_t)j);
    if (it == b1 || *it != (int32_t)j) fail(STMF_ERR_INVALID, "entry (%lld, %lld) is missing", (long long)i, (long long)j);
    int64_t p = it - h_col_idx.begin();
    resolve_err();
    if (!err_valid) objective();
    int32_t jj = (int32_t)j, kk = k;
    CK(cudaMemcpyAsync(cj.p, &jj, sizeof(int32_t), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(ck.p, &kk, sizeof(int32_t), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(cx.p, xr.p + p, sizeof(T), cudaMemcpyDeviceToDevice, st));
    dense_row(i);
    row_cmi(i);
    row_partition();
    eval_batch(i, 0, 1);
    ssync();
    double fv;
    if (!h_chg[op]) {
      fv = err;
    } else if (kExact) {
      fv = fx_to_double(h_acc[op * 2 + 1], h_acc[op * 2], F);
    } else {
      double A = fx_to_double(h_acc[op * 2 + 1], h_acc[op * 2], F);
      if (commit_if_better && !ucol && !vrow && A - margin_of(op, A) >= err) {
        // an attempt that certainly does not decrease the error: its objective is
        // only reported (FitRun._attempt uses it for the decision alone), so the
        // bounded value stands in for numpy's
        *f = A;
        *accepted = 0;
        return;
      }
      set_slot_eval(0, op, 0, k);
      replicas(1);
      fv = h_pwv[0];
    }
    if (ucol) CK(cudaMemcpyAsync(ucol, eval_a(op, 0), sizeof(T) * m, cudaMemcpyDeviceToHost, st));
    if (vrow) CK(cudaMemcpyAsync(vrow, eval_b(op, 0), sizeof(T) * n, cudaMemcpyDeviceToHost, st));
    ssync();
    *f = fv;
    if (commit_if_better) {
      *accepted = fv < err;
      if (*accepted) {
        commit_eval(op, 0, k, kExact ? -1 : 0);
        err = fv;
      }
    }
  }

  void bench_product(int reps, int flush, double* ms, double* errout) override {
    ensure_caches();
    DevBuf<uint8_t> scratch;
    if (flush) scratch.alloc((size_t)256 << 20);
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    float total = 0;
    for (int r = 0; r < reps; r++) {
      if (flush) CK(cudaMemsetAsync(scratch.p, r & 0xff, scratch.n, st));
      CK(cudaEventRecord(e0, st));
      k_product_csr<T><<<warps_grid(m), 256, 0, st>>>(m, n, rank, row_ptr.p, col_idx.p, Ut.p, V.p, t1r.p, t2r.p,
                                                        agr.p);
      CK(cudaMemsetAsync(acc.p, 0, 2 * sizeof(u64), st));
      k_objective<T><<<warps_grid(m), 256, 0, st>>>(m, row_ptr.p, col_idx.p, xr.p, t1r.p, t2r.p, agr.p, 0, Ut.p,
                                                      V.p, acc.p, flags.p, F, exact_limit);
      CK(cudaEventRecord(e1, st));
      CK(cudaEventSynchronize(e1));
      float t;
      CK(cudaEventElapsedTime(&t, e0, e1));
      total += t;
    }
    LAUNCH_CK();
    CK(cudaMemcpyAsync(h_acc, acc.p, 2 * sizeof(u64), cudaMemcpyDeviceToHost, st));
    ssync();
    *ms = total / std::max(reps, 1);
    *errout = fx_to_double(h_acc[1], h_acc[0], F);
    dirty = true;  // the bench overwrote the CSR caches without second-argmax tracking
    cache_k = -1;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }
};

#include <memory>

#include "stmf_maxplus.cuh"
#include "stmf_maxplus_lanes.cuh"
#include "stmf_shard.cuh"

__global__ void k_popcount(int64_t words, const uint32_t* __restrict__ mask, u64* __restrict__ out) {
  u64 c = 0;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < words; w += (int64_t)gridDim.x * blockDim.x)
    c += __popc(mask[w]);
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, c);
}

// config-5 microbench: data generated on the device (seeded counter-based RNG:
// X, U, V ~ U[-1, 1) on the 2^-23 grid, iid mask with P(given) = density)
// layout: 0 = dense tiles (k_maxplus_err), 1 = sampled / compacted (k_maxplus_err_lanes or
// k_maxplus_err_sampled), 2 = k_maxplus_err_lanes demanded,
// -1 = automatic (sampled when density <= 0.35 and r <= 64: fewer bytes and only given
// entries computed; measured crossover, profiles/r02_c5_sampled.md)
template <int RQ>
static void launch_sampled(unsigned grid, cudaStream_t st, int64_t m, int64_t n, const uint32_t* M, const float* vals,
                           const int64_t* off, const float* Urm, const float* Vrm, u64* acc, int* flags, int F,
                           double lim) {
  // STMF_C5_DECODE=list: the code-list decode; default: binary-search decode
  static const bool list = getenv("STMF_C5_DECODE") && !strcmp(getenv("STMF_C5_DECODE"), "list");
  if (list)
    k_maxplus_err_sampled<RQ, false><<<grid, 256, sp_smem_bytes<RQ>(), st>>>(m, n, M, vals, off, Urm, Vrm, acc, flags,
                                                                             F, lim);
  else
    k_maxplus_err_sampled<RQ, true><<<grid, 256, sp_smem_bytes<RQ>(), st>>>(m, n, M, vals, off, Urm, Vrm, acc, flags,
                                                                            F, lim);
}

// k_maxplus_err_lanes<RQ, SPAN>: RQ = 16-byte vectors per factor row, SPAN = columns per chunk
using LanesKernel = void (*)(int64_t, int64_t, const unsigned char*, const int64_t*, const float*, const float*, u64*,
                             int*, int, double, int, int, int);
template <int RQ>
static LanesKernel lanes_kernel_span(int span) {
  switch (span) {
    case 2048: if constexpr (RQ == 1) return k_maxplus_err_lanes<RQ, 2048>; else return nullptr;
    case 1024: return k_maxplus_err_lanes<RQ, 1024>;
    case 512: return k_maxplus_err_lanes<RQ, 512>;
    case 256: return k_maxplus_err_lanes<RQ, 256>;
  }
  return nullptr;
}
static LanesKernel lanes_kernel(int rq, int span) {
  return rq == 1 ? lanes_kernel_span<1>(span) : rq == 2 ? lanes_kernel_span<2>(span) : lanes_kernel_span<4>(span);
}

static void maxplus_bench_impl(int64_t m, int64_t n, int r, double density, uint64_t seed, int reps, int flush,
                               int device, double* out, float* X_out, uint32_t* mask_out, float* U_out,
                               float* V_out, int layout = 0) {
  if (m % kMpTR || n % kMpTC) fail(STMF_ERR_INVALID, "m must be a multiple of %d and n of %d", kMpTR, kMpTC);
  if (r < 1) fail(STMF_ERR_INVALID, "rank must be >= 1");
  if (layout < 0) layout = (density <= 0.35 && r <= 64 && m % kSpT == 0 && n % kSpT == 0) ? 1 : 0;
  if (layout >= 1 && (m % kSpT || n % kSpT)) fail(STMF_ERR_INVALID, "sampled layout: m and n must be multiples of %d", kSpT);
  if (layout >= 1 && r > 64) fail(STMF_ERR_INVALID, "sampled layout: rank must be <= 64");
  // the sampled layout has two kernels: lane-compacted chunks (stmf_maxplus_lanes.cuh: n a multiple of
  // 1024, rank <= 16) and the older 128 x 128 tiles.  layout 1 picks lanes when it applies
  // (STMF_C5_SAMPLED=tiles forces the tile kernel), layout 2 demands it.
  // (m % 128 == 0 is checked above; n % 256 == 0 admits the narrowest chunk)
  const bool lanes_ok = n % kLnMinSpan == 0 && m % kLnRows == 0 && r <= 16;
  if (layout == 2 && !lanes_ok) fail(STMF_ERR_INVALID, "lane-coded layout: n must be a multiple of %d and rank <= 16", kLnMinSpan);
  bool lanes = layout == 2;
  if (layout == 1 && lanes_ok && !(getenv("STMF_C5_SAMPLED") && !strcmp(getenv("STMF_C5_SAMPLED"), "tiles"))) lanes = true;
  if (layout == 2) layout = 1;
  CK(cudaSetDevice(device));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, device));
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  DevBuf<float> X, Ut, V;
  DevBuf<uint32_t> M;
  DevBuf<u64> acc, cnt;
  DevBuf<int> flags;
  DevBuf<uint8_t> scratch;
  int64_t words = m * n / 32;
  X.alloc((size_t)(m * n)); M.alloc((size_t)words); Ut.alloc((size_t)r * m); V.alloc((size_t)r * n);
  acc.alloc(2); cnt.alloc(1); flags.alloc(1);
  unsigned gb = (unsigned)prop.multiProcessorCount * 8;
  k_gen_uniform<<<gb, 256, 0, st>>>(m * n, seed * 4 + 0, X.p); LAUNCH_CK();
  k_gen_uniform<<<gb, 256, 0, st>>>((int64_t)r * m, seed * 4 + 1, Ut.p); LAUNCH_CK();
  k_gen_uniform<<<gb, 256, 0, st>>>((int64_t)r * n, seed * 4 + 2, V.p); LAUNCH_CK();
  uint32_t thr = (uint32_t)std::min(16777216.0, std::max(0.0, density * 16777216.0));
  k_gen_mask<<<gb, 256, 0, st>>>(words, seed * 4 + 3, thr, M.p); LAUNCH_CK();
  CK(cudaMemsetAsync(cnt.p, 0, sizeof(u64), st));
  k_popcount<<<gb, 256, 0, st>>>(words, M.p, cnt.p); LAUNCH_CK();
  if (flush) scratch.alloc((size_t)256 << 20);
  int F = 23;  // every value is a multiple of 2^-23
  double exact_limit = std::ldexp(1.0, 53 - F);
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  dim3 grid((unsigned)(n / kMpTC), (unsigned)(m / kMpTR));
  CK(cudaFuncSetAttribute(k_maxplus_err<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxplusDynSmem));
  CK(cudaFuncSetAttribute(k_maxplus_err<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxplusDynSmem));
  CK(cudaFuncSetAttribute(k_maxplus_err<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxplusDynSmem));
  // k-chunk of the factor slices: the smallest of 4 / 8 / 16 that covers r (STMF_C5_KC forces one)
  int kc_sel = r <= 4 ? 4 : r <= 8 ? 8 : 16;
  if (const char* e = getenv("STMF_C5_KC")) kc_sel = atoi(e) <= 4 ? 4 : atoi(e) <= 8 ? 8 : 16;
  auto kern = kc_sel == 4 ? k_maxplus_err<4> : kc_sel == 8 ? k_maxplus_err<8> : k_maxplus_err<16>;
  // TMA-fed X tiles (STMF_C5_TMA=0: per-thread cp.async copies)
  bool tma = getenv("STMF_C5_TMA") ? atoi(getenv("STMF_C5_TMA")) != 0 : true;
  CUtensorMap xmap{}, umap{}, vmap{};
  if (tma) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      fn = nullptr;
    }
    tma = fn != nullptr;  // no tensor-map encoder in this driver: per-thread copies
  }
  if (tma) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)m};
    cuuint64_t strides[1] = {(cuuint64_t)n * sizeof(float)};
    cuuint32_t box[2] = {(cuuint32_t)kMpTC, (cuuint32_t)kMpTR};
    cuuint32_t estr[2] = {1, 1};
    CUresult cr = encode(&xmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, X.p, dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) fail(STMF_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)cr);
    // factor slices (used when r equals the kernel's k-chunk): Ut is r x m, V is r x n
    int kc = kc_sel;
    if (r % kc == 0) {
      cuuint64_t ud[2] = {(cuuint64_t)m, (cuuint64_t)r}, vd[2] = {(cuuint64_t)n, (cuuint64_t)r};
      cuuint64_t us[1] = {(cuuint64_t)m * sizeof(float)}, vs[1] = {(cuuint64_t)n * sizeof(float)};
      cuuint32_t ub[2] = {(cuuint32_t)kMpTR, (cuuint32_t)kc}, vb[2] = {(cuuint32_t)kMpTC, (cuuint32_t)kc};
      cr = encode(&umap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, Ut.p, ud, us, ub, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (cr == CUDA_SUCCESS)
        cr = encode(&vmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, V.p, vd, vs, vb, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (cr != CUDA_SUCCESS) fail(STMF_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)cr);
    }
    CK(cudaFuncSetAttribute(k_maxplus_err<4, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxplusDynSmem));
    CK(cudaFuncSetAttribute(k_maxplus_err<8, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxplusDynSmem));
    CK(cudaFuncSetAttribute(k_maxplus_err<16, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxplusDynSmem));
  }
  auto kernt = kc_sel == 4 ? k_maxplus_err<4, true> : kc_sel == 8 ? k_maxplus_err<8, true> : k_maxplus_err<16, true>;
  // sampled layout: packed given values per tile + padded row-major factors
  DevBuf<float> vals, Urm, Vrm;
  DevBuf<int64_t> tcnt, toff;
  int rq = 1;
  while (4 * rq < r) rq *= 2;
  unsigned sgrid = 0;
  u64 given_h = 0;
  DevBuf<int> lnmax;
  DevBuf<uint8_t> lnrecs;
  int ln_cpw_log2 = 0, ln_stages = 1, ln_cap = 16, ln_sp = 0;
  size_t ln_smem = 0;
  int64_t ln_bytes = 0;
  if (layout == 1 && lanes) {
    const int RS = 4 * rq;
    // chunk width: the widest SPAN (dividing n) whose largest record fits a shared-memory stage with
    // two blocks per SM (denser matrices get narrower chunks of about as many entries); if even the
    // narrowest does not fit, the narrowest, with the oversized records read from global memory
    if (const char* e = getenv("STMF_C5_STAGES")) ln_stages = std::min(kLnMaxStages, std::max(1, atoi(e)));
    const size_t per_block = (size_t)prop.sharedMemPerMultiprocessor / 2 - 3072;  // static + reserved shared memory
    int64_t nrc = m / kLnRows, nsp = 0, nch = 0, units = 0;
    int maxrec = 0;
    size_t vbytes = 0, budget = 0;
    for (ln_sp = ln_max_span(rq); ln_sp >= kLnMinSpan; ln_sp /= 2) {
      if (n % ln_sp) continue;
      if (const char* e = getenv("STMF_C5_SPAN")) if (atoi(e) != ln_sp && atoi(e) >= kLnMinSpan && n % atoi(e) == 0) continue;
      nsp = n / ln_sp; nch = nrc * nsp;
      tcnt.alloc(nch + 1); toff.alloc(nch + 1); lnmax.alloc(1);
      CK(cudaMemsetAsync(tcnt.p + nch, 0, sizeof(int64_t), st));
      CK(cudaMemsetAsync(lnmax.p, 0, sizeof(int), st));
      k_ln_count<<<gb, 256, 0, st>>>(m, n, ln_sp, M.p, tcnt.p, lnmax.p); LAUNCH_CK();
      CK(cudaMemcpyAsync(&maxrec, lnmax.p, sizeof(int), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      vbytes = sizeof(float4) * rq * ln_sp;
      budget = per_block > vbytes ? per_block - vbytes : 0;
      if ((size_t)kLnWarps * ln_stages * std::max(maxrec, 128) <= budget || ln_sp == kLnMinSpan || getenv("STMF_C5_SPAN")) break;
    }
    size_t tb = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, tcnt.p, toff.p, nch + 1, st));
    DevBuf<uint8_t> tmp;
    tmp.alloc(tb);
    CK(cub::DeviceScan::ExclusiveSum(tmp.p, tb, tcnt.p, toff.p, nch + 1, st));
    CK(cudaMemcpyAsync(&units, toff.p + nch, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    ln_bytes = units * 16;
    lnrecs.alloc((size_t)std::max<int64_t>(ln_bytes, 16));
    CK(cudaMemsetAsync(lnrecs.p, 0, lnrecs.n, st));
    k_ln_fill<<<gb, 256, 0, st>>>(m, n, ln_sp, M.p, X.p, toff.p, lnrecs.p); LAUNCH_CK();
    Urm.alloc((size_t)m * RS); Vrm.alloc((size_t)n * RS);
    k_sp_factor<<<nblk(m * RS, 256), 256, 0, st>>>(m, r, RS, Ut.p, Urm.p); LAUNCH_CK();
    k_sp_factor<<<nblk(n * RS, 256), 256, 0, st>>>(n, r, RS, V.p, Vrm.p); LAUNCH_CK();
    // one record in flight per warp and stage
    ln_cap = std::max(maxrec, 128);
    if ((size_t)kLnWarps * ln_stages * ln_cap > budget) ln_cap = std::max<int>(128, (int)(budget / (kLnWarps * ln_stages)) & ~15);
    const void* kf = (const void*)lanes_kernel(rq, ln_sp);
    if (!kf) fail(STMF_ERR_INVALID, "no lane-coded kernel for rank %d, span %d", r, ln_sp);
    ln_smem = vbytes + (size_t)kLnWarps * ln_stages * ln_cap;
    CK(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ln_smem));
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kf, 32 * kLnWarps, ln_smem));
    per_sm = std::max(per_sm, 1);
    // chunks per warp run: 4 (measured: 0.630 ms vs 0.634 with 8 at 65536^2, shorter runs balance the
    // warps better) when that still gives every resident warp a run
    int cpw = 4;
    if (const char* e = getenv("STMF_C5_CPW")) cpw = std::max(1, atoi(e));
    while (cpw > 1 && (nrc % cpw || (nrc / cpw) * nsp < (int64_t)prop.multiProcessorCount * per_sm * kLnWarps)) cpw /= 2;
    while ((1 << ln_cpw_log2) < cpw) ln_cpw_log2++;
    const int64_t nruns = nrc >> ln_cpw_log2;
    int64_t K = std::max<int64_t>(1, ((int64_t)prop.multiProcessorCount * per_sm) / nsp);
    K = std::min<int64_t>(K, (nruns + kLnWarps - 1) / kLnWarps);
    sgrid = (unsigned)(K * nsp);
    given_h = 1;
    CK(cudaStreamSynchronize(st));
    if (getenv("STMF_C5_VERBOSE"))
      fprintf(stderr, "[stmf c5] lane-coded layout: %lld chunks, records %lld bytes (+ %lld of offsets), largest %d, "
              "span %d, stages %d x %d B, cpw %d, grid %u x 512, %d blocks/SM, smem %zu\n", (long long)nch,
              (long long)ln_bytes, (long long)(nch + 1) * 8, maxrec, ln_sp, ln_stages, ln_cap, cpw, sgrid, per_sm, ln_smem);
  } else if (layout == 1) {
    int RS = sp_stride(rq);
    int64_t T = (m / kSpT) * (n / kSpT);
    tcnt.alloc(T + 1); toff.alloc(T + 1);
    CK(cudaMemsetAsync(tcnt.p + T, 0, sizeof(int64_t), st));
    k_sp_tile_count<<<gb, 256, 0, st>>>(m, n, M.p, tcnt.p); LAUNCH_CK();
    size_t tb = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, tcnt.p, toff.p, T + 1, st));
    DevBuf<uint8_t> tmp;
    tmp.alloc(tb);
    CK(cub::DeviceScan::ExclusiveSum(tmp.p, tb, tcnt.p, toff.p, T + 1, st));
    CK(cudaMemcpyAsync(&given_h, toff.p + T, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    vals.alloc(std::max<u64>(given_h, 1));
    k_sp_tile_fill<<<gb, 256, 0, st>>>(m, n, M.p, X.p, toff.p, vals.p); LAUNCH_CK();
    Urm.alloc((size_t)m * RS); Vrm.alloc((size_t)n * RS);
    k_sp_factor<<<nblk(m * RS, 256), 256, 0, st>>>(m, r, RS, Ut.p, Urm.p); LAUNCH_CK();
    k_sp_factor<<<nblk(n * RS, 256), 256, 0, st>>>(n, r, RS, V.p, Vrm.p); LAUNCH_CK();
    const void* kf = rq == 1 ? (const void*)k_maxplus_err_sampled<1> : rq == 2 ? (const void*)k_maxplus_err_sampled<2>
                   : rq == 4 ? (const void*)k_maxplus_err_sampled<4> : rq == 8 ? (const void*)k_maxplus_err_sampled<8>
                   : (const void*)k_maxplus_err_sampled<16>;
    const void* kfs = rq == 1 ? (const void*)k_maxplus_err_sampled<1, true>
                    : rq == 2 ? (const void*)k_maxplus_err_sampled<2, true>
                    : rq == 4 ? (const void*)k_maxplus_err_sampled<4, true>
                    : rq == 8 ? (const void*)k_maxplus_err_sampled<8, true> : (const void*)k_maxplus_err_sampled<16, true>;
    size_t smem = rq == 1 ? sp_smem_bytes<1>() : rq == 2 ? sp_smem_bytes<2>() : rq == 4 ? sp_smem_bytes<4>()
                : rq == 8 ? sp_smem_bytes<8>() : sp_smem_bytes<16>();
    CK(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CK(cudaFuncSetAttribute(kfs, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kf, 256, smem));
    sgrid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(T, (int64_t)prop.multiProcessorCount * std::max(per_sm, 1)));
    CK(cudaStreamSynchronize(st));
  }
  double total = 0, best = 1e30;
  u64 h[2] = {0, 0};
  for (int rep = 0; rep < std::max(reps, 1); rep++) {
    if (flush) CK(cudaMemsetAsync(scratch.p, rep & 0xff, scratch.n, st));
    CK(cudaMemsetAsync(acc.p, 0, 2 * sizeof(u64), st));
    CK(cudaMemsetAsync(flags.p, 0, sizeof(int), st));
    CK(cudaEventRecord(e0, st));
    if (layout == 1 && lanes) {
      lanes_kernel(rq, ln_sp)<<<sgrid, 32 * kLnWarps, ln_smem, st>>>(m, n, lnrecs.p, toff.p, Urm.p, Vrm.p, acc.p, flags.p,
                                                                     F, exact_limit, ln_cpw_log2, ln_stages, ln_cap);
    } else if (layout == 1) {
      auto L = rq == 1 ? launch_sampled<1> : rq == 2 ? launch_sampled<2> : rq == 4 ? launch_sampled<4>
             : rq == 8 ? launch_sampled<8> : launch_sampled<16>;
      L(sgrid, st, m, n, M.p, vals.p, toff.p, Urm.p, Vrm.p, acc.p, flags.p, F, exact_limit);
    } else if (tma)
      kernt<<<grid, 256, kMaxplusDynSmem, st>>>(m, n, r, X.p, M.p, Ut.p, V.p, acc.p, flags.p, F, exact_limit, xmap,
                                                umap, vmap);
    else
      kern<<<grid, 256, kMaxplusDynSmem, st>>>(m, n, r, X.p, M.p, Ut.p, V.p, acc.p, flags.p, F, exact_limit, xmap,
                                               umap, vmap);
    LAUNCH_CK();
    CK(cudaEventRecord(e1, st));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    total += ms;
    best = std::min(best, (double)ms);
  }
  int hf = 0;
  u64 given = 0;
  CK(cudaMemcpyAsync(h, acc.p, 2 * sizeof(u64), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&hf, flags.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&given, cnt.p, sizeof(u64), cudaMemcpyDeviceToHost, st));
  if (X_out) CK(cudaMemcpyAsync(X_out, X.p, sizeof(float) * m * n, cudaMemcpyDeviceToHost, st));
  if (mask_out) CK(cudaMemcpyAsync(mask_out, M.p, sizeof(uint32_t) * words, cudaMemcpyDeviceToHost, st));
  if (U_out) CK(cudaMemcpyAsync(U_out, Ut.p, sizeof(float) * r * m, cudaMemcpyDeviceToHost, st));
  if (V_out) CK(cudaMemcpyAsync(V_out, V.p, sizeof(float) * r * n, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaStreamDestroy(st);
  if (hf & 6) fail(STMF_ERR_NUMERIC, "exact objective window violated (flags %d)", hf);
  double avg = total / std::max(reps, 1);
  // algorithmic bytes: dense tiles read every value; the sampled layout only the given ones
  double bytes = (layout == 1 ? (double)given * 4.0 : (double)m * n * 4.0) + (double)words * 4.0 +
                 (double)r * (m + n) * 4.0;
  out[0] = avg;
  out[1] = best;
  out[2] = fx_to_double(h[1], h[0], F);
  out[3] = (double)given;
  out[4] = bytes / (avg * 1e-3) / 1e9;                    // algorithmic GB/s
  out[5] = (double)(layout == 1 ? given : m * n) * r / (avg * 1e-3) / 1e9;  // G computed (entry, k) pairs / s
  out[6] = layout == 1 && lanes ? 2 : layout;
  out[7] = bytes;
}

struct stmf_session {
  SessionBase* impl;
};

// contiguous row blocks with about equal given counts
static std::vector<int64_t> balanced_row_starts(const std::vector<int64_t>& nnz, int G) {
  int64_t m = (int64_t)nnz.size(), N = 0;
  for (auto v : nnz) N += v;
  std::vector<int64_t> starts(G + 1, 0);
  starts[G] = m;
  int64_t acc = 0, r = 0;
  for (int s = 1; s < G; s++) {
    int64_t target = N * s / G;
    while (r < m - (G - s) && acc + nnz[r] <= target) acc += nnz[r++];
    r = std::max<int64_t>(r, starts[s - 1] + 1);
    starts[s] = r;
  }
  return starts;
}

static int validate_create(stmf_session** out, int dtype, int64_t m, int64_t n, int rank, const void* X,
                           const uint8_t* mask) {
  if (!out || !X || !mask) return set_err(STMF_ERR_INVALID, "null argument");
  if (m <= 0 || n <= 0) return set_err(STMF_ERR_INVALID, "empty matrix");
  if (rank < 1) return set_err(STMF_ERR_INVALID, "rank must be >= 1");
  if (rank > 255) return set_err(STMF_ERR_INVALID, "rank must be <= 255");
  if (m >= (1ll << 31) || n >= (1ll << 31)) return set_err(STMF_ERR_INVALID, "dimension too large");
  if (dtype != STMF_F64 && dtype != STMF_F32) return set_err(STMF_ERR_INVALID, "unknown dtype %d", dtype);
  return STMF_OK;
}

// ----------------------------------------------------------------------------
// C ABI

#define GUARD(body)                              \
  try {                                          \
    g_err.clear();                               \
    body;                                        \
    return STMF_OK;                              \
  } catch (const StmfError& e) {                 \
    return e.code;                               \
  } catch (const std::bad_alloc&) {              \
    return set_err(STMF_ERR_OOM, "host allocation failed"); \
  }

// every session entry point runs on the session's device (restored on return)
struct DevScope {
  int prev = -1;
  explicit DevScope(int d) {
    if (cudaGetDevice(&prev) == cudaSuccess && prev != d) cudaSetDevice(d);
    else prev = -1;
  }
  ~DevScope() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};
#define NEED(s)                                                         \
  if (!(s) || !(s)->impl) return set_err(STMF_ERR_INVALID, "null session"); \
  DevScope dev_scope_((s)->impl->device_id())

template <typename T>
static void trop_matmul_impl(int64_t m, int rank, int64_t n, const void* U, const void* V, void* P, int32_t* arg,
                             int device) {
  CK(cudaSetDevice(device));
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  DevBuf<T> dU, dV, dP;
  DevBuf<int32_t> dA;
  dU.alloc((size_t)m * rank); dV.alloc((size_t)rank * n);
  if (P) dP.alloc((size_t)m * n);
  if (arg) dA.alloc((size_t)m * n);
  CK(cudaMemcpyAsync(dU.p, U, sizeof(T) * m * rank, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(dV.p, V, sizeof(T) * rank * n, cudaMemcpyHostToDevice, st));
  dim3 grid((unsigned)((n + 31) / 32), (unsigned)((m + 7) / 8));
  k_maxplus_dense<T><<<grid, dim3(32, 8), 0, st>>>(m, rank, n, dU.p, dV.p, dP.p, dA.p);
  LAUNCH_CK();
  if (P) CK(cudaMemcpyAsync(P, dP.p, sizeof(T) * m * n, cudaMemcpyDeviceToHost, st));
  if (arg) CK(cudaMemcpyAsync(arg, dA.p, sizeof(int32_t) * m * n, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  cudaStreamDestroy(st);
}

// ---- evaluation step: rmse, distance correlation ----------
template <typename E>
static void upload_vec(DevBuf<E>& d, const std::vector<E>& h, cudaStream_t st) {
  d.alloc(std::max<size_t>(h.size(), 1));
  if (!h.empty()) CK(cudaMemcpyAsync(d.p, h.data(), sizeof(E) * h.size(), cudaMemcpyHostToDevice, st));
}

// numpy's DOUBLE_pairwise_sum of a[0, len) (device array), len >= 1
static double device_pairwise_sum(const double* a, int64_t len, cudaStream_t st) {
  PWTree t;
  t.build(len);
  if (t.lvl_nodes.empty()) t.lvl_nodes.push_back(0);
  DevBuf<int64_t> loff;
  DevBuf<int32_t> llen, lnode, left, right, lvloff, lvlnodes;
  upload_vec(loff, t.loff, st); upload_vec(llen, t.llen, st); upload_vec(lnode, t.lnode, st);
  upload_vec(left, t.left, st); upload_vec(right, t.right, st); upload_vec(lvloff, t.lvl_off, st);
  upload_vec(lvlnodes, t.lvl_nodes, st);
  DevBuf<double> val;
  val.alloc(t.nnodes);
  int nl = (int)t.loff.size();
  k_pw_leaves8<<<nblk((int64_t)nl * 8, 256), 256, 0, st>>>(nl, loff.p, llen.p, lnode.p,
                                                          reinterpret_cast<const u64*>(a), val.p);
  LAUNCH_CK();
  if (t.H > 0) {
    k_pw_combine<<<1, 1024, 0, st>>>(t.H, lvloff.p, lvlnodes.p, left.p, right.p, val.p);
    LAUNCH_CK();
  }
  double r = 0;
  CK(cudaMemcpyAsync(&r, val.p, sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return r;
}

struct ScopedStream {
  cudaStream_t st = nullptr;
  explicit ScopedStream(int device) {
    CK(cudaSetDevice(device));
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  }
  ~ScopedStream() { if (st) cudaStreamDestroy(st); }
};

// rmse(pred, truth, mask) = sqrt(mean((pred - truth)[mask] ** 2)), 0 if empty (metrics.py:87-95)
static double masked_rmse_impl(int64_t m, int64_t n, const double* pred, const double* truth, const uint8_t* mask,
                               int device) {
  ScopedStream S(device);
  cudaStream_t st = S.st;
  DevBuf<double> dp, dt, sq;
  DevBuf<uint8_t> dm;
  DevBuf<int64_t> rc, ptr;
  dp.alloc((size_t)(m * n)); dt.alloc((size_t)(m * n)); dm.alloc((size_t)(m * n));
  rc.alloc(m); ptr.alloc(m + 1);
  CK(cudaMemcpyAsync(dp.p, pred, sizeof(double) * m * n, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(dt.p, truth, sizeof(double) * m * n, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(dm.p, mask, (size_t)(m * n), cudaMemcpyHostToDevice, st));
  k_count_rows<<<nblk(m * 32, 256), 256, 0, st>>>(m, n, dm.p, rc.p);
  LAUNCH_CK();
  k_scan_ptr<<<1, 1024, 0, st>>>(m, rc.p, ptr.p);
  LAUNCH_CK();
  int64_t N = 0;
  CK(cudaMemcpyAsync(&N, ptr.p + m, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (N == 0) return 0.0;
  sq.alloc(N);
  k_masked_sqdiff<<<nblk(m * 32, 256), 256, 0, st>>>(m, n, dp.p, dt.p, dm.p, ptr.p, sq.p);
  LAUNCH_CK();
  return std::sqrt(device_pairwise_sum(sq.p, N, st) / (double)N);
}

// _centered_distances(x) (metrics.py:120-123) into A (n x n)
static void centered_distances(int64_t n, const double* dx, DevBuf<double>& A, cudaStream_t st) {
  A.alloc((size_t)(n * n));
  unsigned g = nblk(n * n, 256);
  k_absdiff<<<g, 256, 0, st>>>(n, dx, A.p);
  LAUNCH_CK();
  DevBuf<double> cm, rm, scratch;
  cm.alloc(n); rm.alloc(n);
  k_colmean_seq<<<nblk(n, 128), 128, 0, st>>>(n, A.p, cm.p);
  LAUNCH_CK();
  PWTree t;
  t.build(n);
  if (t.lvl_nodes.empty()) t.lvl_nodes.push_back(0);
  DevBuf<int64_t> loff;
  DevBuf<int32_t> llen, lnode, left, right, lvloff, lvlnodes;
  upload_vec(loff, t.loff, st); upload_vec(llen, t.llen, st); upload_vec(lnode, t.lnode, st);
  upload_vec(left, t.left, st); upload_vec(right, t.right, st); upload_vec(lvloff, t.lvl_off, st);
  upload_vec(lvlnodes, t.lvl_nodes, st);
  unsigned nb = (unsigned)std::min<int64_t>(n, 1024);
  scratch.alloc((size_t)nb * t.nnodes);
  k_rowmean_pw<<<nb, 256, 0, st>>>(n, n, A.p, (int)t.loff.size(), loff.p, llen.p, lnode.p, t.H, lvloff.p, lvlnodes.p,
                                   left.p, right.p, t.nnodes, scratch.p, rm.p);
  LAUNCH_CK();
  double tm = device_pairwise_sum(A.p, n * n, st) / (double)(n * n);
  k_center<<<g, 256, 0, st>>>(n, A.p, cm.p, rm.p, tm);
  LAUNCH_CK();
  CK(cudaStreamSynchronize(st));
}

// b_norm(W, mask) (tropical.py:197-211): numpy's pairwise sum of the ascending
// |values|; |v| >= 0, so the bit patterns sort like the values (CUB radix sort)
__global__ void k_abs_bits(int64_t n, const double* __restrict__ v, u64* __restrict__ out) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < n) out[t] = (u64)__double_as_longlong(fabs(v[t]));
}

static double b_norm_impl(int64_t n, const double* vals, int device) {
  ScopedStream S(device);
  cudaStream_t st = S.st;
  DevBuf<double> dv;
  DevBuf<u64> a, b;
  dv.alloc(n); a.alloc(n); b.alloc(n);
  CK(cudaMemcpyAsync(dv.p, vals, sizeof(double) * n, cudaMemcpyHostToDevice, st));
  k_abs_bits<<<nblk(n, 256), 256, 0, st>>>(n, dv.p, a.p);
  LAUNCH_CK();
  size_t bytes = 0;
  CK(cub::DeviceRadixSort::SortKeys(nullptr, bytes, a.p, b.p, n, 0, 63, st));
  DevBuf<uint8_t> tmp;
  tmp.alloc(bytes);
  CK(cub::DeviceRadixSort::SortKeys(tmp.p, bytes, a.p, b.p, n, 0, 63, st));
  g_cub_calls++;
  return device_pairwise_sum(reinterpret_cast<const double*>(b.p), n, st);
}

// distance_correlation(x, y) (metrics.py:98-117)
static double distance_correlation_impl(int64_t n, const double* x, const double* y, int device) {
  ScopedStream S(device);
  cudaStream_t st = S.st;
  DevBuf<double> dx, dy, A, B, P;
  dx.alloc(n); dy.alloc(n);
  CK(cudaMemcpyAsync(dx.p, x, sizeof(double) * n, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(dy.p, y, sizeof(double) * n, cudaMemcpyHostToDevice, st));
  centered_distances(n, dx.p, A, st);
  centered_distances(n, dy.p, B, st);
  int64_t nn = n * n;
  P.alloc((size_t)nn);
  unsigned g = nblk(nn, 256);
  auto mean_prod = [&](const double* a, const double* b) {
    k_mul<<<g, 256, 0, st>>>(nn, a, b, P.p);
    LAUNCH_CK();
    return device_pairwise_sum(P.p, nn, st) / (double)nn;
  };
  double dvar_x = mean_prod(A.p, A.p), dvar_y = mean_prod(B.p, B.p);
  if (dvar_x <= 0.0 || dvar_y <= 0.0) return 0.0;
  double dcov2 = std::max(mean_prod(A.p, B.p), 0.0);
  return std::sqrt(dcov2 / std::sqrt(dvar_x * dvar_y));
}

extern "C" {

const char* stmf_last_error(void) { return g_err.c_str(); }

const char* stmf_version(void) { return "stmf_b200 0.1.0 (sm_100a)"; }

int stmf_create(stmf_session** out, int dtype, int64_t m, int64_t n, int rank, const void* X,
                const uint8_t* mask, int device) {
  if (!out || !X || !mask) return set_err(STMF_ERR_INVALID, "null argument");
  if (m <= 0 || n <= 0) return set_err(STMF_ERR_INVALID, "empty matrix");
  if (rank < 1) return set_err(STMF_ERR_INVALID, "rank must be >= 1");
  if (rank > 255) return set_err(STMF_ERR_INVALID, "rank must be <= 255");
  if (m >= (1ll << 31) || n >= (1ll << 31)) return set_err(STMF_ERR_INVALID, "dimension too large");
  if (dtype != STMF_F64 && dtype != STMF_F32) return set_err(STMF_ERR_INVALID, "unknown dtype %d", dtype);
  *out = nullptr;
  SessionBase* impl = nullptr;
  try {
    g_err.clear();
    if (dtype == STMF_F64) {
      auto* s = new Session<double>();
      impl = s;
      s->dtype = dtype;
      s->init(m, n, rank, (const double*)X, mask, device);
    } else {
      auto* s = new Session<float>();
      impl = s;
      s->dtype = dtype;
      s->init(m, n, rank, (const float*)X, mask, device);
    }
  } catch (const StmfError& e) {
    delete impl;
    return e.code;
  } catch (const std::bad_alloc&) {
    delete impl;
    return set_err(STMF_ERR_OOM, "host allocation failed");
  }
  *out = new stmf_session{impl};
  return STMF_OK;
}

int stmf_bench_maxplus(int64_t m, int64_t n, int rank, double density, uint64_t seed, int reps, int flush_l2,
                       int device, double* out6, float* X_out, uint32_t* mask_out, float* U_out, float* V_out) {
  if (!out6) return set_err(STMF_ERR_INVALID, "null output");
  double o[8];
  GUARD({
    maxplus_bench_impl(m, n, rank, density, seed, reps, flush_l2, device, o, X_out, mask_out, U_out, V_out, 0);
    memcpy(out6, o, sizeof(double) * 6);
  });
}

int stmf_bench_maxplus_layout(int64_t m, int64_t n, int rank, double density, uint64_t seed, int reps, int flush_l2,
                              int device, int layout, double* out8, float* X_out, uint32_t* mask_out, float* U_out,
                              float* V_out) {
  if (!out8) return set_err(STMF_ERR_INVALID, "null output");
  if (layout < -1 || layout > 2) return set_err(STMF_ERR_INVALID, "layout must be -1, 0, 1 or 2");
  GUARD(maxplus_bench_impl(m, n, rank, density, seed, reps, flush_l2, device, out8, X_out, mask_out, U_out, V_out,
                           layout));
}

int stmf_nccl_unique_id(void* out, int64_t* bytes) {
  if (!out || !bytes) return set_err(STMF_ERR_INVALID, "null argument");
  if (*bytes < (int64_t)sizeof(ncclUniqueId)) {
    *bytes = sizeof(ncclUniqueId);
    return set_err(STMF_ERR_INVALID, "buffer too small (%d bytes needed)", (int)sizeof(ncclUniqueId));
  }
  GUARD({
    ncclUniqueId id;
    NCK(NcclApi::get().GetUniqueId(&id));
    memcpy(out, &id, sizeof id);
    *bytes = sizeof id;
  });
}

int stmf_create_sharded(stmf_session** out, int dtype, int64_t m, int64_t n, int rank, const int64_t* row_starts,
                        const int64_t* row_nnz, const void* X_rows, const uint8_t* mask_rows, int world,
                        int shard, const void* nccl_id, int device) {
  int rc = validate_create(out, dtype, m, n, rank, X_rows, mask_rows);
  if (rc) return rc;
  if (dtype != STMF_F32) return set_err(STMF_ERR_INVALID, "sharded fits use binary32 (STMF_F32)");
  if (!row_starts || !row_nnz || world < 1 || shard < 0 || shard >= world)
    return set_err(STMF_ERR_INVALID, "bad shard layout");
  if (world > 1 && !nccl_id) return set_err(STMF_ERR_INVALID, "nccl_id required for world > 1");
  *out = nullptr;
  ShardGroup<float>* g = nullptr;
  try {
    g_err.clear();
    std::vector<int64_t> starts(row_starts, row_starts + world + 1), nnz(row_nnz, row_nnz + m);
    if (starts[0] != 0 || starts[world] != m) fail(STMF_ERR_INVALID, "row_starts must span [0, m]");
    for (int s = 0; s < world; s++)
      if (starts[s + 1] <= starts[s]) fail(STMF_ERR_INVALID, "empty shard %d", s);
    CK(cudaSetDevice(device));
    // an NCCL communicator whenever an id is given (world 1 included: the single-rank
    // communicator runs the same collective calls), else the trivial local group
    Comm* c = nccl_id ? (Comm*)new NcclComm(world, shard, nccl_id) : (Comm*)new LocalComm(1);
    g = new ShardGroup<float>();
    g->dtype = dtype;
    g->init(m, n, rank, starts, nnz, (const float*)X_rows, mask_rows, c, device);
  } catch (const StmfError& e) {
    delete g;
    return e.code;
  } catch (const std::bad_alloc&) {
    delete g;
    return set_err(STMF_ERR_OOM, "host allocation failed");
  }
  *out = new stmf_session{g};
  return STMF_OK;
}

int stmf_create_sim_group(stmf_session** out, int dtype, int64_t m, int64_t n, int rank, const void* X,
                          const uint8_t* mask, int shards, int device) {
  int rc = validate_create(out, dtype, m, n, rank, X, mask);
  if (rc) return rc;
  if (dtype != STMF_F32) return set_err(STMF_ERR_INVALID, "sharded fits use binary32 (STMF_F32)");
  if (shards < 1 || shards > m) return set_err(STMF_ERR_INVALID, "bad shard count %d", shards);
  *out = nullptr;
  ShardGroup<float>* g = nullptr;
  try {
    g_err.clear();
    std::vector<int64_t> nnz(m, 0);
    for (int64_t i = 0; i < m; i++)
      for (int64_t j = 0; j < n; j++) nnz[i] += mask[i * n + j] != 0;
    for (int64_t i = 0; i < m; i++)
      if (!nnz[i]) fail(STMF_ERR_INVALID, "row %lld has no given entries", (long long)i);
    std::vector<int64_t> starts = balanced_row_starts(nnz, shards);
    CK(cudaSetDevice(device));
    g = new ShardGroup<float>();
    g->dtype = dtype;
    g->init(m, n, rank, starts, nnz, (const float*)X, mask, new LocalComm(shards), device);
  } catch (const StmfError& e) {
    delete g;
    return e.code;
  } catch (const std::bad_alloc&) {
    delete g;
    return set_err(STMF_ERR_OOM, "host allocation failed");
  }
  *out = new stmf_session{g};
  return STMF_OK;
}

int stmf_destroy(stmf_session* s) {
  if (!s) return STMF_OK;
  double t0 = now_s();
  {
    DevScope dev_scope_(s->impl ? s->impl->device_id() : 0);
    delete s->impl;
  }
  delete s;
  if (getenv("STMF_TRACE_TEARDOWN")) fprintf(stderr, "[stmf teardown] total %.2f ms\n", (now_s() - t0) * 1e3);
  return STMF_OK;
}

int stmf_info(stmf_session* s, int64_t* out5) {
  NEED(s);
  GUARD(s->impl->info(out5));
}

int stmf_set_factors(stmf_session* s, const void* U, const void* V) {
  NEED(s);
  if (!U) return set_err(STMF_ERR_INVALID, "U is required");
  GUARD(s->impl->set_factors(U, V));
}

int stmf_get_factors(stmf_session* s, void* U, void* V) {
  NEED(s);
  GUARD(s->impl->get_factors(U, V));
}

int stmf_objective(stmf_session* s, double* err) {
  NEED(s);
  GUARD(*err = s->impl->objective());
}

int stmf_run(stmf_session* s, int64_t budget_sweeps, double budget_seconds, double epsilon, double* traj_t,
             double* traj_err, int64_t traj_cap, int64_t* counts) {
  NEED(s);
  if (!counts || (!traj_t) != (!traj_err)) return set_err(STMF_ERR_INVALID, "null output buffer");
  if (epsilon < 0) return set_err(STMF_ERR_INVALID, "epsilon must be >= 0");
  GUARD(s->impl->run(budget_sweeps, budget_seconds, epsilon, traj_t, traj_err, traj_cap, counts));
}

int stmf_replayed_sweeps(stmf_session* s, int64_t* n) {
  NEED(s);
  if (!n) return set_err(STMF_ERR_INVALID, "null argument");
  GUARD(*n = s->impl->replayed_sweeps());
}

int stmf_set_max_attempts(stmf_session* s, int64_t max_attempts) {
  NEED(s);
  GUARD(s->impl->set_max_attempts(max_attempts));
}

int stmf_comm_info(stmf_session* s, int* out3) {
  NEED(s);
  if (!out3) return set_err(STMF_ERR_INVALID, "null argument");
  GUARD(s->impl->comm_info(out3));
}

int stmf_set_audit(stmf_session* s, int on) {
  NEED(s);
  GUARD(s->impl->set_audit(on));
}

int stmf_trajectory(stmf_session* s, double* traj_t, double* traj_err, int64_t cap, int64_t* len) {
  NEED(s);
  if (!len) return set_err(STMF_ERR_INVALID, "null argument");
  GUARD(s->impl->trajectory(traj_t, traj_err, cap, len));
}

int stmf_product_given(stmf_session* s, void* P, int32_t* arg, void* top2) {
  NEED(s);
  GUARD(s->impl->product_given(P, arg, top2));
}

int stmf_col_scores(stmf_session* s, double* scores) {
  NEED(s);
  GUARD(s->impl->col_scores(scores));
}

int stmf_residuate(stmf_session* s, int axis, const void* vec, void* out) {
  NEED(s);
  if (axis != 0 && axis != 1) return set_err(STMF_ERR_INVALID, "axis must be 0 or 1");
  GUARD(s->impl->residuate(axis, vec, out));
}

int stmf_try_update(stmf_session* s, int op, int64_t i, int64_t j, int k, void* ucol, void* vrow, double* f) {
  NEED(s);
  if (op != 0 && op != 1) return set_err(STMF_ERR_INVALID, "op must be 0 (F-ULF) or 1 (F-URF)");
  GUARD(s->impl->try_update(op, i, j, k, ucol, vrow, f, false, nullptr));
}

int stmf_attempt(stmf_session* s, int op, int64_t i, int64_t j, int k, double* f, int* accepted) {
  NEED(s);
  if (op != 0 && op != 1) return set_err(STMF_ERR_INVALID, "op must be 0 (F-ULF) or 1 (F-URF)");
  GUARD(s->impl->try_update(op, i, j, k, nullptr, nullptr, f, true, accepted));
}

int stmf_set_strategy(stmf_session* s, int family, int selection) {
  NEED(s);
  GUARD(s->impl->set_strategy(family, selection));
}

int stmf_row_scores(stmf_session* s, double* scores) {
  NEED(s);
  if (!scores) return set_err(STMF_ERR_INVALID, "null argument");
  GUARD(s->impl->row_scores(scores));
}

int stmf_matrix_candidates(stmf_session* s, int32_t* rows, int32_t* cols, int32_t* ks, double* scores) {
  NEED(s);
  if (!rows || !cols || !ks) return set_err(STMF_ERR_INVALID, "null argument");
  GUARD(s->impl->matrix_candidates(rows, cols, ks, scores));
}

int stmf_masked_rmse(int64_t m, int64_t n, const double* pred, const double* truth, const uint8_t* mask,
                     int device, double* out) {
  if (!pred || !truth || !mask || !out) return set_err(STMF_ERR_INVALID, "null argument");
  if (m < 0 || n < 0) return set_err(STMF_ERR_INVALID, "bad shape");
  if (m == 0 || n == 0) { *out = 0.0; return STMF_OK; }
  GUARD(*out = masked_rmse_impl(m, n, pred, truth, mask, device));
}

int stmf_b_norm(int64_t n, const double* values, int device, double* out) {
  if (!out || (n > 0 && !values)) return set_err(STMF_ERR_INVALID, "null argument");
  if (n <= 0) { *out = 0.0; return STMF_OK; }
  GUARD(*out = b_norm_impl(n, values, device));
}

int stmf_distance_correlation(int64_t len, const double* x, const double* y, int device, double* out) {
  if (!x || !y || !out) return set_err(STMF_ERR_INVALID, "null argument");
  if (len < 2) return set_err(STMF_ERR_INVALID, "need at least two samples");
  GUARD(*out = distance_correlation_impl(len, x, y, device));
}

int stmf_release_memory(int device) {
  GUARD({
    cudaMemPool_t pool;
    CK(cudaSetDevice(device));
    CK(cudaDeviceSynchronize());
    CK(cudaDeviceGetDefaultMemPool(&pool, device));
    CK(cudaMemPoolTrimTo(pool, 0));
  });
}

int stmf_trop_matmul(int dtype, int64_t m, int rank, int64_t n, const void* U, const void* V, void* P,
                     int32_t* arg, int device) {
  if (!U || !V) return set_err(STMF_ERR_INVALID, "null argument");
  if (m <= 0 || n <= 0 || rank < 1) return set_err(STMF_ERR_INVALID, "bad shape");
  if (dtype == STMF_F64) { GUARD(trop_matmul_impl<double>(m, rank, n, U, V, P, arg, device)); }
  if (dtype == STMF_F32) { GUARD(trop_matmul_impl<float>(m, rank, n, U, V, P, arg, device)); }
  return set_err(STMF_ERR_INVALID, "unknown dtype %d", dtype);
}

int stmf_stream(stmf_session* s, void** stream) {
  NEED(s);
  GUARD(*stream = s->impl->stream());
}

int stmf_set_profiling(stmf_session* s, int on) {
  NEED(s);
  GUARD(s->impl->set_profiling(on));
}

int stmf_counters(stmf_session* s, int64_t* out8) {
  NEED(s);
  GUARD(s->impl->counters(out8));
}

int stmf_bench_product(stmf_session* s, int reps, int flush_l2, double* ms, double* err) {
  NEED(s);
  GUARD(s->impl->bench_product(reps, flush_l2, ms, err));
}

}  // extern "C"
