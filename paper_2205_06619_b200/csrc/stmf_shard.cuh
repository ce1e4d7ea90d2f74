// stmf_shard.cuh — row-sharded FastSTMF engine, included by stmf_api.cu.
//
// The work-orientation rows are split into contiguous blocks, one per shard.
// A shard owns the CSR/CSC of its rows, its rows of U and a replica of V.
// Per row visit the owner broadcasts row i: given columns, values, TD_A row
// votes and U_i.  Column scores and TD_A column histograms are all-reduced exactly
// (int64 fixed point / int32).  Residuation statistics of the changed factor index
// are all-gathered and merged.  Per speculative batch:
//   F-ULF: phase A replicated (global statistics), phase B on local rows;
//   F-URF: phase A on local rows, local column minima -> all-reduce MIN -> error
//          pass on local entries;
//   error partials (128-bit fixed point, as 42-bit limbs) -> all-reduce SUM.
// Every reduction is exact, so decisions, factors and trajectories are identical
// for any number of shards (binary32 exact-sum semantics; fp64/numpy semantics is
// single-GPU only).
//
// Comm has two implementations: NCCL (one shard per process, one rank per GPU,
// libnccl dlopen'ed: the process already holds torch's copy) and an in-process
// group of G shards on one device whose collectives are kernels over the G
// buffers (the shard-invariance tests run on one B200 this way).
#pragma once
#include <dlfcn.h>

#include <nccl.h>

namespace stmf {

template <typename V>
__global__ void k_red_min_ptrs(V* const* __restrict__ bufs, int G, int64_t count) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= count) return;
  V v = bufs[0][t];
  for (int g = 1; g < G; g++) v = vmin(v, bufs[g][t]);
  for (int g = 0; g < G; g++) bufs[g][t] = v;
}

template <typename I>
__global__ void k_red_sum_ptrs(I* const* __restrict__ bufs, int G, int64_t count) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= count) return;
  I v = 0;
  for (int g = 0; g < G; g++) v += bufs[g][t];
  for (int g = 0; g < G; g++) bufs[g][t] = v;
}

// merge G shards' top-2 column statistics (shard order; exact)
template <typename T>
__global__ void k_stats_merge(int G, int64_t n, const T* __restrict__ m1s, const T* __restrict__ m2s,
                              const int32_t* __restrict__ a1s, T* __restrict__ m1, T* __restrict__ m2,
                              int32_t* __restrict__ a1) {
  int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= n) return;
  Top2<T> t;
  t.m1 = m1s[c]; t.m2 = m2s[c]; t.a1 = a1s[c];
  for (int g = 1; g < G; g++) {
    Top2<T> u;
    u.m1 = m1s[g * n + c]; u.m2 = m2s[g * n + c]; u.a1 = a1s[g * n + c];
    t = top2_merge(t, u);
  }
  m1[c] = t.m1; m2[c] = t.m2; a1[c] = t.a1;
}

// exact column scores <-> int64 fixed point (values are multiples of 2^-g, < 2^(53-g))
__global__ void k_score_to_fx(int64_t n, const double* __restrict__ s, int64_t* __restrict__ out, double scale) {
  int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c < n) out[c] = (int64_t)(s[c] * scale);
}
__global__ void k_fx_to_score(int64_t n, const int64_t* __restrict__ in, double* __restrict__ s, double inv) {
  int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c < n) s[c] = (double)in[c] * inv;
}

// 128-bit accumulators -> three 42-bit limbs (sums of < 2^21 shards cannot overflow)
__global__ void k_acc_to_limbs(int64_t count, const u64* __restrict__ acc, int64_t* __restrict__ limbs) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= count) return;
  u64 lo = acc[2 * t], hi = acc[2 * t + 1];
  const u64 M = (1ull << 42) - 1;
  limbs[3 * t] = (int64_t)(lo & M);
  limbs[3 * t + 1] = (int64_t)(((lo >> 42) | (hi << 22)) & M);
  limbs[3 * t + 2] = (int64_t)(hi >> 20);
}

// owner of row i packs its broadcast payload
template <typename T>
__global__ void k_pack_row(int64_t nc, int rank, int64_t ml, int64_t il, const int32_t* __restrict__ cols,
                           const T* __restrict__ x, const uint8_t* __restrict__ ag, const T* __restrict__ Ut,
                           int32_t* __restrict__ pcols, T* __restrict__ px, int32_t* __restrict__ prowhist,
                           T* __restrict__ purow, uint8_t* __restrict__ pag) {
  for (int l = threadIdx.x; l < rank; l += blockDim.x) prowhist[l] = 0;
  __syncthreads();
  for (int64_t p = threadIdx.x; p < nc; p += blockDim.x) {
    pcols[p] = cols[p];
    px[p] = x[p];
    pag[p] = ag[p];
    atomicAdd(&prowhist[ag[p]], 1);
  }
  for (int l = threadIdx.x; l < rank; l += blockDim.x) purow[l] = Ut[(int64_t)l * ml + il];
}

template <typename T>
__global__ void k_cand_build_h(int64_t nc, int rank, const int32_t* __restrict__ cols, const T* __restrict__ xrow,
                               const int32_t* __restrict__ rowhist, const int32_t* __restrict__ perm,
                               const int32_t* __restrict__ colhist, int32_t* __restrict__ cj,
                               int32_t* __restrict__ ck, T* __restrict__ cx) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= nc) return;
  int p = perm[t];
  int j = cols[p];
  const int32_t* h = colhist + (int64_t)j * rank;
  int k = 0, best = -1;
  for (int l = 0; l < rank; l++) {
    int v = rowhist[l] + h[l];
    if (v > best) { best = v; k = l; }
  }
  cj[t] = j; ck[t] = k; cx[t] = xrow[p];
}

// F-URF seed with U_ik from the broadcast row (the owner's Ut is not replicated)
template <typename T>
__global__ void k_phaseA_urf_seed_h(int64_t ml, int E, const int32_t* __restrict__ cj, const int32_t* __restrict__ ck,
                                    const T* __restrict__ cx, const T* __restrict__ urow,
                                    const int64_t* __restrict__ col_ptr, const int32_t* __restrict__ row_idx,
                                    const T* __restrict__ xc, T* __restrict__ uI) {
  int q = blockIdx.x;
  if (q >= E) return;
  int j = cj[q];
  T s = sub_rn(cx[q], urow[ck[q]]);
  T* u = uI + ilv_index<T>(q, 0, ml);
  for (int64_t p = col_ptr[j] + threadIdx.x; p < col_ptr[j + 1]; p += blockDim.x) {
    int64_t r = row_idx[p] * Ilv<T>::STRIDE;
    u[r] = vmin(u[r], sub_rn(xc[p], s));
  }
}

}  // namespace stmf

// ----------------------------------------------------------------------------
// collectives over the local shards of this process (+ other processes via NCCL)
struct Comm {
  virtual ~Comm() {}
  virtual int nlocal() = 0;
  virtual void min_f32(std::vector<float*>& b, size_t count, cudaStream_t st) = 0;
  virtual void sum_i64(std::vector<int64_t*>& b, size_t count, cudaStream_t st) = 0;
  virtual void sum_i32(std::vector<int32_t*>& b, size_t count, cudaStream_t st) = 0;
  virtual void max_i32_host(int* v) = 0;  // small host value
  // recv[s] receives world * bytes (shard order) from every shard's send[s]
  virtual void allgather(std::vector<void*>& send, std::vector<void*>& recv, size_t bytes, cudaStream_t st) = 0;
  // root = global shard index (LocalComm: global == local); b[s] of every local
  // shard receives root's bytes
  virtual void broadcast(std::vector<void*>& b, size_t bytes, int root, cudaStream_t st) = 0;
  virtual int world() = 0;
  virtual int first_shard() = 0;  // global index of local shard 0
  // ranks / this rank as the communicator reports them (NCCL: ncclCommCount /
  // ncclCommUserRank; the in-process group: its shard count / 0); kind 0 local, 1 NCCL
  virtual void info(int* nranks, int* me, int* kind) { *nranks = world(); *me = first_shard(); *kind = 0; }
};

struct LocalComm : Comm {
  int G;
  DevBuf<void*> ptrs;
  explicit LocalComm(int g) : G(g) { ptrs.alloc(g); }
  int nlocal() override { return G; }
  int world() override { return G; }
  int first_shard() override { return 0; }
  template <typename V>
  void upload(std::vector<V*>& b, cudaStream_t st) {
    CK(cudaMemcpyAsync(ptrs.p, b.data(), sizeof(void*) * G, cudaMemcpyHostToDevice, st));
  }
  void min_f32(std::vector<float*>& b, size_t count, cudaStream_t st) override {
    if (G == 1 || !count) return;
    upload(b, st);
    k_red_min_ptrs<float><<<nblk(count, 256), 256, 0, st>>>((float* const*)ptrs.p, G, (int64_t)count);
    LAUNCH_CK();
  }
  void sum_i64(std::vector<int64_t*>& b, size_t count, cudaStream_t st) override {
    if (G == 1 || !count) return;
    upload(b, st);
    k_red_sum_ptrs<int64_t><<<nblk(count, 256), 256, 0, st>>>((int64_t* const*)ptrs.p, G, (int64_t)count);
    LAUNCH_CK();
  }
  void sum_i32(std::vector<int32_t*>& b, size_t count, cudaStream_t st) override {
    if (G == 1 || !count) return;
    upload(b, st);
    k_red_sum_ptrs<int32_t><<<nblk(count, 256), 256, 0, st>>>((int32_t* const*)ptrs.p, G, (int64_t)count);
    LAUNCH_CK();
  }
  void max_i32_host(int*) override {}
  void allgather(std::vector<void*>& send, std::vector<void*>& recv, size_t bytes, cudaStream_t st) override {
    for (int d = 0; d < G; d++)
      for (int s = 0; s < G; s++)
        CK(cudaMemcpyAsync((char*)recv[d] + s * bytes, send[s], bytes, cudaMemcpyDeviceToDevice, st));
  }
  void broadcast(std::vector<void*>& b, size_t bytes, int root, cudaStream_t st) override {
    for (int s = 0; s < G; s++)
      if (s != root) CK(cudaMemcpyAsync(b[s], b[root], bytes, cudaMemcpyDeviceToDevice, st));
  }
};

// NCCL entry points resolved at runtime (libnccl.so.2 of the process — torch's)
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*CommCount)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*CommUserRank)(const ncclComm_t, int*) = nullptr;
  bool ok = false;
  static NcclApi& get() {
    static NcclApi a;
    if (!a.ok) {
      void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
      if (!h) fail(STMF_ERR_NCCL, "cannot load libnccl.so.2: %s", dlerror());
      a.GetUniqueId = (decltype(a.GetUniqueId))dlsym(h, "ncclGetUniqueId");
      a.CommInitRank = (decltype(a.CommInitRank))dlsym(h, "ncclCommInitRank");
      a.CommDestroy = (decltype(a.CommDestroy))dlsym(h, "ncclCommDestroy");
      a.AllReduce = (decltype(a.AllReduce))dlsym(h, "ncclAllReduce");
      a.AllGather = (decltype(a.AllGather))dlsym(h, "ncclAllGather");
      a.Broadcast = (decltype(a.Broadcast))dlsym(h, "ncclBroadcast");
      a.GetErrorString = (decltype(a.GetErrorString))dlsym(h, "ncclGetErrorString");
      a.CommCount = (decltype(a.CommCount))dlsym(h, "ncclCommCount");
      a.CommUserRank = (decltype(a.CommUserRank))dlsym(h, "ncclCommUserRank");
      if (!a.GetUniqueId || !a.CommInitRank || !a.AllReduce || !a.AllGather || !a.Broadcast)
        fail(STMF_ERR_NCCL, "libnccl.so.2 lacks required symbols");
      a.ok = true;
    }
    return a;
  }
};

#define NCK(call)                                                                       \
  do {                                                                                  \
    ncclResult_t r_ = (call);                                                           \
    if (r_ != ncclSuccess) fail(STMF_ERR_NCCL, "%s: %s", #call, NcclApi::get().GetErrorString(r_)); \
  } while (0)

struct NcclComm : Comm {
  ncclComm_t comm = nullptr;
  int W, R;
  DevBuf<int> tmp;
  NcclComm(int world, int rank, const void* id) : W(world), R(rank) {
    ncclUniqueId uid;
    memcpy(&uid, id, sizeof uid);
    NCK(NcclApi::get().CommInitRank(&comm, world, uid, rank));
    tmp.alloc(1);
  }
  ~NcclComm() override {
    if (comm) NcclApi::get().CommDestroy(comm);
  }
  int nlocal() override { return 1; }
  int world() override { return W; }
  int first_shard() override { return R; }
  void info(int* nranks, int* me, int* kind) override {
    if (!NcclApi::get().CommCount || !NcclApi::get().CommUserRank) fail(STMF_ERR_NCCL, "libnccl lacks ncclCommCount");
    NCK(NcclApi::get().CommCount(comm, nranks));
    NCK(NcclApi::get().CommUserRank(comm, me));
    *kind = 1;
  }
  void min_f32(std::vector<float*>& b, size_t count, cudaStream_t st) override {
    if (count) NCK(NcclApi::get().AllReduce(b[0], b[0], count, ncclFloat32, ncclMin, comm, st));
  }
  void sum_i64(std::vector<int64_t*>& b, size_t count, cudaStream_t st) override {
    if (count) NCK(NcclApi::get().AllReduce(b[0], b[0], count, ncclInt64, ncclSum, comm, st));
  }
  void sum_i32(std::vector<int32_t*>& b, size_t count, cudaStream_t st) override {
    if (count) NCK(NcclApi::get().AllReduce(b[0], b[0], count, ncclInt32, ncclSum, comm, st));
  }
  void max_i32_host(int* v) override {
    CK(cudaMemcpy(tmp.p, v, sizeof(int), cudaMemcpyHostToDevice));
    NCK(NcclApi::get().AllReduce(tmp.p, tmp.p, 1, ncclInt32, ncclMax, comm, 0));
    CK(cudaMemcpy(v, tmp.p, sizeof(int), cudaMemcpyDeviceToHost));
  }
  void allgather(std::vector<void*>& send, std::vector<void*>& recv, size_t bytes, cudaStream_t st) override {
    NCK(NcclApi::get().AllGather(send[0], recv[0], bytes, ncclUint8, comm, st));
  }
  void broadcast(std::vector<void*>& b, size_t bytes, int root, cudaStream_t st) override {
    NCK(NcclApi::get().Broadcast(b[0], b[0], bytes, ncclUint8, root, comm, st));
  }
};

// ----------------------------------------------------------------------------
template <typename T>
struct Shard {
  int64_t r0 = 0, ml = 0, Nl = 0;
  DevBuf<int64_t> row_ptr, col_ptr;
  DevBuf<int32_t> col_idx, row_idx;
  DevBuf<T> xr, xc;
  std::vector<int64_t> h_row_ptr;
  int64_t max_rownnz = 0;
  DevBuf<T> Ut, V;
  DevBuf<T> t1r, t2r, t1c, t2c;
  DevBuf<uint8_t> agr, agc, a2r, a2c;
  DevBuf<T> Urm, Vcm;  // row-major factor copies (ml x rp, n x rp) for the product passes
  DevBuf<int32_t> rowof_r, colof_c;
  DevBuf<int32_t> long_rows, long_cols;  // lines evaluated block-per-line
  int n_long_rows = 0, n_long_cols = 0;
  DevBuf<double> score;
  DevBuf<int64_t> scorefx;
  DevBuf<int32_t> colhist;
  DevBuf<T> cm1, cm2, rm1, rm2, lm1, lm2, gm1, gm2;
  DevBuf<int32_t> cmarg, rmarg, la1, ga1;
  DevBuf<uint8_t> rowbuf;
  DevBuf<u64> ckeys, ckeys2;
  DevBuf<int32_t> cvals, cperm, cj, ck;
  DevBuf<T> cx, xrow_dense, cmi;
  DevBuf<T> vbuf, ubufA, ubufB, vbufB, dtmpA, dtmpB;
  DevBuf<u64> acc;
  DevBuf<int64_t> limbs;
  DevBuf<int> chg, flags;
  DevBuf<uint8_t> cubtmp;
  size_t cubtmp_bytes = 0;
};

template <typename T>
struct ShardGroup : SessionBase {
  static_assert(sizeof(T) == 4, "sharded fits use binary32 exact-sum semantics");
  int dev = 0, nsm = 148;
  cudaStream_t st = nullptr;
  int64_t m = 0, n = 0;
  int rank = 0, W = 1;
  std::unique_ptr<Comm> comm;
  std::vector<std::unique_ptr<Shard<T>>> sh;
  std::vector<int64_t> row_start;  // W + 1 global row starts
  std::vector<int64_t> row_nnz;    // m global
  int Emax = 512;
  std::vector<int> batch_sched;
  int F = 0;
  double exact_limit = INFINITY;
  bool dirty = true, err_valid = false, have_factors = false;
  int cache_k = -1;  // >= 0: caches valid except for factor index cache_k
  int rp = 4;
  void sync_factor_copies(int k) {  // k < 0: all
    for (auto& s : sh)
      for (int l = (k < 0 ? 0 : k); l < (k < 0 ? rank : k + 1); l++) {
        k_scatter_factor<T><<<nblk(s->ml, 256), 256, 0, st>>>(s->ml, rp, l, s->Ut.p + (size_t)l * s->ml, s->Urm.p);
        LAUNCH_CK();
        k_scatter_factor<T><<<nblk(n, 256), 256, 0, st>>>(n, rp, l, s->V.p + (size_t)l * n, s->Vcm.p);
        LAUNCH_CK();
      }
  }
  std::vector<char> stats_dirty;
  double err = 0;
  u64* h_acc = nullptr;
  int64_t* h_limbs = nullptr;
  int* h_chg = nullptr;
  int* h_flags = nullptr;
  int64_t n_product_passes = 0;
  int unroll = getenv("STMF_UNROLL") ? atoi(getenv("STMF_UNROLL")) : 2;
  int64_t long_thr = getenv("STMF_LONG") ? atoll(getenv("STMF_LONG")) : 4096;
  int group_major = 0;
  size_t off_x = 0, off_h = 0, off_u = 0, off_ag = 0, rowbuf_bytes = 0;
  // adaptive speculation (as the single-device engine): the first batch of a row
  // covers scale x the candidates the row consumed on its previous visit (+ add),
  // floored by batch_floor; later batches grow by `growth`
  std::vector<int64_t> row_depth;
  int batch_floor = 1, sched_add = 1;
  double sched_scale = 0.9, sched_growth = 1.5;
  int e_round = getenv("STMF_EROUND") ? std::max(1, atoi(getenv("STMF_EROUND"))) : kEG;
  int gridX = -1000;

  ~ShardGroup() override {
    pinned_free(h_acc, sizeof(u64) * 4 * Emax);
    pinned_free(h_limbs, sizeof(int64_t) * 6 * Emax);
    pinned_free(h_chg, sizeof(int) * 2 * Emax);
    pinned_free(h_flags, sizeof(int) * 4);
    sh.clear();
    comm.reset();
    if (st) cudaStreamDestroy(st);
  }

  unsigned warps_grid(int64_t lines) const {
    int64_t blocks = (lines * 32 + 255) / 256;
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>(blocks, (int64_t)nsm * 16));
  }
  int nloc() const { return (int)sh.size(); }
  int owner(int64_t i) const {
    return (int)(std::upper_bound(row_start.begin(), row_start.end(), i) - row_start.begin()) - 1;
  }
  Shard<T>* local(int gs) {
    int l = gs - comm->first_shard();
    return (l >= 0 && l < nloc()) ? sh[l].get() : nullptr;
  }

  void info(int64_t* out) override {
    int64_t N = 0;
    for (auto v : row_nnz) N += v;
    out[0] = m; out[1] = n; out[2] = rank; out[3] = N; out[4] = dtype;
  }

  // shards: local row blocks [row_start[first + l], row_start[first + l + 1]) of X_rows
  void init(int64_t m_, int64_t n_, int rank_, const std::vector<int64_t>& starts, const std::vector<int64_t>& nnz,
            const T* X_rows, const uint8_t* mask_rows, Comm* c, int device) {
    m = m_; n = n_; rank = rank_;
    comm.reset(c);
    W = c->world();
    row_start = starts;
    row_nnz = nnz;
    dev = device;
    CK(cudaSetDevice(dev));
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, dev));
    nsm = prop.multiProcessorCount;
    int64_t N = 0;
    for (auto v : nnz) N += v;
    int b0 = (int)std::max<int64_t>(4, std::min<int64_t>(128, 120000000 / std::max<int64_t>(N, 1)));
    for (int b = b0; b < Emax; b *= 4) batch_sched.push_back(b);
    batch_sched.push_back(Emax);
    off_x = ((size_t)4 * n + 15) / 16 * 16;
    off_h = (off_x + sizeof(T) * n + 15) / 16 * 16;
    off_u = (off_h + 4 * (size_t)rank + 15) / 16 * 16;
    off_ag = (off_u + sizeof(T) * rank + 15) / 16 * 16;
    rowbuf_bytes = off_ag + (size_t)n;
    batch_floor = (int)std::max<int64_t>(1, std::min<int64_t>(128, 8000000 / std::max<int64_t>(N, 1)));
    if (batch_floor >= 8) { sched_scale = 1.5; sched_add = 4; sched_growth = 2.0; }
    else { sched_scale = 0.25; sched_add = 1; sched_growth = 1.15; }
    if (const char* e = getenv("STMF_SCHED")) sscanf(e, "%lf,%d,%lf", &sched_scale, &sched_add, &sched_growth);
    row_depth.assign(m, 0);
    const T* Xp = X_rows;
    const uint8_t* Mp = mask_rows;
    int first = c->first_shard();
    for (int l = 0; l < c->nlocal(); l++) {
      auto s = std::make_unique<Shard<T>>();
      s->r0 = starts[first + l];
      s->ml = starts[first + l + 1] - s->r0;
      build_shard(*s, Xp, Mp);
      Xp += s->ml * n;
      Mp += s->ml * n;
      sh.push_back(std::move(s));
    }
    pinned_alloc(&h_acc, sizeof(u64) * 4 * Emax);
    pinned_alloc(&h_limbs, sizeof(int64_t) * 6 * Emax);
    pinned_alloc(&h_chg, sizeof(int) * 2 * Emax);
    pinned_alloc(&h_flags, sizeof(int) * 4);
    {
      double nl = 0;
      for (auto& s : sh) nl += (double)s->Nl;
      group_major = 2.0 * nl * (3 * sizeof(T) + 5) < 0.5 * (double)prop.l2CacheSize ? 1 : 0;
      if (const char* e = getenv("STMF_GROUP_MAJOR")) group_major = atoi(e);
    }
    stats_dirty.assign(rank, 1);
    CK(cudaStreamSynchronize(st));
  }

  void build_shard(Shard<T>& s, const T* X, const uint8_t* mask) {
    int64_t ml = s.ml;
    if (ml <= 0) fail(STMF_ERR_INVALID, "empty shard");
    DevBuf<T> dX;
    DevBuf<uint8_t> dM;
    dX.alloc((size_t)(ml * n));
    dM.alloc((size_t)(ml * n));
    CK(cudaMemcpyAsync(dX.p, X, sizeof(T) * ml * n, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(dM.p, mask, (size_t)(ml * n), cudaMemcpyHostToDevice, st));
    DevBuf<int64_t> rc, cc;
    rc.alloc(ml); cc.alloc(n);
    s.row_ptr.alloc(ml + 1); s.col_ptr.alloc(n + 1);
    k_count_rows<<<nblk(ml * 32, 256), 256, 0, st>>>(ml, n, dM.p, rc.p); LAUNCH_CK();
    k_count_cols<<<nblk(n, 256), 256, 0, st>>>(ml, n, dM.p, cc.p); LAUNCH_CK();
    k_scan_ptr<<<1, 1024, 0, st>>>(ml, rc.p, s.row_ptr.p); LAUNCH_CK();
    k_scan_ptr<<<1, 1024, 0, st>>>(n, cc.p, s.col_ptr.p); LAUNCH_CK();
    s.h_row_ptr.resize(ml + 1);
    CK(cudaMemcpyAsync(s.h_row_ptr.data(), s.row_ptr.p, sizeof(int64_t) * (ml + 1), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    s.Nl = s.h_row_ptr[ml];
    if (s.Nl >= (1ll << 31)) fail(STMF_ERR_INVALID, "more than 2^31 - 1 given entries per shard");
    for (int64_t i = 0; i < ml; i++) {
      int64_t c = s.h_row_ptr[i + 1] - s.h_row_ptr[i];
      if (c != row_nnz[s.r0 + i]) fail(STMF_ERR_INVALID, "row %lld: given count mismatch", (long long)(s.r0 + i));
      if (c == 0) fail(STMF_ERR_INVALID, "row %lld has no given entries", (long long)(s.r0 + i));
      s.max_rownnz = std::max(s.max_rownnz, c);
    }
    int64_t Nl = std::max<int64_t>(s.Nl, 1);
    s.col_idx.alloc(Nl); s.row_idx.alloc(Nl); s.xr.alloc(Nl); s.xc.alloc(Nl);
    k_fill_csr<T><<<nblk(ml * 32, 256), 256, 0, st>>>(ml, n, dX.p, dM.p, s.row_ptr.p, s.col_idx.p, s.xr.p);
    LAUNCH_CK();
    {
      std::vector<int64_t> hcp(n + 1);
      CK(cudaMemcpyAsync(hcp.data(), s.col_ptr.p, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      std::vector<int32_t> lr, lc;
      for (int64_t i = 0; i < ml; i++)
        if (s.h_row_ptr[i + 1] - s.h_row_ptr[i] > long_thr) lr.push_back((int32_t)i);
      for (int64_t j = 0; j < n; j++)
        if (hcp[j + 1] - hcp[j] > long_thr) lc.push_back((int32_t)j);
      s.n_long_rows = (int)lr.size();
      s.n_long_cols = (int)lc.size();
      s.long_rows.alloc(std::max<size_t>(lr.size(), 1));
      s.long_cols.alloc(std::max<size_t>(lc.size(), 1));
      if (!lr.empty()) CK(cudaMemcpy(s.long_rows.p, lr.data(), 4 * lr.size(), cudaMemcpyHostToDevice));
      if (!lc.empty()) CK(cudaMemcpy(s.long_cols.p, lc.data(), 4 * lc.size(), cudaMemcpyHostToDevice));
    }
    s.rowof_r.alloc(Nl); s.colof_c.alloc(Nl);
    k_line_of<<<warps_grid(ml), 256, 0, st>>>(ml, s.row_ptr.p, s.rowof_r.p);
    LAUNCH_CK();
    k_line_of<<<warps_grid(n), 256, 0, st>>>(n, s.col_ptr.p, s.colof_c.p);
    LAUNCH_CK();
    k_fill_csc<T><<<nblk(n, 128), 128, 0, st>>>(ml, n, dX.p, dM.p, s.col_ptr.p, s.row_idx.p, s.xc.p);
    LAUNCH_CK();
    gridX = std::max(gridX, f32_grid_given(X, mask, ml * n));
    s.Ut.alloc((size_t)rank * ml); s.V.alloc((size_t)rank * n);
    s.t1r.alloc(Nl); s.t2r.alloc(Nl); s.agr.alloc(Nl); s.t1c.alloc(Nl); s.t2c.alloc(Nl); s.agc.alloc(Nl);
    s.a2r.alloc(Nl); s.a2c.alloc(Nl);
    rp = (rank + 3) / 4 * 4;
    s.Urm.alloc((size_t)ml * rp); s.Vcm.alloc((size_t)n * rp);
    CK(cudaMemsetAsync(s.Urm.p, 0, sizeof(T) * (size_t)ml * rp, st));
    CK(cudaMemsetAsync(s.Vcm.p, 0, sizeof(T) * (size_t)n * rp, st));
    s.score.alloc(n); s.scorefx.alloc(n); s.colhist.alloc((size_t)n * rank);
    s.cm1.alloc((size_t)rank * n); s.cm2.alloc((size_t)rank * n); s.cmarg.alloc((size_t)rank * n);
    s.rm1.alloc((size_t)rank * ml); s.rm2.alloc((size_t)rank * ml); s.rmarg.alloc((size_t)rank * ml);
    s.lm1.alloc(n); s.lm2.alloc(n); s.la1.alloc(n);
    s.gm1.alloc((size_t)W * n); s.gm2.alloc((size_t)W * n); s.ga1.alloc((size_t)W * n);
    s.rowbuf.alloc(rowbuf_bytes);
    s.ckeys.alloc(n); s.ckeys2.alloc(n); s.cvals.alloc(n); s.cperm.alloc(n);
    s.cj.alloc(n); s.ck.alloc(n); s.cx.alloc(n); s.xrow_dense.alloc(n); s.cmi.alloc((size_t)rank * n);
    s.vbuf.alloc((size_t)Emax * n); s.vbufB.alloc((size_t)Emax * n);
    s.ubufA.alloc((size_t)Emax * ml); s.ubufB.alloc((size_t)Emax * ml);
    s.dtmpA.alloc(ml); s.dtmpB.alloc(n);
    s.acc.alloc(4 * (size_t)Emax); s.limbs.alloc(6 * (size_t)Emax); s.chg.alloc(2 * (size_t)Emax); s.flags.alloc(4);
    size_t b1 = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, b1, s.ckeys.p, s.ckeys2.p, s.cvals.p, s.cperm.p, (int)n, 0, 64, st));
    s.cubtmp_bytes = b1;
    s.cubtmp.alloc(b1);
  }

  template <typename V_>
  std::vector<V_*> ptrs(DevBuf<V_> Shard<T>::*mem, size_t off = 0) {
    std::vector<V_*> v;
    for (auto& s : sh) v.push_back(((*s).*mem).p + off);
    return v;
  }

  void set_factors(const void* Uh, const void* Vh) override {
    const T* U = (const T*)Uh;
    int g = gridX;
    int64_t row = 0;
    for (auto& sp : sh) {
      Shard<T>& s = *sp;
      std::vector<T> ut((size_t)rank * s.ml);
      for (int64_t i = 0; i < s.ml; i++)
        for (int k = 0; k < rank; k++) {
          ut[(size_t)k * s.ml + i] = U[(row + i) * rank + k];
          g = std::max(g, f32_grid((float)U[(row + i) * rank + k]));
        }
      row += s.ml;
      CK(cudaMemcpyAsync(s.Ut.p, ut.data(), sizeof(T) * ut.size(), cudaMemcpyHostToDevice, st));
      CK(cudaStreamSynchronize(st));
    }
    if (Vh) {
      const T* Vp = (const T*)Vh;
      for (int64_t a = 0; a < (int64_t)rank * n; a++) g = std::max(g, f32_grid((float)Vp[a]));
    }
    comm->max_i32_host(&g);
    g = std::max(g, 0);
    if (g > 52) fail(STMF_ERR_NUMERIC, "binary32 data grid 2^-%d is too fine for the exact objective", g);
    F = g;
    exact_limit = std::ldexp(1.0, 53 - g);
    if (Vh) {
      for (auto& s : sh)
        CK(cudaMemcpyAsync(s->V.p, Vh, sizeof(T) * (size_t)rank * n, cudaMemcpyHostToDevice, st));
    } else {
      // V = (-U)^T (x)* R: local column minima, all-reduced (MIN is exact)
      for (auto& s : sh)
        for (int k = 0; k < rank; k++) {
          k_line_min<T><<<warps_grid(n), 256, 0, st>>>(n, s->col_ptr.p, s->row_idx.p, s->xc.p,
                                                        s->Ut.p + (size_t)k * s->ml, s->V.p + (size_t)k * n);
          LAUNCH_CK();
        }
      auto vp = ptrs(&Shard<T>::V);
      comm->min_f32(reinterpret_cast<std::vector<float*>&>(vp), (size_t)rank * n, st);
    }
    CK(cudaStreamSynchronize(st));
    sync_factor_copies(-1);
    std::fill(row_depth.begin(), row_depth.end(), 0);  // a new state: no speculation history
    have_factors = true;
    dirty = true;
    cache_k = -1;
    stats_dirty.assign(rank, 1);
    err_valid = false;
  }

  void get_factors(void* Uh, void* Vh) override {
    if (!have_factors) fail(STMF_ERR_INVALID, "factors not set");
    int64_t row = 0;
    for (auto& sp : sh) {
      Shard<T>& s = *sp;
      std::vector<T> ut((size_t)rank * s.ml);
      CK(cudaMemcpyAsync(ut.data(), s.Ut.p, sizeof(T) * ut.size(), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      if (Uh) {
        T* U = (T*)Uh;
        for (int64_t i = 0; i < s.ml; i++)
          for (int k = 0; k < rank; k++) U[(row + i) * rank + k] = ut[(size_t)k * s.ml + i];
      }
      row += s.ml;
    }
    if (Vh) {
      CK(cudaMemcpyAsync(Vh, sh[0]->V.p, sizeof(T) * (size_t)rank * n, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
    }
  }

  void check_flags() {
    auto fp = ptrs(&Shard<T>::flags);
    comm->sum_i32(fp, 1, st);
    CK(cudaMemcpyAsync(h_flags, sh[0]->flags.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (h_flags[0] & 7) fail(STMF_ERR_NUMERIC, "exact objective window violated (flags %d, grid 2^-%d)", h_flags[0], F);
  }

  void ensure_caches() {
    if (!have_factors) fail(STMF_ERR_INVALID, "factors not set");
    if (dirty) {
      for (auto& sp : sh) {
        Shard<T>& s = *sp;
        CK(cudaMemsetAsync(s.flags.p, 0, sizeof(int), st));
        unsigned gflat = (unsigned)std::max<int64_t>(1, std::min<int64_t>(nblk(s.Nl, 256), (int64_t)nsm * 16));
        k_product2<T><<<gflat, 256, 0, st>>>(s.Nl, s.rowof_r.p, s.col_idx.p, s.ml, n, rank, s.Ut.p, s.V.p, s.Urm.p,
                                             s.Vcm.p, rp, cache_k, s.t1r.p, s.t2r.p, s.agr.p, s.a2r.p);
        LAUNCH_CK();
        k_product2<T><<<gflat, 256, 0, st>>>(s.Nl, s.row_idx.p, s.colof_c.p, s.ml, n, rank, s.Ut.p, s.V.p, s.Urm.p,
                                             s.Vcm.p, rp, cache_k, s.t1c.p, s.t2c.p, s.agc.p, s.a2c.p);
        LAUNCH_CK();
        k_scores<T><<<warps_grid(n), 256, 0, st>>>(n, rank, s.col_ptr.p, s.xc.p, s.t1c.p, s.agc.p, s.score.p,
                                                     s.colhist.p, false, exact_limit, s.flags.p);
        LAUNCH_CK();
        k_score_to_fx<<<nblk(n, 256), 256, 0, st>>>(n, s.score.p, s.scorefx.p, std::ldexp(1.0, F));
        LAUNCH_CK();
      }
      auto sp = ptrs(&Shard<T>::scorefx);
      comm->sum_i64(sp, n, st);
      auto hp = ptrs(&Shard<T>::colhist);
      comm->sum_i32(hp, (size_t)n * rank, st);
      for (auto& s : sh) {
        k_fx_to_score<<<nblk(n, 256), 256, 0, st>>>(n, s->scorefx.p, s->score.p, std::ldexp(1.0, -F));
        LAUNCH_CK();
      }
      check_flags();
      n_product_passes++;
      dirty = false;
      cache_k = -1;
    }
    for (int k = 0; k < rank; k++) {
      if (!stats_dirty[k]) continue;
      for (auto& sp : sh) {
        Shard<T>& s = *sp;
        k_line_stats<T><<<warps_grid(n), 256, 0, st>>>(n, s.col_ptr.p, s.row_idx.p, s.xc.p, s.Ut.p + (size_t)k * s.ml,
                                                         s.lm1.p, s.lm2.p, s.la1.p, (int)s.r0);
        LAUNCH_CK();
        k_line_stats<T><<<warps_grid(s.ml), 256, 0, st>>>(s.ml, s.row_ptr.p, s.col_idx.p, s.xr.p,
                                                            s.V.p + (size_t)k * n, s.rm1.p + (size_t)k * s.ml,
                                                            s.rm2.p + (size_t)k * s.ml, s.rmarg.p + (size_t)k * s.ml);
        LAUNCH_CK();
      }
      std::vector<void*> s1, r1, s2, r2, s3, r3;
      for (auto& s : sh) {
        s1.push_back(s->lm1.p); r1.push_back(s->gm1.p);
        s2.push_back(s->lm2.p); r2.push_back(s->gm2.p);
        s3.push_back(s->la1.p); r3.push_back(s->ga1.p);
      }
      comm->allgather(s1, r1, sizeof(T) * n, st);
      comm->allgather(s2, r2, sizeof(T) * n, st);
      comm->allgather(s3, r3, sizeof(int32_t) * n, st);
      for (auto& s : sh) {
        k_stats_merge<T><<<nblk(n, 256), 256, 0, st>>>(W, n, s->gm1.p, s->gm2.p, s->ga1.p, s->cm1.p + (size_t)k * n,
                                                        s->cm2.p + (size_t)k * n, s->cmarg.p + (size_t)k * n);
        LAUNCH_CK();
      }
      stats_dirty[k] = 0;
    }
  }

  double reduce_acc(int count) {  // count evals' (lo,hi) in acc -> limbs -> all-reduce -> host values
    for (auto& s : sh) {
      k_acc_to_limbs<<<nblk(count, 256), 256, 0, st>>>(count, s->acc.p, s->limbs.p);
      LAUNCH_CK();
    }
    auto lp = ptrs(&Shard<T>::limbs);
    comm->sum_i64(lp, 3 * (size_t)count, st);
    CK(cudaMemcpyAsync(h_limbs, sh[0]->limbs.p, sizeof(int64_t) * 3 * count, cudaMemcpyDeviceToHost, st));
    return 0;
  }
  double limbs_value(int t) const {
    unsigned __int128 v = (unsigned __int128)(u64)h_limbs[3 * t] + ((unsigned __int128)(u64)h_limbs[3 * t + 1] << 42) +
                          ((unsigned __int128)(u64)h_limbs[3 * t + 2] << 84);
    return fx_to_double((u64)(v >> 64), (u64)v, F);
  }

  double objective() override {
    ensure_caches();
    if (!err_valid) {
      for (auto& sp : sh) {
        Shard<T>& s = *sp;
        CK(cudaMemsetAsync(s.acc.p, 0, 2 * sizeof(u64), st));
        CK(cudaMemsetAsync(s.flags.p, 0, sizeof(int), st));
        k_objective<T><<<warps_grid(s.ml), 256, 0, st>>>(s.ml, s.row_ptr.p, s.col_idx.p, s.xr.p, s.t1r.p, s.t2r.p,
                                                           s.agr.p, 0, s.Ut.p, s.V.p, s.acc.p, s.flags.p, F, exact_limit);
        LAUNCH_CK();
      }
      reduce_acc(1);
      check_flags();
      err = limbs_value(0);
      err_valid = true;
    }
    return err;
  }

  // ---- one row visit ----
  int64_t build_candidates(int64_t i) {
    int own = owner(i);
    int64_t nc = row_nnz[i];
    if (Shard<T>* o = local(own)) {
      int64_t il = i - o->r0;
      int64_t beg = o->h_row_ptr[il];
      k_pack_row<T><<<1, 256, 0, st>>>(nc, rank, o->ml, il, o->col_idx.p + beg, o->xr.p + beg, o->agr.p + beg,
                                       o->Ut.p, (int32_t*)o->rowbuf.p, (T*)(o->rowbuf.p + off_x),
                                       (int32_t*)(o->rowbuf.p + off_h), (T*)(o->rowbuf.p + off_u),
                                       o->rowbuf.p + off_ag);
      LAUNCH_CK();
    }
    std::vector<void*> rb;
    for (auto& s : sh) rb.push_back(s->rowbuf.p);
    comm->broadcast(rb, rowbuf_bytes, own, st);
    for (auto& sp : sh) {
      Shard<T>& s = *sp;
      const int32_t* cols = (const int32_t*)s.rowbuf.p;
      const T* xrow = (const T*)(s.rowbuf.p + off_x);
      if (nc <= 4 * kCandThreads && rank <= 256) {
        // one block ranks the candidates (stable merge sort on the score keys), votes
        // and fills the dense row, as in the single-device engine; the extra blocks
        // of the launch fill CM^(-i) (not needed here, but the kernel's contract)
        auto kern = nc <= kCandThreads ? k_cand_row<T, 1> : k_cand_row<T, 4>;
        int64_t need = ((int64_t)rank * n + kCandThreads - 1) / kCandThreads;
        unsigned grid = (unsigned)(1 + std::max<int64_t>(1, std::min<int64_t>(need, nsm)));
        kern<<<grid, kCandThreads, 0, st>>>((int)nc, n, rank, cols, xrow, s.rowbuf.p + off_ag, s.score.p,
                                            s.colhist.p, s.cj.p, s.ck.p, s.cx.p, s.xrow_dense.p, i, s.cm1.p, s.cm2.p,
                                            s.cmarg.p, s.cmi.p, nullptr, nullptr, 0);
        LAUNCH_CK();
        continue;
      }
      k_cand_keys<<<nblk(nc, 256), 256, 0, st>>>(nc, cols, s.score.p, s.ckeys.p, s.cvals.p);
      LAUNCH_CK();
      size_t bytes = s.cubtmp_bytes;
      CK(cub::DeviceRadixSort::SortPairs(s.cubtmp.p, bytes, s.ckeys.p, s.ckeys2.p, s.cvals.p, s.cperm.p, (int)nc, 0,
                                         64, st));
      k_cand_build_h<T><<<nblk(nc, 256), 256, 0, st>>>(nc, rank, cols, xrow, (const int32_t*)(s.rowbuf.p + off_h),
                                                       s.cperm.p, s.colhist.p, s.cj.p, s.ck.p, s.cx.p);
      LAUNCH_CK();
      k_fill<T><<<nblk(n, 256), 256, 0, st>>>(n, s.xrow_dense.p, (T)INFINITY);
      LAUNCH_CK();
      k_scatter_row<T><<<nblk(nc, 256), 256, 0, st>>>(nc, cols, xrow, s.xrow_dense.p);
      LAUNCH_CK();
    }
    return nc;
  }

  void eval_batch(int64_t i, int64_t t0, int E) {
    int64_t G8 = (int64_t)((E + kEG - 1) / kEG) * kEG;
    int ng = (E + kEG - 1) / kEG;
    for (auto& sp : sh) {
      Shard<T>& s = *sp;
      const int32_t* bj = s.cj.p + t0;
      const int32_t* bk = s.ck.p + t0;
      const T* bx = s.cx.p + t0;
      CK(cudaMemsetAsync(s.acc.p, 0, sizeof(u64) * 4 * E, st));
      CK(cudaMemsetAsync(s.chg.p, 0, sizeof(int) * 2 * E, st));
      CK(cudaMemsetAsync(s.flags.p, 0, sizeof(int), st));
      k_phaseA_ulf<T><<<nblk(G8 * n, 256), 256, 0, st>>>(n, E, i, bj, bk, bx, s.V.p, s.cm1.p, s.cm2.p, s.cmarg.p,
                                                          s.xrow_dense.p, s.vbuf.p, s.chg.p);
      LAUNCH_CK();
      k_phaseA_urf_fill<T><<<nblk(G8 * s.ml, 256), 256, 0, st>>>(s.ml, E, bj, bk, s.rm1.p, s.rm2.p, s.rmarg.p,
                                                                   s.ubufA.p);
      LAUNCH_CK();
      k_phaseA_urf_seed_h<T><<<E, 128, 0, st>>>(s.ml, E, bj, bk, bx, (const T*)(s.rowbuf.p + off_u), s.col_ptr.p,
                                                s.row_idx.p, s.xc.p, s.ubufA.p);
      LAUNCH_CK();
      k_chk_ilv<T><<<nblk(G8 * s.ml, 256), 256, 0, st>>>(s.ml, E, bk, s.ubufA.p, s.Ut.p, s.chg.p + E);
      LAUNCH_CK();
      SideB<T> sa{s.ml, s.row_ptr.p, s.col_idx.p, s.xr.p, s.t1r.p, s.t2r.p, s.agr.p, s.vbuf.p, n, s.Ut.p, s.ubufB.p,
                  s.acc.p, s.chg.p, 0, long_thr, group_major};
      SideB<T> sb{n, s.col_ptr.p, s.row_idx.p, s.xc.p, s.t1c.p, s.t2c.p, s.agc.p, s.ubufA.p, s.ml, s.V.p, s.vbufB.p,
                  s.acc.p + 2 * (size_t)E, s.chg.p + E, 1, long_thr, group_major};
      launch_phaseB<T>(unroll, warps_grid((s.ml + n) * ng), st, sa, sb, E, bk, s.flags.p, F, exact_limit,
                       s.long_rows.p, s.n_long_rows, s.long_cols.p, s.n_long_cols, nsm);
      LAUNCH_CK();
    }
    // F-URF: v''_c = min over ALL rows -> all-reduce MIN of the local column minima
    auto vb = ptrs(&Shard<T>::vbufB);
    comm->min_f32(reinterpret_cast<std::vector<float*>&>(vb), (size_t)E * n, st);
    for (auto& sp : sh) {
      Shard<T>& s = *sp;
      const int32_t* bk = s.ck.p + t0;
      SideB<T> none{0, s.row_ptr.p, s.col_idx.p, s.xr.p, s.t1r.p, s.t2r.p, s.agr.p, s.vbuf.p, n, s.Ut.p, s.ubufB.p,
                    s.acc.p, s.chg.p, 0, long_thr, group_major};
      SideB<T> sb{n, s.col_ptr.p, s.row_idx.p, s.xc.p, s.t1c.p, s.t2c.p, s.agc.p, s.ubufA.p, s.ml, s.V.p, s.vbufB.p,
                  s.acc.p + 2 * (size_t)E, s.chg.p + E, 2, long_thr, group_major};
      launch_phaseB<T>(unroll, warps_grid(n * ng), st, none, sb, E, bk, s.flags.p, F, exact_limit, nullptr, 0,
                       s.long_cols.p, s.n_long_cols, nsm);
      LAUNCH_CK();
    }
    reduce_acc(2 * E);
    auto cp = ptrs(&Shard<T>::chg);
    comm->sum_i32(cp, 2 * (size_t)E, st);
    CK(cudaMemcpyAsync(h_chg, sh[0]->chg.p, sizeof(int) * 2 * E, cudaMemcpyDeviceToHost, st));
    check_flags();
  }

  void commit(int op, int q, int k) {
    for (auto& sp : sh) {
      Shard<T>& s = *sp;
      const T* a;
      const T* b;
      if (op == 0) {
        a = s.ubufB.p + (size_t)q * s.ml;
        k_deinterleave<T><<<nblk(n, 256), 256, 0, st>>>(n, q, s.vbuf.p, s.dtmpB.p);
        LAUNCH_CK();
        b = s.dtmpB.p;
      } else {
        k_deinterleave<T><<<nblk(s.ml, 256), 256, 0, st>>>(s.ml, q, s.ubufA.p, s.dtmpA.p);
        LAUNCH_CK();
        a = s.dtmpA.p;
        b = s.vbufB.p + (size_t)q * n;
      }
      CK(cudaMemcpyAsync(s.Ut.p + (size_t)k * s.ml, a, sizeof(T) * s.ml, cudaMemcpyDeviceToDevice, st));
      CK(cudaMemcpyAsync(s.V.p + (size_t)k * n, b, sizeof(T) * n, cudaMemcpyDeviceToDevice, st));
    }
    sync_factor_copies(k);
    cache_k = dirty ? -1 : k;
    dirty = true;
    stats_dirty[k] = 1;
  }

  struct RunState {
    bool wall;
    double t0, budget_seconds;
    int64_t cur_sweep;
    double* tt; double* te; int64_t cap, len;
    int64_t attempts, accepts, visits, evaluated;
  };
  // null trajectory buffers: the trajectory is kept here (growable), read back with
  // stmf_trajectory (as single-device sessions)
  std::vector<double> tj_t, tj_e;
  void trajectory(double* t, double* e, int64_t cap, int64_t* len) override {
    *len = (int64_t)tj_t.size();
    if (!t || !e) return;
    if (cap < *len) fail(STMF_ERR_CAPACITY, "trajectory has %lld samples, capacity %lld", (long long)*len,
                         (long long)cap);
    std::memcpy(t, tj_t.data(), sizeof(double) * tj_t.size());
    std::memcpy(e, tj_e.data(), sizeof(double) * tj_e.size());
  }
  double run_now(RunState& R) { return R.wall ? now_s() - R.t0 : (double)R.cur_sweep; }
  bool out_of_time(RunState& R) {
    // every rank must take the same branch: agree on the wall-clock decision
    int v = R.wall && now_s() - R.t0 >= R.budget_seconds;
    if (R.wall) comm->max_i32_host(&v);
    return v != 0;
  }
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

  void row_visit(RunState& R, int64_t i) {
    ensure_caches();
    int64_t nc = build_candidates(i);
    R.visits++;
    std::vector<int> hk;
    int64_t t0 = 0;
    // the same decisions on every rank, so the same schedule
    int next = row_depth[i] > 0 ? (int)std::max<int64_t>(batch_floor, std::min<int64_t>(
                                      Emax, (int64_t)(sched_scale * row_depth[i]) + sched_add))
                                : batch_sched[0];
    next = round_batch(next, e_round, Emax);
    while (t0 < nc) {
      int E = (int)std::min<int64_t>(nc - t0, next);
      next = round_batch(std::max(next + 1, (int)(next * sched_growth)), e_round, Emax);
      eval_batch(i, t0, E);
      hk.resize(E);
      CK(cudaMemcpyAsync(hk.data(), sh[0]->ck.p + t0, sizeof(int) * E, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      R.evaluated += 2 * (int64_t)E;
      for (int q = 0; q < E; q++)
        for (int op = 0; op < 2; op++) {
          R.attempts++;
          if (!h_chg[op * E + q]) continue;
          double f = limbs_value(op * E + q);
          if (f < err) {
            commit(op, q, hk[q]);
            err = f;
            R.accepts++;
            row_depth[i] = t0 + q + 1;
            traj_append(R, run_now(R), err);
            return;
          }
        }
      if (out_of_time(R)) return;
      t0 += E;
    }
    row_depth[i] = nc;
  }

  void run(int64_t budget_sweeps, double budget_seconds, double epsilon, double* tt, double* te, int64_t cap,
           int64_t* counts) override {
    if (budget_sweeps < 0 && !(budget_seconds > 0)) fail(STMF_ERR_INVALID, "set budget_sweeps or budget_seconds");
    RunState R{};
    if (!tt) { tj_t.clear(); tj_e.clear(); }
    R.wall = budget_seconds > 0;
    R.budget_seconds = budget_seconds;
    R.t0 = now_s();
    R.tt = tt; R.te = te; R.cap = cap;
    int64_t pp0 = n_product_passes;
    objective();
    traj_append(R, run_now(R), err);
    double eps = epsilon * err;
    int64_t sweeps = 0;
    if (err > 0.0) {
      for (;;) {
        if (budget_sweeps >= 0 && sweeps >= budget_sweeps) break;
        if (out_of_time(R)) break;
        R.cur_sweep = sweeps + 1;
        double err_before = err;
        for (int64_t i = 0; i < m; i++) {
          if (out_of_time(R)) break;
          row_visit(R, i);
        }
        sweeps++;
        traj_append(R, run_now(R), err);
        if (err_before - err < eps) break;
      }
    }
    counts[0] = R.len; counts[1] = R.attempts; counts[2] = R.accepts; counts[3] = sweeps;
    counts[4] = R.visits; counts[5] = R.evaluated; counts[6] = 0; counts[7] = n_product_passes - pp0;
  }

  void col_scores(double* out) override {
    ensure_caches();
    CK(cudaMemcpyAsync(out, sh[0]->score.p, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  }
  void product_given(void*, int32_t*, void*) override { fail(STMF_ERR_INVALID, "not available on sharded sessions"); }
  void residuate(int, const void*, void*) override { fail(STMF_ERR_INVALID, "not available on sharded sessions"); }
  void try_update(int, int64_t, int64_t, int, void*, void*, double*, bool, int*) override {
    fail(STMF_ERR_INVALID, "not available on sharded sessions");
  }
  void bench_product(int, int, double*, double*) override { fail(STMF_ERR_INVALID, "not available on sharded sessions"); }
  void* stream() override { return (void*)st; }
  int device_id() const override { return dev; }
  void comm_info(int* out3) override { comm->info(&out3[0], &out3[1], &out3[2]); }
  void set_profiling(int) override {}
  void counters(int64_t* out) override {
    for (int i = 0; i < 8; i++) out[i] = 0;
    out[0] = g_launches.load();
    out[1] = g_cub_calls.load();
    out[5] = n_product_passes;
  }
};
