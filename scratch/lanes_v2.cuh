// stmf_maxplus_lanes.cuh — config-5 kernel for low densities, second generation:
// the "lane-coded" sampled layout.  Included by stmf_api.cu after stmf_maxplus.cuh.
//
//   err = sum over given (i, j) of |X_ij - max_k (U_ik + V_kj)|   (tropical.py:214-222 in
//   binary32 with the exact-sum semantics of the fit's objective)
//
// What the first sampled kernel (k_maxplus_err_sampled) paid for: a per-tile decode of the
// bit mask into (row, column) codes and two bank-conflicted gathers of staged factor rows
// per given entry (98 thread instructions per entry, 21% of HBM at 65536^2 / rank 4 / 10%).
// A first lane-owned variant that still walked mask bits in the kernel (FLO + bit clear + a
// divergent word advance + two POPC per entry) reached 25% (profiles/r02_c5_lanes_v1.jsonl):
// bound by the quarter-rate bit instructions.  This layout moves the whole decode into the
// (untimed, once per matrix) format build:
//
//  * A chunk = 8 rows x 1024 columns is one warp's unit of work.  Lane l owns the chunk's
//    given entries whose column c has c mod 32 == l.  The span's V rows sit in shared
//    memory in natural order (16 RQ bytes per column), so the 8 lanes of a quarter-warp
//    always read 8 different 16-byte bank groups: the per-entry V gather is conflict free
//    by construction.
//  * A chunk is one record: [33 x u16 lane offsets][the values, lane-major][one byte code
//    per value: (row in chunk) << 5 | (column in span) >> 5].  A lane walks its own
//    contiguous run of values and codes: no bit scans, no ballots, no popcounts.  The
//    record replaces the bit mask (the codes carry the positions): 5 bytes per given entry
//    + 80 per chunk, less than the mask + values (m n / 8 + 4 given) below 12% density.
//  * The U rows of the chunk (8 x 16 RQ bytes, one or a few cache lines) are read through
//    L1 per entry.
//  * Records are 16-byte aligned and ordered span-major, row-chunks ascending, so a warp's
//    run of chunks is one contiguous byte range; each warp streams its records through a
//    ring of shared-memory stages filled by 1-D bulk async copies (cp.async.bulk ...
//    mbarrier::complete_tx): whole records in flight, no register-staged loads.
//
// Lanes of a warp finish a chunk when the fullest lane does: at 10% density a lane holds
// Binomial(256, 0.1) entries, so ~72% of the lane slots are busy.
#pragma once

namespace stmf {

constexpr int kLnSpan = 1024;    // columns per chunk
constexpr int kLnRows = 8;       // rows per chunk (3 code bits; 5 for the column / 32)
constexpr int kLnMaxStages = 4;
constexpr int kLnHeader = 80;    // 33 u16 lane offsets, padded to 16 bytes

__device__ __forceinline__ void ln_mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n LNWAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra LNWAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// record bytes of a chunk with n given entries (16-byte multiple)
__host__ __device__ __forceinline__ int ln_record_bytes(int n) {
  return kLnHeader + 4 * ((n + 3) & ~3) + ((n + 15) & ~15);
}

template <bool STAGED, typename V>
__device__ __forceinline__ V ln_ld(unsigned sa, const unsigned char* ga) {
  V v;
  if constexpr (STAGED) {
    if constexpr (sizeof(V) == 4) asm volatile("ld.shared.b32 %0, [%1];" : "=r"(*reinterpret_cast<unsigned*>(&v)) : "r"(sa));
    else if constexpr (sizeof(V) == 2) asm volatile("ld.shared.u16 %0, [%1];" : "=h"(*reinterpret_cast<unsigned short*>(&v)) : "r"(sa));
    else {
      unsigned t;
      asm volatile("ld.shared.u8 %0, [%1];" : "=r"(t) : "r"(sa));
      v = (V)t;
    }
  } else {
    v = __ldg(reinterpret_cast<const V*>(ga));
  }
  return v;
}
__device__ __forceinline__ float4 ln_lds4(unsigned a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}

// one chunk: the record is at shared address rs (STAGED) or global pointer rg; urow = the
// chunk's first U row (row-major, stride 4 RQ floats); vlane = shared address of V column
// `lane` of the span (column c of the lane's entries is lane + 32 * (code & 31))
template <int RQ, bool STAGED>
__device__ __forceinline__ double ln_chunk(unsigned rs, const unsigned char* __restrict__ rg,
                                           const float4* __restrict__ urow, unsigned vlane, int lane, double part) {
  const int o0 = ln_ld<STAGED, unsigned short>(rs + 2 * lane, rg + 2 * lane);
  const int o1 = ln_ld<STAGED, unsigned short>(rs + 2 * lane + 2, rg + 2 * lane + 2);
  const int n = ln_ld<STAGED, unsigned short>(rs + 64, rg + 64);
  const int cnt = o1 - o0;
  const int maxc = __reduce_max_sync(0xffffffffu, cnt);
  const int np = (n + 3) & ~3;
  unsigned xs = rs + kLnHeader + 4 * o0, cs = rs + kLnHeader + 4 * np + o0;
  const unsigned char* xg = rg + kLnHeader + 4 * o0;
  const unsigned char* cg = rg + kLnHeader + 4 * np + o0;
  asm volatile("" : "+r"(xs), "+r"(cs), "+r"(vlane));  // keep the addresses in registers
  for (int it = 0; it < maxc; ++it) {
    if (it < cnt) {
      const float x = ln_ld<STAGED, float>(xs + 4 * it, xg + 4 * it);
      const unsigned code = ln_ld<STAGED, unsigned char>(cs + it, cg + it);
      const float4* ur = urow + (code >> 5) * RQ;
      const unsigned va = vlane + (code & 31u) * (32 * 16);
      float p0 = -CUDART_INF_F, p1 = -CUDART_INF_F;
#pragma unroll
      for (int q = 0; q < RQ; q++) {
        const float4 v = ln_lds4(va + q * (kLnSpan * 16)), u = __ldg(ur + q);
        const float2 a = fadd2(make_float2(u.x, u.y), make_float2(v.x, v.y));
        const float2 c = fadd2(make_float2(u.z, u.w), make_float2(v.z, v.w));
        if (q == 0) {
          p0 = fmaxf(a.x, a.y);
          p1 = fmaxf(c.x, c.y);
        } else {
          p0 = max3f(p0, a.x, a.y);
          p1 = max3f(p1, c.x, c.y);
        }
      }
      part = __dadd_rn(part, (double)fabsf(__fsub_rn(x, fmaxf(p0, p1))));
    }
  }
  return part;
}

// grid = K * (n / 1024) blocks of 256 threads (block b: span b % nspans); factors row-major
// with stride 4 RQ (padding -inf).  recs = the chunk records, coff[id] = start of record id in
// 16-byte units (id = span * (m / 8) + row-chunk).  cpw = chunks per warp run (power of two
// dividing m / 8).
template <int RQ>
__global__ void __launch_bounds__(256)
k_maxplus_err_lanes(int64_t m, int64_t n, const unsigned char* __restrict__ recs, const int64_t* __restrict__ coff,
                    const float* __restrict__ Urm, const float* __restrict__ Vrm, u64* __restrict__ acc,
                    int* __restrict__ flags, int F, double exact_limit, int cpw_log2, int nstage, int stage_cap) {
  extern __shared__ __align__(128) unsigned char ln_smem[];
  float4* Vs = reinterpret_cast<float4*>(ln_smem);  // [RQ][1024]
  unsigned char* stg = ln_smem + sizeof(float4) * RQ * kLnSpan;
  __shared__ __align__(8) uint64_t bars[8][kLnMaxStages];
  __shared__ int64_t meta_off[8][kLnMaxStages];
  __shared__ int meta_bytes[8][kLnMaxStages];
  __shared__ double red[8];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int nspans = (int)(n / kLnSpan);
  const int cs = (int)(blockIdx.x % nspans), kb = (int)(blockIdx.x / nspans), K = (int)(gridDim.x / nspans);
  const int64_t nrc = m / kLnRows;
  const int cpw = 1 << cpw_log2;
  for (int c = tid; c < kLnSpan; c += 256) {
    const float4* src = reinterpret_cast<const float4*>(Vrm + ((int64_t)cs * kLnSpan + c) * (4 * RQ));
#pragma unroll
    for (int q2 = 0; q2 < RQ; q2++) Vs[q2 * kLnSpan + c] = __ldg(src + q2);
  }
  if (lane == 0) {
    for (int s = 0; s < nstage; s++)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[wid][s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();

  // this warp's runs: run r covers row-chunks [r cpw, (r + 1) cpw) of span cs
  const int64_t nruns = nrc >> cpw_log2;
  const int64_t r0 = (int64_t)kb * 8 + wid, rstep = (int64_t)K * 8;
  const int64_t nR = r0 < nruns ? (nruns - r0 + rstep - 1) / rstep : 0;
  const int64_t nT = nR << cpw_log2;
  auto chunk_rc = [&](int64_t t) { return ((r0 + (t >> cpw_log2) * rstep) << cpw_log2) + (t & (cpw - 1)); };
  auto load_offs = [&](int64_t run_i) -> int64_t {  // lane l: offset l of the run's cpw + 1 record offsets
    if (run_i >= nR || lane > cpw) return 0;
    return __ldg(coff + (int64_t)cs * nrc + ((r0 + run_i * rstep) << cpw_log2) + lane);
  };
  int64_t offC = load_offs(0), offN = load_offs(1);
  unsigned char* mystg = stg + (size_t)wid * nstage * stage_cap;
  // producer: record of chunk t into stage s (= t mod nstage)
  auto issue = [&](int64_t t, int s) {
    if (t >= nT) return;
    const int l = (int)(t & (cpw - 1));
    if (l == 0 && t > 0) {
      offC = offN;
      offN = load_offs((t >> cpw_log2) + 1);
    }
    const int64_t o0 = __shfl_sync(0xffffffffu, offC, l), o1 = __shfl_sync(0xffffffffu, offC, l + 1);
    const int bytes = (int)(o1 - o0) * 16;
    if (lane == 0) {
      meta_off[wid][s] = o0;
      meta_bytes[wid][s] = bytes;
      if (bytes <= stage_cap) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bars[wid][s])),
                     "r"((unsigned)bytes)
                     : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(mystg + (size_t)s * stage_cap)),
            "l"(recs + o0 * 16), "r"((unsigned)bytes), "r"(smem_u32(&bars[wid][s]))
            : "memory");
      }
    }
  };
  {
    int s = 0;
    for (int64_t t = 0; t < nstage; t++, s++) issue(t, s);
  }
  __syncwarp();

  const unsigned vlane = smem_u32(Vs) + lane * 16;
  const unsigned stg_s = smem_u32(mystg);
  double part = 0.0;
  unsigned phase = 0;
  int s = 0;
  for (int64_t t = 0; t < nT; t++) {
    const float4* urow = reinterpret_cast<const float4*>(Urm + chunk_rc(t) * kLnRows * (4 * RQ));
    const int bytes = meta_bytes[wid][s];
    if (bytes <= stage_cap) {
      ln_mbar_wait(&bars[wid][s], (phase >> s) & 1u);
      phase ^= 1u << s;
      part = ln_chunk<RQ, true>(stg_s + s * stage_cap, nullptr, urow, vlane, lane, part);
    } else {  // a record larger than a stage: read straight from global memory
      part = ln_chunk<RQ, false>(0, recs + meta_off[wid][s] * 16, urow, vlane, lane, part);
    }
    __syncwarp();
    issue(t + nstage, s);
    __syncwarp();
    s = s + 1 == nstage ? 0 : s + 1;
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
constexpr size_t ln_smem_bytes(int nstage, int stage_cap) {
  return sizeof(float4) * RQ * kLnSpan + (size_t)8 * nstage * stage_cap;
}

// format build (not timed, once per matrix).  Chunk id = span * (m / 8) + row-chunk; a warp
// per chunk; lane l counts / writes the entries of its column class c mod 32 == l, rows
// ascending, columns ascending.  cnt[id] = the record's size in 16-byte units.
__device__ __forceinline__ int ln_lane_count(const uint32_t* __restrict__ mrow0, int64_t wpr, int lane) {
  int c = 0;
  for (int r = 0; r < kLnRows; r++)
    for (int w = 0; w < kLnSpan / 32; w++) c += (mrow0[r * wpr + w] >> lane) & 1u;
  return c;
}

__global__ void k_ln_count(int64_t m, int64_t n, const uint32_t* __restrict__ mask, int64_t* __restrict__ cnt,
                           int* __restrict__ maxrec) {
  const int lane = threadIdx.x & 31;
  const int64_t nrc = m / kLnRows, nch = nrc * (n / kLnSpan), wpr = n / 32;
  for (int64_t id = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; id < nch;
       id += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t cs = id / nrc, rc = id - cs * nrc;
    int c = ln_lane_count(mask + rc * kLnRows * wpr + cs * (kLnSpan / 32), wpr, lane);
    c = __reduce_add_sync(0xffffffffu, c);
    if (lane == 0) {
      const int bytes = ln_record_bytes(c);
      cnt[id] = bytes / 16;
      atomicMax(maxrec, bytes);
    }
  }
}

__global__ void k_ln_fill(int64_t m, int64_t n, const uint32_t* __restrict__ mask, const float* __restrict__ X,
                          const int64_t* __restrict__ coff, unsigned char* __restrict__ recs) {
  const int lane = threadIdx.x & 31;
  const int64_t nrc = m / kLnRows, nch = nrc * (n / kLnSpan), wpr = n / 32;
  for (int64_t id = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; id < nch;
       id += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t cs = id / nrc, rc = id - cs * nrc;
    const uint32_t* mrow0 = mask + rc * kLnRows * wpr + cs * (kLnSpan / 32);
    const int c = ln_lane_count(mrow0, wpr, lane);
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31), off = incl - c;
    unsigned char* rec = recs + coff[id] * 16;
    unsigned short* hdr = reinterpret_cast<unsigned short*>(rec);
    hdr[lane] = (unsigned short)off;
    if (lane == 31) hdr[32] = (unsigned short)total;
    float* xv = reinterpret_cast<float*>(rec + kLnHeader);
    unsigned char* cd = rec + kLnHeader + 4 * ((total + 3) & ~3);
    int pos = off;
    for (int r = 0; r < kLnRows; r++)
      for (int w = 0; w < kLnSpan / 32; w++)
        if ((mrow0[r * wpr + w] >> lane) & 1u) {
          xv[pos] = X[(rc * kLnRows + r) * n + cs * kLnSpan + w * 32 + lane];
          cd[pos] = (unsigned char)((r << 5) | w);
          pos++;
        }
  }
}

}  // namespace stmf
