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
//  * A chunk = 4 rows x SPAN columns is one warp's unit of work; SPAN (2048 ... 256, at most
//    1024 above rank 4) is chosen per matrix as the widest whose largest chunk record still
//    fits a shared-memory stage, so denser matrices get narrower chunks of about the same
//    number of entries.  (SPAN = 2048 up to ~12% density at rank <= 4.)  A chunk is one warp's
//    unit of work.  Lane l = 8 q + j owns the given entries of row q of the chunk whose
//    column c has c mod 8 == j; its U row lives in registers.  The span's V rows sit in
//    shared memory in natural order (16 bytes per column and plane), so the 8 lanes of a
//    quarter-warp always read 8 different 16-byte bank groups: the per-entry V gather is
//    conflict free by construction.
//  * A chunk is one record: [header: 32 u16 lane counts, total, iterations, 32 u8 lane
//    ranks][u16 slot base per iteration][the values][one byte code per value: (column in
//    span) >> 3].  Values and codes are stored "iteration-major, compacted": first the first
//    entry of every lane that has one, then the second of every lane that has two, ...,
//    within an iteration in order of decreasing lane count (the lane's rank).  Lanes with
//    more entries rank first, so the lanes active in iteration `it` are exactly ranks
//    0 .. A_it - 1 and lane l reads slot base[it] + rank[l]: consecutive floats and bytes
//    across the active lanes (no shared-memory bank conflicts), no padding in memory, and
//    no ballot / popcount / bit scan in the kernel (the first lane-owned variants spent
//    their time in exactly those quarter-rate instructions).  The record replaces the bit
//    mask (the codes carry the positions): 5 bytes per given entry + ~200 per chunk, less
//    than the mask + values (m n / 8 + 4 given) below 12% density.
//  * Records are 16-byte aligned and ordered span-major, row-chunks ascending, so a warp's
//    run of chunks is one contiguous byte range; each warp streams its records through a
//    ring of shared-memory stages filled by 1-D bulk async copies (cp.async.bulk ...
//    mbarrier::complete_tx): whole records in flight, no register-staged loads.
//
// Lanes of a warp finish a chunk when the fullest lane does: at 10% density and rank <= 4 a
// lane holds Binomial(256, 0.1) entries, so ~72% of the lane slots are busy.
#pragma once

namespace stmf {

constexpr int kLnRows = 4;       // rows per chunk (one per quarter-warp)
constexpr int kLnMaxStages = 2;
constexpr int kLnWarps = 16;     // warps per block (one V span staged per block)
constexpr int kLnHeader = 112;   // 32 u16 lane counts, total, iterations, 32 u8 lane ranks; padded to 16 bytes
// widest chunk: 8 column classes x 256 codes (rank <= 4) or x 128 (the V span must fit shared memory)
__host__ __device__ constexpr int ln_max_span(int rq) { return rq == 1 ? 2048 : 1024; }
constexpr int kLnMinSpan = 256;

__device__ __forceinline__ void ln_mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n LNWAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra LNWAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// record bytes of a chunk with n given entries in maxc iterations (16-byte multiple)
__host__ __device__ __forceinline__ int ln_record_bytes(int n, int maxc) {
  return kLnHeader + ((2 * maxc + 15) & ~15) + 4 * ((n + 3) & ~3) + ((n + 15) & ~15);
}

// small loads from the record: shared memory by 32-bit shared address (STAGED) or global.
// The narrow ones return the zero-extended value in a 32-bit register (no re-masking).
template <bool STAGED>
__device__ __forceinline__ unsigned ln_ld_u8(unsigned sa, const unsigned char* ga) {
  unsigned t;
  if constexpr (STAGED) asm volatile("ld.shared.u8 %0, [%1];" : "=r"(t) : "r"(sa));
  else asm volatile("ld.global.nc.u8 %0, [%1];" : "=r"(t) : "l"(ga));
  return t;
}
template <bool STAGED>
__device__ __forceinline__ unsigned ln_ld_u16(unsigned sa, const unsigned char* ga) {
  unsigned t;
  if constexpr (STAGED) asm volatile("ld.shared.u16 %0, [%1];" : "=r"(t) : "r"(sa));
  else asm volatile("ld.global.nc.u16 %0, [%1];" : "=r"(t) : "l"(ga));
  return t;
}
template <bool STAGED>
__device__ __forceinline__ float ln_ld_f32(unsigned sa, const unsigned char* ga) {
  float t;
  if constexpr (STAGED) asm volatile("ld.shared.f32 %0, [%1];" : "=f"(t) : "r"(sa));
  else asm volatile("ld.global.nc.f32 %0, [%1];" : "=f"(t) : "l"(ga));
  return t;
}
// four consecutive u16 (8-byte aligned)
template <bool STAGED>
__device__ __forceinline__ uint2 ln_ld_b64(unsigned sa, const unsigned char* ga) {
  uint2 t;
  if constexpr (STAGED) asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(t.x), "=r"(t.y) : "r"(sa));
  else asm volatile("ld.global.nc.v2.u32 {%0, %1}, [%2];" : "=r"(t.x), "=r"(t.y) : "l"(ga));
  return t;
}
__device__ __forceinline__ float4 ln_lds4(unsigned a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}

// one chunk: the record is at shared address rs (STAGED) or global pointer rg; uu = the
// lane's U row; vlane = shared address of V column j = lane & 7 of the span (the column of
// an entry is j + 8 * code)
template <int RQ, int SPAN, bool STAGED>
__device__ __forceinline__ double ln_entry(unsigned xs, unsigned cs, const unsigned char* __restrict__ xg,
                                           const unsigned char* __restrict__ cg, unsigned base,
                                           const float4 (&uu)[RQ], unsigned vlane, double part) {
  const float x = ln_ld_f32<STAGED>(xs + 4 * base, xg + 4 * base);
  const unsigned code = ln_ld_u8<STAGED>(cs + base, cg + base);
  const unsigned va = vlane + code * 128u;
  float p0 = -CUDART_INF_F, p1 = -CUDART_INF_F;
#pragma unroll
  for (int q = 0; q < RQ; q++) {
    const float4 v = ln_lds4(va + q * (SPAN * 16)), u = uu[q];
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
  return __dadd_rn(part, (double)fabsf(__fsub_rn(x, fmaxf(p0, p1))));
}

template <int RQ, int SPAN, bool STAGED>
__device__ __forceinline__ double ln_chunk(unsigned rs, const unsigned char* __restrict__ rg, const float4 (&uu)[RQ],
                                           unsigned vlane, int lane, double part) {
  const int cnt = (int)ln_ld_u16<STAGED>(rs + 2 * lane, rg + 2 * lane);
  const int n = (int)ln_ld_u16<STAGED>(rs + 64, rg + 64);
  const int maxc = (int)ln_ld_u16<STAGED>(rs + 66, rg + 66);
  const unsigned rank = ln_ld_u8<STAGED>(rs + 68 + lane, rg + 68 + lane);
  const int nb = (2 * maxc + 15) & ~15, np4 = 4 * ((n + 3) & ~3);
  unsigned bs = rs + kLnHeader, xs = rs + kLnHeader + nb + 4 * rank, cs = rs + kLnHeader + nb + np4 + rank;
  const unsigned char* bg = rg + kLnHeader;
  const unsigned char* xg = rg + kLnHeader + nb + 4 * rank;
  const unsigned char* cg = rg + kLnHeader + nb + np4 + rank;
  asm volatile("" : "+r"(bs), "+r"(xs), "+r"(cs), "+r"(vlane));  // keep the addresses in registers
  // four iterations per step: their slot bases are one 8-byte load (the base array is padded to
  // 16 bytes, so the load stays inside the record)
  for (int it = 0; it < maxc; it += 4) {
    const uint2 b4 = ln_ld_b64<STAGED>(bs + 2 * it, bg + 2 * it);
    if (it < cnt) part = ln_entry<RQ, SPAN, STAGED>(xs, cs, xg, cg, b4.x & 0xffffu, uu, vlane, part);
    if (it + 1 < cnt) part = ln_entry<RQ, SPAN, STAGED>(xs, cs, xg, cg, b4.x >> 16, uu, vlane, part);
    if (it + 2 < cnt) part = ln_entry<RQ, SPAN, STAGED>(xs, cs, xg, cg, b4.y & 0xffffu, uu, vlane, part);
    if (it + 3 < cnt) part = ln_entry<RQ, SPAN, STAGED>(xs, cs, xg, cg, b4.y >> 16, uu, vlane, part);
  }
  return part;
}

// grid = K * (n / SPAN) blocks of 32 kLnWarps threads (block b: span b % nspans); factors row-major
// with stride 4 RQ (padding -inf).  recs = the chunk records, coff[id] = start of record id in
// 16-byte units (id = span * (m / 4) + row-chunk).  cpw = chunks per warp run (power of two
// dividing m / 4).
template <int RQ, int SPAN>
__global__ void __launch_bounds__(32 * kLnWarps, RQ <= 2 ? 2 : 1)
k_maxplus_err_lanes(int64_t m, int64_t n, const unsigned char* __restrict__ recs, const int64_t* __restrict__ coff,
                    const float* __restrict__ Urm, const float* __restrict__ Vrm, u64* __restrict__ acc,
                    int* __restrict__ flags, int F, double exact_limit, int cpw_log2, int nstage, int stage_cap) {
  extern __shared__ __align__(128) unsigned char ln_smem[];
  float4* Vs = reinterpret_cast<float4*>(ln_smem);  // [RQ][SPAN]
  unsigned char* stg = ln_smem + sizeof(float4) * RQ * SPAN;
  __shared__ __align__(8) uint64_t bars[kLnWarps][kLnMaxStages];
  __shared__ int64_t meta_off[kLnWarps][kLnMaxStages];
  __shared__ int meta_bytes[kLnWarps][kLnMaxStages];
  __shared__ double red[kLnWarps];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, q = lane >> 3, j = lane & 7;
  const int nspans = (int)(n / SPAN);
  const int cs = (int)(blockIdx.x % nspans), kb = (int)(blockIdx.x / nspans), K = (int)(gridDim.x / nspans);
  const int64_t nrc = m / kLnRows;
  const int cpw = 1 << cpw_log2;
  for (int c = tid; c < SPAN; c += 32 * kLnWarps) {
    const float4* src = reinterpret_cast<const float4*>(Vrm + ((int64_t)cs * SPAN + c) * (4 * RQ));
#pragma unroll
    for (int q2 = 0; q2 < RQ; q2++) Vs[q2 * SPAN + c] = __ldg(src + q2);
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
  const int64_t r0 = (int64_t)kb * kLnWarps + wid, rstep = (int64_t)K * kLnWarps;
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

  // the lane's U row of a chunk, prefetched one chunk ahead
  float4 uuN[RQ];
  auto prefetch = [&](int64_t t) {
    if (t >= nT) return;
    const float4* ur = reinterpret_cast<const float4*>(Urm + (chunk_rc(t) * kLnRows + q) * (4 * RQ));
#pragma unroll
    for (int q2 = 0; q2 < RQ; q2++) uuN[q2] = __ldg(ur + q2);
  };
  prefetch(0);
  const unsigned vlane = smem_u32(Vs) + j * 16;
  const unsigned stg_s = smem_u32(mystg);
  double part = 0.0;
  unsigned phase = 0;
  int s = 0;
  for (int64_t t = 0; t < nT; t++) {
    float4 uu[RQ];
#pragma unroll
    for (int q2 = 0; q2 < RQ; q2++) uu[q2] = uuN[q2];
    prefetch(t + 1);
    const int bytes = meta_bytes[wid][s];
    if (bytes <= stage_cap) {
      ln_mbar_wait(&bars[wid][s], (phase >> s) & 1u);
      phase ^= 1u << s;
      part = ln_chunk<RQ, SPAN, true>(stg_s + s * stage_cap, nullptr, uu, vlane, lane, part);
    } else {  // a record larger than a stage: read straight from global memory
      part = ln_chunk<RQ, SPAN, false>(0, recs + meta_off[wid][s] * 16, uu, vlane, lane, part);
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
    for (int w = 0; w < kLnWarps; w++) sum = __dadd_rn(sum, red[w]);
    int fl = 0;
    if (!(sum < exact_limit)) fl |= 4;
    u64 hi, lo;
    fx_from_double(sum, F, hi, lo, fl);
    fx_atomic_add(acc, hi, lo);
    if (fl) atomicOr(flags, fl);
  }
}

// format build (not timed, once per matrix).  Chunk id = span * (m / 4) + row-chunk; a warp
// per chunk; lane l = 8 q + j counts / writes the entries of row q with column class
// c mod 8 == j, columns ascending.  cnt[id] = the record's size in 16-byte units.
// A lane's bits of mask word w: 0x01010101 << j (columns w * 32 + j + 8 t, t = 0..3).
__device__ __forceinline__ int ln_lane_count(const uint32_t* __restrict__ mrow, int span, int j) {
  int c = 0;
  for (int w = 0; w < span / 32; w++) c += __popc(mrow[w] & (0x01010101u << j));
  return c;
}

__global__ void k_ln_count(int64_t m, int64_t n, int span, const uint32_t* __restrict__ mask, int64_t* __restrict__ cnt,
                           int* __restrict__ maxrec) {
  const int lane = threadIdx.x & 31, q = lane >> 3, j = lane & 7;
  const int64_t nrc = m / kLnRows, nch = nrc * (n / span), wpr = n / 32;
  for (int64_t id = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; id < nch;
       id += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t cs = id / nrc, rc = id - cs * nrc;
    const int c = ln_lane_count(mask + (rc * kLnRows + q) * wpr + cs * (span / 32), span, j);
    const int total = __reduce_add_sync(0xffffffffu, c), maxc = __reduce_max_sync(0xffffffffu, c);
    if (lane == 0) {
      const int bytes = ln_record_bytes(total, maxc);
      cnt[id] = bytes / 16;
      atomicMax(maxrec, bytes);
    }
  }
}

__global__ void k_ln_fill(int64_t m, int64_t n, int span, const uint32_t* __restrict__ mask, const float* __restrict__ X,
                          const int64_t* __restrict__ coff, unsigned char* __restrict__ recs) {
  const int lane = threadIdx.x & 31, q = lane >> 3, j = lane & 7;
  const int64_t nrc = m / kLnRows, nch = nrc * (n / span), wpr = n / 32;
  for (int64_t id = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; id < nch;
       id += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t cs = id / nrc, rc = id - cs * nrc, row = rc * kLnRows + q;
    const uint32_t* mrow = mask + row * wpr + cs * (span / 32);
    const float* xrow = X + row * n + cs * span;
    const int c = ln_lane_count(mrow, span, j);
    const int total = __reduce_add_sync(0xffffffffu, c), maxc = __reduce_max_sync(0xffffffffu, c);
    // rank: lanes by decreasing count, ties by lane
    int rank = 0;
    for (int l = 0; l < 32; l++) {
      const int cl = __shfl_sync(0xffffffffu, c, l);
      rank += (cl > c) || (cl == c && l < lane);
    }
    unsigned char* rec = recs + coff[id] * 16;
    unsigned short* hdr = reinterpret_cast<unsigned short*>(rec);
    hdr[lane] = (unsigned short)c;
    if (lane == 0) { hdr[32] = (unsigned short)total; hdr[33] = (unsigned short)maxc; }
    rec[68 + lane] = (unsigned char)rank;
    // base[it] = sum over lanes of min(count, it): the slots used by earlier iterations
    unsigned short* bases = reinterpret_cast<unsigned short*>(rec + kLnHeader);
    for (int it0 = 0; it0 < maxc; it0 += 32) {
      const int it = it0 + lane;
      int b = 0;
      for (int l = 0; l < 32; l++) b += min(__shfl_sync(0xffffffffu, c, l), it);
      if (it < maxc) bases[it] = (unsigned short)b;
    }
    __syncwarp();
    const int nb = (2 * maxc + 15) & ~15;
    float* xv = reinterpret_cast<float*>(rec + kLnHeader + nb);
    unsigned char* cd = rec + kLnHeader + nb + 4 * ((total + 3) & ~3);
    // the lane's entries in column order: entry number e goes to slot base[e] + rank
    int e = 0;
    for (int w = 0; w < span / 32; w++) {
      uint32_t cur = mrow[w] & (0x01010101u << j);
      while (cur) {
        const int b = __ffs(cur) - 1;
        cur &= cur - 1;
        const int col = w * 32 + b, slot = bases[e] + rank;
        xv[slot] = xrow[col];
        cd[slot] = (unsigned char)(col >> 3);
        e++;
      }
    }
  }
}

}  // namespace stmf
