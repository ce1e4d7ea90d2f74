// stmf_maxplus_lanes.cuh — config-5 kernel for low densities, second generation:
// the "lane-compacted" sampled layout.  Included by stmf_api.cu after stmf_maxplus.cuh.
//
//   err = sum over given (i, j) of |X_ij - max_k (U_ik + V_kj)|   (tropical.py:214-222 in
//   binary32 with the exact-sum semantics of the fit's objective)
//
// What the first sampled kernel (k_maxplus_err_sampled) paid for: a per-tile decode of the
// mask into (row, column) codes and two bank-conflicted gathers of staged factor rows per
// given entry (98 thread instructions per entry, 21% of HBM at 65536^2 / rank 4 / 10%).
// Here the work is laid out so that neither is needed:
//
//  * A chunk = 4 rows x 1024 columns is one warp's unit.  Lane l = 8 q + j owns row q of
//    the chunk and the 128 consecutive columns [128 j, 128 j + 128) of the span, i.e. ONE
//    aligned uint4 of the ordinary row-major bit-packed mask (no custom bit order).  Its
//    U row lives in registers.
//  * The span's V rows are staged in shared memory transposed, V row c at slot
//    (c mod 128) * 8 + c / 128, so the 8 lanes of a quarter-warp always hit 8 different
//    16-byte bank groups: the per-entry V gather is conflict free by construction.
//  * The chunk's given values are stored "iteration-major, compacted": first the first
//    given value of every lane that has one (in lane order), then the second of every lane
//    that has two, ...  In iteration `it` lane l reads slot base_it + popc(ballot(it < cnt)
//    & lanemask_lt): consecutive lanes read consecutive floats, with no padding in memory.
//    Chunks start 16-byte aligned (<= 3 pad values per chunk) and are ordered span-major,
//    row-chunks ascending, so one warp's run of chunks is one contiguous byte range.
//  * Each warp streams its chunks through a ring of shared-memory stages filled by 1-D bulk
//    async copies (cp.async.bulk ... mbarrier::complete_tx): enough bytes in flight to
//    cover HBM latency without register-staged loads.
//
// Algorithmic bytes are those of the sampled layout: m n / 8 (mask) + 4 given + factors;
// the chunk offsets add 8 bytes per 4096 entries (0.06 bit per entry).
#pragma once

namespace stmf {

constexpr int kLnSpan = 1024;    // columns per chunk (8 lanes x 128 bits)
constexpr int kLnRows = 4;       // rows per chunk (4 quarter-warps)
constexpr int kLnMaxStages = 4;

__device__ __forceinline__ void ln_mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n LNWAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra LNWAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ float ln_lds(unsigned a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ float4 ln_lds4(unsigned a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}

// one lane's entries of a chunk.  w..w3: the lane's four mask words bit-reversed (so the
// lowest column is the leading one); the chunk's compacted values are at shared address
// sv_s (STAGED) or global pointer sv_g; vtop = shared address of the lane's V slot for
// bit 31 of the current (reversed) word, so bit position p (from the LSB) is at vtop - 128 p
template <int RQ, bool STAGED>
__device__ __forceinline__ double ln_chunk(unsigned sv_s, const float* __restrict__ sv_g, uint32_t w, uint32_t w1,
                                           uint32_t w2, uint32_t w3, const float4 (&uu)[RQ], unsigned vtop, int cnt,
                                           int maxc, unsigned ltmask, double part) {
  asm volatile("" : "+r"(sv_s), "+r"(vtop));  // keep both addresses in registers (no rematerialisation in the loop)
  int base = 0;
  for (int it = 0; it < maxc; ++it) {
    const bool act = it < cnt;
    const unsigned bal = __ballot_sync(0xffffffffu, act);
    if (act) {
      // next nonzero word of the lane's 128 bits (terminates: the lane still has entries)
      asm volatile(
          "{\n .reg .pred p;\n"
          " LNADV_%=:\n setp.ne.u32 p, %0, 0;\n @p bra LNDONE_%=;\n"
          " mov.u32 %0, %1;\n mov.u32 %1, %2;\n mov.u32 %2, %3;\n mov.u32 %3, 0;\n add.u32 %4, %4, 4096;\n"
          " bra LNADV_%=;\n LNDONE_%=:\n}"
          : "+r"(w), "+r"(w1), "+r"(w2), "+r"(w3), "+r"(vtop));
      const int p = 31 - __clz(w);
      w &= (1u << p) - 1u;
      const int rank = __popc(bal & ltmask);
      const float x = STAGED ? ln_lds(sv_s + 4u * (base + rank)) : __ldg(sv_g + base + rank);
      const unsigned va = vtop - 128u * p;
      float p0 = -CUDART_INF_F, p1 = -CUDART_INF_F;
#pragma unroll
      for (int q = 0; q < RQ; q++) {
        const float4 v = ln_lds4(va + q * (kLnSpan * 16)), u = uu[q];
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
    base += __popc(bal);
  }
  return part;
}

// grid = K * (n / 1024) blocks of 256 threads (block b: span b % nspans); factors row-major
// with stride 4 RQ (padding -inf).  cpw = chunks per warp run (power of two dividing m / 4).
template <int RQ>
__global__ void __launch_bounds__(256)
k_maxplus_err_lanes(int64_t m, int64_t n, const uint32_t* __restrict__ mask, const float* __restrict__ vals,
                    const int64_t* __restrict__ coff, const float* __restrict__ Urm, const float* __restrict__ Vrm,
                    u64* __restrict__ acc, int* __restrict__ flags, int F, double exact_limit, int cpw_log2,
                    int nstage, int stage_cap) {
  extern __shared__ __align__(128) unsigned char ln_smem[];
  float4* Vs = reinterpret_cast<float4*>(ln_smem);  // [RQ][1024] transposed slots
  float* stg = reinterpret_cast<float*>(ln_smem + sizeof(float4) * RQ * kLnSpan);
  __shared__ __align__(8) uint64_t bars[8][kLnMaxStages];
  __shared__ int64_t meta_off[8][kLnMaxStages];
  __shared__ int meta_bytes[8][kLnMaxStages];
  __shared__ double red[8];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, q = lane >> 3, j = lane & 7;
  const int nspans = (int)(n / kLnSpan);
  const int cs = (int)(blockIdx.x % nspans), kb = (int)(blockIdx.x / nspans), K = (int)(gridDim.x / nspans);
  const int64_t nrc = m / kLnRows, wpr = n / 32;
  const int cpw = 1 << cpw_log2;
  // the span's V rows, transposed so that lane j's columns land in bank group j
  for (int s = tid; s < kLnSpan; s += 256) {
    const int c = (s & 7) * 128 + (s >> 3);
    const float4* src = reinterpret_cast<const float4*>(Vrm + ((int64_t)cs * kLnSpan + c) * (4 * RQ));
#pragma unroll
    for (int q2 = 0; q2 < RQ; q2++) Vs[q2 * kLnSpan + s] = __ldg(src + q2);
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
  auto load_offs = [&](int64_t run_i) -> int64_t {  // lane l: offset l of the run's cpw + 1 chunk offsets
    if (run_i >= nR || lane > cpw) return 0;
    return __ldg(coff + (int64_t)cs * nrc + ((r0 + run_i * rstep) << cpw_log2) + lane);
  };
  int64_t offC = load_offs(0), offN = load_offs(1);
  float* mystg = stg + (size_t)wid * nstage * stage_cap;
  // producer: chunk t into stage t % nstage
  auto issue = [&](int64_t t, int s) {
    if (t >= nT) return;
    const int l = (int)(t & (cpw - 1));
    if (l == 0 && t > 0) {
      offC = offN;
      offN = load_offs((t >> cpw_log2) + 1);
    }
    const int64_t o0 = __shfl_sync(0xffffffffu, offC, l), o1 = __shfl_sync(0xffffffffu, offC, l + 1);
    const int bytes = (int)(o1 - o0) * 4;
    if (lane == 0) {
      meta_off[wid][s] = o0;
      meta_bytes[wid][s] = bytes;
      if (bytes > 0 && bytes <= stage_cap * 4) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bars[wid][s])),
                     "r"((unsigned)bytes)
                     : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(mystg + (size_t)s * stage_cap)),
            "l"(vals + o0), "r"((unsigned)bytes), "r"(smem_u32(&bars[wid][s]))
            : "memory");
      }
    }
  };
  {
    int s = 0;
    for (int64_t t = 0; t < nstage; t++, s++) issue(t, s);
  }
  __syncwarp();

  // mask words and U row of a chunk (prefetched one chunk ahead)
  uint4 mwN = make_uint4(0, 0, 0, 0);
  float4 uuN[RQ];
  auto prefetch = [&](int64_t t) {
    if (t >= nT) return;
    const int64_t row = chunk_rc(t) * kLnRows + q;
    mwN = __ldg(reinterpret_cast<const uint4*>(mask + row * wpr + (int64_t)cs * (kLnSpan / 32)) + j);
#pragma unroll
    for (int q2 = 0; q2 < RQ; q2++) uuN[q2] = __ldg(reinterpret_cast<const float4*>(Urm + row * (4 * RQ)) + q2);
  };
  prefetch(0);
  unsigned ltmask;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(ltmask));
  const unsigned vtop0 = smem_u32(Vs) + j * 16 + 31 * 128;  // slot of (bit 31 of reversed word 0) = column 0... +31
  const unsigned stg_s = smem_u32(mystg);
  double part = 0.0;
  unsigned phase = 0;
  int s = 0;
  for (int64_t t = 0; t < nT; t++) {
    const uint4 mw = mwN;
    float4 uu[RQ];
#pragma unroll
    for (int q2 = 0; q2 < RQ; q2++) uu[q2] = uuN[q2];
    prefetch(t + 1);
    const int cnt = __popc(mw.x) + __popc(mw.y) + __popc(mw.z) + __popc(mw.w);
    const int maxc = __reduce_max_sync(0xffffffffu, cnt);
    const int bytes = meta_bytes[wid][s];
    if (bytes > 0 && bytes <= stage_cap * 4) {
      ln_mbar_wait(&bars[wid][s], (phase >> s) & 1u);
      phase ^= 1u << s;
      part = ln_chunk<RQ, true>(stg_s + 4u * s * stage_cap, nullptr, __brev(mw.x), __brev(mw.y), __brev(mw.z),
                                __brev(mw.w), uu, vtop0, cnt, maxc, ltmask, part);
    } else if (bytes > 0) {  // a chunk larger than a stage: its values straight from global memory
      part = ln_chunk<RQ, false>(0, vals + meta_off[wid][s], __brev(mw.x), __brev(mw.y), __brev(mw.z), __brev(mw.w),
                                 uu, vtop0, cnt, maxc, ltmask, part);
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
  return sizeof(float4) * RQ * kLnSpan + sizeof(float) * 8 * (size_t)nstage * stage_cap;
}

// data preparation (not timed).  Chunk id = span * (m / 4) + row-chunk; a warp per chunk.
// cnt[id] = the chunk's given count rounded up to 4 values (16-byte aligned chunk starts).
__global__ void k_ln_count(int64_t m, int64_t n, const uint32_t* __restrict__ mask, int64_t* __restrict__ cnt,
                           int* __restrict__ maxchunk) {
  const int lane = threadIdx.x & 31, q = lane >> 3, j = lane & 7;
  const int64_t nrc = m / kLnRows, nch = nrc * (n / kLnSpan), wpr = n / 32;
  for (int64_t id = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; id < nch;
       id += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t cs = id / nrc, rc = id - cs * nrc;
    const uint4 mw = *(reinterpret_cast<const uint4*>(mask + (rc * kLnRows + q) * wpr + cs * (kLnSpan / 32)) + j);
    int c = __popc(mw.x) + __popc(mw.y) + __popc(mw.z) + __popc(mw.w);
    c = __reduce_add_sync(0xffffffffu, c);
    c = (c + 3) & ~3;
    if (lane == 0) {
      cnt[id] = c;
      atomicMax(maxchunk, c);
    }
  }
}

__global__ void k_ln_fill(int64_t m, int64_t n, const uint32_t* __restrict__ mask, const float* __restrict__ X,
                          const int64_t* __restrict__ coff, float* __restrict__ vals) {
  const int lane = threadIdx.x & 31, q = lane >> 3, j = lane & 7;
  const int64_t nrc = m / kLnRows, nch = nrc * (n / kLnSpan), wpr = n / 32;
  const unsigned lt = (1u << lane) - 1u;
  for (int64_t id = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; id < nch;
       id += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t cs = id / nrc, rc = id - cs * nrc, row = rc * kLnRows + q;
    const uint4 mw = *(reinterpret_cast<const uint4*>(mask + row * wpr + cs * (kLnSpan / 32)) + j);
    const uint32_t w[4] = {mw.x, mw.y, mw.z, mw.w};
    const float* xr = X + row * n + cs * kLnSpan + j * 128;
    float* out = vals + coff[id];
    int wi = 0, base = 0;
    uint32_t cur = w[0];
    for (;;) {
      while (cur == 0 && wi < 3) cur = w[++wi];
      const bool act = cur != 0;
      const unsigned bal = __ballot_sync(0xffffffffu, act);
      if (!bal) break;
      if (act) {
        const int b = __ffs(cur) - 1;
        cur &= cur - 1;
        out[base + __popc(bal & lt)] = xr[wi * 32 + b];
      }
      base += __popc(bal);
    }
  }
}

}  // namespace stmf
