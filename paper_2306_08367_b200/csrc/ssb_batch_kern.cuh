// The batched scan kernel (design in ssb_batch.cuh) and its launch templates;
// instantiated per batch size in ssb_batch_q{2,3,4}.cu (parallel compilation).
#pragma once

#include "ssb_batch.cuh"

namespace laq {
namespace scan {

// ---------------------------------------------------------------------------
// the batched scan
// ---------------------------------------------------------------------------

__device__ __forceinline__ uint32_t lds_u16(uint32_t addr) {
  uint16_t v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(addr));
  return static_cast<uint32_t>(v);
}
__device__ __forceinline__ uint2 lds_u64(uint32_t addr) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
  return v;
}

// Lane q of a row's accumulator (lo: lanes 0-1, hi: lanes 2-3).
__device__ __forceinline__ uint32_t lane_of(uint32_t lo, uint32_t hi, int q) {
  const uint32_t w = q < 2 ? lo : hi;
  return (q & 1) ? (w >> 16) : (w & 0xFFFFu);
}

// Accumulator layouts.  DW = 64: 4 x 16-bit lanes in (lo, hi), fail = 4096.
// DW = 32 (narrow decode, up to 3 queries): 3 x 10-bit lanes in lo alone, fail
// = B.fail32 (a power of two >= every G; the host checks that G - 1 + (links +
// filters + 1) fails fit 10 bits): one 4-byte decode load per link instead of
// 8 bytes (half the shared-memory wavefronts of the decode).
template <int DW>
__device__ __forceinline__ uint32_t lane_w(uint32_t lo, uint32_t hi, int q) {
  if constexpr (DW == 64) return lane_of(lo, hi, q);
  else return (lo >> (10 * q)) & 0x3FFu;
}
template <int DW>
__device__ __forceinline__ void add_fail(const BatchScan& B, uint32_t& lo, uint32_t& hi, int q, bool f) {
  if constexpr (DW == 64) {
    const uint32_t a = f ? (kLaneFail << (16 * (q & 1))) : 0u;
    if (q < 2) lo += a;
    else hi += a;
  } else {
    lo += f ? (B.fail32 << (10 * q)) : 0u;
  }
}

// Predicated (branch-free) shared atomic add and L2 gathers.
__device__ __forceinline__ void reds_add_if(bool p, uint32_t addr, uint32_t v) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q red.shared.add.u32 [%0], %1;\n}" ::"r"(addr), "r"(v),
               "r"(static_cast<uint32_t>(p))
               : "memory");
}
__device__ __forceinline__ uint32_t ldg_u8_if(bool p, const void* ptr, uint32_t dflt) {
  uint32_t v;
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\tmov.b32 %0, %3;\n\t@q ld.global.nc.u8 %0, [%1];\n}"
               : "=r"(v)
               : "l"(ptr), "r"(static_cast<uint32_t>(p)), "r"(dflt));
  return v;
}
__device__ __forceinline__ uint32_t ldg_u16_if(bool p, const void* ptr, uint32_t dflt) {
  uint32_t v;
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\tmov.b32 %0, %3;\n\t@q ld.global.nc.u16 %0, [%1];\n}"
               : "=r"(v)
               : "l"(ptr), "r"(static_cast<uint32_t>(p)), "r"(dflt));
  return v;
}

// Bulk L2 prefetch on the TMA engine (one instruction moves a warp's 512-byte
// slice of a column; no LSU wavefronts, no registers).
__device__ __forceinline__ void bulk_prefetch_l2(const Col& c, int64_t row0, int64_t n) {
  const int64_t rows = min(static_cast<int64_t>(128), n - row0);
  if (rows <= 0) return;
  const uint32_t bytes = static_cast<uint32_t>((rows * 4 + 15) & ~int64_t{15});
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(static_cast<const int32_t*>(c.p) + row0),
               "r"(bytes)
               : "memory");
}

// Row loads without the bounds test (steps whose rows are all in range).
__device__ __forceinline__ int4 ld4_nb(const Col& c, int64_t row0) {
  return __ldcs(reinterpret_cast<const int4*>(static_cast<const int32_t*>(c.p) + row0));
}

// Four rows per thread.  Each row's accumulator starts at B.init (kLaneFail in
// the lanes of queries that match nothing) or all-fail past the end; a fact
// filter adds kLaneFail to the lanes of the queries it rejects.  Every lookup
// is branch-free: a key outside the probe range is clamped to slot `size`,
// whose id is the miss tuple; L2 gathers are predicated instructions.  Decode
// tables are replicated B.dec_rep times with the copies interleaved per
// entry, lane l reading copy l % dec_rep (no bank conflicts between copies).
// MODE 0: per-thread register sums (every query has one group); MODE 1: u32
// (count, sum) bins; MODE 2: u32 sum bins only -- the measure is positive, so
// a group is present iff its sum is non-zero (half the shared atomics).
template <int NQ, int NL, int NF, int MODE, int DW, bool JP, bool TAIL>
__device__ __forceinline__ void batch_rows(const BatchScan& B, int64_t row0, const int4 (&kv)[NL],
                                           const int4 (&fv)[NF > 0 ? NF : 1], const int4& mv, uint32_t s_base,
                                           uint32_t dec_base, uint32_t (&r_cnt)[NQ],
                                           unsigned long long (&r_sum)[NQ]) {
  const uint32_t FL = DW == 64 ? kLaneFail : B.fail32;
  uint32_t lo[4], hi[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const bool past = TAIL && row0 + r >= B.n;
    lo[r] = past ? B.fail_lo : B.init_lo;
    hi[r] = DW == 32 ? 0u : (past ? B.fail_hi : B.init_hi);
  }
#pragma unroll
  for (int f = 0; f < NF; ++f)
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const uint32_t flo = static_cast<uint32_t>(B.ff_lo[f][q]);
      const uint32_t span = static_cast<uint32_t>(B.ff_hi[f][q]) - flo;
#pragma unroll
      for (int r = 0; r < 4; ++r)
        add_fail<DW>(B, lo[r], hi[r], q, static_cast<uint32_t>(comp(fv[f], r)) - flo > span);
    }
  const uint32_t sh = B.dec_shift;  // log2(entry bytes * dec_rep)
  uint32_t jid[4];
#pragma unroll
  for (int j = 0; j < NL; ++j) {
    const BatchLink& L = B.link[j];
    uint32_t sl[4], id[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) sl[r] = min(static_cast<uint32_t>(comp(kv[j], r)) - L.base, L.size);
    if (L.fmt == kIdSmemU8) {
#pragma unroll
      for (int r = 0; r < 4; ++r) id[r] = lds_u8(s_base + L.id_byte + sl[r]);
    } else if (L.fmt == kIdSmemU16) {
#pragma unroll
      for (int r = 0; r < 4; ++r) id[r] = lds_u16(s_base + L.id_byte + 2 * sl[r]);
    } else {
      // gathered through L2 only for rows some query still keeps (and, with a
      // staged any-pass bitmap, whose slot passes for some query)
      bool go[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        bool alive = false;
#pragma unroll
        for (int q = 0; q < NQ; ++q) alive = alive || lane_w<DW>(lo[r], hi[r], q) < FL;
        go[r] = alive;
      }
      if (L.bm_byte >= 0) {
#pragma unroll
        for (int r = 0; r < 4; ++r)
          go[r] = go[r] && ((lds_u32(s_base + L.bm_byte + 4 * (sl[r] >> 5)) >> (sl[r] & 31)) & 1u);
      }
      if (L.fmt == kIdGlobU8) {
#pragma unroll
        for (int r = 0; r < 4; ++r) id[r] = ldg_u8_if(go[r], static_cast<const uint8_t*>(L.ids) + sl[r], L.miss);
      } else {
#pragma unroll
        for (int r = 0; r < 4; ++r) id[r] = ldg_u16_if(go[r], static_cast<const uint16_t*>(L.ids) + sl[r], L.miss);
      }
    }
    if (JP && j == 0) {  // the pair's first id waits for link 1 (compile-time after unrolling)
#pragma unroll
      for (int r = 0; r < 4; ++r) jid[r] = id[r];
      continue;
    }
    if (JP && j == 1) {
#pragma unroll
      for (int r = 0; r < 4; ++r) id[r] += jid[r] * B.n_tup1;
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      if constexpr (DW == 64) {
        const uint2 d = lds_u64(dec_base + L.dec_byte + (id[r] << sh));
        lo[r] += d.x;
        hi[r] += d.y;
      } else {
        lo[r] += lds_u32(dec_base + L.dec_byte + (id[r] << sh));
      }
    }
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const uint32_t m = static_cast<uint32_t>(comp(mv, r));
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const uint32_t g = lane_w<DW>(lo[r], hi[r], q);
      const bool ok = g < FL;
      if constexpr (MODE == 0) {
        r_cnt[q] += ok ? 1u : 0u;
        r_sum[q] += ok ? static_cast<unsigned long long>(static_cast<long long>(static_cast<int32_t>(m))) : 0ull;
      } else if constexpr (MODE == 1) {
        const uint32_t ad = s_base + B.bins_byte[q] + 4u * g;
        reds_add_if(ok, ad, 1u);
        reds_add_if(ok, ad + 4u * static_cast<uint32_t>(B.G[q]), m);
      } else {
        reds_add_if(ok, s_base + B.bins_byte[q] + 4u * g, m);
      }
    }
  }
}

// MODE 2 spill: sum bins only; the count slot gets 1 per non-empty bin (a
// presence tally: non-zero iff the group has rows, all laq_plan_emit reads).
__device__ __forceinline__ void spill_sums32(uint32_t* b32, int64_t G, unsigned long long* acc, int t, int nt) {
  for (int64_t g = t; g < G; g += nt) {
    const uint32_t v = b32[g];
    if (v) {
      atomicAdd(acc + 2 * g, 1ull);
      atomicAdd(acc + 2 * g + 1, static_cast<unsigned long long>(v));
      b32[g] = 0;
    }
  }
}

template <int NQ, int MODE>
__device__ __forceinline__ void spill_all(const BatchScan& B, unsigned char* smem, int tid) {
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    uint32_t* b = reinterpret_cast<uint32_t*>(smem + B.bins_byte[q]);
    if constexpr (MODE == 1) spill_bins32(b, B.G[q], B.acc[q], tid, kDirectThreads);
    else spill_sums32(b, B.G[q], B.acc[q], tid, kDirectThreads);
  }
}

template <int NQ, int NL, int NF, int MODE, int DW, bool JP>
__global__ void __launch_bounds__(kDirectThreads, 1) scan_batch_kernel(const __grid_constant__ BatchScan B) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int tid = threadIdx.x;
  auto stage = [&](const void* src, int byte, int bytes) {
    const uint4* s = static_cast<const uint4*>(src);
    uint4* d = reinterpret_cast<uint4*>(smem + byte);
    for (int w = tid; w < bytes / 16; w += kDirectThreads) d[w] = __ldg(s + w);
  };
  const int rep = 1 << (B.dec_shift - (DW == 64 ? 3 : 2));
#pragma unroll
  for (int j = 0; j < NL; ++j) {
    const BatchLink& L = B.link[j];
    if (L.fmt == kIdSmemU8 || L.fmt == kIdSmemU16) stage(L.ids, L.id_byte, L.id_bytes);
    // Entry x of link j's table; with JP, link 1's table is the pair's joint
    // table (x = id0 * n_tup1 + id1: the sum of both links' entries, i.e. the
    // lanes the two separate adds would give) and link 0 stages none (n_dec 0).
    auto entry = [&](int x) -> unsigned long long {
      if (JP && j == 1)
        return __ldg(B.link[0].dec + x / static_cast<int>(B.n_tup1)) + __ldg(L.dec + x % static_cast<int>(B.n_tup1));
      return __ldg(L.dec + x);
    };
    if constexpr (DW == 64) {
      unsigned long long* d = reinterpret_cast<unsigned long long*>(smem + L.dec_byte);
      for (int w = tid; w < L.n_dec * rep; w += kDirectThreads) d[w] = entry(w / rep);  // entry-interleaved copies
    } else {
      // 16-bit lanes (fail = 4096 per failing link) -> 10-bit lanes (fail = B.fail32)
      uint32_t* d = reinterpret_cast<uint32_t*>(smem + L.dec_byte);
      for (int w = tid; w < L.n_dec * rep; w += kDirectThreads) {
        const unsigned long long e = entry(w / rep);
        uint32_t v = 0;
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          const uint32_t x = static_cast<uint32_t>(e >> (16 * q)) & 0xFFFFu;
          v |= (x >= kLaneFail ? B.fail32 : x) << (10 * q);
        }
        d[w] = v;
      }
    }
    if (L.bm_byte >= 0) stage(L.bm, L.bm_byte, L.bm_bytes);
  }
  if constexpr (MODE != 0) {
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      uint32_t* b = reinterpret_cast<uint32_t*>(smem + B.bins_byte[q]);
      for (int64_t g = tid; g < (MODE == 1 ? 2 : 1) * B.G[q]; g += kDirectThreads) b[g] = 0;
    }
  }
  __syncthreads();

  const uint32_t s_base = smem_u32(smem);
  const uint32_t dec_base = s_base + (DW == 64 ? 8u : 4u) * static_cast<uint32_t>(tid & (rep - 1));
  uint32_t r_cnt[NQ];
  unsigned long long r_sum[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) r_cnt[q] = 0, r_sum[q] = 0;

  const int64_t step = static_cast<int64_t>(gridDim.x) * kDirectThreads * 4;
  const int64_t iters = (B.n + step - 1) / step;
  const int64_t full = B.n / step;
  int64_t row0 = (static_cast<int64_t>(blockIdx.x) * kDirectThreads + tid) * 4;
  // prefetch > 0: prefetch.global.L2 by every 8th lane; prefetch < 0: TMA bulk
  // prefetch of the warp's slice by lane 0, |prefetch| steps ahead
  const bool pf_lane = B.prefetch > 0 && (tid & 7) == 0;
  const bool pf_bulk = B.prefetch < 0 && (tid & 31) == 0;
  const int64_t pf_rows = static_cast<int64_t>(B.prefetch < 0 ? -B.prefetch : B.prefetch) * step;

  int4 kvA[NL], fvA[NF > 0 ? NF : 1], mvA = make_int4(0, 0, 0, 0);
  int4 kvB[NL], fvB[NF > 0 ? NF : 1], mvB = make_int4(0, 0, 0, 0);
  auto load = [&](int4 (&kv)[NL], int4 (&fv)[NF > 0 ? NF : 1], int4& mv, int64_t r, bool inb) {
    if (inb) {  // every row of the step exists: no per-load bounds test
#pragma unroll
      for (int j = 0; j < NL; ++j) kv[j] = ld4_nb(B.fkc[j], r);
#pragma unroll
      for (int f = 0; f < NF; ++f) fv[f] = ld4_nb(B.ffc[f], r);
      if (B.has_measure) mv = ld4_nb(B.mc, r);
    } else {
#pragma unroll
      for (int j = 0; j < NL; ++j) kv[j] = dld<0>(B.fkc[j], r, B.n);
#pragma unroll
      for (int f = 0; f < NF; ++f) fv[f] = dld<0>(B.ffc[f], r, B.n);
      if (B.has_measure) mv = dld<0>(B.mc, r, B.n);
    }
  };
  load(kvA, fvA, mvA, row0, full > 0);
  int64_t until_flush = B.flush_every;
  auto one = [&](int64_t it, const int4 (&kv)[NL], const int4 (&fv)[NF > 0 ? NF : 1], const int4& mv,
                 int4 (&nkv)[NL], int4 (&nfv)[NF > 0 ? NF : 1], int4& nmv) {
    load(nkv, nfv, nmv, row0 + step, it + 1 < full);
    if (pf_lane && row0 + pf_rows < B.n) {
#pragma unroll
      for (int j = 0; j < NL; ++j) prefetch_l2<0>(B.fkc[j], row0 + pf_rows);
#pragma unroll
      for (int f = 0; f < NF; ++f) prefetch_l2<0>(B.ffc[f], row0 + pf_rows);
      if (B.has_measure) prefetch_l2<0>(B.mc, row0 + pf_rows);
    }
    if (pf_bulk && row0 + pf_rows < B.n) {
#pragma unroll
      for (int j = 0; j < NL; ++j) bulk_prefetch_l2(B.fkc[j], row0 + pf_rows, B.n);
#pragma unroll
      for (int f = 0; f < NF; ++f) bulk_prefetch_l2(B.ffc[f], row0 + pf_rows, B.n);
      if (B.has_measure) bulk_prefetch_l2(B.mc, row0 + pf_rows, B.n);
    }
    if (it < full)
      batch_rows<NQ, NL, NF, MODE, DW, JP, false>(B, row0, kv, fv, mv, s_base, dec_base, r_cnt, r_sum);
    else
      batch_rows<NQ, NL, NF, MODE, DW, JP, true>(B, row0, kv, fv, mv, s_base, dec_base, r_cnt, r_sum);
    if constexpr (MODE != 0) {
      if (--until_flush == 0) {
        until_flush = B.flush_every;
        if (it + 1 < iters) {
          __syncthreads();
          spill_all<NQ, MODE>(B, smem, tid);
          __syncthreads();
        }
      }
    }
    row0 += step;
  };
  for (int64_t it = 0; it < iters; it += 2) {
    one(it, kvA, fvA, mvA, kvB, fvB, mvB);
    if (it + 1 < iters) one(it + 1, kvB, fvB, mvB, kvA, fvA, mvA);
  }
  if constexpr (MODE == 0) {
#pragma unroll
    for (int q = 0; q < NQ; ++q) flush_single(r_cnt[q], r_sum[q], B.acc[q]);
  } else {
    __syncthreads();
    spill_all<NQ, MODE>(B, smem, tid);
  }
}

// ---------------------------------------------------------------------------
// Software-pipelined form for batches whose LAST probe link is gathered
// through L2 (SF=100 Q4.x: the 1.4M-slot part ids; SF=10 Q2.x).  Two rows per
// thread; iteration i runs stage A of its own rows (fact filters, the staged
// links, then ISSUES the predicated L2 gather of the last link) and stage B of
// iteration i-1's rows (that gather's decode + the bins), so each gather has a
// whole iteration of other work to hide behind.  Fact columns are register
// double-buffered 8-byte vectors and prefetched into L2 two steps ahead.
// ---------------------------------------------------------------------------
struct PipeState {
  uint32_t lo[2], hi[2], id[2], m[2];
};

__device__ __forceinline__ int comp2(const int2& v, int i) { return i == 0 ? v.x : v.y; }

__device__ __forceinline__ int2 ld2(const Col& c, int64_t row0, int64_t n, bool inb) {
  const int2* p = reinterpret_cast<const int2*>(static_cast<const int32_t*>(c.p) + row0);
  return inb || row0 < n ? __ldcs(p) : make_int2(0, 0);  // columns are padded past the end
}

template <int NQ, int NL, int NF, bool TAIL>
__device__ __forceinline__ void pipe_stage_a(const BatchScan& B, int64_t row0, const int2 (&kv)[NL],
                                             const int2 (&fv)[NF > 0 ? NF : 1], const int2& mv, uint32_t s_base,
                                             uint32_t dec_base, PipeState& st) {
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const bool past = TAIL && row0 + r >= B.n;
    st.lo[r] = past ? B.fail_lo : B.init_lo;
    st.hi[r] = past ? B.fail_hi : B.init_hi;
    st.m[r] = static_cast<uint32_t>(comp2(mv, r));
  }
#pragma unroll
  for (int f = 0; f < NF; ++f)
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const uint32_t flo = static_cast<uint32_t>(B.ff_lo[f][q]);
      const uint32_t span = static_cast<uint32_t>(B.ff_hi[f][q]) - flo;
      const uint32_t add = kLaneFail << (16 * (q & 1));
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const uint32_t a = static_cast<uint32_t>(comp2(fv[f], r)) - flo > span ? add : 0u;
        if (q < 2) st.lo[r] += a;
        else st.hi[r] += a;
      }
    }
  const uint32_t sh = B.dec_shift;
#pragma unroll
  for (int j = 0; j < NL; ++j) {
    const BatchLink& L = B.link[j];
    uint32_t sl[2], id[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) sl[r] = min(static_cast<uint32_t>(comp2(kv[j], r)) - L.base, L.size);
    if (L.fmt == kIdSmemU8) {
#pragma unroll
      for (int r = 0; r < 2; ++r) id[r] = lds_u8(s_base + L.id_byte + sl[r]);
    } else if (L.fmt == kIdSmemU16) {
#pragma unroll
      for (int r = 0; r < 2; ++r) id[r] = lds_u16(s_base + L.id_byte + 2 * sl[r]);
    } else {
      bool go[2];
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        bool alive = false;
#pragma unroll
        for (int q = 0; q < NQ; ++q) alive = alive || lane_of(st.lo[r], st.hi[r], q) < kLaneFail;
        go[r] = alive;
        if (L.bm_byte >= 0)
          go[r] = go[r] && ((lds_u32(s_base + L.bm_byte + 4 * (sl[r] >> 5)) >> (sl[r] & 31)) & 1u);
      }
#pragma unroll
      for (int r = 0; r < 2; ++r)
        id[r] = L.fmt == kIdGlobU8 ? ldg_u8_if(go[r], static_cast<const uint8_t*>(L.ids) + sl[r], L.miss)
                                   : ldg_u16_if(go[r], static_cast<const uint16_t*>(L.ids) + sl[r], L.miss);
    }
    if (j == NL - 1) {  // the last link's decode waits for stage B (one iteration later)
#pragma unroll
      for (int r = 0; r < 2; ++r) st.id[r] = id[r];
    } else {
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const uint2 d = lds_u64(dec_base + L.dec_byte + (id[r] << sh));
        st.lo[r] += d.x;
        st.hi[r] += d.y;
      }
    }
  }
}

template <int NQ, int NL, int MODE>
__device__ __forceinline__ void pipe_stage_b(const BatchScan& B, const PipeState& st, uint32_t s_base,
                                             uint32_t dec_base) {
  const BatchLink& L = B.link[NL - 1];
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const uint2 d = lds_u64(dec_base + L.dec_byte + (st.id[r] << B.dec_shift));
    const uint32_t lo = st.lo[r] + d.x, hi = st.hi[r] + d.y;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const uint32_t g = lane_of(lo, hi, q);
      const bool ok = g < kLaneFail;
      if constexpr (MODE == 1) {
        const uint32_t ad = s_base + B.bins_byte[q] + 4u * g;
        reds_add_if(ok, ad, 1u);
        reds_add_if(ok, ad + 4u * static_cast<uint32_t>(B.G[q]), st.m[r]);
      } else {
        reds_add_if(ok, s_base + B.bins_byte[q] + 4u * g, st.m[r]);
      }
    }
  }
}

template <int NQ, int NL, int NF, int MODE>
__global__ void __launch_bounds__(kDirectThreads, 1) scan_batch_pipe_kernel(const __grid_constant__ BatchScan B) {
  static_assert(MODE == 1 || MODE == 2, "bins modes only");
  extern __shared__ __align__(16) unsigned char smem[];
  const int tid = threadIdx.x;
  auto stage = [&](const void* src, int byte, int bytes) {
    const uint4* s = static_cast<const uint4*>(src);
    uint4* d = reinterpret_cast<uint4*>(smem + byte);
    for (int w = tid; w < bytes / 16; w += kDirectThreads) d[w] = __ldg(s + w);
  };
  const int rep = 1 << (B.dec_shift - 3);
#pragma unroll
  for (int j = 0; j < NL; ++j) {
    const BatchLink& L = B.link[j];
    if (L.fmt == kIdSmemU8 || L.fmt == kIdSmemU16) stage(L.ids, L.id_byte, L.id_bytes);
    unsigned long long* d = reinterpret_cast<unsigned long long*>(smem + L.dec_byte);
    for (int w = tid; w < L.n_dec * rep; w += kDirectThreads) d[w] = __ldg(L.dec + w / rep);
    if (L.bm_byte >= 0) stage(L.bm, L.bm_byte, L.bm_bytes);
  }
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    uint32_t* b = reinterpret_cast<uint32_t*>(smem + B.bins_byte[q]);
    for (int64_t g = tid; g < (MODE == 1 ? 2 : 1) * B.G[q]; g += kDirectThreads) b[g] = 0;
  }
  __syncthreads();
  const uint32_t s_base = smem_u32(smem);
  const uint32_t dec_base = s_base + 8u * static_cast<uint32_t>(tid & (rep - 1));

  const int64_t step = static_cast<int64_t>(gridDim.x) * kDirectThreads * 2;
  const int64_t iters = (B.n + step - 1) / step;
  const int64_t full = B.n / step;
  int64_t row0 = (static_cast<int64_t>(blockIdx.x) * kDirectThreads + tid) * 2;
  const bool pf_lane = B.prefetch && (tid & 15) == 0;  // one 128-byte line per 16 lanes
  const int64_t pf_rows = static_cast<int64_t>(B.prefetch) * step;

  int2 kvA[NL], fvA[NF > 0 ? NF : 1], mvA = make_int2(0, 0);
  int2 kvB[NL], fvB[NF > 0 ? NF : 1], mvB = make_int2(0, 0);
  auto load = [&](int2 (&kv)[NL], int2 (&fv)[NF > 0 ? NF : 1], int2& mv, int64_t r, bool inb) {
#pragma unroll
    for (int j = 0; j < NL; ++j) kv[j] = ld2(B.fkc[j], r, B.n, inb);
#pragma unroll
    for (int f = 0; f < NF; ++f) fv[f] = ld2(B.ffc[f], r, B.n, inb);
    if (B.has_measure) mv = ld2(B.mc, r, B.n, inb);
  };
  PipeState sA, sB;
  load(kvA, fvA, mvA, row0, full > 0);
  int64_t until_flush = B.flush_every;
  // iteration it: loads for it+1, stage A(it), stage B(it-1)
  auto one = [&](int64_t it, const int2 (&kv)[NL], const int2 (&fv)[NF > 0 ? NF : 1], const int2& mv,
                 int2 (&nkv)[NL], int2 (&nfv)[NF > 0 ? NF : 1], int2& nmv, PipeState& cur, const PipeState& prev) {
    if (it + 1 < iters) load(nkv, nfv, nmv, row0 + step, it + 1 < full);
    if (pf_lane && row0 + pf_rows < B.n) {
#pragma unroll
      for (int j = 0; j < NL; ++j) prefetch_l2<0>(B.fkc[j], row0 + pf_rows);
#pragma unroll
      for (int f = 0; f < NF; ++f) prefetch_l2<0>(B.ffc[f], row0 + pf_rows);
      if (B.has_measure) prefetch_l2<0>(B.mc, row0 + pf_rows);
    }
    if (it < full) pipe_stage_a<NQ, NL, NF, false>(B, row0, kv, fv, mv, s_base, dec_base, cur);
    else pipe_stage_a<NQ, NL, NF, true>(B, row0, kv, fv, mv, s_base, dec_base, cur);
    if (it > 0) {
      pipe_stage_b<NQ, NL, MODE>(B, prev, s_base, dec_base);
      if (--until_flush == 0) {
        until_flush = B.flush_every;
        __syncthreads();
        spill_all<NQ, MODE>(B, smem, tid);
        __syncthreads();
      }
    }
    row0 += step;
  };
  for (int64_t it = 0; it < iters; it += 2) {
    one(it, kvA, fvA, mvA, kvB, fvB, mvB, sA, sB);
    if (it + 1 < iters) one(it + 1, kvB, fvB, mvB, kvA, fvA, mvA, sB, sA);
  }
  if (iters > 0) pipe_stage_b<NQ, NL, MODE>(B, (iters & 1) ? sA : sB, s_base, dec_base);
  __syncthreads();
  spill_all<NQ, MODE>(B, smem, tid);
}

template <int NQ, int NL, int NF, int MODE>
void launch_batch_t(laq_ctx* ctx, const BatchScan& B, size_t smem, int grid) {
  if constexpr (MODE != 0) {
    if (B.pipe) {
      auto kern = scan_batch_pipe_kernel<NQ, NL, NF, MODE>;
      LAQ_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
      const int64_t blocks_needed = (B.n + kDirectThreads * 2 - 1) / (kDirectThreads * 2);
      const int g = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(grid, blocks_needed)));
      kern<<<g, kDirectThreads, smem, ctx->stream>>>(B);
      return;
    }
  }
  auto kern = scan_batch_kernel<NQ, NL, NF, MODE, 64, false>;
  if constexpr (NQ <= 3 && NL <= 3) {
    if (B.dec32) kern = scan_batch_kernel<NQ, NL, NF, MODE, 32, false>;
  }
  if constexpr (MODE == 2 && NL >= 2) {  // joint pair: the positive-measure (sum-bin) batches only
    if (B.joint01) {
      kern = scan_batch_kernel<NQ, NL, NF, MODE, 64, true>;
      if constexpr (NQ <= 3 && NL <= 3) {
        if (B.dec32) kern = scan_batch_kernel<NQ, NL, NF, MODE, 32, true>;
      }
    }
  }
  LAQ_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  const int64_t blocks_needed = (B.n + kDirectThreads * 4 - 1) / (kDirectThreads * 4);
  const int g = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(grid, blocks_needed)));
  kern<<<g, kDirectThreads, smem, ctx->stream>>>(B);
}

template <int NQ, int NL, int NF>
void launch_batch_m(laq_ctx* ctx, const BatchScan& B, int mode, size_t smem, int grid) {
  if (mode == 0) launch_batch_t<NQ, NL, NF, 0>(ctx, B, smem, grid);
  else if (mode == 1) launch_batch_t<NQ, NL, NF, 1>(ctx, B, smem, grid);
  else launch_batch_t<NQ, NL, NF, 2>(ctx, B, smem, grid);
}

template <int NQ, int NL>
void launch_batch_f(laq_ctx* ctx, const BatchScan& B, int nf, int mode, size_t smem, int grid) {
  switch (nf) {
    case 0: launch_batch_m<NQ, NL, 0>(ctx, B, mode, smem, grid); break;
    case 1: launch_batch_m<NQ, NL, 1>(ctx, B, mode, smem, grid); break;
    case 2: launch_batch_m<NQ, NL, 2>(ctx, B, mode, smem, grid); break;
    default: fail(LAQ_ERR_UNSUPPORTED, "batched scan: at most 2 fact filter columns");
  }
}

template <int NQ>
void launch_batch_q(laq_ctx* ctx, const BatchScan& B, int nl, int nf, int mode, size_t smem, int grid) {
  switch (nl) {
    case 1: launch_batch_f<NQ, 1>(ctx, B, nf, mode, smem, grid); break;
    case 2: launch_batch_f<NQ, 2>(ctx, B, nf, mode, smem, grid); break;
    case 3: launch_batch_f<NQ, 3>(ctx, B, nf, mode, smem, grid); break;
    case 4: launch_batch_f<NQ, 4>(ctx, B, nf, mode, smem, grid); break;
    case 5: launch_batch_f<NQ, 5>(ctx, B, nf, mode, smem, grid); break;
    case 6: launch_batch_f<NQ, 6>(ctx, B, nf, mode, smem, grid); break;
    default: fail(LAQ_ERR_UNSUPPORTED, "batched scan: 1..6 links");
  }
}

}  // namespace scan
}  // namespace laq
