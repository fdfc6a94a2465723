// Batched query scan kernels (design in ssb_batch.cuh): the device dictionary
// build of per-link code tuples and the one-pass scan of a batch of queries.
// Host side: laq_batch_* in ssb.cu.
#include "ssb_batch.cuh"

namespace laq {
namespace scan {

// ---------------------------------------------------------------------------
// dictionary build
// ---------------------------------------------------------------------------

__device__ __forceinline__ unsigned long long dict_key(const DictLink& L, int nq, int64_t s) {
  unsigned long long k = 0;
#pragma unroll
  for (int q = 0; q < kBatchMaxQ; ++q)
    if (q < nq && L.code[q]) {
      const int32_t c = __ldg(L.code[q] + s);
      const uint32_t lane = c >= 0 ? static_cast<uint32_t>(c) : kLaneFail;
      k |= static_cast<unsigned long long>(lane) << (16 * q);
    }
  return k;
}

__device__ __forceinline__ uint32_t dict_hash(unsigned long long k, int bits) {
  return static_cast<uint32_t>((k * 0x9E3779B97F4A7C15ull) >> (64 - bits));
}

__device__ __forceinline__ bool dict_any_pass(const DictLink& L, int nq, unsigned long long key) {
  bool any = false;
#pragma unroll
  for (int q = 0; q < kBatchMaxQ; ++q)
    if (q < nq && L.code[q]) any = any || ((key >> (16 * q)) & 0xFFFFull) < kLaneFail;
  return any;
}

// Phase 1: insert every slot's tuple.  Consecutive slots mostly repeat a
// tuple, so one lane per distinct key of the warp inserts (match_any), and the
// CAS is only tried on an empty entry.
__global__ void dict_insert_kernel(const DictArgs d) {
  const int64_t total = d.start[d.nl];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    int j = 0;
    while (i >= d.start[j + 1]) ++j;
    const DictLink& L = d.l[j];
    const int64_t s = i - d.start[j];
    const bool in = s < L.slots;
    const unsigned long long key = in ? dict_key(L, d.nq, s) : kDictEmpty;
    const unsigned peers = __match_any_sync(0xffffffffu, key);
    if (!in || static_cast<int>(__ffs(peers)) - 1 != static_cast<int>(threadIdx.x & 31)) continue;
    const uint32_t mask = (1u << L.hbits) - 1u;
    uint32_t h = dict_hash(key, L.hbits);
    bool done = false;
    for (uint32_t p = 0; p <= mask && !done; ++p, h = (h + 1) & mask) {
      unsigned long long cur = *reinterpret_cast<volatile unsigned long long*>(L.hkeys + h);
      if (cur == key) {
        done = true;
      } else if (cur == kDictEmpty) {
        cur = atomicCAS(L.hkeys + h, kDictEmpty, key);
        done = cur == kDictEmpty || cur == key;
      }
    }
    if (!done) atomicOr(d.overflow, 1);
  }
}

// Phase 2 (one CTA per link): number the occupied entries -> tuple ids; write
// the decode table and the miss entry (id = number of tuples).
__global__ void __launch_bounds__(1024) dict_rank_kernel(const DictArgs d) {
  const DictLink& L = d.l[blockIdx.x];
  const int hs = 1 << L.hbits;
  const int per = (hs + 1023) / 1024;
  const int b = threadIdx.x * per, e = min(b + per, hs);
  int cnt = 0;
  for (int x = b; x < e; ++x) cnt += L.hkeys[x] != kDictEmpty ? 1 : 0;
  __shared__ int wsum[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int inc = cnt;
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += v;
  }
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    int w = wsum[lane];
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += v;
    }
    wsum[lane] = w;  // inclusive
  }
  __syncthreads();
  int id = (warp ? wsum[warp - 1] : 0) + inc - cnt;
  for (int x = b; x < e; ++x) {
    const unsigned long long k = L.hkeys[x];
    if (k == kDictEmpty) continue;
    L.hid[x] = id;
    if (id < L.dec_cap) L.dec[id] = k;
    ++id;
  }
  if (threadIdx.x == 1023) {
    const int n = id;  // tuples; the miss id is n
    const int lim = L.idw == 1 ? 256 : 65536;
    if (n + 1 > L.dec_cap || n + 1 > lim) atomicOr(d.overflow, 1);
    else L.dec[n] = L.miss;
    d.n_dec[blockIdx.x] = n + 1;
  }
}

// Phase 3: every slot's tuple id (and the any-pass bitmap: one warp ballot per
// 32 slots; links start at multiples of 32 flattened slots).
__global__ void dict_assign_kernel(const DictArgs d) {
  const int64_t total = d.start[d.nl];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    int j = 0;
    while (i >= d.start[j + 1]) ++j;
    const DictLink& L = d.l[j];
    const int64_t s = i - d.start[j];
    const bool in = s < L.slots;
    unsigned long long key = 0;
    if (in) {
      key = dict_key(L, d.nq, s);
      const uint32_t mask = (1u << L.hbits) - 1u;
      uint32_t h = dict_hash(key, L.hbits);
      int id = -1;
      for (uint32_t p = 0; p <= mask; ++p, h = (h + 1) & mask) {
        const unsigned long long k = L.hkeys[h];
        if (k == key) {
          id = L.hid[h];
          break;
        }
        if (k == kDictEmpty) break;
      }
      if (id < 0) atomicOr(d.overflow, 2);
      if (L.idw == 1) static_cast<uint8_t*>(L.ids)[s] = static_cast<uint8_t>(id);
      else static_cast<uint16_t*>(L.ids)[s] = static_cast<uint16_t>(id);
    }
    if (L.bm) {
      const unsigned bits = __ballot_sync(0xffffffffu, in && dict_any_pass(L, d.nq, key));
      if ((threadIdx.x & 31) == 0) L.bm[s >> 5] = bits;
    }
  }
}

void launch_dict_build(laq_ctx* ctx, const DictArgs& d) {
  const int64_t total = d.start[d.nl];
  if (total == 0) return;
  const int g = grid_for(total, 256, ctx->sm_count * 8);
  dict_insert_kernel<<<g, 256, 0, ctx->stream>>>(d);
  launched(ctx);
  dict_rank_kernel<<<d.nl, 1024, 0, ctx->stream>>>(d);
  launched(ctx);
  dict_assign_kernel<<<g, 256, 0, ctx->stream>>>(d);
  launched(ctx);
}

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

// Shared-memory addresses are s_base + a byte offset read from the kernel
// parameters (constant bank operands, no registers held across the loop).
template <int NL, int NF, int MODE, bool TAIL>
__device__ __forceinline__ void batch_rows(const BatchScan& B, int64_t row0, const int4 (&kv)[NL],
                                           const int4 (&fv)[NF > 0 ? NF : 1], const int4& mv, uint32_t s_base,
                                           uint32_t (&r_cnt)[kBatchMaxQ],
                                           unsigned long long (&r_sum)[kBatchMaxQ]) {
  const int nq = B.nq;
  uint32_t lo[4], hi[4], fm[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    lo[r] = hi[r] = 0;
    fm[r] = TAIL && row0 + r >= B.n ? 0xFu : B.reject_mask;  // bit q: query q rejects the row
  }
#pragma unroll
  for (int f = 0; f < NF; ++f) {
#pragma unroll
    for (int q = 0; q < kBatchMaxQ; ++q) {
      if (q >= nq) break;
      const int32_t flo = B.ff_lo[f][q];
      const uint32_t span = static_cast<uint32_t>(B.ff_hi[f][q]) - static_cast<uint32_t>(flo);
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const uint32_t off = static_cast<uint32_t>(comp(fv[f], r)) - static_cast<uint32_t>(flo);
        fm[r] |= off > span ? (1u << q) : 0u;
      }
    }
  }
#pragma unroll
  for (int j = 0; j < NL; ++j) {
    const BatchLink& L = B.link[j];
    const uint32_t base = L.base, size = L.size, miss = L.miss;
    const int fmt = L.fmt;
    uint32_t id[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const uint32_t s = static_cast<uint32_t>(comp(kv[j], r)) - base;
      const bool in = s < size;
      if (fmt == kIdSmemU8) {
        id[r] = in ? lds_u8(s_base + L.id_byte + s) : miss;
      } else if (fmt == kIdSmemU16) {
        id[r] = in ? lds_u16(s_base + L.id_byte + 2 * s) : miss;
      } else {
        // gathered through L2 only while some query still keeps the row
        bool alive = false;
#pragma unroll
        for (int q = 0; q < kBatchMaxQ; ++q)
          if (q < nq) alive = alive || (lane_of(lo[r], hi[r], q) < kLaneFail && !((fm[r] >> q) & 1u));
        bool go = in && alive;
        if (go && L.bm_byte >= 0) go = (lds_u32(s_base + L.bm_byte + 4 * (s >> 5)) >> (s & 31)) & 1u;
        id[r] = miss;
        if (go)
          id[r] = fmt == kIdGlobU8 ? static_cast<uint32_t>(__ldg(static_cast<const uint8_t*>(L.ids) + s))
                                   : static_cast<uint32_t>(__ldg(static_cast<const uint16_t*>(L.ids) + s));
      }
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const uint2 d = lds_u64(s_base + L.dec_byte + 8 * id[r]);
      lo[r] += d.x;
      hi[r] += d.y;
    }
  }
#pragma unroll
  for (int q = 0; q < kBatchMaxQ; ++q) {
    if (q >= nq) break;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const uint32_t g = lane_of(lo[r], hi[r], q);
      const bool ok = g < kLaneFail && !((fm[r] >> q) & 1u);
      if constexpr (MODE == 0) {
        r_cnt[q] += ok ? 1u : 0u;
        r_sum[q] += ok && B.has_measure ? static_cast<unsigned long long>(static_cast<long long>(comp(mv, r))) : 0ull;
      } else {
        if (ok) {
          const uint32_t ad = s_base + B.bins_byte[q] + 4u * g;
          reds_add(ad, 1u);
          if (B.has_measure) reds_add(ad + 4u * static_cast<uint32_t>(B.G[q]), static_cast<uint32_t>(comp(mv, r)));
        }
      }
    }
  }
}

template <int NL, int NF, int MODE>
__global__ void __launch_bounds__(kDirectThreads, 1) scan_batch_kernel(const __grid_constant__ BatchScan B) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int tid = threadIdx.x;
  auto stage = [&](const void* src, int byte, int bytes) {
    const uint4* s = static_cast<const uint4*>(src);
    uint4* d = reinterpret_cast<uint4*>(smem + byte);
    for (int w = tid; w < bytes / 16; w += kDirectThreads) d[w] = __ldg(s + w);
  };
#pragma unroll
  for (int j = 0; j < NL; ++j) {
    const BatchLink& L = B.link[j];
    if (L.fmt == kIdSmemU8 || L.fmt == kIdSmemU16) stage(L.ids, L.id_byte, L.id_bytes);
    stage(L.dec, L.dec_byte, L.dec_bytes);
    if (L.bm_byte >= 0) stage(L.bm, L.bm_byte, L.bm_bytes);
  }
  if constexpr (MODE == 1) {
    for (int q = 0; q < B.nq; ++q) {
      uint32_t* b = reinterpret_cast<uint32_t*>(smem + B.bins_byte[q]);
      for (int64_t g = tid; g < 2 * B.G[q]; g += kDirectThreads) b[g] = 0;
    }
  }
  __syncthreads();

  const uint32_t s_base = smem_u32(smem);
  uint32_t r_cnt[kBatchMaxQ];
  unsigned long long r_sum[kBatchMaxQ];
#pragma unroll
  for (int q = 0; q < kBatchMaxQ; ++q) r_cnt[q] = r_sum[q] = 0;

  const int64_t step = static_cast<int64_t>(gridDim.x) * kDirectThreads * 4;
  const int64_t iters = (B.n + step - 1) / step;
  const int64_t full = B.n / step;
  int64_t row0 = (static_cast<int64_t>(blockIdx.x) * kDirectThreads + tid) * 4;
  const bool pf_lane = B.prefetch && (tid & 7) == 0;
  const int64_t pf_rows = static_cast<int64_t>(B.prefetch) * step;

  int4 kvA[NL], fvA[NF > 0 ? NF : 1], mvA = make_int4(0, 0, 0, 0);
  int4 kvB[NL], fvB[NF > 0 ? NF : 1], mvB = make_int4(0, 0, 0, 0);
  auto load = [&](int4 (&kv)[NL], int4 (&fv)[NF > 0 ? NF : 1], int4& mv, int64_t r) {
#pragma unroll
    for (int j = 0; j < NL; ++j) kv[j] = dld<0>(B.fkc[j], r, B.n);
#pragma unroll
    for (int f = 0; f < NF; ++f) fv[f] = dld<0>(B.ffc[f], r, B.n);
    if (B.has_measure) mv = dld<0>(B.mc, r, B.n);
  };
  load(kvA, fvA, mvA, row0);
  int64_t until_flush = B.flush_every;
  auto one = [&](int64_t it, const int4 (&kv)[NL], const int4 (&fv)[NF > 0 ? NF : 1], const int4& mv,
                 int4 (&nkv)[NL], int4 (&nfv)[NF > 0 ? NF : 1], int4& nmv) {
    load(nkv, nfv, nmv, row0 + step);
    if (pf_lane && row0 + pf_rows < B.n) {
#pragma unroll
      for (int j = 0; j < NL; ++j) prefetch_l2<0>(B.fkc[j], row0 + pf_rows);
#pragma unroll
      for (int f = 0; f < NF; ++f) prefetch_l2<0>(B.ffc[f], row0 + pf_rows);
      if (B.has_measure) prefetch_l2<0>(B.mc, row0 + pf_rows);
    }
    if (it < full)
      batch_rows<NL, NF, MODE, false>(B, row0, kv, fv, mv, s_base, r_cnt, r_sum);
    else
      batch_rows<NL, NF, MODE, true>(B, row0, kv, fv, mv, s_base, r_cnt, r_sum);
    if constexpr (MODE == 1) {
      if (--until_flush == 0) {
        until_flush = B.flush_every;
        if (it + 1 < iters) {
          __syncthreads();
          for (int q = 0; q < B.nq; ++q)
            spill_bins32(reinterpret_cast<uint32_t*>(smem + B.bins_byte[q]), B.G[q], B.acc[q], tid, kDirectThreads);
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
    for (int q = 0; q < kBatchMaxQ; ++q)
      if (q < B.nq) flush_single(r_cnt[q], r_sum[q], B.acc[q]);
  } else {
    __syncthreads();
    for (int q = 0; q < B.nq; ++q)
      spill_bins32(reinterpret_cast<uint32_t*>(smem + B.bins_byte[q]), B.G[q], B.acc[q], tid, kDirectThreads);
  }
}

template <int NL, int NF, int MODE>
void launch_batch_t(laq_ctx* ctx, const BatchScan& B, size_t smem, int grid) {
  auto kern = scan_batch_kernel<NL, NF, MODE>;
  LAQ_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  const int64_t blocks_needed = (B.n + kDirectThreads * 4 - 1) / (kDirectThreads * 4);
  const int g = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(grid, blocks_needed)));
  kern<<<g, kDirectThreads, smem, ctx->stream>>>(B);
}

template <int NL, int NF>
void launch_batch_m(laq_ctx* ctx, const BatchScan& B, int mode, size_t smem, int grid) {
  if (mode == 0) launch_batch_t<NL, NF, 0>(ctx, B, smem, grid);
  else launch_batch_t<NL, NF, 1>(ctx, B, smem, grid);
}

template <int NL>
void launch_batch_f(laq_ctx* ctx, const BatchScan& B, int nf, int mode, size_t smem, int grid) {
  switch (nf) {
    case 0: launch_batch_m<NL, 0>(ctx, B, mode, smem, grid); break;
    case 1: launch_batch_m<NL, 1>(ctx, B, mode, smem, grid); break;
    case 2: launch_batch_m<NL, 2>(ctx, B, mode, smem, grid); break;
    default: fail(LAQ_ERR_UNSUPPORTED, "batched scan: at most 2 fact filter columns");
  }
}

void launch_batch(laq_ctx* ctx, const BatchScan& B, int nl, int nf, int mode, size_t smem, int grid) {
  switch (nl) {
    case 1: launch_batch_f<1>(ctx, B, nf, mode, smem, grid); break;
    case 2: launch_batch_f<2>(ctx, B, nf, mode, smem, grid); break;
    case 3: launch_batch_f<3>(ctx, B, nf, mode, smem, grid); break;
    case 4: launch_batch_f<4>(ctx, B, nf, mode, smem, grid); break;
    case 5: launch_batch_f<5>(ctx, B, nf, mode, smem, grid); break;
    case 6: launch_batch_f<6>(ctx, B, nf, mode, smem, grid); break;
    default: fail(LAQ_ERR_UNSUPPORTED, "batched scan: 1..6 links");
  }
  launched(ctx);
}

}  // namespace scan
}  // namespace laq
