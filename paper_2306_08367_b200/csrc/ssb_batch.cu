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
    if (n + 1 > L.dec_cap || n + 1 > lim) {
      atomicOr(d.overflow, 1);
    } else {
      L.dec[n] = L.miss;
      if (L.idw == 1) static_cast<uint8_t*>(L.ids)[L.size] = static_cast<uint8_t>(n);
      else static_cast<uint16_t*>(L.ids)[L.size] = static_cast<uint16_t>(n);
    }
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

template <int NQ>
void launch_batch_q(laq_ctx* ctx, const BatchScan& B, int nl, int nf, int mode, size_t smem, int grid);
extern template void launch_batch_q<2>(laq_ctx*, const BatchScan&, int, int, int, size_t, int);
extern template void launch_batch_q<3>(laq_ctx*, const BatchScan&, int, int, int, size_t, int);
extern template void launch_batch_q<4>(laq_ctx*, const BatchScan&, int, int, int, size_t, int);

void launch_batch(laq_ctx* ctx, const BatchScan& B, int nl, int nf, int mode, size_t smem, int grid) {
  switch (B.nq) {
    case 2: launch_batch_q<2>(ctx, B, nl, nf, mode, smem, grid); break;
    case 3: launch_batch_q<3>(ctx, B, nl, nf, mode, smem, grid); break;
    case 4: launch_batch_q<4>(ctx, B, nl, nf, mode, smem, grid); break;
    default: fail(LAQ_ERR_UNSUPPORTED, "batched scan: 2..4 queries");
  }
  launched(ctx);
}

}  // namespace scan
}  // namespace laq
