// K2+K3 fast path: fused join + predict over slot-ordered partials.
//
// For DIRECT probes the key -> slot map is arithmetic (slot = key - base), so
// instead of  slot -> dim row -> P_j[row]  (two dependent gathers into two
// tables) the partials are re-laid out once per call in slot order,
// Pslot_j[slot] = P_j[row(slot)], next to a 1-bit-per-slot existence bitmap.
// A fact row then costs, per dimension, one bitmap test (shared memory when
// the bitmaps fit) and one 8-byte gather that is only issued for rows still
// alive.  That halves the gather footprint (L1 hit rate) and the dependent
// latency chain of the generic star kernel.
//
// Survivor compaction: single-pass decoupled look-back over 4096-row tiles,
// the tile aggregate published before the predictions are computed, the
// walk resolved after; predictions staged in shared memory and written in
// coalesced runs (l == 1) or directly (l <= 8).
#pragma once

#include <cub/block/block_scan.cuh>

#include "probe.cuh"

namespace laq {
namespace slot {

constexpr int kMaxLinks = 8;
constexpr int kThreads = 256;
constexpr int kItems = 16;
constexpr int kTile = kThreads * kItems;  // 4096 rows
constexpr int kSmemBitmapWords = 4 * 1024;  // 16 KB of staged existence bitmaps

struct Args {
  int64_t n;
  int64_t l;
  const int32_t* fk[kMaxLinks];
  int64_t base[kMaxLinks];
  int64_t size[kMaxLinks];
  const uint32_t* bits[kMaxLinks];  // existence bitmap per link
  const double* pslot[kMaxLinks];   // slot-ordered partials (size x l)
  int smem_off[kMaxLinks];          // >= 0: bitmap staged in smem at this word offset
  int smem_words;
  double* y;
  int64_t* survivors;
  unsigned long long* tile_state;
  int* tile_counter;
  int64_t* nnz;
  int64_t n_tiles;
};

#define LAQ_SLOT_AGG (1ull << 62)
#define LAQ_SLOT_INC (2ull << 62)
#define LAQ_SLOT_VAL ((1ull << 62) - 1)

__device__ __forceinline__ unsigned long long resolve(unsigned long long* state, int64_t tile, unsigned long long total) {
  const int lane = threadIdx.x & 31;
  if (tile == 0) return 0;
  unsigned long long prefix = 0;
  int64_t p = tile - 1;
  while (true) {
    const int64_t idx = p - lane;
    unsigned long long s;
    do {
      s = idx >= 0 ? *reinterpret_cast<volatile unsigned long long*>(state + idx) : LAQ_SLOT_INC;
    } while (!__all_sync(0xffffffffu, (s & ~LAQ_SLOT_VAL) != 0));
    const unsigned inc = __ballot_sync(0xffffffffu, (s & ~LAQ_SLOT_VAL) == LAQ_SLOT_INC);
    const int stop = inc ? __ffs(inc) - 1 : 31;
    unsigned long long v = lane <= stop ? (s & LAQ_SLOT_VAL) : 0;
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    prefix += v;
    if (inc) break;
    p -= 32;
  }
  if (lane == 0) atomicExch(state + tile, LAQ_SLOT_INC | (prefix + total));
  return prefix;
}

template <int NL>
__global__ void __launch_bounds__(kThreads) predict_slot_kernel(const Args a) {
  using Scan = cub::BlockScan<int, kThreads>;
  extern __shared__ __align__(16) uint32_t s_bits[];
  __shared__ typename Scan::TempStorage scan_tmp;
  __shared__ int64_t s_tile;
  __shared__ unsigned long long s_prefix;
  __shared__ double s_y[kTile];

  for (int w = threadIdx.x; w < a.smem_words; w += kThreads) {
#pragma unroll
    for (int j = 0; j < NL; ++j)
      if (a.smem_off[j] >= 0 && w >= a.smem_off[j] && w < a.smem_off[j] + (a.size[j] + 31) / 32)
        s_bits[w] = __ldg(a.bits[j] + (w - a.smem_off[j]));
  }
  const bool stage_y = a.l == 1;

  while (true) {
    if (threadIdx.x == 0) s_tile = atomicAdd(a.tile_counter, 1);
    __syncthreads();
    const int64_t tile = s_tile;
    if (tile >= a.n_tiles) break;
    const int64_t row0 = tile * kTile + static_cast<int64_t>(threadIdx.x) * kItems;
    const int64_t left = a.n - row0;
    const int valid = left >= kItems ? kItems : (left > 0 ? static_cast<int>(left) : 0);

    uint32_t slot[NL][kItems];
    bool alive[kItems];
#pragma unroll
    for (int i = 0; i < kItems; ++i) alive[i] = i < valid;
#pragma unroll
    for (int j = 0; j < NL; ++j) {
      int32_t k[kItems];
      if (valid == kItems) {
#pragma unroll
        for (int q = 0; q < kItems / 4; ++q) {
          const int4 v = __ldcs(reinterpret_cast<const int4*>(a.fk[j] + row0) + q);
          k[4 * q] = v.x; k[4 * q + 1] = v.y; k[4 * q + 2] = v.z; k[4 * q + 3] = v.w;
        }
      } else {
#pragma unroll
        for (int i = 0; i < kItems; ++i) k[i] = i < valid ? a.fk[j][row0 + i] : 0;
      }
      const uint32_t base = static_cast<uint32_t>(a.base[j]), size = static_cast<uint32_t>(a.size[j]);
      const int off = a.smem_off[j];
#pragma unroll
      for (int i = 0; i < kItems; ++i) {
        const uint32_t s = static_cast<uint32_t>(k[i]) - base;
        bool ok = alive[i] && k[i] >= 0 && s < size;
        if (ok) {
          const uint32_t word = off >= 0 ? s_bits[off + (s >> 5)] : __ldg(a.bits[j] + (s >> 5));
          ok = (word >> (s & 31)) & 1u;
        }
        alive[i] = ok;
        slot[j][i] = s;
      }
    }

    int count = 0;
#pragma unroll
    for (int i = 0; i < kItems; ++i) count += alive[i] ? 1 : 0;
    int excl, total;
    Scan(scan_tmp).ExclusiveSum(count, excl, total);
    if (threadIdx.x == 0)
      atomicExch(a.tile_state + tile, (tile == 0 ? LAQ_SLOT_INC : LAQ_SLOT_AGG) | static_cast<unsigned long long>(total));

    if (stage_y) {
      int local = excl;
#pragma unroll
      for (int i = 0; i < kItems; ++i) {
        if (!alive[i]) continue;
        double acc = __dadd_rn(0.0, __ldg(a.pslot[0] + slot[0][i]));  // 0 + 1*x (spmm_dense)
#pragma unroll
        for (int j = 1; j < NL; ++j) acc = __dadd_rn(acc, __ldg(a.pslot[j] + slot[j][i]));  // fusion.cpp:73-76
        s_y[local++] = acc;
      }
    }
    if (threadIdx.x < 32) {
      const unsigned long long prefix = resolve(a.tile_state, tile, static_cast<unsigned long long>(total));
      if (threadIdx.x == 0) {
        s_prefix = prefix;
        if (tile == a.n_tiles - 1) *a.nnz = static_cast<int64_t>(prefix) + total;
      }
    }
    __syncthreads();
    const int64_t prefix = static_cast<int64_t>(s_prefix);
    if (stage_y) {
      for (int t = threadIdx.x; t < total; t += kThreads) __stcs(a.y + prefix + t, s_y[t]);
    }
    if (!stage_y || a.survivors) {
      int64_t pos = prefix + excl;
#pragma unroll
      for (int i = 0; i < kItems; ++i) {
        if (!alive[i]) continue;
        if (a.survivors) a.survivors[pos] = row0 + i;
        if (!stage_y) {
          for (int64_t c = 0; c < a.l; ++c) {
            double acc = __dadd_rn(0.0, __ldg(a.pslot[0] + static_cast<int64_t>(slot[0][i]) * a.l + c));
#pragma unroll
            for (int j = 1; j < NL; ++j)
              acc = __dadd_rn(acc, __ldg(a.pslot[j] + static_cast<int64_t>(slot[j][i]) * a.l + c));
            __stcs(a.y + pos * a.l + c, acc);
          }
        }
        ++pos;
      }
    }
    __syncthreads();
  }
}

// Build slot-ordered partials + existence bitmap for one link.
__global__ void scatter_slots_kernel(const int32_t* __restrict__ row_slot, int64_t rows, const double* __restrict__ P,
                                     int64_t l, double* __restrict__ pslot, uint32_t* __restrict__ bits) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = row_slot[r];
    for (int64_t c = 0; c < l; ++c) pslot[s * l + c] = P[r * l + c];
    atomicOr(bits + (s >> 5), 1u << (s & 31));
  }
}

}  // namespace slot
}  // namespace laq
