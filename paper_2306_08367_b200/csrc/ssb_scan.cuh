// K4 scan kernels: the fused filter -> star probe -> group-id -> exact int64
// (count, sum) aggregation over the fact table.  Included by the launch units.
//
// scan_pipe_kernel (primary, sm_100a), warp-specialised:
//   * one persistent CTA per SM: 1 producer warp + 16 consumer warps,
//     static round-robin over 2048-row tiles;
//   * the producer streams every touched int32 fact column of a tile into
//     shared memory with cp.async.bulk (the TMA bulk-copy engine, SASS
//     UBLKCP) completing on a per-stage "full" mbarrier, S stages ahead;
//     consumer warps release a stage through a per-stage "empty" mbarrier, so
//     no CTA-wide barrier sits in the steady-state loop;
//   * small per-link code tables (<= 48K slots, int16) are staged in shared
//     memory once per CTA; larger ones (e.g. part at SF>=10) are gathered
//     from L2 through the read-only path;
//   * links are probed in ascending pass-fraction order (chosen on the host),
//     so gathers into a big dimension only happen for rows that survived the
//     cheap, selective shared-memory ones;
//   * predicates are pre-lowered to closed int32 intervals (branch-free);
//   * per-group (count, sum) bins live in shared memory as 32-bit counters
//     (native ATOMS.ADD; 64-bit shared atomics are CAS loops on this part),
//     spilled into the global 64-bit accumulator before they could wrap.
// scan_stream_kernel (default): register double-buffered 16-byte loads of 4 rows
//   per thread.  Opt-in (LAQ_PACK=1): fact columns whose value range fits 8 or
//   16 bits are read byte-packed relative to their minimum (Q1.x: 6 bytes per
//   row instead of 16); slower as measured, see ssb.cu.
// scan_ldg_kernel (fallback): plain vectorised loads, any 4-byte alignment.
#pragma once

#include "probe.cuh"

namespace laq {
namespace scan {

constexpr int kMaxLinks = 8;
constexpr int kMaxFactFilters = 4;
constexpr int kMaxFactGroups = 4;
constexpr int kConsumerWarps = 16;
constexpr int kPipeThreads = 32 * (kConsumerWarps + 1);
constexpr int kTile = 4 * 32 * kConsumerWarps;  // 2048 rows
constexpr int kMaxStages = 8;

struct LinkProbe {
  int kind;
  int64_t base, size;
  const int64_t* keys;
  const int32_t* code;  // per slot, global
  int smem_off;         // >= 0: int16 code table staged in smem at this element offset
  // direct kernel: the table's format and where it is staged
  int fmt;              // kFmtGlobal / kFmtS16 / kFmtU8 / kFmtBit
  int smem_byte;        // byte offset of the staged table (fmt != kFmtGlobal)
  int smem_bytes;       // staged bytes (multiple of 16)
  const void* packed;   // the compact table in global memory (fmt != kFmtGlobal)
};

// Code-table formats of the direct kernel (a link's code is its contribution to
// the group id, -1 = the dim row fails the filters or the key has no row):
//   global int32 (gathered through L2), shared int16, shared uint8 (255 = -1;
//   the contribution fits 0..254), shared bitmap (the link filters only:
//   contribution 0, bit = passes).
enum : int { kFmtGlobal = 0, kFmtS16 = 1, kFmtU8 = 2, kFmtBit = 3 };

// A fact predicate lowered to  lo <= v <= hi  over int32 (or InSet).
struct FactFilter {
  const int32_t* col;
  int32_t lo, hi;
  int inset;
  const int64_t* set;
  int set_len;
};

struct FactGroup {
  const int32_t* col;
  int64_t mn, stride;
};

// A fact column as the stream kernel reads it: int32, or byte-packed (1 or 2
// bytes per row) relative to the column minimum `off` when the value range fits.
struct Col {
  const void* p;
  int w;         // bytes per row: 1, 2 or 4; 0 = bit-packed
  int32_t off;   // value = stored + off (w < 4)
  int bits = 0;  // w == 0: bits per row (1..32) of a little-endian bitstream
};

struct ScanArgs {
  int64_t n;
  const int32_t* fk[kMaxLinks];
  LinkProbe link[kMaxLinks];
  FactFilter ff[kMaxFactFilters];
  int n_fgroups;
  FactGroup fg[kMaxFactGroups];
  const int32_t* measure;  // nullptr: count only
  // stream kernel views of the same columns (packed where the range allows)
  Col fkc[kMaxLinks];
  Col ffc[kMaxFactFilters];
  Col mc;
  int64_t n_groups;
  unsigned long long* acc;  // [2*G]: count, sum
  // pipe kernel layout
  int stages;
  int smem_tab_elems;   // int16 elements of staged code tables
  int narrow_bins;      // 1: u32 (count, sum) bins, spilled every flush_every tiles
  int64_t flush_every;  // tiles per CTA after which u32 bins could overflow
  int prefetch;         // direct kernel: L2 prefetch distance in grid steps (0: off)
};

__device__ __forceinline__ bool pred_eval(int kind, int64_t v, int64_t lo, int64_t hi, const int64_t* set, int n) {
  switch (kind) {  // predicate.hpp:84-93
    case LAQ_PRED_LT: return v < lo;
    case LAQ_PRED_LE: return v <= lo;
    case LAQ_PRED_EQ: return v == lo;
    case LAQ_PRED_GE: return v >= lo;
    case LAQ_PRED_GT: return v > lo;
    case LAQ_PRED_BETWEEN: return v >= lo && v <= hi;
    default: {  // InSet: binary search over the sorted set (predicate.hpp:90)
      int a = 0, b = n;
      while (a < b) {
        const int m = (a + b) >> 1;
        const int64_t s = set[m];
        if (s == v) return true;
        if (s < v) a = m + 1; else b = m;
      }
      return false;
    }
  }
}

__device__ __forceinline__ bool filter_ok(const FactFilter& f, int32_t v) {
  if (f.inset) return pred_eval(LAQ_PRED_INSET, v, 0, 0, f.set, f.set_len);
  return v >= f.lo && v <= f.hi;
}

__device__ __forceinline__ int32_t hash_code(const LinkProbe& p, int32_t key) {
  const uint64_t mask = static_cast<uint64_t>(p.size) - 1;
  uint64_t h = static_cast<uint64_t>(static_cast<int64_t>(key)) * 0x9E3779B97F4A7C15ull;
  h ^= h >> 29;
  for (uint64_t s = h & mask;; s = (s + 1) & mask) {
    const int64_t k = __ldg(p.keys + s);
    if (k == key) return __ldg(p.code + s);
    if (k < 0) return -1;
  }
}

__device__ __forceinline__ int comp(const int4& v, int i) { return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w; }

// Probe one link for 4 rows; the 4 lookups are independent (issued together).
__device__ __forceinline__ void probe4(const LinkProbe& p, const int4& k, const int16_t* s_tab, bool (&alive)[4],
                                       int32_t (&gid)[4]) {
  int32_t c[4];
  if (p.kind == PROBE_HASH) {
#pragma unroll
    for (int i = 0; i < 4; ++i) c[i] = alive[i] ? hash_code(p, comp(k, i)) : -1;
  } else {
    const uint32_t base = static_cast<uint32_t>(p.base), size = static_cast<uint32_t>(p.size);
    uint32_t s[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) s[i] = static_cast<uint32_t>(comp(k, i)) - base;  // keys >= base >= 0
    if (p.smem_off >= 0) {
      const int16_t* t = s_tab + p.smem_off;
#pragma unroll
      for (int i = 0; i < 4; ++i) c[i] = (alive[i] && s[i] < size) ? static_cast<int32_t>(t[s[i]]) : -1;
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i) c[i] = (alive[i] && s[i] < size) ? __ldg(p.code + s[i]) : -1;
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    alive[i] = alive[i] && c[i] >= 0;
    gid[i] += c[i];
  }
}

// ---------------------------------------------------------------------------
// PTX helpers: mbarrier + bulk async copy (TMA engine, 1-D)
// ---------------------------------------------------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "LAQ_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra LAQ_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// Block-wide reduction of the single-group (count, sum) pair into acc[0..1].
__device__ __forceinline__ void flush_single(unsigned long long cnt, unsigned long long sum, unsigned long long* acc) {
  for (int o = 16; o; o >>= 1) {
    cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    sum += __shfl_xor_sync(0xffffffffu, sum, o);
  }
  if ((threadIdx.x & 31) == 0 && cnt) {
    atomicAdd(acc, cnt);
    atomicAdd(acc + 1, sum);
  }
}

// Shared 32-bit bins -> global accumulator (and reset).
__device__ __forceinline__ void spill_bins32(uint32_t* b32, int64_t G, unsigned long long* acc, int t, int nt) {
  for (int64_t g = t; g < G; g += nt) {
    const uint32_t c = b32[g];
    if (c) {
      atomicAdd(acc + 2 * g, static_cast<unsigned long long>(c));
      atomicAdd(acc + 2 * g + 1, static_cast<unsigned long long>(b32[G + g]));
      b32[g] = 0;
      b32[G + g] = 0;
    }
  }
}

// ---------------------------------------------------------------------------
// the warp-specialised, TMA-fed scan
// ---------------------------------------------------------------------------

template <int NL, int NF, int MODE>
__global__ void __launch_bounds__(kPipeThreads, 1) scan_pipe_kernel(const ScanArgs a) {
  constexpr int NCmax = NL + NF + 1;
  extern __shared__ __align__(128) unsigned char smem[];
  const int nc = NL + NF + (a.measure ? 1 : 0);
  const int S = a.stages;
  const int stage_bytes = nc * kTile * 4;
  unsigned char* stage_base = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * stage_bytes);
  uint64_t* empty = full + kMaxStages;
  int16_t* s_tab = reinterpret_cast<int16_t*>(empty + kMaxStages);
  unsigned char* bins_base = reinterpret_cast<unsigned char*>(s_tab) + ((a.smem_tab_elems * 2 + 15) & ~15);
  uint32_t* b32 = reinterpret_cast<uint32_t*>(bins_base);  // [G] counts, [G] sums
  unsigned long long* b64 = reinterpret_cast<unsigned long long*>(bins_base);

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int64_t n_tiles = (a.n + kTile - 1) / kTile;
  const int64_t my_tiles = n_tiles > blockIdx.x ? (n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // Stage code tables (int16) and zero the bins.
#pragma unroll
  for (int j = 0; j < NL; ++j) {
    const LinkProbe& p = a.link[j];
    if (p.smem_off >= 0)
      for (int64_t s = tid; s < p.size; s += kPipeThreads) s_tab[p.smem_off + s] = static_cast<int16_t>(__ldg(p.code + s));
  }
  if constexpr (MODE == 1) {
    const int64_t words = a.narrow_bins ? 2 * a.n_groups : 4 * a.n_groups;
    for (int64_t g = tid; g < words; g += kPipeThreads) b32[g] = 0;
  }
  __syncthreads();

  if (warp == kConsumerWarps) {
    // ===== producer warp: one elected lane streams the tiles =====
    if (lane == 0) {
      const int32_t* cols[NCmax];
#pragma unroll
      for (int j = 0; j < NL; ++j) cols[j] = a.fk[j];
#pragma unroll
      for (int f = 0; f < NF; ++f) cols[NL + f] = a.ff[f].col;
      cols[NL + NF] = a.measure;
      const uint64_t policy = evict_first_policy();
      int st = 0;
      uint32_t phase = 0;
      for (int64_t i = 0; i < my_tiles; ++i) {
        if (i >= S) {
          mbar_wait(empty + st, phase ^ 1);  // consumers released this stage
          // order the consumers' generic-proxy reads of the stage before the
          // async-proxy (TMA) writes that refill it
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
        const int64_t row0 = (blockIdx.x + i * gridDim.x) * kTile;
        const int64_t rows = min(static_cast<int64_t>(kTile), a.n - row0);
        const uint32_t bytes = static_cast<uint32_t>((rows * 4 + 15) & ~15ll);
        mbar_arrive_expect_tx(full + st, bytes * nc);
#pragma unroll
        for (int c = 0; c < NCmax; ++c)
          if (c < nc) bulk_g2s(stage_base + st * stage_bytes + c * kTile * 4, cols[c] + row0, bytes, full + st, policy);
        if (++st == S) {
          st = 0;
          phase ^= 1;
        }
      }
    }
  } else {
    // ===== consumer warps: 4 consecutive rows per thread per tile =====
    unsigned long long r_cnt = 0, r_sum = 0;
    int st = 0;
    uint32_t phase = 0;
    int64_t since_flush = 0;
    for (int64_t i = 0; i < my_tiles; ++i) {
      mbar_wait(full + st, phase);
      const int64_t row0 = (blockIdx.x + i * gridDim.x) * kTile + tid * 4;
      const unsigned char* sb = stage_base + st * stage_bytes + tid * 16;
      int4 kv[NL > 0 ? NL : 1], fv[NF > 0 ? NF : 1], mv;
#pragma unroll
      for (int j = 0; j < NL; ++j) kv[j] = *reinterpret_cast<const int4*>(sb + j * kTile * 4);
#pragma unroll
      for (int f = 0; f < NF; ++f) fv[f] = *reinterpret_cast<const int4*>(sb + (NL + f) * kTile * 4);
      if (a.measure) mv = *reinterpret_cast<const int4*>(sb + (NL + NF) * kTile * 4);

      const int64_t left = a.n - row0;  // rows of this thread's 4 that exist
      const int valid = left >= 4 ? 4 : (left > 0 ? static_cast<int>(left) : 0);
      bool alive[4];
      int32_t gid[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        alive[r] = r < valid;
        gid[r] = 0;
      }
      // Fact filters are closed int32 intervals here (InSet plans use the fallback kernel).
#pragma unroll
      for (int f = 0; f < NF; ++f) {
        const int32_t lo = a.ff[f].lo, hi = a.ff[f].hi;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int32_t v = comp(fv[f], r);
          alive[r] = alive[r] & (v >= lo) & (v <= hi);
        }
      }
#pragma unroll
      for (int j = 0; j < NL; ++j)
        if (alive[0] | alive[1] | alive[2] | alive[3]) probe4(a.link[j], kv[j], s_tab, alive, gid);
      for (int g = 0; g < a.n_fgroups; ++g)
#pragma unroll
        for (int r = 0; r < 4; ++r)
          if (alive[r])
            gid[r] += static_cast<int32_t>((static_cast<int64_t>(__ldg(a.fg[g].col + row0 + r)) - a.fg[g].mn) *
                                           a.fg[g].stride);
      if constexpr (MODE == 0) {
        // Branch-free: 4-row partials in 32 bits, one 64-bit add per tile.
        int32_t c4 = 0;
        long long s4 = 0;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          c4 += alive[r] ? 1 : 0;
          s4 += alive[r] ? (a.measure ? comp(mv, r) : 0) : 0;
        }
        r_cnt += static_cast<unsigned long long>(c4);
        r_sum += static_cast<unsigned long long>(static_cast<long long>(s4));
      } else {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          if (!alive[r]) continue;
          const int32_t v = a.measure ? comp(mv, r) : 0;
          if constexpr (MODE == 1) {
            if (a.narrow_bins) {
              atomicAdd(b32 + gid[r], 1u);
              if (a.measure) atomicAdd(b32 + a.n_groups + gid[r], static_cast<uint32_t>(v));
            } else {
              atomicAdd(b64 + gid[r], 1ull);
              if (a.measure)
                atomicAdd(b64 + a.n_groups + gid[r], static_cast<unsigned long long>(static_cast<long long>(v)));
            }
          } else {
            atomicAdd(a.acc + 2 * gid[r], 1ull);
            if (a.measure) atomicAdd(a.acc + 2 * gid[r] + 1, static_cast<unsigned long long>(static_cast<long long>(v)));
          }
        }
      }
      // Release the stage only after its data has been consumed (WAR vs the next bulk copy).
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + st);
      if (++st == S) {
        st = 0;
        phase ^= 1;
      }
      if constexpr (MODE == 1) {
        if (a.narrow_bins && ++since_flush == a.flush_every && i + 1 < my_tiles) {
          // All consumer warps flush together (named barrier 1, producer excluded).
          since_flush = 0;
          asm volatile("bar.sync 1, %0;" ::"n"(32 * kConsumerWarps));
          spill_bins32(b32, a.n_groups, a.acc, tid, 32 * kConsumerWarps);
          asm volatile("bar.sync 1, %0;" ::"n"(32 * kConsumerWarps));
        }
      }
    }
    if constexpr (MODE == 0) flush_single(r_cnt, r_sum, a.acc);
  }

  if constexpr (MODE == 1) {
    __syncthreads();
    if (a.narrow_bins) {
      spill_bins32(b32, a.n_groups, a.acc, tid, kPipeThreads);
    } else {
      for (int64_t g = tid; g < a.n_groups; g += kPipeThreads) {
        const unsigned long long c = b64[g];
        if (c) {
          atomicAdd(a.acc + 2 * g, c);
          atomicAdd(a.acc + 2 * g + 1, b64[a.n_groups + g]);
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// fallback: vectorised-load scan (any alignment), shared 64-bit bins
// ---------------------------------------------------------------------------

__device__ __forceinline__ int4 ld4(const int32_t* p, int64_t row0, int64_t n, bool vec) {
  if (vec && row0 + 4 <= n) return __ldcs(reinterpret_cast<const int4*>(p + row0));
  int4 v;
  v.x = row0 + 0 < n ? p[row0 + 0] : 0;
  v.y = row0 + 1 < n ? p[row0 + 1] : 0;
  v.z = row0 + 2 < n ? p[row0 + 2] : 0;
  v.w = row0 + 3 < n ? p[row0 + 3] : 0;
  return v;
}

template <int NL, int NF, int MODE>
__global__ void __launch_bounds__(256) scan_ldg_kernel(const ScanArgs a, const bool vec) {
  extern __shared__ unsigned long long s_bins[];  // MODE 1: [G] counts then [G] sums
  if constexpr (MODE == 1) {
    for (int64_t g = threadIdx.x; g < 2 * a.n_groups; g += blockDim.x) s_bins[g] = 0;
    __syncthreads();
  }
  unsigned long long r_cnt = 0, r_sum = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * 4;
  for (int64_t row0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * 4; row0 < a.n; row0 += stride) {
    int4 fk[NL > 0 ? NL : 1], fv[NF > 0 ? NF : 1], mv;
#pragma unroll
    for (int j = 0; j < NL; ++j) fk[j] = ld4(a.fk[j], row0, a.n, vec);
#pragma unroll
    for (int f = 0; f < NF; ++f) fv[f] = ld4(a.ff[f].col, row0, a.n, vec);
    if (a.measure) mv = ld4(a.measure, row0, a.n, vec);
    int32_t gid[4];
    bool alive[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      alive[i] = row0 + i < a.n;
      gid[i] = 0;
    }
#pragma unroll
    for (int f = 0; f < NF; ++f)
#pragma unroll
      for (int i = 0; i < 4; ++i) alive[i] = alive[i] && filter_ok(a.ff[f], comp(fv[f], i));
#pragma unroll
    for (int j = 0; j < NL; ++j) {
      LinkProbe p = a.link[j];
      p.smem_off = -1;
      probe4(p, fk[j], nullptr, alive, gid);
    }
    for (int g = 0; g < a.n_fgroups; ++g) {
      const int4 v = ld4(a.fg[g].col, row0, a.n, vec);
#pragma unroll
      for (int i = 0; i < 4; ++i)
        gid[i] += static_cast<int32_t>((static_cast<int64_t>(comp(v, i)) - a.fg[g].mn) * a.fg[g].stride);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (!alive[i]) continue;
      const unsigned long long val = a.measure ? static_cast<unsigned long long>(static_cast<long long>(comp(mv, i))) : 0ull;
      if constexpr (MODE == 0) {
        r_cnt += 1;
        r_sum += val;
      } else if constexpr (MODE == 1) {
        atomicAdd(s_bins + gid[i], 1ull);
        if (a.measure) atomicAdd(s_bins + a.n_groups + gid[i], val);
      } else {
        atomicAdd(a.acc + 2 * gid[i], 1ull);
        if (a.measure) atomicAdd(a.acc + 2 * gid[i] + 1, val);
      }
    }
  }
  if constexpr (MODE == 0) {
    flush_single(r_cnt, r_sum, a.acc);
  } else if constexpr (MODE == 1) {
    __syncthreads();
    for (int64_t g = threadIdx.x; g < a.n_groups; g += blockDim.x) {
      const unsigned long long c = s_bins[g];
      if (c) {
        atomicAdd(a.acc + 2 * g, c);
        atomicAdd(a.acc + 2 * g + 1, s_bins[a.n_groups + g]);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// stream: resident-table streaming scan (vectorised loads, register double
// buffering), shared-memory code tables + 32-bit bins like the pipe kernel,
// but with many more warps per SM to hide the L2 gathers of big dimensions.
// ---------------------------------------------------------------------------

constexpr int kStreamThreads = 256;

__device__ __forceinline__ int4 ld4_padded(const int32_t* p, int64_t row0, int64_t n) {
  // Columns on this path are 16-byte aligned with >= 16 readable bytes past the end.
  return row0 < n ? __ldcs(reinterpret_cast<const int4*>(p + row0)) : make_int4(0, 0, 0, 0);
}

// 4 consecutive rows of a (possibly packed) column; row0 is a multiple of 4 and
// every allocation on this path has >= 16 readable bytes past the end.  The raw
// words are kept as loaded (the register double buffer) and unpacked only when
// the rows are processed, an iteration later, so the load latency stays hidden.
__device__ __forceinline__ int4 ld4_raw(const Col& c, int64_t row0, int64_t n) {
  if (row0 >= n) return make_int4(0, 0, 0, 0);
  if (c.w == 1) {
    const uint32_t v = __ldcs(reinterpret_cast<const unsigned int*>(static_cast<const uint8_t*>(c.p) + row0));
    return make_int4(static_cast<int32_t>(v), 0, 0, 0);
  }
  if (c.w == 2) {
    const uint2 v = __ldcs(reinterpret_cast<const uint2*>(static_cast<const uint16_t*>(c.p) + row0));
    return make_int4(static_cast<int32_t>(v.x), static_cast<int32_t>(v.y), 0, 0);
  }
  return __ldcs(reinterpret_cast<const int4*>(static_cast<const int32_t*>(c.p) + row0));
}
__device__ __forceinline__ int4 unpack4(const int4& r, const Col& c) {
  if (c.w == 1) {
    const uint32_t v = static_cast<uint32_t>(r.x);
    return make_int4(static_cast<int32_t>(v & 0xffu) + c.off, static_cast<int32_t>((v >> 8) & 0xffu) + c.off,
                     static_cast<int32_t>((v >> 16) & 0xffu) + c.off, static_cast<int32_t>(v >> 24) + c.off);
  }
  if (c.w == 2) {
    const uint32_t x = static_cast<uint32_t>(r.x), y = static_cast<uint32_t>(r.y);
    return make_int4(static_cast<int32_t>(x & 0xffffu) + c.off, static_cast<int32_t>(x >> 16) + c.off,
                     static_cast<int32_t>(y & 0xffffu) + c.off, static_cast<int32_t>(y >> 16) + c.off);
  }
  return r;
}

// PK: some column is byte-packed (width dispatch per load); false: every column
// is int32 and the loads are plain 16-byte vectors (no per-load width branch).
template <int NL, int NF, int MODE, bool PK>
__device__ __forceinline__ int4 ld_batch(const Col& c, int64_t row0, int64_t n) {
  if constexpr (PK) return ld4_raw(c, row0, n);
  else return ld4_padded(static_cast<const int32_t*>(c.p), row0, n);
}
template <bool PK>
__device__ __forceinline__ int4 unpack_batch(const int4& r, const Col& c) {
  if constexpr (PK) return unpack4(r, c);
  else return r;
}

template <int NL, int NF, int MODE, bool PK>
__global__ void __launch_bounds__(kStreamThreads) scan_stream_kernel(const ScanArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  int16_t* s_tab = reinterpret_cast<int16_t*>(smem);
  uint32_t* b32 = reinterpret_cast<uint32_t*>(smem + ((a.smem_tab_elems * 2 + 15) & ~15));
  unsigned long long* b64 = reinterpret_cast<unsigned long long*>(b32);
  const int tid = threadIdx.x;

#pragma unroll
  for (int j = 0; j < NL; ++j) {
    const LinkProbe& p = a.link[j];
    if (p.smem_off >= 0)
      for (int64_t s = tid; s < p.size; s += kStreamThreads) s_tab[p.smem_off + s] = static_cast<int16_t>(__ldg(p.code + s));
  }
  if constexpr (MODE == 1) {
    const int64_t words = a.narrow_bins ? 2 * a.n_groups : 4 * a.n_groups;
    for (int64_t g = tid; g < words; g += kStreamThreads) b32[g] = 0;
  }
  __syncthreads();

  const int64_t step = static_cast<int64_t>(gridDim.x) * kStreamThreads * 4;
  const int64_t iters = (a.n + step - 1) / step;  // uniform across the block (barriers below)
  int64_t row0 = (static_cast<int64_t>(blockIdx.x) * kStreamThreads + tid) * 4;

  int4 kv[NL > 0 ? NL : 1], fv[NF > 0 ? NF : 1], mv = make_int4(0, 0, 0, 0);
#pragma unroll
  for (int j = 0; j < NL; ++j) kv[j] = ld_batch<NL, NF, MODE, PK>(a.fkc[j], row0, a.n);
#pragma unroll
  for (int f = 0; f < NF; ++f) fv[f] = ld_batch<NL, NF, MODE, PK>(a.ffc[f], row0, a.n);
  if (a.measure) mv = ld_batch<NL, NF, MODE, PK>(a.mc, row0, a.n);

  unsigned long long r_cnt = 0, r_sum = 0;
  for (int64_t it = 0; it < iters; ++it) {
    // Prefetch the next rows while this batch is probed (register double buffer).
    const int64_t nrow0 = row0 + step;
    int4 nkv[NL > 0 ? NL : 1], nfv[NF > 0 ? NF : 1], nmv = make_int4(0, 0, 0, 0);
#pragma unroll
    for (int j = 0; j < NL; ++j) nkv[j] = ld_batch<NL, NF, MODE, PK>(a.fkc[j], nrow0, a.n);
#pragma unroll
    for (int f = 0; f < NF; ++f) nfv[f] = ld_batch<NL, NF, MODE, PK>(a.ffc[f], nrow0, a.n);
    if (a.measure) nmv = ld_batch<NL, NF, MODE, PK>(a.mc, nrow0, a.n);

    const int64_t left = a.n - row0;
    const int valid = left >= 4 ? 4 : (left > 0 ? static_cast<int>(left) : 0);
    bool alive[4];
    int32_t gid[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      alive[r] = r < valid;
      gid[r] = 0;
    }
#pragma unroll
    for (int f = 0; f < NF; ++f) {
      const int32_t lo = a.ff[f].lo, hi = a.ff[f].hi;
      const int4 fu = unpack_batch<PK>(fv[f], a.ffc[f]);
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int32_t v = comp(fu, r);
        alive[r] = alive[r] & (v >= lo) & (v <= hi);
      }
    }
#pragma unroll
    for (int j = 0; j < NL; ++j)
      if (alive[0] | alive[1] | alive[2] | alive[3]) probe4(a.link[j], unpack_batch<PK>(kv[j], a.fkc[j]), s_tab, alive, gid);
    const int4 mu = unpack_batch<PK>(mv, a.mc);
    for (int g = 0; g < a.n_fgroups; ++g)
#pragma unroll
      for (int r = 0; r < 4; ++r)
        if (alive[r])
          gid[r] += static_cast<int32_t>((static_cast<int64_t>(__ldg(a.fg[g].col + row0 + r)) - a.fg[g].mn) *
                                         a.fg[g].stride);
    if constexpr (MODE == 0) {
      int32_t c4 = 0;
      long long s4 = 0;
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        c4 += alive[r] ? 1 : 0;
        s4 += alive[r] ? comp(mu, r) : 0;
      }
      r_cnt += static_cast<unsigned long long>(c4);
      r_sum += static_cast<unsigned long long>(s4);
    } else {
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        if (!alive[r]) continue;
        const int32_t v = comp(mu, r);
        if constexpr (MODE == 1) {
          if (a.narrow_bins) {
            atomicAdd(b32 + gid[r], 1u);
            if (a.measure) atomicAdd(b32 + a.n_groups + gid[r], static_cast<uint32_t>(v));
          } else {
            atomicAdd(b64 + gid[r], 1ull);
            if (a.measure) atomicAdd(b64 + a.n_groups + gid[r], static_cast<unsigned long long>(static_cast<long long>(v)));
          }
        } else {
          atomicAdd(a.acc + 2 * gid[r], 1ull);
          if (a.measure) atomicAdd(a.acc + 2 * gid[r] + 1, static_cast<unsigned long long>(static_cast<long long>(v)));
        }
      }
      if constexpr (MODE == 1) {
        if (a.narrow_bins && (it + 1) % a.flush_every == 0 && it + 1 < iters) {
          __syncthreads();
          spill_bins32(b32, a.n_groups, a.acc, tid, kStreamThreads);
          __syncthreads();
        }
      }
    }
#pragma unroll
    for (int j = 0; j < NL; ++j) kv[j] = nkv[j];
#pragma unroll
    for (int f = 0; f < NF; ++f) fv[f] = nfv[f];
    mv = nmv;
    row0 = nrow0;
  }

  if constexpr (MODE == 0) {
    flush_single(r_cnt, r_sum, a.acc);
  } else if constexpr (MODE == 1) {
    __syncthreads();
    if (a.narrow_bins) {
      spill_bins32(b32, a.n_groups, a.acc, tid, kStreamThreads);
    } else {
      for (int64_t g = tid; g < a.n_groups; g += kStreamThreads) {
        const unsigned long long c = b64[g];
        if (c) {
          atomicAdd(a.acc + 2 * g, c);
          atomicAdd(a.acc + 2 * g + 1, b64[a.n_groups + g]);
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// direct: the stream kernel's data flow with the per-row instruction count cut
// to what the query needs, for plans whose links are all DIRECT probe tables
// and whose group id comes from the links only (every SSB query).  Measured on
// Q2.1 (ncu source page) the stream kernel issued ~410 warp instructions per
// 128 rows: per-row generic->shared address construction (S2R SR_CgaCtaId),
// 64-bit row bounds, a 64-bit modulo per iteration for the bin-spill test and
// the runtime probe-kind dispatch.  Here: shared code tables and bins are
// addressed with 32-bit shared-window addresses computed once, full grid
// steps run without row bounds (one bounded tail step), the spill test is a
// countdown, and each probe is  slot = key - base; slot < size ? table[slot]
// : -1  with the table format a warp-uniform branch per link.
//
// One 1024-thread CTA per SM (the register file holds 1024 threads at <= 64
// registers anyway), so the SM's whole shared memory holds ONE copy of the
// code tables, in the most compact format each link allows (int16, uint8,
// or a pass bitmap for filter-only links): at SF=100 the 200K-slot supplier
// table (Q3.x: uint8, 200 KB) and the 1.4M-slot part table (Q4.x: bitmap,
// 175 KB) come out of L2 gathers into shared memory.
// ---------------------------------------------------------------------------

constexpr int kDirectThreads = 1024;

__device__ __forceinline__ int32_t lds_s16(uint32_t addr) {
  int16_t v;
  asm volatile("ld.shared.s16 %0, [%1];" : "=h"(v) : "r"(addr));
  return static_cast<int32_t>(v);
}
__device__ __forceinline__ uint32_t lds_u8(uint32_t addr) {
  uint16_t v;
  asm volatile("ld.shared.u8 %0, [%1];" : "=h"(v) : "r"(addr));
  return static_cast<uint32_t>(v);
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ void reds_add(uint32_t addr, uint32_t v) {
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

// One 128-byte line per 8 lanes (8 lanes x 4 rows x 4 B) of a column.
template <int PKM>
__device__ __forceinline__ void prefetch_l2(const Col& c, int64_t row0) {
  if constexpr (PKM == 2) return;  // bit-packed (transfer format): no prefetch
  const uint8_t* p = static_cast<const uint8_t*>(c.p) + (PKM == 1 ? row0 * c.w : row0 * 4);
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// Direct-kernel column access by packing mode PKM: 0 int32, 1 byte-packed
// (widths 1/2/4), 2 bit-packed.  Modes 0/1: a lane owns 4 consecutive rows
// row0..row0+3.  Mode 2: the warp's 128 rows are 4 groups of 32 and a lane owns
// row (group r, lane) -- the raw registers hold the lane's word of each group
// (a group of 32 rows x b bits is b consecutive 32-bit words), unpacked with
// two shuffles and a funnel shift.  Row order inside a step is irrelevant to
// the aggregation, so the mapping only has to be consistent across columns.
template <int PKM>
__device__ __forceinline__ int64_t drow(int64_t row0, int r) {
  if constexpr (PKM == 2) {
    const int lane = threadIdx.x & 31;
    return row0 - 3 * lane + 32 * r;  // warp base (row0 - 4 lane) + 32 r + lane
  } else {
    return row0 + r;
  }
}
template <int PKM>
__device__ __forceinline__ int4 dld(const Col& c, int64_t row0, int64_t n) {
  if constexpr (PKM == 0) {
    return ld4_padded(static_cast<const int32_t*>(c.p), row0, n);
  } else if constexpr (PKM == 1) {
    return ld4_raw(c, row0, n);
  } else {
    const int lane = threadIdx.x & 31;
    const int64_t wbase = row0 - 4 * lane;
    if (wbase >= n || lane >= c.bits) return make_int4(0, 0, 0, 0);
    const uint32_t* w = static_cast<const uint32_t*>(c.p) + (wbase >> 5) * c.bits + lane;
    const int b = c.bits;
    return make_int4(static_cast<int32_t>(__ldcs(w)), static_cast<int32_t>(__ldcs(w + b)),
                     static_cast<int32_t>(__ldcs(w + 2 * b)), static_cast<int32_t>(__ldcs(w + 3 * b)));
  }
}
__device__ __forceinline__ int32_t bit_extract(uint32_t word, int bits, int off) {
  const int lane = threadIdx.x & 31;
  const int bit = lane * bits;
  const int wi = bit >> 5, sh = bit & 31;
  const uint32_t lo = __shfl_sync(0xffffffffu, word, wi);
  const uint32_t hi = __shfl_sync(0xffffffffu, word, (wi + 1) & 31);
  const uint32_t v = __funnelshift_r(lo, hi, sh);
  const uint32_t mask = bits >= 32 ? 0xffffffffu : ((1u << bits) - 1u);
  return static_cast<int32_t>(v & mask) + off;
}
template <int PKM>
__device__ __forceinline__ int4 dunpack(const int4& r, const Col& c) {
  if constexpr (PKM == 0) {
    return r;
  } else if constexpr (PKM == 1) {
    return unpack4(r, c);
  } else {
    return make_int4(bit_extract(static_cast<uint32_t>(r.x), c.bits, c.off),
                     bit_extract(static_cast<uint32_t>(r.y), c.bits, c.off),
                     bit_extract(static_cast<uint32_t>(r.z), c.bits, c.off),
                     bit_extract(static_cast<uint32_t>(r.w), c.bits, c.off));
  }
}

template <int NL, int NF, int MODE, int PKM, bool TAIL>
__device__ __forceinline__ void direct_rows(const ScanArgs& a, int64_t row0, const int4 (&kv)[NL > 0 ? NL : 1],
                                            const int4 (&fv)[NF > 0 ? NF : 1], const int4& mv,
                                            const uint32_t (&tab_addr)[NL > 0 ? NL : 1], uint32_t bins,
                                            unsigned long long& r_cnt, unsigned long long& r_sum) {
  bool alive[4];
  int32_t gid[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    alive[r] = TAIL ? drow<PKM>(row0, r) < a.n : true;
    gid[r] = 0;
  }
#pragma unroll
  for (int f = 0; f < NF; ++f) {
    const int32_t lo = a.ff[f].lo, hi = a.ff[f].hi;
    const int4 fu = dunpack<PKM>(fv[f], a.ffc[f]);
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int32_t v = comp(fu, r);
      alive[r] = alive[r] & (v >= lo) & (v <= hi);
    }
  }
#pragma unroll
  for (int j = 0; j < NL; ++j) {
    const uint32_t base = static_cast<uint32_t>(a.link[j].base), size = static_cast<uint32_t>(a.link[j].size);
    const int4 k = dunpack<PKM>(kv[j], a.fkc[j]);
    const int fmt = a.link[j].fmt;
    int32_t c[4];
    uint32_t s[4];
    bool ok[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      s[r] = static_cast<uint32_t>(comp(k, r)) - base;
      ok[r] = alive[r] && s[r] < size;
      c[r] = -1;
    }
    if (fmt == kFmtS16) {
#pragma unroll
      for (int r = 0; r < 4; ++r)
        if (ok[r]) c[r] = lds_s16(tab_addr[j] + 2 * s[r]);
    } else if (fmt == kFmtU8) {
#pragma unroll
      for (int r = 0; r < 4; ++r)
        if (ok[r]) {
          const uint32_t v = lds_u8(tab_addr[j] + s[r]);
          c[r] = v == 255u ? -1 : static_cast<int32_t>(v);
        }
    } else if (fmt == kFmtBit) {
#pragma unroll
      for (int r = 0; r < 4; ++r)
        if (ok[r]) c[r] = ((lds_u32(tab_addr[j] + 4 * (s[r] >> 5)) >> (s[r] & 31)) & 1u) ? 0 : -1;
    } else {
      const int32_t* code = a.link[j].code;
#pragma unroll
      for (int r = 0; r < 4; ++r)
        if (ok[r]) c[r] = __ldg(code + s[r]);
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      alive[r] = alive[r] & (c[r] >= 0);
      gid[r] += c[r];
    }
  }
  const int4 mu = dunpack<PKM>(mv, a.mc);
  if constexpr (MODE == 0) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      r_cnt += alive[r] ? 1u : 0u;
      r_sum += alive[r] ? static_cast<unsigned long long>(static_cast<long long>(comp(mu, r))) : 0ull;
    }
  } else {
    const uint32_t sum_off = static_cast<uint32_t>(a.n_groups) * 4u;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      if (alive[r]) {
        const uint32_t ad = bins + 4u * static_cast<uint32_t>(gid[r]);
        reds_add(ad, 1u);
        if (a.measure) reds_add(ad + sum_off, static_cast<uint32_t>(comp(mu, r)));
      }
    }
  }
}

// MODE 0 (one group: register accumulation) or MODE 1 with narrow (u32) bins.
// Shared memory: [staged code tables (a.smem_tab_elems bytes)] [u32 bins 2G].
template <int NL, int NF, int MODE, int PKM>
__global__ void __launch_bounds__(kDirectThreads, 1) scan_direct_kernel(const ScanArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint32_t* b32 = reinterpret_cast<uint32_t*>(smem + a.smem_tab_elems);
  const int tid = threadIdx.x;
#pragma unroll
  for (int j = 0; j < NL; ++j) {
    const LinkProbe& p = a.link[j];
    if (p.fmt != kFmtGlobal) {
      const uint4* src = static_cast<const uint4*>(p.packed);
      uint4* dst = reinterpret_cast<uint4*>(smem + p.smem_byte);
      for (int w = tid; w < p.smem_bytes / 16; w += kDirectThreads) dst[w] = __ldg(src + w);
    }
  }
  if constexpr (MODE == 1)
    for (int64_t g = tid; g < 2 * a.n_groups; g += kDirectThreads) b32[g] = 0;
  __syncthreads();

  const uint32_t s_base = smem_u32(smem);
  const uint32_t bins = smem_u32(b32);
  uint32_t tab_addr[NL > 0 ? NL : 1];
#pragma unroll
  for (int j = 0; j < NL; ++j) tab_addr[j] = s_base + static_cast<uint32_t>(a.link[j].smem_byte);

  const int64_t step = static_cast<int64_t>(gridDim.x) * kDirectThreads * 4;
  const int64_t iters = (a.n + step - 1) / step;  // uniform across the block
  const int64_t full = a.n / step;                // steps with every row in range
  int64_t row0 = (static_cast<int64_t>(blockIdx.x) * kDirectThreads + tid) * 4;
  const bool pf_lane = PKM != 2 && a.prefetch && (tid & 7) == 0;
  const int64_t pf_rows = static_cast<int64_t>(a.prefetch) * step;

  // Two register buffers used in turn (the loop is unrolled by two so the
  // double buffer needs no register moves).
  int4 kvA[NL > 0 ? NL : 1], fvA[NF > 0 ? NF : 1], mvA = make_int4(0, 0, 0, 0);
  int4 kvB[NL > 0 ? NL : 1], fvB[NF > 0 ? NF : 1], mvB = make_int4(0, 0, 0, 0);
  auto load = [&](int4 (&kv)[NL > 0 ? NL : 1], int4 (&fv)[NF > 0 ? NF : 1], int4& mv, int64_t r) {
#pragma unroll
    for (int j = 0; j < NL; ++j) kv[j] = dld<PKM>(a.fkc[j], r, a.n);
#pragma unroll
    for (int f = 0; f < NF; ++f) fv[f] = dld<PKM>(a.ffc[f], r, a.n);
    if (a.measure) mv = dld<PKM>(a.mc, r, a.n);
  };
  load(kvA, fvA, mvA, row0);

  unsigned long long r_cnt = 0, r_sum = 0;
  int64_t until_flush = a.narrow_bins ? a.flush_every : INT64_MAX;
  // One grid step: prefetch the next rows into the other buffer, process these.
  auto one = [&](int64_t it, const int4 (&kv)[NL > 0 ? NL : 1], const int4 (&fv)[NF > 0 ? NF : 1], const int4& mv,
                 int4 (&nkv)[NL > 0 ? NL : 1], int4 (&nfv)[NF > 0 ? NF : 1], int4& nmv) {
    load(nkv, nfv, nmv, row0 + step);
    if (pf_lane && row0 + pf_rows < a.n) {  // the rows `prefetch` steps ahead into L2 (no registers held)
#pragma unroll
      for (int j = 0; j < NL; ++j) prefetch_l2<PKM>(a.fkc[j], row0 + pf_rows);
#pragma unroll
      for (int f = 0; f < NF; ++f) prefetch_l2<PKM>(a.ffc[f], row0 + pf_rows);
      if (a.measure) prefetch_l2<PKM>(a.mc, row0 + pf_rows);
    }
    if (it < full) direct_rows<NL, NF, MODE, PKM, false>(a, row0, kv, fv, mv, tab_addr, bins, r_cnt, r_sum);
    else direct_rows<NL, NF, MODE, PKM, true>(a, row0, kv, fv, mv, tab_addr, bins, r_cnt, r_sum);
    if constexpr (MODE == 1) {
      if (--until_flush == 0) {
        until_flush = a.flush_every;
        if (it + 1 < iters) {
          __syncthreads();
          spill_bins32(b32, a.n_groups, a.acc, tid, kDirectThreads);
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
    flush_single(r_cnt, r_sum, a.acc);
  } else {
    __syncthreads();
    spill_bins32(b32, a.n_groups, a.acc, tid, kDirectThreads);
  }
}

}  // namespace scan
}  // namespace laq
