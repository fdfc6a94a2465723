// K5/K7: tensor-core contractions for the wide shapes of the paper's complexity
// analysis (BASELINE configs[4], SURVEY.md §8a rows 12-15, §8d "GEMM"):
//
//   prefuse   P_j = B_j (M_j L)          fusion.cpp:31-36, 50-62  (A = dim rows, dense)
//   non-fused Y   = materialize(I_j,B_j) L   laqops.cpp:338-374 + mlops.cpp:248-250
//                                             (A = gathered join rows, T never written)
//   apply     Y   = sum_j P_j[i_j]       fusion.cpp:64-77 (fp32 partials, memory-bound)
//
// C[m x n] (fp32) = A[m x K] . W[K x n]: A rows are 32-feature blocks of the dims'
// split tables (tc.cuh layout, one 128-byte line per row and block), gathered by
// row maps (or the identity), W in the same split block layout (W^T rows = output
// columns).  Scaled fp16x2 split (tc.cuh), hi.hi + hi.lo + lo.hi with fp32
// accumulation in TMEM, unscaled exactly in the epilogue;
// accuracy is checked condition-aware at 1e-5.
//
// Persistent kernel, one CTA per SM, output tiles 128 x BN (BN <= 256).  Tile order:
// row-tile-major when the split W fits L2 (each A tile is fetched from HBM once and
// re-read from L2 by the CTAs computing its other column tiles), else column-major
// (a W panel is reused from L2 by consecutive CTAs):
//   warps 0-7   epilogue: tcgen05.ld (thread = row, 32 columns per load), unscale,
//               transpose through a swizzled 4 KB shared tile so every store
//               instruction writes four full 128-byte row segments of C;
//   warps 8-11  producers: per stage (one 32-feature K block) the 128 A lines
//               (gathered rows: cp.async, cp.async.mbarrier.arrive.noinc) and the
//               BN W lines (dense: ONE TMA tile load, 128B-swizzled by the tensor
//               map, issued by one thread with expect_tx on the same barrier);
//   warp 12     TMEM owner + MMA issuer: 3 x (1..2) tcgen05.mma per stage into
//               one of two TMEM accumulators.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <string>
#include <utility>
#include <vector>

#include "common.cuh"
#include "tc.cuh"

namespace laq {
namespace gemm {

constexpr int kRows = 128;
constexpr int kEpiWarps = 8;
constexpr int kProdWarps = 4, kProdWarp0 = 8, kMmaWarp = 12;
constexpr int kThreads = 13 * 32;
constexpr int kMaxDims = 8;
constexpr int kMaxBlocks = 64;  // K <= 2048
constexpr uint32_t kABytes = kRows * 128u;

struct Args {
  CUtensorMap wmap;                   // W as a 2-D fp16 tensor [n_blocks * n_pad rows][64], box {64, BN}, 128B swizzle
  CUtensorMap amap[kMaxBlocks];       // identity rows: A block b as [rows][64], box {64, 128}
  int w_tma;                          // 1: W tiles by TMA (wmap), 0: by cp.async
  int a_tma;                          // 1: A tiles by TMA too (identity rows, prefuse); one producer thread
  const tc::elem* block[kMaxBlocks];  // A block b: [rows_j x 64]
  int block_dim[kMaxBlocks];
  int block_steps[kMaxBlocks];
  int n_blocks;
  int n_dims;
  const int32_t* idx[kMaxDims];  // row maps (nullptr = identity)
  int64_t m;                     // output rows
  int64_t n;                     // output columns
  int BN;                        // tile columns (multiple of 16, <= 256)
  const tc::elem* w;        // [n_blocks][n_pad][64]
  int64_t n_pad;                 // W rows per block (n rounded up to BN)
  float* c;                      // [m x n]
  float unscale;                 // 1 / (s_A s_W), a power of two
  int stages;
  int64_t m_tiles, n_tiles;
  int m_major;  // tile order: 1 = all column tiles of a row tile together (W resident in L2)
};

__host__ __device__ inline uint32_t stage_bytes(int BN) { return kABytes + static_cast<uint32_t>(BN) * 128u; }
constexpr uint32_t kBarBytes = 256;  // mbarriers + TMEM slot (after the stages)
// stages | barriers | 8 x 4 KB epilogue staging tiles | 1 KB alignment slack
__host__ __device__ inline uint32_t smem_bytes(int BN, int S) {
  return S * stage_bytes(BN) + kBarBytes + kEpiWarps * 4096u + 1024;
}

__global__ void __launch_bounds__(kThreads, 1) gemm_kernel(const __grid_constant__ Args a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int S = a.stages, BN = a.BN, NB = a.n_blocks;
  const uint32_t SB = stage_bytes(BN);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * SB);
  uint64_t* empty = full + S;
  uint64_t* acc_full = empty + S;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  const uint32_t sbase = tc::smem_u32(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n_tiles_total = a.m_tiles * a.n_tiles;

  if (warp == kMmaWarp) {
    if (lane == 0) {
      for (int s = 0; s < S; ++s) {
        // cp.async arrivals of the producer warps + the TMA issuer's expect_tx arrive
        tc::mbar_init(&full[s], a.a_tma ? 1 : kProdWarps * 32 + a.w_tma);
        tc::mbar_init(&empty[s], 1);
      }
      for (int b = 0; b < 2; ++b) {
        tc::mbar_init(&acc_full[b], 1);
        tc::mbar_init(&acc_empty[b], kEpiWarps);
      }
      tc::fence_mbar_init();
    }
    __syncwarp();
    tc::tmem_alloc<512>(tmem_slot);
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp >= kProdWarp0 && warp < kProdWarp0 + kProdWarps && a.a_tma) {
    // ================= TMA producer (identity rows: A and W tiles dense) =================
    if (warp == kProdWarp0 && lane == 0) {
      int it = 0;
      for (int64_t t = blockIdx.x; t < n_tiles_total; t += gridDim.x) {
        const int64_t nt = a.m_major ? t % a.n_tiles : t / a.m_tiles, mt = a.m_major ? t / a.n_tiles : t % a.m_tiles;
        for (int b = 0; b < NB; ++b, ++it) {
          const int s = it % S;
          tc::mbar_wait(&empty[s], ((it / S) & 1) ^ 1);
          const uint32_t st = sbase + s * SB;
          tc::mbar_arrive_expect_tx(&full[s], kABytes + static_cast<uint32_t>(BN) * 128u);
          tc::tma_load_2d(&a.amap[b], &full[s], st, 0, static_cast<int32_t>(mt * kRows));  // rows past m: zero fill
          tc::tma_load_2d(&a.wmap, &full[s], st + kABytes, 0, static_cast<int32_t>(b * a.n_pad + nt * BN));
        }
      }
    }
  } else if (warp >= kProdWarp0 && warp < kProdWarp0 + kProdWarps) {
    // ================= cp.async producers =================
    const int pw = warp - kProdWarp0;
    __shared__ int32_t s_rows[kProdWarps][kMaxDims][32];
    const int sub = lane >> 3, chunk = lane & 7;
    int it = 0;  // global stage counter
    for (int64_t t = blockIdx.x; t < n_tiles_total; t += gridDim.x) {
      const int64_t nt = a.m_major ? t % a.n_tiles : t / a.m_tiles, mt = a.m_major ? t / a.n_tiles : t % a.m_tiles;
      // this warp's 32 A rows: resolve every dim's source row
      {
        int64_t g = mt * kRows + 32 * pw + lane;
        if (g >= a.m) g = a.m - 1;
        for (int j = 0; j < a.n_dims; ++j) s_rows[pw][j][lane] = a.idx[j] ? __ldg(a.idx[j] + g) : static_cast<int32_t>(g);
      }
      __syncwarp();
      for (int b = 0; b < NB; ++b, ++it) {
        const int s = it % S;
        tc::mbar_wait(&empty[s], ((it / S) & 1) ^ 1);
        const uint32_t st = sbase + s * SB;
        // A: 32 rows x 128 B of block b
        const tc::elem* ab = a.block[b] + chunk * 8;
        const int j = a.block_dim[b];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int r = 32 * pw + 4 * q + sub;
          tc::cp_async16(st + tc::sw128_off(r, chunk), ab + static_cast<int64_t>(s_rows[pw][j][4 * q + sub]) * 64);
        }
        // W: BN rows of block b (contiguous in global)
        if (a.w_tma) {
          if (pw == 0 && lane == 0) {
            tc::mbar_arrive_expect_tx(&full[s], static_cast<uint32_t>(BN) * 128u);
            tc::tma_load_2d(&a.wmap, &full[s], st + kABytes, 0, static_cast<int32_t>(b * a.n_pad + nt * BN));
          }
        } else {
          const tc::elem* wb = a.w + (static_cast<int64_t>(b) * a.n_pad + nt * BN) * 64 + chunk * 8;
          for (int r = pw * 4 + sub; r < BN; r += 16)
            tc::cp_async16(st + kABytes + tc::sw128_off(r, chunk), wb + static_cast<int64_t>(r) * 64);
        }
        tc::cp_async_arrive_noinc(&full[s]);
      }
      __syncwarp();  // s_rows reuse
    }
  } else if (warp == kMmaWarp) {
    // ================= MMA issuer =================
    if (lane == 0) {
      const uint32_t idesc = tc::idesc_f16_f32(kRows, BN);
      int it = 0, tl = 0;
      for (int64_t t = blockIdx.x; t < n_tiles_total; t += gridDim.x, ++tl) {
        const int ab = tl & 1;
        tc::mbar_wait(&acc_empty[ab], ((tl >> 1) & 1) ^ 1);
        tc::tc_fence_after();
        const uint32_t d = tmem + ab * 256;
        uint32_t acc = 0;
        for (int b = 0; b < NB; ++b, ++it) {
          const int s = it % S;
          tc::mbar_wait(&full[s], (it / S) & 1);
          tc::fence_proxy_async();
          tc::tc_fence_after();
          const uint32_t st = sbase + s * SB;
#pragma unroll
          for (int pr = 0; pr < 3; ++pr) {  // hi.hi, hi.lo, lo.hi
            const uint32_t pa = pr == 2 ? 64u : 0u, pb = pr == 1 ? 64u : 0u;
            for (int k = 0; k < a.block_steps[b]; ++k) {
              tc::mma_f16(d, tc::sdesc_sw128(st + pa + k * 32u), tc::sdesc_sw128(st + kABytes + pb + k * 32u), idesc,
                           acc);
              acc = 1;
            }
          }
          tc::mma_commit(&empty[s]);
        }
        tc::mma_commit(&acc_full[ab]);
      }
    }
    __syncwarp();
  } else {
    // ================= epilogue (warps 0-7) =================
    const int q = warp & 3, hh = warp >> 2;  // TMEM lane group, column half
    int tl = 0;
    for (int64_t t = blockIdx.x; t < n_tiles_total; t += gridDim.x, ++tl) {
      const int64_t nt = a.m_major ? t % a.n_tiles : t / a.m_tiles, mt = a.m_major ? t / a.n_tiles : t % a.m_tiles;
      const int ab = tl & 1;
      tc::mbar_wait(&acc_full[ab], (tl >> 1) & 1);
      tc::tc_fence_after();
      const int64_t row0 = mt * kRows + 32 * q;
      const uint32_t t0 = tmem + (static_cast<uint32_t>(32 * q) << 16) + ab * 256;
      const uint32_t stg = sbase + S * SB + kBarBytes + warp * 4096u;  // this warp's 32 x 32 fp32 staging tile
      for (int c0 = 32 * hh; c0 < BN; c0 += 64) {
        uint32_t v[32];
        tc::tmem_ld32(t0 + c0, v);
        tc::tmem_ld_wait();
        // thread = row -> staging (16-byte chunk c4 of row r at c4 ^ (r & 7): conflict-free)
#pragma unroll
        for (int c4 = 0; c4 < 8; ++c4)
          tc::sts128(stg + lane * 128u + ((c4 ^ (lane & 7)) << 4),
                     make_float4(__uint_as_float(v[4 * c4]) * a.unscale, __uint_as_float(v[4 * c4 + 1]) * a.unscale,
                                 __uint_as_float(v[4 * c4 + 2]) * a.unscale, __uint_as_float(v[4 * c4 + 3]) * a.unscale));
        __syncwarp();
        // staging -> C: each group of 8 lanes writes one full 128-byte row segment
        const int64_t col = nt * BN + c0 + 4 * (lane & 7);
#pragma unroll
        for (int qq = 0; qq < 8; ++qq) {
          const int r = 4 * qq + (lane >> 3);
          const float4 x = tc::lds128(stg + r * 128u + (((lane & 7) ^ (r & 7)) << 4));
          const int64_t grow = row0 + r;
          if (grow >= a.m) continue;
          float* dst = a.c + grow * a.n + col;
          if (col + 4 <= a.n && (a.n & 3) == 0) {
            __stcs(reinterpret_cast<float4*>(dst), x);
          } else {
            if (col < a.n) __stcs(dst, x.x);
            if (col + 1 < a.n) __stcs(dst + 1, x.y);
            if (col + 2 < a.n) __stcs(dst + 2, x.z);
            if (col + 3 < a.n) __stcs(dst + 3, x.w);
          }
        }
        __syncwarp();
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&acc_empty[ab]);
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc::tc_fence_after();
    tc::tmem_dealloc<512>(tmem);
  }
}

// Y[m] = sum_j P_j[i_j[m]] in fp32, association ((P_0 + P_1) + ...) as fusion.cpp:73-76.
__global__ void apply_f32_kernel(int n_parts, const int32_t* const* __restrict__ idx, int64_t rows,
                                 const float* const* __restrict__ P, int64_t l, float* __restrict__ y) {
  const int64_t total = rows * l;
  if ((l & 3) == 0) {
    const int64_t l4 = l >> 2;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < rows * l4; e += (int64_t)gridDim.x * blockDim.x) {
      const int64_t r = e / l4, c = e - r * l4;
      float4 acc = __ldg(reinterpret_cast<const float4*>(P[0] + static_cast<int64_t>(__ldg(idx[0] + r)) * l) + c);
      for (int j = 1; j < n_parts; ++j) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(P[j] + static_cast<int64_t>(__ldg(idx[j] + r)) * l) + c);
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
      }
      __stcs(reinterpret_cast<float4*>(y) + e, acc);
    }
    return;
  }
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / l, c = e - r * l;
    float acc = __ldg(P[0] + static_cast<int64_t>(__ldg(idx[0] + r)) * l + c);
    for (int j = 1; j < n_parts; ++j) acc += __ldg(P[j] + static_cast<int64_t>(__ldg(idx[j] + r)) * l + c);
    __stcs(y + e, acc);
  }
}

}  // namespace gemm
}  // namespace laq

using namespace laq;

// A-side operand: the dims' feature tables in the split block layout plus the
// global feature index of every (block, column) position.
struct laq_tc_features {
  int n_dims = 0;
  int64_t k = 0;
  double scale = 1.0;  // s_A
  int64_t dim_rows[gemm::kMaxDims] = {};
  int n_blocks = 0;
  int block_dim[gemm::kMaxBlocks] = {}, block_steps[gemm::kMaxBlocks] = {};
  DevMem<tc::elem> blocks[gemm::kMaxBlocks];
  CUtensorMap amap[gemm::kMaxBlocks];  // block b as a TMA tensor (identity-row GEMMs)
  bool amap_ok = false;
  std::vector<int64_t> perm;  // 32 * n_blocks entries, -1 = padding
  DevMem<int64_t> dperm;
};

extern "C" {

int laq_tc_features_create(laq_ctx* ctx, int32_t n_dims, const double* const* d_dims, const int64_t* h_dim_rows,
                           const int64_t* h_dim_cols, const int64_t* const* h_placements, int64_t k,
                           laq_tc_features** out) {
  return guard(ctx, [&] {
    if (n_dims < 1 || n_dims > gemm::kMaxDims) fail(LAQ_ERR_UNSUPPORTED, "tc features: 1..8 dimension tables");
    std::vector<int> seen(static_cast<size_t>(std::max<int64_t>(k, 0)), 0);
    for (int j = 0; j < n_dims; ++j)
      for (int64_t c = 0; c < h_dim_cols[j]; ++c) {
        const int64_t g = h_placements[j][c];
        if (g < 0 || g >= k) fail(LAQ_ERR_MAPPING, "column map: target index out of range");
        if (seen[g]++) fail(LAQ_ERR_MAPPING, "fusion: overlapping target columns");
      }
    auto* f = new laq_tc_features();
    try {
      f->n_dims = n_dims;
      f->k = k;
      std::vector<std::pair<int, int64_t>> src;
      for (int j = 0; j < n_dims; ++j) {
        f->dim_rows[j] = h_dim_rows[j];
        for (int64_t f0 = 0; f0 < h_dim_cols[j]; f0 += 32) {
          if (f->n_blocks == gemm::kMaxBlocks) fail(LAQ_ERR_UNSUPPORTED, "tc features: more than 2048 features");
          const int64_t w = std::min<int64_t>(32, h_dim_cols[j] - f0);
          f->block_dim[f->n_blocks] = j;
          f->block_steps[f->n_blocks] = w > 16 ? 2 : 1;
          ++f->n_blocks;
          src.emplace_back(j, f0);
          for (int64_t c = 0; c < 32; ++c) f->perm.push_back(c < w ? h_placements[j][f0 + c] : -1);
        }
      }
      const int g = ctx->sm_count * 8;
      double amax = 0.0;
      for (int j = 0; j < n_dims; ++j) amax = std::max(amax, absmax_f64(ctx, d_dims[j], h_dim_rows[j] * h_dim_cols[j]));
      f->scale = tc::pow2_scale(amax);
      for (int b = 0; b < f->n_blocks; ++b) {
        const int j = src[b].first;
        const int64_t r = h_dim_rows[j];
        f->blocks[b] = DevMem<tc::elem>(static_cast<size_t>(std::max<int64_t>(r, 1) * 64));
        if (r > 0) {
          tc::split_block_kernel<<<g, 256, 0, ctx->stream>>>(d_dims[j], r, h_dim_cols[j], src[b].second, f->scale,
                                                             f->blocks[b].get());
          launched(ctx);
        }
      }
      f->amap_ok = true;
      for (int b = 0; b < f->n_blocks; ++b)
        f->amap_ok = f->amap_ok && tc::encode_rows128(&f->amap[b], f->blocks[b].get(),
                                                      static_cast<uint64_t>(std::max<int64_t>(h_dim_rows[src[b].first], 1)),
                                                      gemm::kRows);
      f->dperm = DevMem<int64_t>(f->perm.size());
      LAQ_CUDA(cudaMemcpyAsync(f->dperm.get(), f->perm.data(), f->perm.size() * sizeof(int64_t),
                               cudaMemcpyHostToDevice, ctx->stream));
      sync(ctx);
    } catch (...) {
      delete f;
      throw;
    }
    *out = f;
  });
}

int laq_tc_features_destroy(laq_tc_features* f) {
  delete f;
  return LAQ_OK;
}

int laq_tc_gemm(laq_ctx* ctx, const laq_tc_features* f, const int32_t* const* d_rows, int64_t m, const double* d_W,
                int64_t n, float* d_out) {
  return guard(ctx, [&] {
    if (n < 1) fail(LAQ_ERR_SHAPE, "tc gemm: output width must be positive");
    if (!d_rows) {
      if (f->n_dims != 1) fail(LAQ_ERR_SHAPE, "tc gemm: identity rows need a single dimension table");
      if (m != f->dim_rows[0]) fail(LAQ_ERR_SHAPE, "tc gemm: identity rows must cover the dimension table");
    }
    if (m == 0) return;
    const int BN = static_cast<int>(std::min<int64_t>(256, (n + 15) / 16 * 16));
    const int64_t n_tiles = (n + BN - 1) / BN;
    const int64_t n_pad = n_tiles * BN;
    // W (k x n fp64) -> split blocks in the features' column order
    DevBuf<tc::elem> w(ctx, static_cast<size_t>(f->n_blocks * n_pad * 64));
    LAQ_CUDA(cudaMemsetAsync(w.get(), 0, static_cast<size_t>(f->n_blocks * n_pad * 64) * 2, ctx->stream));
    // split_w1_kernel writes [n_blocks][n][64]; lay each block out with stride n_pad
    const double sw = tc::pow2_scale(absmax_f64(ctx, d_W, f->k * n));
    for (int b = 0; b < f->n_blocks; ++b) {
      tc::split_w1_kernel<<<grid_for(n * 32, 256, ctx->sm_count * 8), 256, 0, ctx->stream>>>(
          d_W, n, f->dperm.get() + 32 * b, 1, sw, w.get() + static_cast<int64_t>(b) * n_pad * 64);
      launched(ctx);
    }
    gemm::Args a{};
    for (int b = 0; b < f->n_blocks; ++b) {
      a.block[b] = f->blocks[b].get();
      a.block_dim[b] = f->block_dim[b];
      a.block_steps[b] = f->block_steps[b];
    }
    a.n_blocks = f->n_blocks;
    a.n_dims = f->n_dims;
    for (int j = 0; j < f->n_dims; ++j) a.idx[j] = d_rows ? d_rows[j] : nullptr;
    a.m = m;
    a.n = n;
    a.BN = BN;
    a.w = w.get();
    a.n_pad = n_pad;
    a.w_tma = !std::getenv("LAQ_GEMM_NO_TMA") &&
              tc::encode_rows128(&a.wmap, w.get(), static_cast<uint64_t>(f->n_blocks * n_pad), static_cast<uint32_t>(BN));
    a.a_tma = a.w_tma && !d_rows && f->amap_ok && !std::getenv("LAQ_GEMM_NO_TMA_A");
    if (a.a_tma)
      for (int b = 0; b < f->n_blocks; ++b) a.amap[b] = f->amap[b];
    a.c = d_out;
    a.unscale = static_cast<float>(1.0 / (f->scale * sw));
    a.m_tiles = (m + gemm::kRows - 1) / gemm::kRows;
    a.n_tiles = n_tiles;
    a.m_major = f->n_blocks * n_pad * 128 <= (int64_t{64} << 20) ? 1 : 0;
    int S = 0;
    for (int s = 8; s >= 2; --s)
      if (gemm::smem_bytes(BN, s) <= 220 * 1024) { S = s; break; }
    a.stages = S;
    const uint32_t bytes = gemm::smem_bytes(BN, S);
    LAQ_CUDA(cudaFuncSetAttribute(gemm::gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>(a.m_tiles * a.n_tiles, ctx->sm_count));
    gemm::gemm_kernel<<<grid, gemm::kThreads, bytes, ctx->stream>>>(a);
    launched(ctx);
  });
}

int laq_apply_fused_linear_f32(laq_ctx* ctx, int32_t n_parts, const int32_t* const* d_idx, int64_t rows,
                               const float* const* d_partials, int64_t l, float* d_out) {
  return guard(ctx, [&] {
    if (n_parts < 1 || n_parts > gemm::kMaxDims) fail(LAQ_ERR_SHAPE, "apply_fused_linear: 1..8 partials");
    if (rows == 0 || l == 0) return;
    DevBuf<const void*> ptrs(ctx, 2 * n_parts);
    std::vector<const void*> h(2 * n_parts);
    for (int j = 0; j < n_parts; ++j) {
      h[j] = d_idx[j];
      h[n_parts + j] = d_partials[j];
    }
    LAQ_CUDA(cudaMemcpyAsync(ptrs.get(), h.data(), h.size() * sizeof(void*), cudaMemcpyHostToDevice, ctx->stream));
    const int64_t work = (l & 3) == 0 ? rows * (l / 4) : rows * l;
    gemm::apply_f32_kernel<<<grid_for(work, 256, ctx->sm_count * 16), 256, 0, ctx->stream>>>(
        n_parts, reinterpret_cast<const int32_t* const*>(ptrs.get()), rows,
        reinterpret_cast<const float* const*>(ptrs.get() + n_parts), l, d_out);
    launched(ctx);
    sync(ctx);  // the host pointer table must outlive its async copy
  });
}

}  // extern "C"
