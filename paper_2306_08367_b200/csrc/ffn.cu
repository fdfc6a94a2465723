// K6: the non-fused 2-layer FFN over a star join on the 5th-generation tensor cores
// (BASELINE configs[2]; SURVEY.md §8a row 17, §8d "GEMM"):
//
//     Y = ReLU(T . W1) . W2,   T[m] = [B_0[row_0(m)] | B_1[row_1(m)] | ...]
//
// T is the reference's materialize (laqops.cpp:338-374) and the two products its
// predict_linear / dense_matmul (mlops.cpp:248-250, matrix.cpp:158-174).  The
// reference has no FFN; cfg3 composes these pinned functions with a ReLU.  T is
// never written to HBM: each 128-row tile of T is gathered straight from the
// dimension feature tables into shared memory and multiplied there.
//
// Numerics: fp64 inputs are stored once as a bf16x3 split
// (x = hi + lo + O(2^-18|x|)); every tile runs hi.hi + hi.lo + lo.hi on tcgen05
// with fp32 accumulation in TMEM, then ReLU and layer 2 in fp32 on the CUDA cores.
// Accuracy is judged condition-aware at 1e-5 (tests/test_gpu_ffn.py).
//
// Kernel structure (persistent, one CTA per SM, 288 threads):
//   warps 0-3  epilogue: tcgen05.ld the 128 x h accumulator (thread = row),
//              ReLU, dot with W2 (shared memory), coalesced fp32 stores;
//   warps 4-7  gather producers: resolve dim rows (row maps, or fact keys through
//              the probe tables) two tiles ahead, then 16-byte cp.async of the
//              hi/lo feature chunks into the K-major SW128 stage, cp.async.wait +
//              proxy fence + mbarrier arrive;
//   warp 8     TMEM owner + MMA issuer (one elected lane): 3 x K/16 tcgen05.mma
//              per tile into one of two TMEM accumulators, tcgen05.commit frees
//              the stage and hands the accumulator to the epilogue.
// W1 (hi/lo, K-major) stays resident in shared memory for the whole kernel.
#include <algorithm>
#include <vector>

#include "probe.cuh"
#include "tc.cuh"

namespace laq {
namespace ffn {

constexpr int kRows = 128;  // tile rows = UMMA M = TMEM lanes
constexpr int kEpiWarps = 4, kProdWarps = 4;
constexpr int kThreads = (kEpiWarps + kProdWarps + 1) * 32;
constexpr int kMaxDims = 4;
constexpr int kMaxL = 8;
constexpr int kProdThreads = kProdWarps * 32;

struct Args {
  int n_dims;
  int64_t n;  // rows processed (fact rows in probe mode, join rows otherwise)
  const int32_t* idx[kMaxDims];  // row maps, or fact keys (probe mode)
  ProbeView probe[kMaxDims];
  int probe_mode;
  const __nv_bfloat16* hi[kMaxDims];  // [rows_j x 8*chunks_j] row-major
  const __nv_bfloat16* lo[kMaxDims];
  int chunks[kMaxDims];  // 16-byte chunks per dim row
  int chunk0[kMaxDims];  // first global chunk of dim j in the T row
  int C;                 // chunks per T row (K_pad / 8)
  int KB;                // 64-wide K blocks
  int ksteps;            // K_pad / 16
  int N;                 // hidden width (UMMA N)
  int l;
  const __nv_bfloat16* w1hi;  // [N x K_pad] (W1^T, K-major)
  const __nv_bfloat16* w1lo;
  const float* w2;  // [N x l]
  float* y;         // [n x l]
  int stages;
  int64_t n_tiles;
  unsigned long long* miss;  // probe mode: rows missing some dimension
};

struct Smem {  // offsets into the 1024-aligned dynamic buffer
  uint32_t b, a, w2, bars, stage_bytes;
};

__host__ __device__ inline Smem layout(int KB, int N, int l, int S) {
  Smem m;
  m.b = 0;
  m.a = static_cast<uint32_t>(KB) * 2u * N * 128u;
  m.stage_bytes = static_cast<uint32_t>(KB) * 2u * kRows * 128u;
  m.w2 = m.a + S * m.stage_bytes;
  m.bars = (m.w2 + N * l * 4u + 15u) & ~15u;
  return m;
}
__host__ __device__ inline uint32_t smem_bytes(int KB, int N, int l, int S) {
  // barriers: full[S], empty[S], acc_full[2], acc_empty[2] + tmem slot; +1 KB alignment slack
  return layout(KB, N, l, S).bars + (2 * S + 4) * 8 + 16 + 1024;
}

// Resolve dim rows of this producer thread's row for one tile (row maps or probe).
__device__ __forceinline__ void load_keys(const Args& a, int64_t tile, int lane_row, int32_t (&k)[kMaxDims]) {
  int64_t r = tile * kRows + lane_row;
  if (r >= a.n) r = a.n - 1;
#pragma unroll
  for (int j = 0; j < kMaxDims; ++j)
    if (j < a.n_dims) k[j] = __ldg(a.idx[j] + r);
}

template <int kLag>
__global__ void __launch_bounds__(kThreads, 1) ffn_kernel(const Args a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int S = a.stages, KB = a.KB, N = a.N, l = a.l;
  const Smem L = layout(KB, N, l, S);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bars);
  uint64_t* empty = full + S;
  uint64_t* acc_full = empty + S;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  float* s_w2 = reinterpret_cast<float*>(smem + L.w2);
  const uint32_t sbase = tc::smem_u32(smem);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // ---- one-time setup: W1 (hi, lo) -> SW128 K-major blocks; W2 -> smem --------
  {
    const int C = a.C;
    const int total = N * C * 2;
    for (int e = threadIdx.x; e < total; e += kThreads) {
      const int n = e / (2 * C), rem = e - n * 2 * C, p = rem >= C, c = rem - p * C;
      const uint4 v = *reinterpret_cast<const uint4*>((p ? a.w1lo : a.w1hi) + static_cast<int64_t>(n) * C * 8 + c * 8);
      *reinterpret_cast<uint4*>(smem + L.b + ((c >> 3) * 2 + p) * N * 128u + tc::sw128_off(n, c & 7)) = v;
    }
    for (int e = threadIdx.x; e < N * l; e += kThreads) s_w2[e] = a.w2[e];
  }
  if (warp == 8) {
    if (lane == 0) {
      for (int s = 0; s < S; ++s) {
        tc::mbar_init(&full[s], kProdThreads);
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
  tc::fence_proxy_async();  // W1 st.shared -> async proxy
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp >= kEpiWarps && warp < kEpiWarps + kProdWarps) {
    // ================= gather producers =================
    const int pw = warp - kEpiWarps;  // rows 32*pw .. 32*pw+31 of every tile
    const int C = a.C, items = 32 * 2 * C;
    __shared__ int32_t s_rows[kProdWarps][kMaxDims][32];
    int32_t k1[kMaxDims] = {}, k2[kMaxDims] = {}, r1[kMaxDims] = {};
    int64_t tile = blockIdx.x;
    const int64_t step = gridDim.x;
    unsigned long long misses = 0;
    // prologue: keys for tiles 0 and 1, rows for tile 0
    if (tile < a.n_tiles) load_keys(a, tile, 32 * pw + lane, k1);
    if (tile + step < a.n_tiles) load_keys(a, tile + step, 32 * pw + lane, k2);
#pragma unroll
    for (int j = 0; j < kMaxDims; ++j)
      if (j < a.n_dims) r1[j] = a.probe_mode ? a.probe[j].row(k1[j]) : k1[j];
    int it = 0;
    for (; tile < a.n_tiles; tile += step, ++it) {
      const int s = it % S;
      const uint32_t ph = (it / S) & 1;
      // rows of this tile (resolved last iteration) -> shared
      const bool live = tile * kRows + 32 * pw + lane < a.n;
#pragma unroll
      for (int j = 0; j < kMaxDims; ++j)
        if (j < a.n_dims) {
          int32_t r = r1[j];
          if (r < 0) {
            misses += live ? 1 : 0;
            r = 0;
          }
          s_rows[pw][j][lane] = r;
        }
      // look ahead: rows of tile+1 (keys loaded last iteration), keys of tile+2
#pragma unroll
      for (int j = 0; j < kMaxDims; ++j)
        if (j < a.n_dims) r1[j] = a.probe_mode ? a.probe[j].row(k2[j]) : k2[j];
      if (tile + 2 * step < a.n_tiles) load_keys(a, tile + 2 * step, 32 * pw + lane, k2);
      __syncwarp();

      tc::mbar_wait(&empty[s], ph ^ 1);
      const uint32_t abase = sbase + L.a + s * L.stage_bytes;
      for (int e = lane; e < items; e += 32) {
        const int rl = e / (2 * C), rem = e - rl * 2 * C, p = rem >= C, c = rem - p * C;
        int j = 0;
#pragma unroll
        for (int q = 1; q < kMaxDims; ++q)
          if (q < a.n_dims && c >= a.chunk0[q]) j = q;
        const int cj = c - a.chunk0[j];
        const int64_t drow = s_rows[pw][j][rl];
        const __nv_bfloat16* src = (p ? a.lo[j] : a.hi[j]) + drow * (a.chunks[j] * 8) + cj * 8;
        const int r = 32 * pw + rl;
        tc::cp_async16(abase + ((c >> 3) * 2 + p) * (kRows * 128u) + tc::sw128_off(r, c & 7), src);
      }
      tc::cp_async_commit();
      if (it >= kLag) {
        tc::cp_async_wait<kLag>();
        tc::fence_proxy_async();
        tc::mbar_arrive(&full[(it - kLag) % S]);
      }
      __syncwarp();  // s_rows reuse
    }
    tc::cp_async_wait<0>();
    tc::fence_proxy_async();
    for (int t = std::max(0, it - kLag); t < it; ++t) tc::mbar_arrive(&full[t % S]);
    if (a.probe_mode) {
      for (int o = 16; o; o >>= 1) misses += __shfl_xor_sync(0xffffffffu, misses, o);
      if (lane == 0 && misses) atomicAdd(a.miss, misses);
    }
  } else if (warp == kEpiWarps + kProdWarps) {
    // ================= MMA issuer =================
    if (lane == 0) {
      const uint32_t idesc = tc::idesc_bf16_f32(kRows, N);
      int it = 0;
      for (int64_t tile = blockIdx.x; tile < a.n_tiles; tile += gridDim.x, ++it) {
        const int s = it % S, ab = it & 1;
        tc::mbar_wait(&acc_empty[ab], ((it >> 1) & 1) ^ 1);
        tc::mbar_wait(&full[s], (it / S) & 1);
        tc::tc_fence_after();
        const uint32_t d = tmem + ab * N;
        const uint32_t abase = sbase + L.a + s * L.stage_bytes;
        uint32_t acc = 0;
#pragma unroll
        for (int pr = 0; pr < 3; ++pr) {  // hi.hi, hi.lo, lo.hi
          const int pa = pr == 2, pb = pr == 1;
          for (int ks = 0; ks < a.ksteps; ++ks) {
            const int kb = ks >> 2;
            const uint32_t koff = (ks & 3) * 32u;
            const uint64_t ad = tc::sdesc_sw128(abase + (kb * 2 + pa) * (kRows * 128u) + koff);
            const uint64_t bd = tc::sdesc_sw128(sbase + L.b + (kb * 2 + pb) * (N * 128u) + koff);
            tc::mma_bf16(d, ad, bd, idesc, acc);
            acc = 1;
          }
        }
        tc::mma_commit(&empty[s]);
        tc::mma_commit(&acc_full[ab]);
      }
    }
    __syncwarp();
  } else {
    // ================= epilogue (warps 0-3) =================
    int it = 0;
    for (int64_t tile = blockIdx.x; tile < a.n_tiles; tile += gridDim.x, ++it) {
      const int ab = it & 1;
      tc::mbar_wait(&acc_full[ab], (it >> 1) & 1);
      tc::tc_fence_after();
      float y[kMaxL];
#pragma unroll
      for (int c = 0; c < kMaxL; ++c) y[c] = 0.f;
      const uint32_t t0 = tmem + (static_cast<uint32_t>(32 * warp) << 16) + ab * N;
      for (int c0 = 0; c0 < N; c0 += 32) {
        uint32_t v[32];
        tc::tmem_ld32(t0 + c0, v);
        tc::tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const float h = fmaxf(__uint_as_float(v[i]), 0.f);
          const float* w = s_w2 + (c0 + i) * l;
#pragma unroll
          for (int c = 0; c < kMaxL; ++c)
            if (c < l) y[c] = fmaf(h, w[c], y[c]);
        }
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&acc_empty[ab]);
      const int64_t row = tile * kRows + 32 * warp + lane;
      if (row < a.n) {
#pragma unroll
        for (int c = 0; c < kMaxL; ++c)
          if (c < l) __stcs(a.y + row * l + c, y[c]);
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 8) {
    tc::tc_fence_after();
    tc::tmem_dealloc<512>(tmem);
  }
}

// ---- layout preparation --------------------------------------------------------
// dim table B_j (rows x cols fp64) -> hi/lo bf16 [rows x kpad], zero padded.
__global__ void split_table_kernel(const double* __restrict__ B, int64_t rows, int64_t cols, int64_t kpad,
                                   __nv_bfloat16* __restrict__ hi, __nv_bfloat16* __restrict__ lo) {
  const int64_t total = rows * kpad;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / kpad, c = e - r * kpad;
    __nv_bfloat16 h = __float2bfloat16(0.f), q = __float2bfloat16(0.f);
    if (c < cols) tc::split_bf16(B[r * cols + c], h, q);
    hi[e] = h;
    lo[e] = q;
  }
}
// W1 (k x n fp64, row-major) -> W1^T hi/lo [n x kpad]; T column q holds global
// feature perm[q] (-1 = padding).
__global__ void split_w1_kernel(const double* __restrict__ W, int64_t n, const int64_t* __restrict__ perm,
                                int64_t kpad, __nv_bfloat16* __restrict__ hi, __nv_bfloat16* __restrict__ lo) {
  const int64_t total = n * kpad;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t col = e / kpad, q = e - col * kpad;
    __nv_bfloat16 h = __float2bfloat16(0.f), o = __float2bfloat16(0.f);
    const int64_t g = perm[q];
    if (g >= 0) tc::split_bf16(W[g * n + col], h, o);
    hi[e] = h;
    lo[e] = o;
  }
}
__global__ void to_f32_kernel(const double* __restrict__ x, int64_t n, float* __restrict__ y) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    y[e] = static_cast<float>(x[e]);
}
__global__ void iota_kernel(int64_t* __restrict__ out, int64_t n) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    out[e] = e;
}

}  // namespace ffn
}  // namespace laq

using namespace laq;

struct laq_ffn {
  int n_dims = 0;
  int64_t dim_rows[ffn::kMaxDims] = {};
  int chunks[ffn::kMaxDims] = {}, chunk0[ffn::kMaxDims] = {};
  int C = 0, KB = 0, ksteps = 0, N = 0, l = 0, stages = 0;
  int64_t k = 0;
  DevMem<__nv_bfloat16> hi[ffn::kMaxDims], lo[ffn::kMaxDims];
  DevMem<__nv_bfloat16> w1hi, w1lo;
  DevMem<float> w2;
  DevMem<unsigned long long> miss;
};

namespace laq {
namespace {

ffn::Args make_args(const laq_ffn* f, int64_t n, float* y) {
  ffn::Args a{};
  a.n_dims = f->n_dims;
  a.n = n;
  for (int j = 0; j < f->n_dims; ++j) {
    a.hi[j] = f->hi[j].get();
    a.lo[j] = f->lo[j].get();
    a.chunks[j] = f->chunks[j];
    a.chunk0[j] = f->chunk0[j];
  }
  a.C = f->C;
  a.KB = f->KB;
  a.ksteps = f->ksteps;
  a.N = f->N;
  a.l = f->l;
  a.w1hi = f->w1hi.get();
  a.w1lo = f->w1lo.get();
  a.w2 = f->w2.get();
  a.y = y;
  a.stages = f->stages;
  a.n_tiles = (n + ffn::kRows - 1) / ffn::kRows;
  a.miss = f->miss.get();
  return a;
}

void launch_ffn(laq_ctx* ctx, const laq_ffn* f, const ffn::Args& a) {
  if (a.n_tiles == 0) return;
  const uint32_t bytes = ffn::smem_bytes(f->KB, f->N, f->l, f->stages);
  const unsigned grid = static_cast<unsigned>(std::min<int64_t>(a.n_tiles, ctx->sm_count));
  if (f->stages >= 4) {
    LAQ_CUDA(cudaFuncSetAttribute(ffn::ffn_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    ffn::ffn_kernel<2><<<grid, ffn::kThreads, bytes, ctx->stream>>>(a);
  } else {
    LAQ_CUDA(cudaFuncSetAttribute(ffn::ffn_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    ffn::ffn_kernel<1><<<grid, ffn::kThreads, bytes, ctx->stream>>>(a);
  }
  launched(ctx);
}

}  // namespace
}  // namespace laq

extern "C" {

int laq_ffn_create(laq_ctx* ctx, int32_t n_dims, const double* const* d_dims, const int64_t* h_dim_rows,
                   const int64_t* h_dim_cols, const int64_t* const* h_placements, int64_t k, const double* d_W1,
                   int64_t h, const double* d_W2, int64_t l, laq_ffn** out) {
  return guard(ctx, [&] {
    if (n_dims < 1 || n_dims > ffn::kMaxDims) fail(LAQ_ERR_UNSUPPORTED, "ffn: 1..4 dimension tables");
    if (h < 32 || h > 256 || h % 32) fail(LAQ_ERR_UNSUPPORTED, "ffn: hidden width must be a multiple of 32 in [32,256]");
    if (l < 1 || l > ffn::kMaxL) fail(LAQ_ERR_UNSUPPORTED, "ffn: output width 1..8");
    // placements must tile [0,k) exactly (check_placements, fusion.cpp:11-25)
    std::vector<int> seen(static_cast<size_t>(std::max<int64_t>(k, 0)), 0);
    int64_t covered = 0;
    for (int j = 0; j < n_dims; ++j)
      for (int64_t c = 0; c < h_dim_cols[j]; ++c) {
        const int64_t g = h_placements[j][c];
        if (g < 0 || g >= k) fail(LAQ_ERR_SHAPE, "ffn: placement outside the feature width");
        if (seen[g]++) fail(LAQ_ERR_MAPPING, "ffn: overlapping placements");
        ++covered;
      }
    if (covered != k) fail(LAQ_ERR_SHAPE, "ffn: placements do not cover the feature width");
    auto* f = new laq_ffn();
    try {
      f->n_dims = n_dims;
      f->k = k;
      f->N = static_cast<int>(h);
      f->l = static_cast<int>(l);
      // T row = concatenation of the dims' (8-padded) feature chunks
      std::vector<int64_t> perm;
      for (int j = 0; j < n_dims; ++j) {
        const int64_t kp = (h_dim_cols[j] + 7) / 8 * 8;
        f->chunk0[j] = static_cast<int>(perm.size() / 8);
        f->chunks[j] = static_cast<int>(kp / 8);
        for (int64_t c = 0; c < kp; ++c) perm.push_back(c < h_dim_cols[j] ? h_placements[j][c] : -1);
      }
      while (perm.size() % 16) perm.push_back(-1);
      const int64_t kpad = static_cast<int64_t>(perm.size());
      if (kpad > 128) fail(LAQ_ERR_UNSUPPORTED, "ffn: gathered width > 128 features (use materialize + gemm)");
      f->C = static_cast<int>(kpad / 8);
      f->KB = (f->C + 7) / 8;
      f->ksteps = static_cast<int>(kpad / 16);
      int S = 0;
      for (int s = 6; s >= 2; --s)
        if (ffn::smem_bytes(f->KB, f->N, f->l, s) <= 224 * 1024) { S = s; break; }
      if (S == 0) fail(LAQ_ERR_UNSUPPORTED, "ffn: W1 tile does not fit shared memory");
      f->stages = S;
      const int g = ctx->sm_count * 8;
      for (int j = 0; j < n_dims; ++j) {
        const int64_t r = h_dim_rows[j], kp = f->chunks[j] * 8;
        f->dim_rows[j] = r;
        f->hi[j] = DevMem<__nv_bfloat16>(static_cast<size_t>(std::max<int64_t>(r * kp, 1)));
        f->lo[j] = DevMem<__nv_bfloat16>(static_cast<size_t>(std::max<int64_t>(r * kp, 1)));
        if (r > 0) {
          ffn::split_table_kernel<<<g, 256, 0, ctx->stream>>>(d_dims[j], r, h_dim_cols[j], kp, f->hi[j].get(),
                                                              f->lo[j].get());
          launched(ctx);
        }
      }
      DevBuf<int64_t> dperm(ctx, perm.size());
      LAQ_CUDA(cudaMemcpyAsync(dperm.get(), perm.data(), perm.size() * sizeof(int64_t), cudaMemcpyHostToDevice,
                               ctx->stream));
      f->w1hi = DevMem<__nv_bfloat16>(static_cast<size_t>(h * kpad));
      f->w1lo = DevMem<__nv_bfloat16>(static_cast<size_t>(h * kpad));
      ffn::split_w1_kernel<<<g, 256, 0, ctx->stream>>>(d_W1, h, dperm.get(), kpad, f->w1hi.get(), f->w1lo.get());
      launched(ctx);
      f->w2 = DevMem<float>(static_cast<size_t>(h * l));
      ffn::to_f32_kernel<<<g, 256, 0, ctx->stream>>>(d_W2, h * l, f->w2.get());
      launched(ctx);
      f->miss = DevMem<unsigned long long>(1);
      sync(ctx);  // dperm is freed with the stream; host vector outlives the copy
    } catch (...) {
      delete f;
      throw;
    }
    *out = f;
  });
}

int laq_ffn_destroy(laq_ffn* f) {
  delete f;
  return LAQ_OK;
}

int laq_ffn_predict_rows(laq_ctx* ctx, const laq_ffn* f, const int32_t* const* d_rows, int64_t rows, float* d_out) {
  return guard(ctx, [&] {
    ffn::Args a = make_args(f, rows, d_out);
    for (int j = 0; j < f->n_dims; ++j) a.idx[j] = d_rows[j];
    a.probe_mode = 0;
    launch_ffn(ctx, f, a);
  });
}

int laq_ffn_predict_star(laq_ctx* ctx, const laq_ffn* f, const laq_probe* probe, const int32_t* const* d_fks,
                         int64_t n_fact, float* d_out, int64_t* d_survivors, int64_t* h_nnz) {
  return guard(ctx, [&] {
    if (probe_links(probe) != f->n_dims) fail(LAQ_ERR_SHAPE, "ffn: probe / feature table count differs");
    // Optimistic pass: every fact row probed inside the kernel, Y written at the
    // fact row; misses counted.  With no miss the output is already the
    // (ascending, complete) survivor list.
    ffn::Args a = make_args(f, n_fact, d_out);
    for (int j = 0; j < f->n_dims; ++j) {
      a.idx[j] = d_fks[j];
      a.probe[j] = probe_view(probe, j);
    }
    a.probe_mode = 1;
    LAQ_CUDA(cudaMemsetAsync(f->miss.get(), 0, sizeof(unsigned long long), ctx->stream));
    launch_ffn(ctx, f, a);
    LAQ_CUDA(cudaMemcpyAsync(ctx->h_pinned, f->miss.get(), sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    sync(ctx);
    if (ctx->h_pinned[0] == 0) {
      if (d_survivors && n_fact > 0) {
        ffn::iota_kernel<<<grid_for(n_fact, 256, ctx->sm_count * 8), 256, 0, ctx->stream>>>(d_survivors, n_fact);
        launched(ctx);
      }
      *h_nnz = n_fact;
      return;
    }
    // Some fact rows drop out: compact the join (int32 row maps), then rerun on them.
    std::vector<DevBuf<int32_t>> maps;
    std::vector<int32_t*> mp;
    for (int j = 0; j < f->n_dims; ++j) {
      maps.emplace_back(ctx, static_cast<size_t>(std::max<int64_t>(n_fact, 1)));
      mp.push_back(maps.back().get());
    }
    int64_t* d_nnz = ctx->d_flags + 21;
    int rc = laq_probe_join_rows(ctx, probe, d_fks, n_fact, mp.data(), d_survivors, d_nnz);
    if (rc) fail(rc, ctx->err);
    LAQ_CUDA(cudaMemcpyAsync(ctx->h_pinned, d_nnz, sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    sync(ctx);
    const int64_t nnz = ctx->h_pinned[0];
    ffn::Args b = make_args(f, nnz, d_out);
    for (int j = 0; j < f->n_dims; ++j) b.idx[j] = mp[j];
    b.probe_mode = 0;
    launch_ffn(ctx, f, b);
    *h_nnz = nnz;
  });
}

}  // extern "C"
