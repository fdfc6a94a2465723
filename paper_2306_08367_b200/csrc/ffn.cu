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
// Numerics: fp64 inputs are stored once as a scaled fp16x2
// split (tc.cuh split_f16: x*s = hi + lo + O(2^-22)); every tile runs hi.hi + hi.lo
// + lo.hi on tcgen05 with fp32 accumulation in TMEM, the epilogue unscales by the
// exact power of two 1/(s_A s_W1), then ReLU and layer 2 in fp32 on the CUDA cores.
// Accuracy is judged condition-aware at 1e-5 (tests/test_gpu_ffn.py).  (A bf16
// split keeps only 16 significant bits, 1.5e-5 per element: measured to fail.)
//
// HBM layout: every dimension's features are cut into blocks of 32 columns; block b
// is an fp16 table [rows_j x 64] whose row is (hi[32] | lo[32]) -- exactly one
// 128-byte line, the unit one TMA gather moves.  W1 uses the same block layout
// (W1^T rows = hidden units), so inside a 128-byte swizzled smem row the hi
// operand sits at byte 0 and the lo operand at byte 64.
//
// Kernel structure (persistent, one CTA per SM, 416 threads):
//   warps 0-7   epilogue: warp w reads TMEM lanes 32(w%4).. (thread = tile row) and
//               every other 32-column chunk of the 128 x h accumulator (tcgen05.ld),
//               ReLU, dot with W2 (broadcast shared loads, 4 independent FMA
//               chains); the two column halves meet through shared memory and a
//               named barrier; coalesced fp32 stores;
//   warps 8-11  gather producers: each lane resolves one row (row maps, or fact
//               keys through the probe tables, two tiles ahead); then every warp
//               instruction moves 4 feature lines (4 rows x 128 B) with 16-byte
//               cp.async into the SW128 stage; cp.async.mbarrier.arrive.noinc
//               signals the stage when the thread's copies land (no blocking);
//   warp 12     TMEM owner + MMA issuer (one lane): 3 x K/16 tcgen05.mma per tile
//               into one of two TMEM accumulators; tcgen05.commit frees the stage
//               and hands the accumulator to the epilogue.
// Measured alternative (not used): TMA tile::gather4 (4 rows per instruction)
// was issue-bound at ~1.5 TB/s on B200 because the per-lane row indices force
// the uniform-datapath TMA instruction into a serialised per-lane loop.
// W1 (hi/lo) stays resident in shared memory for the whole kernel.
#include <algorithm>
#include <cstdlib>
#include <string>
#include <utility>
#include <vector>

#include "probe.cuh"
#include "tc.cuh"

namespace laq {
namespace ffn {

constexpr int kRows = 128;  // tile rows = UMMA M = TMEM lanes
constexpr int kEpiWarps = 8;
constexpr int kProdWarps = 4, kProdWarp0 = 8, kMmaWarp = 12;
constexpr int kThreads = 13 * 32;
constexpr int kMaxDims = 4;
constexpr int kMaxBlocks = 8;  // 32-feature blocks (K <= 256)
constexpr int kMaxL = 8;
constexpr uint32_t kBlockBytes = kRows * 128u;  // one feature block of a stage

struct Args {
  const tc::elem* block[kMaxBlocks];  // block b: [rows x 64] fp16 = (hi32 | lo32)
  int n_blocks;
  int block_dim[kMaxBlocks];    // dimension owning block b
  int block_steps[kMaxBlocks];  // 16-feature MMA steps in block b (1 or 2)
  int n_dims;
  int64_t n;                     // rows processed (fact rows in probe mode, join rows otherwise)
  const int32_t* idx[kMaxDims];  // row maps, or fact keys (probe mode)
  ProbeView probe[kMaxDims];
  int probe_mode;
  int N;                    // hidden width (UMMA N)
  int l;
  const tc::elem* w1;  // [n_blocks][N][64] (hi32 | lo32)
  const float* w2;          // [N x LP] (l padded to a power of two with zeros)
  float* y;                 // [n x l]
  float unscale;            // 1 / (s_A s_W1), a power of two
  int stages;
  int64_t n_tiles;
  unsigned long long* miss;  // probe mode: rows missing some dimension
  int diag;  // A/B diagnostics: 1 no gathers, 2 no MMAs, 3 no gathers + no epilogue, 4 no gathers + TMEM loads only
};

struct Smem {  // offsets into the 1024-aligned dynamic buffer
  uint32_t b, a, w2, bars, stage_bytes;
};

// cg = 2 (CTA pair): each CTA holds N/2 rows of every W1 block (its half of B).
__host__ __device__ inline Smem layout(int nb, int N, int lp, int S, int cg = 1) {
  Smem m;
  m.b = 0;
  m.a = static_cast<uint32_t>(nb) * (N / cg) * 128u;
  m.stage_bytes = static_cast<uint32_t>(nb) * kBlockBytes;
  m.w2 = m.a + S * m.stage_bytes;
  m.bars = (m.w2 + N * lp * 4u + 15u) & ~15u;
  return m;
}
__host__ __device__ inline uint32_t smem_bytes(int nb, int N, int lp, int S, int cg = 1) {
  // barriers: full[S], empty[S], acc_full[2], acc_empty[2] + tmem slot; +1 KB alignment slack
  return layout(nb, N, lp, S, cg).bars + (2 * S + 4) * 8 + 16 + 1024;
}

// Key (or row-map entry) of fact row `g` for every dim, clamped to n-1.
__device__ __forceinline__ void load_keys(const Args& a, int64_t g, int32_t (&k)[kMaxDims]) {
  if (g >= a.n) g = a.n - 1;
#pragma unroll
  for (int j = 0; j < kMaxDims; ++j)
    if (j < a.n_dims) k[j] = __ldg(a.idx[j] + g);
}
__device__ __forceinline__ void resolve(const Args& a, const int32_t (&k)[kMaxDims], int32_t (&r)[kMaxDims]) {
#pragma unroll
  for (int j = 0; j < kMaxDims; ++j)
    if (j < a.n_dims) r[j] = a.probe_mode ? a.probe[j].row(k[j]) : k[j];
}

// CG = 1: one CTA per SM, M = 128 UMMAs.  CG = 2: a CTA pair (cluster of 2)
// runs M = 256 UMMAs (cta_group::2) over 256-row tiles: each CTA gathers its
// 128 rows and holds half of W1, so every SM's shared memory serves half of
// the B operand reads; only the leader issues MMAs; the peer's producers
// report through a relay arrive on the leader's stage barrier, its epilogue
// warps release the accumulator on the leader's barrier.
template <int LP, int CG>
__global__ void __launch_bounds__(kThreads, 1) ffn_kernel(const __grid_constant__ Args a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int S = a.stages, NB = a.n_blocks, N = a.N, l = a.l;
  const Smem L = layout(NB, N, LP, S, CG);
  const uint32_t rank = CG == 2 ? tc::cluster_rank() : 0u;
  const bool leader = rank == 0;
  const int64_t tile0 = CG == 2 ? blockIdx.x / 2 : blockIdx.x;   // tiles of kRows * CG rows
  const int64_t tstep = CG == 2 ? gridDim.x / 2 : gridDim.x;
  const int64_t row_off = static_cast<int64_t>(rank) * kRows;    // this CTA's rows within a tile
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bars);
  uint64_t* empty = full + S;
  uint64_t* acc_full = empty + S;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  float* s_w2 = reinterpret_cast<float*>(smem + L.w2);
  const uint32_t sbase = tc::smem_u32(smem);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // ---- one-time setup: W1 blocks -> SW128 K-major rows; W2 -> smem ----------------
  const int NH = N / CG;  // W1 rows (hidden units) this CTA holds per block
  for (int e = threadIdx.x; e < NB * NH * 8; e += kThreads) {
    const int c = e & 7, row = e >> 3;  // row = b * NH + n_local
    const int b = row / NH, nl = row - b * NH;
    const int64_t src = static_cast<int64_t>(b) * N + static_cast<int64_t>(rank) * NH + nl;
    const uint4 v = *reinterpret_cast<const uint4*>(a.w1 + src * 64 + c * 8);
    *reinterpret_cast<uint4*>(smem + L.b + tc::sw128_off(row, c)) = v;  // NH is a multiple of 8
  }
  for (int e = threadIdx.x; e < N * LP; e += kThreads) s_w2[e] = a.w2[e] * a.unscale;  // exact (power of two)
  if (warp == kMmaWarp) {
    if (lane == 0) {
      for (int s = 0; s < S; ++s) {
        // the leader's stage barrier also counts the peer's relay arrive
        tc::mbar_init(&full[s], kProdWarps * 32 + (CG == 2 && leader ? 1 : 0));
        tc::mbar_init(&empty[s], 1);
      }
      for (int b = 0; b < 2; ++b) {
        tc::mbar_init(&acc_full[b], 1);
        tc::mbar_init(&acc_empty[b], kEpiWarps * CG);  // the leader's counts both CTAs' epilogues
      }
      tc::fence_mbar_init();
    }
    __syncwarp();
    if constexpr (CG == 2) tc::tmem_alloc2<512>(tmem_slot);
    else tc::tmem_alloc<512>(tmem_slot);
  }
  tc::fence_proxy_async();  // W1 st.shared -> async proxy
  tc::tc_fence_before();
  __syncthreads();
  if constexpr (CG == 2) tc::cluster_sync();  // both CTAs' barriers exist before any remote arrive
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp >= kProdWarp0 && warp < kProdWarp0 + kProdWarps) {
    // ================= cp.async gather producers =================
    const int pw = warp - kProdWarp0;  // tile rows 32*pw .. 32*pw+31
    __shared__ int32_t s_rows[kProdWarps][kMaxDims][32];
    int32_t k1[kMaxDims] = {}, k2[kMaxDims] = {}, r1[kMaxDims] = {};
    int64_t tile = tile0;
    const int64_t step = tstep;
    const int64_t TR = static_cast<int64_t>(kRows) * CG;  // rows per tile
    const int64_t my = row_off + 32 * pw + lane;          // this lane's row within a tile
    unsigned long long misses = 0;
    // prologue: keys of the first two tiles, rows of the first
    if (tile < a.n_tiles) load_keys(a, tile * TR + my, k1);
    if (tile + step < a.n_tiles) load_keys(a, (tile + step) * TR + my, k2);
    resolve(a, k1, r1);
    const int sub = lane >> 3, chunk = lane & 7;  // 4 rows x 8 16-byte chunks per instruction
    for (int it = 0; tile < a.n_tiles; tile += step, ++it) {
      const int s = it % S;
      const bool live = tile * TR + my < a.n;
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
      // look ahead: rows of the next tile (keys loaded an iteration ago), keys two ahead
      resolve(a, k2, r1);
      if (tile + 2 * step < a.n_tiles) load_keys(a, (tile + 2 * step) * TR + my, k2);
      __syncwarp();

      tc::mbar_wait(&empty[s], ((it / S) & 1) ^ 1);
      if (a.diag != 1 && a.diag < 3) {
        const uint32_t abase = sbase + L.a + s * L.stage_bytes;
        for (int b = 0; b < NB; ++b) {
          const tc::elem* base = a.block[b] + chunk * 8;
          const int j = a.block_dim[b];
          const uint32_t dbase = abase + b * kBlockBytes;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int rl = 4 * q + sub, r = 32 * pw + rl;
            const int64_t drow = s_rows[pw][j][rl];
            tc::cp_async16(dbase + tc::sw128_off(r, chunk), base + drow * 64);
          }
        }
      }
      tc::cp_async_arrive_noinc(&full[s]);
      __syncwarp();  // s_rows reuse
    }
    if (a.probe_mode) {
      for (int o = 16; o; o >>= 1) misses += __shfl_xor_sync(0xffffffffu, misses, o);
      if (lane == 0 && misses) atomicAdd(a.miss, misses);
    }
  } else if (warp == kMmaWarp && CG == 2 && !leader) {
    // ================= peer relay (CTA pair) =================
    // When this CTA's producers have filled stage s, tell the leader (its MMA
    // reads this CTA's half of A and B from this shared memory).
    if (lane == 0) {
      int it = 0;
      for (int64_t tile = tile0; tile < a.n_tiles; tile += tstep, ++it) {
        const int s = it % S;
        tc::mbar_wait(&full[s], (it / S) & 1);
        tc::fence_proxy_async();  // cp.async (generic proxy) writes -> the leader's tensor-core reads
        tc::mbar_arrive_cluster(tc::mapa(&full[s], 0));
      }
    }
    __syncwarp();
  } else if (warp == kMmaWarp) {
    // ================= MMA issuer =================
    if (lane == 0) {
      const uint32_t idesc = tc::idesc_f16_f32(kRows * CG, N);
      int it = 0;
      for (int64_t tile = tile0; tile < a.n_tiles; tile += tstep, ++it) {
        const int s = it % S, ab = it & 1;
        tc::mbar_wait(&acc_empty[ab], ((it >> 1) & 1) ^ 1);
        tc::mbar_wait(&full[s], (it / S) & 1);
        tc::fence_proxy_async();  // cp.async (generic proxy) writes -> tensor core reads
        tc::tc_fence_after();
        const uint32_t d = tmem + ab * N;
        const uint32_t abase = sbase + L.a + s * L.stage_bytes;
        uint32_t acc = 0;
#pragma unroll
        for (int pr = 0; pr < (a.diag == 2 ? 0 : 3); ++pr) {  // hi.hi, hi.lo, lo.hi
          const uint32_t pa = pr == 2 ? 64u : 0u, pb = pr == 1 ? 64u : 0u;
          for (int b = 0; b < NB; ++b)
            for (int st = 0; st < a.block_steps[b]; ++st) {
              const uint64_t ad = tc::sdesc_sw128(abase + b * kBlockBytes + pa + st * 32u);
              const uint64_t bd = tc::sdesc_sw128(sbase + L.b + b * ((N / CG) * 128u) + pb + st * 32u);
              if constexpr (CG == 2) tc::mma_f16_pair(d, ad, bd, idesc, acc);
              else tc::mma_f16(d, ad, bd, idesc, acc);
              acc = 1;
            }
        }
        if constexpr (CG == 2) {
          tc::mma_commit_pair(&empty[s]);
          tc::mma_commit_pair(&acc_full[ab]);
        } else {
          tc::mma_commit(&empty[s]);
          tc::mma_commit(&acc_full[ab]);
        }
      }
    }
    __syncwarp();
  } else {
    // ================= epilogue (warps 0-7) =================
    __shared__ float s_red[2][4][32][kMaxL];
    const int q = warp & 3, hh = warp >> 2;  // TMEM lane group, column half
    const uint32_t w2a = tc::smem_u32(s_w2);
    int it = 0;
    // the accumulator is released on the leader's barrier (a cluster address for the peer)
    const uint32_t rel[2] = {CG == 2 ? tc::mapa(&acc_empty[0], 0) : 0u, CG == 2 ? tc::mapa(&acc_empty[1], 0) : 0u};
    for (int64_t tile = tile0; tile < a.n_tiles; tile += tstep, ++it) {
      const int ab = it & 1;
      tc::mbar_wait(&acc_full[ab], (it >> 1) & 1);
      tc::tc_fence_after();
      // 4 independent accumulation chains, two per packed f32x2 register (FFMA2)
      constexpr int LQ = LP == 1 ? 1 : LP / 2;
      float2 y2[2][LQ];
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int c = 0; c < LQ; ++c) y2[u][c] = make_float2(0.f, 0.f);
      const uint32_t t0 = tmem + (static_cast<uint32_t>(32 * q) << 16) + ab * N;
      bool released = false;
      // this warp's chunks: c0 = 32*hh, 32*hh + 64, ... (two per TMEM wait)
      for (int c0 = 32 * hh; c0 < (a.diag >= 3 ? (a.diag == 3 ? 0 : N) : N); c0 += 128) {
        uint32_t v[64];
        const bool two = c0 + 64 < N;
        tc::tmem_ld32(t0 + c0, *reinterpret_cast<uint32_t(*)[32]>(v));
        if (two) tc::tmem_ld32(t0 + c0 + 64, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
        tc::tmem_ld_wait_regs(*reinterpret_cast<uint32_t(*)[32]>(v));
        if (two) tc::reg_fence(*reinterpret_cast<uint32_t(*)[32]>(v + 32));
        if (c0 + 128 >= N) {
          // last TMEM read of this warp for the tile: release the accumulator
          // before the arithmetic, so the MMA warp can start the tile after next
          tc::tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if constexpr (CG == 2) tc::mbar_arrive_cluster(rel[ab]);
            else tc::mbar_arrive(&acc_empty[ab]);
          }
          released = true;
        }
        if (a.diag == 4) {
          y2[0][0].x += __uint_as_float(v[0] ^ v[17] ^ v[33] ^ v[63]);
          continue;
        }
#pragma unroll
        for (int i0 = 0; i0 < 64; i0 += 4) {
          if (i0 < 32 || two) {
            const int col = c0 + (i0 < 32 ? i0 : i0 + 32);
            float w[4 * LP];  // W2 rows col .. col+3, pre-multiplied by the unscale (broadcast loads)
#pragma unroll
            for (int qq = 0; qq < LP; ++qq) {
              const float4 t = tc::lds128_const(w2a + (col * LP + 4 * qq) * 4u);
              w[4 * qq] = t.x; w[4 * qq + 1] = t.y; w[4 * qq + 2] = t.z; w[4 * qq + 3] = t.w;
            }
            // ReLU(acc * s) = s * ReLU(acc) for the power-of-two s > 0 folded into W2
            float h[4];
#pragma unroll
            for (int ii = 0; ii < 4; ++ii) h[ii] = fmaxf(__uint_as_float(v[i0 + ii]), 0.f);
            if constexpr (LP == 1) {
              y2[0][0] = tc::ffma2(make_float2(h[0], h[1]), make_float2(w[0], w[1]), y2[0][0]);
              y2[1][0] = tc::ffma2(make_float2(h[2], h[3]), make_float2(w[2], w[3]), y2[1][0]);
            } else {
#pragma unroll
              for (int ii = 0; ii < 4; ++ii)
#pragma unroll
                for (int c = 0; c < LQ; ++c)
                  y2[ii & 1][c] = tc::ffma2(make_float2(h[ii], h[ii]), make_float2(w[ii * LP + 2 * c], w[ii * LP + 2 * c + 1]),
                                            y2[ii & 1][c]);
            }
          }
        }
      }
      if (!released) {
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (CG == 2) tc::mbar_arrive_cluster(rel[ab]);
          else tc::mbar_arrive(&acc_empty[ab]);
        }
      }
      float yy[LP];
      if constexpr (LP == 1) {
        yy[0] = (y2[0][0].x + y2[0][0].y) + (y2[1][0].x + y2[1][0].y);
      } else {
#pragma unroll
        for (int c = 0; c < LQ; ++c) {
          yy[2 * c] = y2[0][c].x + y2[1][c].x;
          yy[2 * c + 1] = y2[0][c].y + y2[1][c].y;
        }
      }
      if (hh == 1) {
#pragma unroll
        for (int c = 0; c < LP; ++c) s_red[ab][q][lane][c] = yy[c];
      }
      asm volatile("bar.sync %0, 64;" ::"r"(1 + q) : "memory");  // the two warps of lane group q
      if (hh == 0) {
        const int64_t row = tile * (static_cast<int64_t>(kRows) * CG) + row_off + 32 * q + lane;
        if (row < a.n) {
#pragma unroll
          for (int c = 0; c < LP; ++c)
            if (c < l) __stcs(a.y + row * l + c, yy[c] + s_red[ab][q][lane][c]);
        }
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if constexpr (CG == 2) tc::cluster_sync();  // the pair is done with TMEM and each other's barriers
  if (warp == kMmaWarp) {
    tc::tc_fence_after();
    if constexpr (CG == 2) tc::tmem_dealloc2<512>(tmem);
    else tc::tmem_dealloc<512>(tmem);
  }
}

// ---- layout preparation (feature blocks / W1: tc::split_block_kernel, tc::split_w1_kernel) ----
// W2 (h x l fp64) -> fp32 [h x lp], zero columns l..lp-1.
__global__ void w2_pad_kernel(const double* __restrict__ x, int64_t h, int64_t l, int64_t lp, float* __restrict__ y) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < h * lp; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / lp, c = e - r * lp;
    y[e] = c < l ? static_cast<float>(x[r * l + c]) : 0.f;
  }
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
  int n_blocks = 0;
  int block_dim[ffn::kMaxBlocks] = {}, block_steps[ffn::kMaxBlocks] = {};
  int N = 0, l = 0, lp = 1, stages = 0;
  int64_t k = 0;
  double unscale = 1.0;
  DevMem<tc::elem> blocks[ffn::kMaxBlocks];  // [rows_j x 64] (hi32 | lo32)
  DevMem<tc::elem> w1;  // [n_blocks][N][64]
  DevMem<float> w2;
  DevMem<unsigned long long> miss;
};

namespace laq {
namespace {

ffn::Args make_args(const laq_ffn* f, int64_t n, float* y) {
  ffn::Args a{};
  a.n_blocks = f->n_blocks;
  for (int b = 0; b < f->n_blocks; ++b) {
    a.block[b] = f->blocks[b].get();
    a.block_dim[b] = f->block_dim[b];
    a.block_steps[b] = f->block_steps[b];
  }
  a.n_dims = f->n_dims;
  a.n = n;
  a.N = f->N;
  a.l = f->l;
  a.w1 = f->w1.get();
  a.w2 = f->w2.get();
  a.y = y;
  a.unscale = static_cast<float>(f->unscale);
  a.stages = f->stages;
  a.n_tiles = (n + ffn::kRows - 1) / ffn::kRows;
  a.miss = f->miss.get();
  const char* d = std::getenv("LAQ_FFN_DIAG");
  a.diag = d ? std::atoi(d) : 0;
  return a;
}

template <int LP>
void launch_lp(laq_ctx* ctx, const ffn::Args& a, unsigned grid, uint32_t bytes, int cg) {
  if (cg == 2) {  // CTA pairs: clusters of 2 on neighbouring SMs
    auto kern = ffn::ffn_kernel<LP, 2>;
    LAQ_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(ffn::kThreads);
    cfg.dynamicSmemBytes = bytes;
    cfg.stream = ctx->stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    LAQ_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
    return;
  }
  LAQ_CUDA(cudaFuncSetAttribute(ffn::ffn_kernel<LP, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  ffn::ffn_kernel<LP, 1><<<grid, ffn::kThreads, bytes, ctx->stream>>>(a);
}

void launch_ffn(laq_ctx* ctx, const laq_ffn* f, const ffn::Args& a0) {
  if (a0.n_tiles == 0) return;
  // LAQ_FFN_2CTA=1: M = 256 UMMAs on CTA pairs (cta_group::2) over 256-row tiles.
  const char* e = std::getenv("LAQ_FFN_2CTA");
  const int cg = e && std::string(e) == "1" ? 2 : 1;
  ffn::Args a = a0;
  a.n_tiles = (a.n + int64_t{ffn::kRows} * cg - 1) / (int64_t{ffn::kRows} * cg);
  const uint32_t bytes = ffn::smem_bytes(f->n_blocks, f->N, f->lp, f->stages, cg);
  const unsigned grid = static_cast<unsigned>(cg * std::min<int64_t>(a.n_tiles, ctx->sm_count / cg));
  switch (f->lp) {
    case 1: launch_lp<1>(ctx, a, grid, bytes, cg); break;
    case 2: launch_lp<2>(ctx, a, grid, bytes, cg); break;
    case 4: launch_lp<4>(ctx, a, grid, bytes, cg); break;
    default: launch_lp<8>(ctx, a, grid, bytes, cg); break;
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
      while (f->lp < f->l) f->lp *= 2;
      // 32-feature blocks per dimension; W1 rows permuted to the block order
      std::vector<int64_t> perm;
      std::vector<std::pair<int, int64_t>> src;  // (dim, first feature)
      for (int j = 0; j < n_dims; ++j)
        for (int64_t f0 = 0; f0 < h_dim_cols[j]; f0 += 32) {
          if (f->n_blocks == ffn::kMaxBlocks)
            fail(LAQ_ERR_UNSUPPORTED, "ffn: more than 8 32-feature blocks (use materialize + gemm)");
          const int64_t w = std::min<int64_t>(32, h_dim_cols[j] - f0);
          f->block_dim[f->n_blocks] = j;
          f->block_steps[f->n_blocks] = w > 16 ? 2 : 1;
          ++f->n_blocks;
          src.emplace_back(j, f0);
          for (int64_t c = 0; c < 32; ++c) perm.push_back(c < w ? h_placements[j][f0 + c] : -1);
        }
      int S = 0;
      for (int s = 6; s >= 2; --s)
        if (ffn::smem_bytes(f->n_blocks, f->N, f->lp, s) <= 212 * 1024) { S = s; break; }
      if (S == 0) fail(LAQ_ERR_UNSUPPORTED, "ffn: W1 tile does not fit shared memory");
      f->stages = S;
      const int g = ctx->sm_count * 8;
      double amax = 0.0;
      for (int j = 0; j < n_dims; ++j) amax = std::max(amax, absmax_f64(ctx, d_dims[j], h_dim_rows[j] * h_dim_cols[j]));
      const double sa = tc::pow2_scale(amax), sw = tc::pow2_scale(absmax_f64(ctx, d_W1, k * h));
      f->unscale = 1.0 / (sa * sw);
      for (int b = 0; b < f->n_blocks; ++b) {
        const int j = src[b].first;
        const int64_t r = h_dim_rows[j];
        f->blocks[b] = DevMem<tc::elem>(static_cast<size_t>(std::max<int64_t>(r, 1) * 64));
        if (r > 0) {
          tc::split_block_kernel<<<g, 256, 0, ctx->stream>>>(d_dims[j], r, h_dim_cols[j], src[b].second, sa,
                                                              f->blocks[b].get());
          launched(ctx);
        } else {
          LAQ_CUDA(cudaMemsetAsync(f->blocks[b].get(), 0, 128, ctx->stream));
        }
      }
      DevBuf<int64_t> dperm(ctx, perm.size());
      LAQ_CUDA(cudaMemcpyAsync(dperm.get(), perm.data(), perm.size() * sizeof(int64_t), cudaMemcpyHostToDevice,
                               ctx->stream));
      f->w1 = DevMem<tc::elem>(static_cast<size_t>(f->n_blocks * h * 64));
      tc::split_w1_kernel<<<g, 256, 0, ctx->stream>>>(d_W1, h, dperm.get(), f->n_blocks, sw, f->w1.get());
      launched(ctx);
      f->w2 = DevMem<float>(static_cast<size_t>(h * f->lp));
      ffn::w2_pad_kernel<<<g, 256, 0, ctx->stream>>>(d_W2, h, l, f->lp, f->w2.get());
      launched(ctx);
      f->miss = DevMem<unsigned long long>(1);
      sync(ctx);  // the host perm vector must outlive its async copy
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
