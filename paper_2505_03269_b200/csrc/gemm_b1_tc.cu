// gemm_b1_tc.cu -- 1-bit-mode complex beamformer GEMM on the sm_100a tensor cores (kind::i8).
//
// The paper's 1-bit tensor-core path (b1 mma with XOR/AND + popc) does not
// exist natively on sm_100a: ptxas lowers `mma.sync ... .b1 ... .popc` to 8 legacy
// IMMA.16832.U8 + LOP3 masks per m16n8k256 (cuobjdump -sass; profiles/).  This kernel keeps
// HBM traffic at one bit per component and feeds the 5th-generation tensor cores instead:
//
//   * the packed words are expanded IN SHARED MEMORY to unsigned bytes 2u, u in {0, 1}, by
//     bit-plane masking, byte i of plane j = 2 * bit (8i + j) of the word.  This is a fixed
//     permutation of the 32 K-elements of a word, applied identically to both operands, so
//     every dot product is unchanged;
//   * tcgen05.mma.kind::i8 (unsigned, int32 accumulate in TMEM) then computes scaled
//     AND-popcounts 4 P(A & B) = sum_k (2u_a)(2u_b) exactly (PAPER.md:265-270 AND form);
//   * the complex +-1 result follows from the single-AND identities (reading R1b),
//     with a = 2u - 1 and |X| the popcount of a row/column:
//         acc_r = P(A_r & B_r) + P(A_i & ~B_i)          acc_i = P(A_r & B_i) + P(A_i & B_r)
//         Re = 4 acc_r - 2|A_r| - 2|A_i| - 2|B_r| + 2|B_i|
//         Im = 4 acc_i - 2(|A_r| + |A_i| + |B_r| + |B_i|) + 2K
//     ~B_i is formed during expansion, the paper's "Im(b) = -Im(b) in local registers"
//     (PAPER.md:154-159).  Padding bits are 0 in A, so the 1s of ~B_i in the padding never
//     contribute; no K_pad term is needed.
//
// Roles (persistent CTA per SM, 416 threads):
//   warp 0      TMEM allocator + single-thread MMA issuer (2 MMAs of N = 256 per K=32 step)
//   warps 1-4   epilogue: tcgen05.ld, + row term + column term (one IADD3), TMA store of int32
//   warps 5-8   expanders for A_r, A_i (one weight row per thread; also |A_r| + |A_i|)
//   warps 9-12  expanders for B_r, B_i, ~B_i (one data column per thread; also |B_r|, |B_i|)
// The popcounts travel expanders -> epilogue through smem with their own full/empty mbarriers.
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "kernels.h"
#include "ptx.cuh"

namespace tcbf {
namespace {

constexpr int BM = 128;
constexpr int BN = 128;
constexpr int KB_WORDS = 4;            // 128 bits per K block -> 128 expanded bytes per row
constexpr int TILE_BYTES = 128 * 128;  // one expanded operand tile (rows x 128 B)
constexpr int STAGES = 2;
constexpr int STAGE_BYTES = 5 * TILE_BYTES;  // A_r, A_i, ~B_i, B_r, B_i
constexpr int EPI_BYTES = 4 * 2 * 4096;
constexpr int COLSUM_BYTES = 2 * 3 * 128 * 4;  // [2 acc buf][|A_r|+|A_i| rows, |B_r|, |B_i| cols][128]
constexpr int BAR_OFFSET = STAGES * STAGE_BYTES + EPI_BYTES + COLSUM_BYTES;
constexpr int SMEM_BYTES = 1024 + BAR_OFFSET + 256;
constexpr int NUM_THREADS = 13 * 32;
constexpr int NUM_EXPANDERS = 256;
constexpr int EXPANDER_WARPS = NUM_EXPANDERS / 32;  // barrier arrivals are aggregated per warp
constexpr uint32_t TMEM_COLS = 512;  // 2 buffers x (acc_r, acc_i) x 128 columns
static_assert(SMEM_BYTES <= 232448, "smem budget");

// Bit-plane expansion to bytes in {0, 2}: byte i of plane j = 2 * bit (8i + j) of the word.
// With both operands scaled by 2 the tensor core accumulates 4 * P(A & B) directly.
__device__ __forceinline__ uint4 planes_lo(uint32_t w) {
  const uint32_t m = 0x02020202u;
  return make_uint4((w << 1) & m, w & m, (w >> 1) & m, (w >> 2) & m);
}
__device__ __forceinline__ uint4 planes_hi(uint32_t w) {
  const uint32_t m = 0x02020202u;
  return make_uint4((w >> 3) & m, (w >> 4) & m, (w >> 5) & m, (w >> 6) & m);
}

__device__ __forceinline__ void expand_word(uint8_t* row_base, int row, int q, uint32_t w) {
  // word q of the K block -> chunks 2q (planes 0-3) and 2q+1 (planes 4-7), 128-byte swizzle
  uint4 c0 = planes_lo(w);
  uint4 c1 = planes_hi(w);
  const int sw = row & 7;
  *reinterpret_cast<uint4*>(row_base + (((2 * q) ^ sw) << 4)) = c0;
  *reinterpret_cast<uint4*>(row_base + (((2 * q + 1) ^ sw) << 4)) = c1;
}

// expands w and its complement (planes of ~w are planes of w xor 0x02020202)
__device__ __forceinline__ void expand_word_pair(uint8_t* base, uint8_t* base_c, int row, int q, uint32_t w) {
  const uint32_t m = 0x02020202u;
  uint4 c0 = planes_lo(w);
  uint4 c1 = planes_hi(w);
  const int sw = row & 7;
  const int p0 = ((2 * q) ^ sw) << 4, p1 = ((2 * q + 1) ^ sw) << 4;
  *reinterpret_cast<uint4*>(base + p0) = c0;
  *reinterpret_cast<uint4*>(base + p1) = c1;
  *reinterpret_cast<uint4*>(base_c + p0) = make_uint4(c0.x ^ m, c0.y ^ m, c0.z ^ m, c0.w ^ m);
  *reinterpret_cast<uint4*>(base_c + p1) = make_uint4(c1.x ^ m, c1.y ^ m, c1.z ^ m, c1.w ^ m);
}

template <bool TMA_STORE>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    cgemm_b1_tc_kernel(const __grid_constant__ CUtensorMap tmC, GemmB1Args p, int tiles_m, int tiles_n,
                       int num_tiles) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* epi_base = smem + STAGES * STAGE_BYTES;
  int* colsum = reinterpret_cast<int*>(epi_base + EPI_BYTES);  // [2 buf][2 plane][BN]
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + BAR_OFFSET);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull_bar = empty_bar + STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint64_t* sfull_bar = tempty_bar + 2;   // popcount sums of a tile written (256 expanders)
  uint64_t* sempty_bar = sfull_bar + 2;   // popcount sums consumed (4 epilogue warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sempty_bar + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int num_kb = p.Kw / KB_WORDS;
  const int num_items = num_tiles * p.splits;  // (tile, K split) work items

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], EXPANDER_WARPS);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], 4);
      // every thread arrives after its own colsum accesses (no reliance on a warp-level
      // sync before a single-lane arrive; keeps compute-sanitizer racecheck exact)
      mbar_init(&sfull_bar[s], EXPANDER_WARPS * 32);
      mbar_init(&sempty_bar[s], 4 * 32);
    }
    fence_barrier_init();
    if (TMA_STORE) tma_prefetch_desc(&tmC);
  }
  if (warp == 0) {
    tmem_alloc(tmem_slot, TMEM_COLS);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ MMA issuer (converged warp, one
    // elected lane issues: descriptors stay in uniform registers)
    {
      // kind::i8, unsigned A and B, int32 D, K-major, M = 128, N = 2 BN: one MMA covers both
      // accumulators [D_r | D_i] (contiguous TMEM columns) against two stacked data tiles, so A
      // is read from smem once per pair of sub-products (the stage holds ~B_i, B_r, B_i in row
      // order: A_r x [B_r; B_i] and A_i x [~B_i; B_r])
      constexpr uint32_t IDESC = (2u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)((2 * BN) >> 3) << 17) |
                                 ((uint32_t)(BM >> 4) << 24);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int item = blockIdx.x; item < num_items; item += gridDim.x, ++it) {
        const int sp = item % p.splits;
        const int kb0 = sp * p.kb_per_split, kb1 = min(num_kb, kb0 + p.kb_per_split);
        const int abuf = it & 1;
        mbar_wait(&tempty_bar[abuf], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_re = tmem_base + abuf * 2 * BN;  // D_i follows at d_re + BN
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint8_t* st = smem + stage * STAGE_BYTES;
          // K advance per MMA: 32 bytes (+2 in the descriptor address field)
          const uint64_t ar0 = smem_desc_k128(st, 0), ai0 = smem_desc_k128(st + TILE_BYTES, 0);
          const uint64_t b_cr0 = smem_desc_k128(st + 2 * TILE_BYTES, 0);  // [~B_i; B_r]
          const uint64_t b_ri0 = smem_desc_k128(st + 3 * TILE_BYTES, 0);  // [B_r; B_i]
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {  // K = 32 bytes per MMA
              const uint32_t acc = ((kb - kb0) | kk) ? 1u : 0u;
              if (TCBF_ABLATE(p, 2)) continue;
              mma_i8_ss(d_re, ar0 + (uint64_t)(2 * kk), b_ri0 + (uint64_t)(2 * kk), IDESC, acc);  // [P(A_r & B_r) | P(A_r & B_i)]
              mma_i8_ss(d_re, ai0 + (uint64_t)(2 * kk), b_cr0 + (uint64_t)(2 * kk), IDESC, 1u);   // [P(A_i & ~B_i) | P(A_i & B_r)]
            }
            mma_commit(&empty_bar[stage]);
          }
          __syncwarp();
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        if (elect_one()) mma_commit(&tfull_bar[abuf]);
        __syncwarp();
      }
    }
  } else if (warp <= 4) {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;
    const int ew = warp - 1;
    uint8_t* stg = epi_base + ew * 8192;
    int sbuf = 0;
    int it = 0;
    for (int item = blockIdx.x; item < num_items; item += gridDim.x, ++it) {
      const int t = item / p.splits;
      int b, mt, nt;
      tile_coords(t, tiles_m, tiles_n, p.group_m, b, mt, nt);
      const int m0 = mt * BM;
      const int n0 = nt * BN;
      const int cb = it & 1;
      // popcounts |A_r|+|A_i| (rows) and |B_r|, |B_i| (columns), accumulated by the expanders
      mbar_wait(&sfull_bar[cb], (it >> 1) & 1);
      const int m = m0 + q * 32 + lane;
      const int rterm = colsum[(cb * 3 + 0) * 128 + q * 32 + lane];  // -2 (|A_r| + |A_i|)
      const int* cterm_re = colsum + (cb * 3 + 1) * 128;           // 2 (|B_i| - |B_r|)
      const int* cterm_im = colsum + (cb * 3 + 2) * 128;           // 2K - 2 (|B_r| + |B_i|)
      const int abuf = it & 1;
      mbar_wait(&tfull_bar[abuf], (it >> 1) & 1);
      tc_fence_after();
      constexpr int CHUNKS = BN / 32;
      const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + abuf * 2 * BN;
      uint32_t vbuf[2][32];
      tmem_ld_32x32b_x32(tbase, vbuf[0]);
#pragma unroll
      for (int ch = 0; ch < 2 * CHUNKS; ++ch) {
        const int part = ch / CHUNKS;
        const int c = ch % CHUNKS;
        tmem_wait_ld();
        if (ch + 1 < 2 * CHUNKS) {
          tmem_ld_32x32b_x32(tbase + (ch + 1) * 32, vbuf[(ch + 1) & 1]);
        } else {  // all TMEM reads of this tile done: release the accumulator buffer
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty_bar[abuf]);
        }
        uint32_t* v = vbuf[ch & 1];
        const int* cterm = (part == 0 ? cterm_re : cterm_im) + c * 32;
        int ct[32];
#pragma unroll
        for (int j = 0; j < 8; ++j) {  // broadcast 128-bit smem loads
          const int4 t4 = *reinterpret_cast<const int4*>(cterm + 4 * j);
          ct[4 * j] = t4.x; ct[4 * j + 1] = t4.y; ct[4 * j + 2] = t4.z; ct[4 * j + 3] = t4.w;
        }
        if (ch == 2 * CHUNKS - 1) mbar_arrive(&sempty_bar[cb]);  // last read of this tile's terms
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = (uint32_t)((int)v[j] + ct[j] + rterm);  // Re / Im, R1b
        if (TCBF_ABLATE(p, 1)) continue;
        if constexpr (TMA_STORE) {
          if (lane == 0) bulk_wait_group_read<1>();
          __syncwarp();
          uint8_t* buf = stg + sbuf * 4096;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int pos = j ^ (lane & 7);
            *reinterpret_cast<uint4*>(buf + lane * 128 + pos * 16) =
                make_uint4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            if (p.splits > 1) tma_reduce_add_3d(&tmC, buf, n0 + c * 32, m0 + q * 32, 2 * b + part);
            else tma_store_3d(&tmC, buf, n0 + c * 32, m0 + q * 32, 2 * b + part);
            bulk_commit_group();
          }
          sbuf ^= 1;
        } else {
          if (m < p.M) {
            int32_t* row = p.out + ((size_t)(2 * b + part) * p.M + m) * (size_t)p.N;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const int n = n0 + c * 32 + j;
              if (n < p.N) {
                if (p.splits > 1) atomicAdd(row + n, (int32_t)v[j]);
                else row[n] = (int32_t)v[j];
              }
            }
          }
        }
      }
    }
    if constexpr (TMA_STORE) {
      if (lane == 0) bulk_wait_group<0>();
      __syncwarp();
    }
  } else {
    // ------------------------------------------------------------ expanders
    const int e = threadIdx.x - 5 * 32;  // 0..255
    const bool a_side = e < 128;
    const int row = a_side ? e : e - 128;
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    const uint4 zero = make_uint4(0, 0, 0, 0);
    // row pointers of this thread's operand row/column for tile t (nullptr when out of range)
    auto row_ptrs = [&](int t, const uint4*& pr, const uint4*& pi) {
      int b, mt, nt;
      tile_coords(t, tiles_m, tiles_n, p.group_m, b, mt, nt);
      pr = pi = nullptr;
      if (a_side) {
        const int m = mt * BM + row;
        if (m < p.M) {
          pr = reinterpret_cast<const uint4*>(p.w + ((size_t)(2 * b) * p.M + m) * p.Kw);
          pi = reinterpret_cast<const uint4*>(p.w + ((size_t)(2 * b + 1) * p.M + m) * p.Kw);
        }
      } else {
        const int n = nt * BN + row;
        if (n < p.N) {
          pr = reinterpret_cast<const uint4*>(p.x + ((size_t)(2 * b) * p.N + n) * p.Kw);
          pi = reinterpret_cast<const uint4*>(p.x + ((size_t)(2 * b + 1) * p.N + n) * p.Kw);
        }
      }
    };
    const uint4* src_r;
    const uint4* src_i;
    auto item_range = [&](int item, int& kb0, int& kb1) {
      const int sp = item % p.splits;
      kb0 = sp * p.kb_per_split;
      kb1 = min(num_kb, kb0 + p.kb_per_split);
    };
    row_ptrs(blockIdx.x / p.splits, src_r, src_i);
    int kb0, kb1;
    item_range(blockIdx.x, kb0, kb1);
    uint4 nr = (blockIdx.x < (unsigned)num_items && src_r) ? __ldg(src_r + kb0) : zero;
    uint4 ni = (blockIdx.x < (unsigned)num_items && src_i) ? __ldg(src_i + kb0) : zero;
    for (int item = blockIdx.x; item < num_items; item += gridDim.x, ++it) {
      int pc_r = 0, pc_i = 0;  // popcounts of this row / column over the item's K range
      const bool valid = src_r != nullptr;
      const uint4* next_r = nullptr;
      const uint4* next_i = nullptr;
      const int in = item + gridDim.x;
      int nkb0 = 0, nkb1 = 0;
      if (in < num_items) {
        row_ptrs(in / p.splits, next_r, next_i);
        item_range(in, nkb0, nkb1);
      }
      for (int kb = kb0; kb < kb1; ++kb) {
        const uint4 wr = nr, wi = ni;
        if (kb + 1 < kb1) {
          nr = valid ? __ldg(src_r + kb + 1) : zero;
          ni = valid ? __ldg(src_i + kb + 1) : zero;
        } else {  // first K block of this thread's next work item
          nr = next_r ? __ldg(next_r + nkb0) : zero;
          ni = next_i ? __ldg(next_i + nkb0) : zero;
        }
        pc_r += __popc(wr.x) + __popc(wr.y) + __popc(wr.z) + __popc(wr.w);
        pc_i += __popc(wi.x) + __popc(wi.y) + __popc(wi.z) + __popc(wi.w);
        mbar_wait(&empty_bar[stage], phase ^ 1);
        uint8_t* st = smem + stage * STAGE_BYTES;
        if (TCBF_ABLATE(p, 4)) {
        } else if (a_side) {
          uint8_t* ar = st + row * 128;
          uint8_t* ai = st + TILE_BYTES + row * 128;
          expand_word(ar, row, 0, wr.x); expand_word(ar, row, 1, wr.y);
          expand_word(ar, row, 2, wr.z); expand_word(ar, row, 3, wr.w);
          expand_word(ai, row, 0, wi.x); expand_word(ai, row, 1, wi.y);
          expand_word(ai, row, 2, wi.z); expand_word(ai, row, 3, wi.w);
        } else {
          uint8_t* bc = st + 2 * TILE_BYTES + row * 128;
          uint8_t* br = st + 3 * TILE_BYTES + row * 128;
          uint8_t* bi = st + 4 * TILE_BYTES + row * 128;
          expand_word(br, row, 0, wr.x); expand_word(br, row, 1, wr.y);
          expand_word(br, row, 2, wr.z); expand_word(br, row, 3, wr.w);
          expand_word_pair(bi, bc, row, 0, wi.x); expand_word_pair(bi, bc, row, 1, wi.y);
          expand_word_pair(bi, bc, row, 2, wi.z); expand_word_pair(bi, bc, row, 3, wi.w);
        }
        fence_proxy_async_smem();  // each thread's generic-proxy smem writes -> async proxy
        __syncwarp();
        if (lane == 0) mbar_arrive(&full_bar[stage]);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      // publish this tile's popcounts for the epilogue's single-AND correction (R1b)
      const int cb = it & 1;
      mbar_wait(&sempty_bar[cb], ((it >> 1) & 1) ^ 1);
      if (a_side) {
        colsum[(cb * 3 + 0) * 128 + row] = -2 * (pc_r + pc_i);
      } else {
        colsum[(cb * 3 + 1) * 128 + row] = 2 * (pc_i - pc_r);
        // logical K positions of this item's range (padding bits are 0 and count nothing)
        const int k_s = max(0, min(p.K, kb1 * 128) - kb0 * 128);
        colsum[(cb * 3 + 2) * 128 + row] = 2 * k_s - 2 * (pc_r + pc_i);
      }
      mbar_arrive(&sfull_bar[cb]);
      src_r = next_r;
      src_i = next_i;
      kb0 = nkb0;
      kb1 = nkb1;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem_base, TMEM_COLS);
  }
}

template <bool TMA_STORE>
cudaError_t launch_tc(const CUtensorMap& tmC, const GemmB1Args& a, int num_sms, cudaStream_t stream) {
  auto kern = cgemm_b1_tc_kernel<TMA_STORE>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
  if (e != cudaSuccess) return e;
  const int tiles_m = (a.M + BM - 1) / BM, tiles_n = (a.N + BN - 1) / BN;
  const long long nt = (long long)tiles_m * tiles_n * a.B;
  if (nt > 0x7fffffffLL) return cudaErrorInvalidValue;
  const int grid = (int)(nt < num_sms ? nt : num_sms);
  kern<<<grid, NUM_THREADS, SMEM_BYTES, stream>>>(tmC, a, tiles_m, tiles_n, (int)nt);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_gemm_b1_tc(const CUtensorMap& tmC, const GemmB1Args& args, bool tma_store, int num_sms,
                              cudaStream_t stream) {
  return tma_store ? launch_tc<true>(tmC, args, num_sms, stream) : launch_tc<false>(tmC, args, num_sms, stream);
}

}  // namespace tcbf
