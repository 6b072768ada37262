// gemm_b1_2cta.cu -- 1-bit-mode complex beamformer GEMM with CTA pairs (tcgen05 cta_group::2, kind::i8).
//
// Same method as gemm_b1_tc.cu (bit-plane expansion to bytes {0, 2}, int8 tensor-core
// AND-popcounts, the single-AND correction R1b -- PAPER.md:215-272), but each 2-CTA cluster
// computes a 256 x 128 complex tile with M=256 MMAs:
//   * CTA r expands its own 128 weight rows (A_r, A_i) and only HALF of the 128 data columns
//     (64 columns: B_r, B_i, ~B_i); the tensor cores of the pair exchange the B halves, so the
//     per-SM expansion work and shared-memory operand traffic drop by ~30% (energy);
//   * the leader's MMA waits on a full barrier that both CTAs' expander warps arrive on
//     (remote arrives for the peer), issues tcgen05.mma.cta_group::2, and multicasts its commits;
//   * the B-side expanders publish their 64 column correction terms into BOTH CTAs' shared
//     memory (local + shared::cluster stores) and arrive on both CTAs' barriers; each CTA's
//     epilogue corrects and stores its own 128 rows x 128 columns.
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "kernels.h"
#include "ptx.cuh"

namespace tcbf {
namespace {

constexpr int BN = 128;                  // pair tile: 256 rows x 128 columns
constexpr int BH = 64;                   // data columns expanded by each CTA
constexpr int A_TILE = 128 * 128;        // 128 rows x 128 B
constexpr int B_TILE = BH * 128;         // 64 rows x 128 B
constexpr int STAGES = 3;
constexpr int STAGE_BYTES = 2 * A_TILE + 3 * B_TILE;  // A_r, A_i, B_r, B_i, ~B_i
constexpr int EPI_BYTES = 4 * 2 * 4096;
constexpr int TERM_BYTES = 2 * 3 * 128 * 4;           // [2 bufs][row term, col re, col im][128]
constexpr int BAR_OFFSET = STAGES * STAGE_BYTES + EPI_BYTES + TERM_BYTES;
constexpr int SMEM_BYTES = 1024 + BAR_OFFSET + 256;
constexpr int A_WARPS = 4, B_WARPS = 2;
constexpr int EXP_WARPS = A_WARPS + B_WARPS;
constexpr int NUM_THREADS = (1 + 4 + EXP_WARPS) * 32;  // MMA, epilogue, expanders
constexpr uint32_t TMEM_COLS = 512;
static_assert(SMEM_BYTES <= 232448, "smem budget");
static_assert(STAGE_BYTES % 1024 == 0, "stage alignment");

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa_shared(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void st_cluster_s32(uint32_t cluster_addr, int v) {
  asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(cluster_addr), "r"(v) : "memory");
}
// cluster-scope acquire wait (the peer CTA's writes are released with .release.cluster arrives)
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  auto try_once = [&]() {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
  };
  if (try_once()) return;
  const long long t0 = clock64();
  while (!try_once()) {
    if (clock64() - t0 > (1ll << 34)) __trap();
  }
}
__device__ __forceinline__ void mma_i8_2sm(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_commit_2sm_mc(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}" ::"r"(
          smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ uint4 planes_lo(uint32_t w) {
  const uint32_t m = 0x02020202u;
  return make_uint4((w << 1) & m, w & m, (w >> 1) & m, (w >> 2) & m);
}
__device__ __forceinline__ uint4 planes_hi(uint32_t w) {
  const uint32_t m = 0x02020202u;
  return make_uint4((w >> 3) & m, (w >> 4) & m, (w >> 5) & m, (w >> 6) & m);
}
__device__ __forceinline__ void expand_word(uint8_t* row_base, int row, int q, uint32_t w) {
  const int sw = row & 7;
  *reinterpret_cast<uint4*>(row_base + (((2 * q) ^ sw) << 4)) = planes_lo(w);
  *reinterpret_cast<uint4*>(row_base + (((2 * q + 1) ^ sw) << 4)) = planes_hi(w);
}
__device__ __forceinline__ void expand_word_pair(uint8_t* base, uint8_t* base_c, int row, int q, uint32_t w) {
  const uint32_t m = 0x02020202u;
  const uint4 c0 = planes_lo(w), c1 = planes_hi(w);
  const int sw = row & 7;
  const int p0 = ((2 * q) ^ sw) << 4, p1 = ((2 * q + 1) ^ sw) << 4;
  *reinterpret_cast<uint4*>(base + p0) = c0;
  *reinterpret_cast<uint4*>(base + p1) = c1;
  *reinterpret_cast<uint4*>(base_c + p0) = make_uint4(c0.x ^ m, c0.y ^ m, c0.z ^ m, c0.w ^ m);
  *reinterpret_cast<uint4*>(base_c + p1) = make_uint4(c1.x ^ m, c1.y ^ m, c1.z ^ m, c1.w ^ m);
}

template <bool TMA_STORE>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    cgemm_b1_2cta_kernel(const __grid_constant__ CUtensorMap tmC, GemmB1Args p, int tiles_m, int tiles_n,
                         int num_tiles) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* epi_base = smem + STAGES * STAGE_BYTES;
  int* terms = reinterpret_cast<int*>(epi_base + EPI_BYTES);
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + BAR_OFFSET);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull_bar = empty_bar + STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint64_t* sfull_bar = tempty_bar + 2;
  uint64_t* sempty_bar = sfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sempty_bar + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const uint32_t peer = rank ^ 1u;
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1;
  const int npairs = gridDim.x >> 1;
  const int num_kb = p.Kw / 4;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 2 * EXP_WARPS);  // (leader's) both CTAs' expander warps
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], 2 * 4);         // (leader's) both CTAs' epilogue warps
      mbar_init(&sfull_bar[s], EXP_WARPS + B_WARPS);  // local expanders + peer B-side expanders
      mbar_init(&sempty_bar[s], 2 * 4);         // both CTAs' epilogue warps
    }
    fence_barrier_init();
    if (TMA_STORE) tma_prefetch_desc(&tmC);
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ MMA issuer (leader)
    if (leader && lane == 0) {
      constexpr uint32_t IDESC = (2u << 4) | ((uint32_t)(BN >> 3) << 17) | ((256u >> 4) << 24);  // u8 x u8 -> s32
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = pair; t < num_tiles; t += npairs, ++it) {
        const int abuf = it & 1;
        mbar_wait_cluster(&tempty_bar[abuf], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_re = tmem_base + abuf * 2 * BN;
        const uint32_t d_im = d_re + BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait_cluster(&full_bar[stage], phase);
          tc_fence_after();
          uint8_t* st = smem + stage * STAGE_BYTES;
          uint8_t* sAr = st;
          uint8_t* sAi = st + A_TILE;
          uint8_t* sBr = st + 2 * A_TILE;
          uint8_t* sBi = sBr + B_TILE;
          uint8_t* sBc = sBi + B_TILE;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint32_t off = kk * 32;
            const uint64_t ar = smem_desc_k128(sAr, off), ai = smem_desc_k128(sAi, off);
            const uint64_t br = smem_desc_k128(sBr, off), bi = smem_desc_k128(sBi, off);
            const uint64_t bc = smem_desc_k128(sBc, off);
            const uint32_t acc = (kb | kk) ? 1u : 0u;
            mma_i8_2sm(d_re, ar, br, IDESC, acc);  // P(A_r & B_r)
            mma_i8_2sm(d_re, ai, bc, IDESC, 1u);   // P(A_i & ~B_i)
            mma_i8_2sm(d_im, ar, bi, IDESC, acc);  // P(A_r & B_i)
            mma_i8_2sm(d_im, ai, br, IDESC, 1u);   // P(A_i & B_r)
          }
          mma_commit_2sm_mc(&empty_bar[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        mma_commit_2sm_mc(&tfull_bar[abuf]);
      }
    }
  } else if (warp <= 4) {
    // ------------------------------------------------------------ epilogue (both CTAs)
    const int q = warp & 3;
    constexpr int CHUNKS = BN / 32;
    uint8_t* stg = epi_base + (warp - 1) * 8192;
    int sbuf = 0;
    int it = 0;
    const uint32_t tempty_leader[2] = {mapa_shared(&tempty_bar[0], 0), mapa_shared(&tempty_bar[1], 0)};
    const uint32_t sempty_peer[2] = {mapa_shared(&sempty_bar[0], peer), mapa_shared(&sempty_bar[1], peer)};
    for (int t = pair; t < num_tiles; t += npairs, ++it) {
      int b, mt, nt;
      tile_coords(t, tiles_m, tiles_n, p.group_m, b, mt, nt);
      const int m0 = mt * 256 + (int)rank * 128;
      const int n0 = nt * BN;
      const int cb = it & 1;
      mbar_wait_cluster(&sfull_bar[cb], (it >> 1) & 1);
      const int rterm = terms[(cb * 3 + 0) * 128 + q * 32 + lane];
      const int* cterm_re = terms + (cb * 3 + 1) * 128;
      const int* cterm_im = terms + (cb * 3 + 2) * 128;
      const int abuf = it & 1;
      mbar_wait(&tfull_bar[abuf], (it >> 1) & 1);
      tc_fence_after();
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
        } else {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(tempty_leader[abuf]);
        }
        uint32_t* v = vbuf[ch & 1];
        const int* cterm = (part == 0 ? cterm_re : cterm_im) + c * 32;
        int ct[32];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int4 t4 = *reinterpret_cast<const int4*>(cterm + 4 * j);
          ct[4 * j] = t4.x; ct[4 * j + 1] = t4.y; ct[4 * j + 2] = t4.z; ct[4 * j + 3] = t4.w;
        }
        if (ch == 2 * CHUNKS - 1) {  // this tile's terms consumed: tell both CTAs' B-expanders
          __syncwarp();
          if (lane == 0) {
            mbar_arrive(&sempty_bar[cb]);
            mbar_arrive_cluster(sempty_peer[cb]);
          }
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = (uint32_t)((int)v[j] + ct[j] + rterm);
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
            tma_store_3d(&tmC, buf, n0 + c * 32, m0 + q * 32, 2 * b + part);
            bulk_commit_group();
          }
          sbuf ^= 1;
        } else {
          const int m = m0 + q * 32 + lane;
          if (m < p.M) {
            int32_t* rowp = p.out + ((size_t)(2 * b + part) * p.M + m) * (size_t)p.N;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const int n = n0 + c * 32 + j;
              if (n < p.N) rowp[n] = (int32_t)v[j];
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
    // ------------------------------------------------------------ expanders (both CTAs)
    const int e = threadIdx.x - 5 * 32;  // 0..191
    const bool a_side = e < 128;
    const int row = a_side ? e : e - 128;  // A: weight row within this CTA's 128; B: column within half
    const uint32_t full_leader0 = mapa_shared(&full_bar[0], 0);
    const uint32_t sfull_peer[2] = {mapa_shared(&sfull_bar[0], peer), mapa_shared(&sfull_bar[1], peer)};
    const uint32_t terms_peer = mapa_shared(terms, peer);
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    const uint4 zero = make_uint4(0, 0, 0, 0);
    for (int t = pair; t < num_tiles; t += npairs, ++it) {
      int b, mt, nt;
      tile_coords(t, tiles_m, tiles_n, p.group_m, b, mt, nt);
      const uint4* src_r = nullptr;
      const uint4* src_i = nullptr;
      if (a_side) {
        const int m = mt * 256 + (int)rank * 128 + row;
        if (m < p.M) {
          src_r = reinterpret_cast<const uint4*>(p.w + ((size_t)(2 * b) * p.M + m) * p.Kw);
          src_i = reinterpret_cast<const uint4*>(p.w + ((size_t)(2 * b + 1) * p.M + m) * p.Kw);
        }
      } else {
        const int n = nt * BN + (int)rank * BH + row;
        if (n < p.N) {
          src_r = reinterpret_cast<const uint4*>(p.x + ((size_t)(2 * b) * p.N + n) * p.Kw);
          src_i = reinterpret_cast<const uint4*>(p.x + ((size_t)(2 * b + 1) * p.N + n) * p.Kw);
        }
      }
      int pc_r = 0, pc_i = 0;
      uint4 nr = src_r ? __ldg(src_r) : zero;
      uint4 ni = src_i ? __ldg(src_i) : zero;
      for (int kb = 0; kb < num_kb; ++kb) {
        const uint4 wr = nr, wi = ni;
        if (kb + 1 < num_kb) {
          nr = src_r ? __ldg(src_r + kb + 1) : zero;
          ni = src_i ? __ldg(src_i + kb + 1) : zero;
        }
        pc_r += __popc(wr.x) + __popc(wr.y) + __popc(wr.z) + __popc(wr.w);
        pc_i += __popc(wi.x) + __popc(wi.y) + __popc(wi.z) + __popc(wi.w);
        mbar_wait(&empty_bar[stage], phase ^ 1);
        uint8_t* st = smem + stage * STAGE_BYTES;
        if (a_side) {
          uint8_t* ar = st + row * 128;
          uint8_t* ai = st + A_TILE + row * 128;
          expand_word(ar, row, 0, wr.x); expand_word(ar, row, 1, wr.y);
          expand_word(ar, row, 2, wr.z); expand_word(ar, row, 3, wr.w);
          expand_word(ai, row, 0, wi.x); expand_word(ai, row, 1, wi.y);
          expand_word(ai, row, 2, wi.z); expand_word(ai, row, 3, wi.w);
        } else {
          uint8_t* br = st + 2 * A_TILE + row * 128;
          uint8_t* bi = br + B_TILE;
          uint8_t* bc = bi + B_TILE;
          expand_word(br, row, 0, wr.x); expand_word(br, row, 1, wr.y);
          expand_word(br, row, 2, wr.z); expand_word(br, row, 3, wr.w);
          expand_word_pair(bi, bc, row, 0, wi.x); expand_word_pair(bi, bc, row, 1, wi.y);
          expand_word_pair(bi, bc, row, 2, wi.z); expand_word_pair(bi, bc, row, 3, wi.w);
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(full_leader0 + stage * 8);  // the leader's full barrier
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      // correction terms (R1b): rows -> local; the 64 columns of this half -> both CTAs
      const int cb = it & 1;
      mbar_wait(&sempty_bar[cb], ((it >> 1) & 1) ^ 1);
      if (a_side) {
        terms[(cb * 3 + 0) * 128 + row] = -2 * (pc_r + pc_i);
      } else {
        const int col = (int)rank * BH + row;
        const int tre = 2 * (pc_i - pc_r), tim = 2 * p.K - 2 * (pc_r + pc_i);
        terms[(cb * 3 + 1) * 128 + col] = tre;
        terms[(cb * 3 + 2) * 128 + col] = tim;
        st_cluster_s32(terms_peer + ((cb * 3 + 1) * 128 + col) * 4, tre);
        st_cluster_s32(terms_peer + ((cb * 3 + 2) * 128 + col) * 4, tim);
      }
      __syncwarp();
      if (lane == 0) {
        mbar_arrive_cluster(mapa_shared(&sfull_bar[cb], rank));
        if (!a_side) mbar_arrive_cluster(sfull_peer[cb]);
      }
    }
  }

  tc_fence_before();
  cluster_sync();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS)
                 : "memory");
  }
}

template <bool TMA_STORE>
cudaError_t launch2(const CUtensorMap& tmC, const GemmB1Args& a, int num_sms, cudaStream_t s) {
  auto kern = cgemm_b1_2cta_kernel<TMA_STORE>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
  if (e != cudaSuccess) return e;
  const int tiles_m = (a.M + 255) / 256, tiles_n = (a.N + BN - 1) / BN;
  const long long nt = (long long)tiles_m * tiles_n * a.B;
  if (nt > 0x7fffffffLL) return cudaErrorInvalidValue;
  const int pairs = (int)(nt < num_sms / 2 ? nt : num_sms / 2);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(NUM_THREADS);
  cfg.dynamicSmemBytes = SMEM_BYTES;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, kern, tmC, a, tiles_m, tiles_n, (int)nt);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_gemm_b1_2cta(const CUtensorMap& tmC, const GemmB1Args& args, bool tma_store, int num_sms,
                                cudaStream_t stream) {
  return tma_store ? launch2<true>(tmC, args, num_sms, stream) : launch2<false>(tmC, args, num_sms, stream);
}

}  // namespace tcbf
