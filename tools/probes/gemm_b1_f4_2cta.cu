// gemm_b1_f4_2cta.cu -- 1-bit-mode complex beamformer GEMM on the fp4 tensor cores with CTA pairs
// (tcgen05.mma.cta_group::2.kind::mxf4).
//
// Same method as gemm_b1_f4.cu (sign bits expanded in shared memory to +-1 e2m1 nibbles, unit
// block scales, [D_r | D_i] += A_r [B_r ; B_i] + A_i [-B_i ; B_r], Im - 2 K_pad -- PAPER.md:143-159,
// 170-172, 249-259, reading R1c), but a 2-CTA cluster computes a 256-beam x 128-sample tile with
// M = 256 MMAs.  The N = 256 stacked data operand is split between the pair by rows:
//     [B_r ; B_i]   -> CTA 0 holds B_r,  CTA 1 holds B_i   (tile T0, same smem offset)
//     [-B_i ; B_r]  -> CTA 0 holds -B_i, CTA 1 holds B_r   (tile T1)
// so each CTA expands its own 128 weight rows (A_r, A_i) and TWO data tiles instead of three, and
// each MMA reads 8 KB of its CTA's shared memory per 128 x 256 x 64 share instead of 12 KB: ~20%
// less shared-memory traffic per useful op, which bounds the 1-CTA kernel on compute-bound shapes
// (DESIGN.md §4).  TMEM per CTA: its 128 rows of [D_r | D_i] (256 columns) + unit scale factors.
//
// Roles (per CTA, 544 threads): warp 0 TMEM allocator + (leader) single-thread MMA issuer;
// warps 1-8 epilogue (tcgen05.ld, fp32 -> int32, Im - 2 K_pad, 32 x 32 TMA store boxes);
// warps 9-16 expanders (threads 0-127: weight rows, 128-255: data columns), packed words loaded two
// K blocks ahead in registers.  The leader's full barrier counts both CTAs' expander warps; its
// commits are multicast to both CTAs' empty / tile-full barriers; both CTAs' epilogues release TMEM
// on the leader's tile-empty barrier.
//
// MEASURED SLOWER than the 1-CTA kernel (square 8192^3: 1.33 vs 0.82 ms; radio 1-bit 2.23 vs 1.60 ms),
// so it is opt-in (TCBF_B1_KERNEL=f4pair): with MMAs and expansion both skipped (TCBF_DEBUG=6) the
// pair's skeleton -- register look-ahead word loads plus the per-K-block cluster barrier round trip
// -- already takes 1.05 ms against 0.44 ms for the 1-CTA kernel's TMA-fed skeleton; a third stage
// made it slower (1.60 ms); without word loads (TCBF_DEBUG bit 3) the full pipeline still takes 0.92 ms.
// Bit-exact (tests/test_gpu_parity.py, b1_kernel = f4pair).
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "kernels.h"
#include "ptx.cuh"

namespace tcbf {
namespace {

constexpr int BN = 128;                  // data columns per pair tile (complex)
constexpr int KBW = 8;                   // 256 bits per K block -> 128 bytes of nibbles per row
constexpr int TILE_BYTES = 128 * 128;    // one expanded operand tile
constexpr int STAGES = 2;
constexpr int STAGE_BYTES = 4 * TILE_BYTES;  // A_r, A_i, T0, T1
constexpr int EPI_WARPS = 8;
constexpr int EXP_WARP0 = 1 + EPI_WARPS;
constexpr int EXPANDER_WARPS = 8;
constexpr int NUM_THREADS = (EXP_WARP0 + EXPANDER_WARPS) * 32;
constexpr int EPI_BOX = 32 * 32 * 4;
constexpr int EPI_OFFSET = STAGES * STAGE_BYTES;
constexpr int EPI_BYTES = EPI_WARPS * 2 * EPI_BOX;
constexpr int BAR_OFFSET = EPI_OFFSET + EPI_BYTES;
constexpr int SMEM_BYTES = 1024 + BAR_OFFSET + 256;
constexpr uint32_t TMEM_COLS = 512;
constexpr uint32_t SF_COL = 256;
constexpr int REG_PF = 2;
static_assert(SMEM_BYTES <= 232448, "smem budget");

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
__device__ __forceinline__ void mma_mxf4_2sm(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                             uint32_t sfa, uint32_t sfb, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t}" ::"r"(
          d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(sfa), "r"(sfb)
      : "memory");
}
__device__ __forceinline__ void mma_commit_2sm_mc(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}" ::"r"(
          smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tmem_st_32x32b_x32_same(uint32_t taddr, uint32_t v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, "
      "%1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1};" ::"r"(taddr),
      "r"(v)
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// output word j (4 per packed word) of the +-1 e2m1 expansion: nibble i <- bit (4i + j)
template <int J>
__device__ __forceinline__ uint32_t nib_pm1(uint32_t w) {
  return ((w << (3 - J)) & 0x88888888u) ^ 0xAAAAAAAAu;  // bit 1 -> 0x2 (+1), bit 0 -> 0xA (-1)
}
template <int J>
__device__ __forceinline__ uint32_t nib_neg(uint32_t w) {
  return ((w << (3 - J)) & 0x88888888u) ^ 0x22222222u;  // bit 1 -> 0xA (-1), bit 0 -> 0x2 (+1)
}
template <bool NEG>
__device__ __forceinline__ void expand(uint8_t* row_base, int row, const uint4& lo, const uint4& hi) {
  const uint32_t w[KBW] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
#pragma unroll
  for (int q = 0; q < KBW; ++q) {
    const uint4 v = NEG ? make_uint4(nib_neg<0>(w[q]), nib_neg<1>(w[q]), nib_neg<2>(w[q]), nib_neg<3>(w[q]))
                        : make_uint4(nib_pm1<0>(w[q]), nib_pm1<1>(w[q]), nib_pm1<2>(w[q]), nib_pm1<3>(w[q]));
    *reinterpret_cast<uint4*>(row_base + ((q ^ (row & 7)) << 4)) = v;  // 128-byte swizzle
  }
}

template <bool TMA_STORE>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    cgemm_b1_f4_2cta_kernel(const __grid_constant__ CUtensorMap tmC, GemmB1Args p, int tiles_m, int tiles_n,
                            int num_tiles) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* epi_base = smem + EPI_OFFSET;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + BAR_OFFSET);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull_bar = empty_bar + STAGES;
  uint64_t* tempty_bar = tfull_bar + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1;
  const int npairs = gridDim.x >> 1;
  const int num_kb = p.Kw / KBW;
  const int two_kpad = 2 * (32 * p.Kw - p.K);

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 2 * EXPANDER_WARPS);  // (leader's) both CTAs' expander warps
      mbar_init(&empty_bar[s], 1);
    }
    mbar_init(tfull_bar, 1);
    mbar_init(tempty_bar, 2 * EPI_WARPS);           // (leader's) both CTAs' epilogue warps
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
  if (warp >= 1 && warp <= 4) {  // unit block scales in this CTA's TMEM: columns 256..511 = 0x7F
    const uint32_t lanes = (uint32_t)((warp & 3) * 32) << 16;
#pragma unroll
    for (uint32_t c = SF_COL; c < TMEM_COLS; c += 32) tmem_st_32x32b_x32_same(tmem_base + lanes + c, 0x7F7F7F7Fu);
    tmem_wait_st();
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();

  if (warp == 0) {
    // ------------------------------------------------------------ MMA issuer (leader)
    if (leader && lane == 0) {
      // kind::mxf4 block32: A, B e2m1, UE8M0 scales, fp32 D, K-major, M = 256 (pair), N = 256
      constexpr uint32_t IDESC = (1u << 7) | (1u << 10) | ((uint32_t)((2 * BN) >> 3) << 17) | (1u << 23) |
                                 ((uint32_t)(256 >> 4) << 24);
      const uint32_t sfa = tmem_base + SF_COL, sfb = tmem_base + SF_COL + 128;
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = pair; t < num_tiles; t += npairs, ++it) {
        mbar_wait_cluster(tempty_bar, (it & 1) ^ 1);
        tc_fence_after();
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait_cluster(&full_bar[stage], phase);
          tc_fence_after();
          uint8_t* st = smem + stage * STAGE_BYTES;
#pragma unroll
          for (int kk = 0; kk < KBW / 2; ++kk) {  // K = 64 elements (32 bytes) per MMA
            const uint32_t off = kk * 32;
            const uint64_t ar = smem_desc_k128(st, off), ai = smem_desc_k128(st + TILE_BYTES, off);
            const uint64_t t0 = smem_desc_k128(st + 2 * TILE_BYTES, off);  // [B_r ; B_i]
            const uint64_t t1 = smem_desc_k128(st + 3 * TILE_BYTES, off);  // [-B_i ; B_r]
            const uint32_t acc = (kb | kk) ? 1u : 0u;
            if (p.debug & 2) continue;
            mma_mxf4_2sm(tmem_base, ar, t0, IDESC, sfa, sfb, acc);  // [Re(a)Re(b) | Re(a)Im(b)]
            mma_mxf4_2sm(tmem_base, ai, t1, IDESC, sfa, sfb, 1u);   // [-Im(a)Im(b) | Im(a)Re(b)]
          }
          mma_commit_2sm_mc(&empty_bar[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        mma_commit_2sm_mc(tfull_bar);
      }
    }
  } else if (warp <= EPI_WARPS) {
    // ------------------------------------------------------------ epilogue (both CTAs)
    const int q = warp & 3;            // TMEM lane quarter
    const int part = (warp - 1) >> 2;  // 0: Re (columns 0..127), 1: Im (128..255)
    constexpr int CHUNKS = BN / 32;
    uint8_t* bufs = epi_base + (warp - 1) * 2 * EPI_BOX;
    const uint32_t tempty_leader = mapa_shared(tempty_bar, 0);
    int sbuf = 0;
    int it = 0;
    for (int t = pair; t < num_tiles; t += npairs, ++it) {
      int b, mt, nt;
      tile_coords(t, tiles_m, tiles_n, p.group_m, b, mt, nt);
      const int m0 = mt * 256 + (int)rank * 128;
      const int n0 = nt * BN;
      mbar_wait(tfull_bar, it & 1);
      tc_fence_after();
      const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + part * BN;
      const int corr = part == 0 ? 0 : two_kpad;
      uint32_t vbuf[2][32];
      tmem_ld_32x32b_x32(tbase, vbuf[0]);
#pragma unroll
      for (int c = 0; c < CHUNKS; ++c) {
        tmem_wait_ld();
        if (c + 1 < CHUNKS) {
          tmem_ld_32x32b_x32(tbase + (c + 1) * 32, vbuf[(c + 1) & 1]);
        } else {  // all TMEM reads of this warp done: the pair's next MMAs may start
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(tempty_leader);
        }
        uint32_t* vv = vbuf[c & 1];
#pragma unroll
        for (int j = 0; j < 32; ++j) vv[j] = (uint32_t)(__float2int_rn(__uint_as_float(vv[j])) - corr);
        if (p.debug & 1) continue;
        if constexpr (TMA_STORE) {  // 32 x 32 boxes, 128-byte swizzle, double-buffered per warp
          uint8_t* buf = bufs + sbuf * EPI_BOX;
          if (lane == 0) bulk_wait_group_read<1>();
          __syncwarp();
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int pos = j ^ (lane & 7);
            *reinterpret_cast<uint4*>(buf + lane * 128 + pos * 16) =
                make_uint4(vv[4 * j], vv[4 * j + 1], vv[4 * j + 2], vv[4 * j + 3]);
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
              if (n < p.N) rowp[n] = (int32_t)vv[j];
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
    const int e = threadIdx.x - EXP_WARP0 * 32;  // 0..255
    const bool a_side = e < 128;
    const int row = a_side ? e : e - 128;
    const uint32_t full_leader0 = mapa_shared(&full_bar[0], 0);
    int stage = 0;
    uint32_t phase = 0;
    const uint4 zero = make_uint4(0, 0, 0, 0);
    auto row_ptrs = [&](int t, const uint4*& pr, const uint4*& pi) {
      int b, mt, nt;
      tile_coords(t, tiles_m, tiles_n, p.group_m, b, mt, nt);
      pr = pi = nullptr;
      if (a_side) {
        const int m = mt * 256 + (int)rank * 128 + row;
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
    // the thread's K blocks over all its tiles form one flat stream, loaded REG_PF blocks ahead
    int lt = pair, lkb = 0;
    const uint4* lr = nullptr;
    const uint4* li = nullptr;
    if (lt < num_tiles) row_ptrs(lt, lr, li);
    auto load_next = [&](uint4 (&d)[4]) {
      const bool ok = lr != nullptr && !(p.debug & 8);  // ablation bit 3: no word loads
      d[0] = ok ? __ldg(lr + 2 * lkb) : zero;
      d[1] = ok ? __ldg(lr + 2 * lkb + 1) : zero;
      d[2] = ok ? __ldg(li + 2 * lkb) : zero;
      d[3] = ok ? __ldg(li + 2 * lkb + 1) : zero;
      if (++lkb == num_kb) {
        lkb = 0;
        lt += npairs;
        lr = li = nullptr;
        if (lt < num_tiles) row_ptrs(lt, lr, li);
      }
    };
    uint4 ring[REG_PF][4];
#pragma unroll
    for (int u = 0; u < REG_PF; ++u) load_next(ring[u]);
    const int my_tiles = pair < num_tiles ? (num_tiles - 1 - pair) / npairs + 1 : 0;
    const int total = my_tiles * num_kb;
    for (int base = 0; base < total; base += REG_PF) {
#pragma unroll
      for (int u = 0; u < REG_PF; ++u) {
        if (base + u >= total) break;
        const uint4 r0 = ring[u][0], r1 = ring[u][1], i0 = ring[u][2], i1 = ring[u][3];
        load_next(ring[u]);
        mbar_wait(&empty_bar[stage], phase ^ 1);
        uint8_t* st = smem + stage * STAGE_BYTES;
        if (!(p.debug & 4)) {
          if (a_side) {
            expand<false>(st + row * 128, row, r0, r1);               // A_r
            expand<false>(st + TILE_BYTES + row * 128, row, i0, i1);  // A_i
          } else if (rank == 0) {
            expand<false>(st + 2 * TILE_BYTES + row * 128, row, r0, r1);  // T0 = B_r
            expand<true>(st + 3 * TILE_BYTES + row * 128, row, i0, i1);   // T1 = -B_i
          } else {
            expand<false>(st + 2 * TILE_BYTES + row * 128, row, i0, i1);  // T0 = B_i
            expand<false>(st + 3 * TILE_BYTES + row * 128, row, r0, r1);  // T1 = B_r
          }
        }
        fence_proxy_async_smem();  // generic-proxy smem writes -> async proxy (the MMAs)
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(full_leader0 + stage * 8);  // the leader's full barrier
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
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
cudaError_t launch_pair(const CUtensorMap& tmC, const GemmB1Args& a, int num_sms, cudaStream_t s) {
  auto kern = cgemm_b1_f4_2cta_kernel<TMA_STORE>;
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

cudaError_t launch_gemm_b1_f4_2cta(const CUtensorMap& tmC, const GemmB1Args& args, bool tma_store, int num_sms,
                                   cudaStream_t stream) {
  return tma_store ? launch_pair<true>(tmC, args, num_sms, stream) : launch_pair<false>(tmC, args, num_sms, stream);
}

}  // namespace tcbf
