// gram_tc.cu -- 3xTF32 Gram tiles on the 5th-generation tensor cores
// (tcgen05.mma kind::tf32, accumulators in TMEM), the filter stage of the
// certified kNN search (knn.cu).
//
// Each point x is split as x = hi + lo with hi = tf32(x), lo = tf32(x - hi);
// g_ij ~ hi_i.hi_j + hi_i.lo_j + lo_i.hi_j (three MMAs into one fp32
// accumulator), which carries ~fp32 accuracy.  The approximation only
// filters candidates: the neighbour lists are re-ranked with the canonical
// fp64 distance, so results stay bit-exact (see knn.cu).
//
// Tile: 128 query rows x 128 candidate rows per CTA, K staged 32 at a time.
// Shared memory holds K-major operand tiles in the canonical SWIZZLE_NONE
// "core matrix" layout: an 8-row x 16-byte core matrix is 128 contiguous
// bytes; the 8 core matrices of a 32-wide k chunk follow each other (LBO =
// 128 B) and 8-row groups are 1024 B apart (SBO).  One elected thread issues
// the MMAs; tcgen05.commit arrives on an mbarrier that every thread waits on
// before the shared-memory stage is refilled.
#include <math_constants.h>

#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdlib>
#include <string>

#include "common.cuh"

namespace cpcag_cuda {

namespace tc {

constexpr int kM = 128;                 // query rows per tile (UMMA M)
constexpr int kN = 128;                 // candidate rows per tile (UMMA N)
constexpr int kKc = 32;                 // k per stage (one 128-byte row per point)
constexpr int kTileBytes = kM * kKc * 4;  // 16 KiB per operand tile

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// UMMA shared-memory descriptor, K-major, SWIZZLE_NONE.
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo_bytes >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1) << 46;  // descriptor version (sm100)
  // base offset 0, lbo mode 0, layout type 0 (SWIZZLE_NONE)
  return d;
}

// Instruction descriptor: D f32, A/B tf32, both K-major, M x N.
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
         (static_cast<uint32_t>(M >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                   smem_u32(mbar))
               : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(mbar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* mbar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(mbar)),
      "r"(phase)
      : "memory");
}

__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
}

__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(taddr), "r"(ncols) : "memory");
}

// 32 consecutive fp32 columns of this thread's TMEM lane.
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int q = 0; q < 32; ++q) v[q] = __uint_as_float(r[q]);
}

// One column: lane l gets TMEM lane (base lane + l) at column taddr (waits).
__device__ __forceinline__ float tmem_ld1(uint32_t taddr) {
  uint32_t r;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];\n" : "=r"(r) : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
  return __uint_as_float(r);
}

// Split form of tmem_ld32: issue, then wait (tcgen05.wait::ld covers every
// outstanding load of the thread), so the next chunk loads while this one is
// processed.
__device__ __forceinline__ void tmem_ld32_issue(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }

// Copies rows [row0, row0 + 128) x k [k0, k0 + 32) of a point-major fp32
// matrix (leading dimension ld, rows >= nrows read as zero) into the core
// matrix layout at dst.  128 threads, 16-byte chunks.
__device__ __forceinline__ void stage_tile(unsigned char* dst, const float* __restrict__ src, i64 ld, i64 nrows,
                                           i64 row0, i64 k0) {
#pragma unroll
  for (int q = 0; q < (kM * 8) / 128; ++q) {
    const int id = threadIdx.x + 128 * q;
    const int r = id >> 3, kc = id & 7;
    const i64 gr = row0 + r;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (gr < nrows) v = *reinterpret_cast<const float4*>(src + gr * ld + k0 + kc * 4);
    *reinterpret_cast<float4*>(dst + ((r >> 3) * 8 + kc) * 128 + (r & 7) * 16) = v;
  }
}

}  // namespace tc

// G(i, j) for a 128 x 128 tile: 3xTF32 Gram of points i (rows of H/L) and j.
// H, L: n x dp fp32 point-major (dp multiple of 32).  G row-major n x n.
__global__ void __launch_bounds__(128) gram_tf32x3_k(const float* __restrict__ H, const float* __restrict__ L, i64 n,
                                                     i64 dp, float* __restrict__ G) {
  using namespace tc;
  extern __shared__ __align__(1024) unsigned char smem[];
  unsigned char* Ah = smem;
  unsigned char* Al = smem + kTileBytes;
  unsigned char* Bh = smem + 2 * kTileBytes;
  unsigned char* Bl = smem + 3 * kTileBytes;
  __shared__ uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const i64 i0 = static_cast<i64>(blockIdx.x) * kM, j0 = static_cast<i64>(blockIdx.y) * kN;
  if (warp == 0) tmem_alloc(&tmem_base, kN);
  if (threadIdx.x == 0) {
    mbar_init(&mbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = tmem_base;
  constexpr uint32_t idesc = idesc_tf32(kM, kN);
  uint32_t phase = 0;
  for (i64 k0 = 0; k0 < dp; k0 += kKc) {
    stage_tile(Ah, H, dp, n, i0, k0);
    stage_tile(Al, L, dp, n, i0, k0);
    stage_tile(Bh, H, dp, n, j0, k0);
    stage_tile(Bl, L, dp, n, j0, k0);
    fence_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
      fence_after();
      const uint32_t ah = smem_u32(Ah), al = smem_u32(Al), bh = smem_u32(Bh), bl = smem_u32(Bl);
#pragma unroll
      for (int kk = 0; kk < kKc / 8; ++kk) {
        const uint32_t off = kk * 256;  // two core matrices (8 tf32) per MMA
        const uint32_t acc = (k0 > 0 || kk > 0) ? 1u : 0u;
        mma_tf32(tmem, umma_desc(ah + off, 128, 1024), umma_desc(bh + off, 128, 1024), idesc, acc);
        mma_tf32(tmem, umma_desc(ah + off, 128, 1024), umma_desc(bl + off, 128, 1024), idesc, 1u);
        mma_tf32(tmem, umma_desc(al + off, 128, 1024), umma_desc(bh + off, 128, 1024), idesc, 1u);
      }
      mma_commit(&mbar);
    }
    mbar_wait(&mbar, phase);
    phase ^= 1u;
    fence_after();
  }
  // Epilogue: warp w owns TMEM lanes [32w, 32w + 32) = rows i0 + 32w + lane.
  const i64 gi = i0 + 32 * warp + lane;
#pragma unroll 1
  for (int c0 = 0; c0 < kN; c0 += 32) {
    float v[32];
    tmem_ld32(tmem + (static_cast<uint32_t>(32 * warp) << 16) + c0, v);
    if (gi < n)
#pragma unroll
      for (int q = 0; q < 32; ++q) {
        const i64 gj = j0 + c0 + q;
        if (gj < n) G[gi * n + gj] = v[q];
      }
  }
  fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, kN);
}

// ------------------------------------------------------------------ pipelined filter (TMA + warp roles)
// The certified filter on the tensor cores, Blackwell-style:
//   warp 0    TMA producer: 2D tensor loads (SWIZZLE_128B, one 32-float k
//             chunk = one 128-byte row per point) of A-hi, A-lo, B-hi, B-lo
//             into a 3-stage ring, full/empty mbarriers;
//   warp 1    MMA issuer: 3 tcgen05.mma kind::tf32 per k8 step into one of
//             two TMEM accumulators (2 x 128 columns), commit -> empty[stage]
//             and, after the last k chunk, -> tmem_full[acc];
//   warps 2-5 epilogue (TMEM lane quarter w % 4 = 32 query rows each):
//             distances + top-kCand insertion for tile t while the MMAs of
//             tile t+1 run; arrive tmem_empty[acc].
namespace tc2 {
constexpr int kTile = 128 * 32 * 4;        // 16 KiB: 128 rows x 128 B (an A plane chunk)
constexpr int kThreads = 192;

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* mbar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(tc::smem_u32(mbar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* mbar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(tc::smem_u32(mbar)) : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* mbar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          tc::smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(tc::smem_u32(mbar))
      : "memory");
}
// mbarrier wait with a watchdog: a pipeline that never completes (a bad
// descriptor, a lost transaction) traps after ~10 s instead of hanging.
__device__ __forceinline__ void mbar_wait_guarded(uint64_t* mbar, uint32_t phase) {
  uint32_t done = 0;
  unsigned long long t0 = 0;
  for (uint32_t spin = 0;; ++spin) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}\n"
        : "=r"(done)
        : "r"(tc::smem_u32(mbar)), "r"(phase)
        : "memory");
    if (done) return;
    if ((spin & 1023u) == 0u) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
      if (t0 == 0) t0 = t;
      else if (t - t0 > 10000000000ull) asm volatile("trap;");
    }
  }
}
// TMA 2D load with an L2 cache policy (createpolicy): the query block A is
// re-read once per candidate tile and must survive in L2 (evict_last); the
// candidate stream B is consumed by the concurrently running CTAs within a
// short window (evict_first), so it must not push A out.
__device__ __forceinline__ void tma_load_2d_hint(void* dst, const CUtensorMap* map, uint64_t* mbar, int c0, int c1,
                                                 uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3}], "
      "[%4], %5;\n" ::"r"(tc::smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(tc::smem_u32(mbar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
// K-major SWIZZLE_128B operand: rows of 128 B, 8-row atoms 1024 B apart.
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>(1) << 16;            // LBO (unused for swizzled K-major)
  d |= static_cast<uint64_t>(1024 >> 4) << 32;    // SBO
  d |= static_cast<uint64_t>(1) << 46;            // sm100 descriptor version
  d |= static_cast<uint64_t>(2) << 61;            // SWIZZLE_128B
  return d;
}
}  // namespace tc2

// NT = candidate rows per tile (UMMA N): 128 (3-stage ring of 64 KiB) or
// 256 (2-stage ring of 96 KiB; each A chunk then serves twice the
// candidates, 65 instead of 48 flops per staged byte).
//
// KC = candidates kept per query (32: first pass over every point, 3-stage
// ring; 64: second pass over the queries the first pass could not certify,
// 2-stage ring so the longer lists fit).  qidx (null = identity) maps the
// nq query rows of mapH / mapL to point indices; outputs are indexed by
// query row: cand[(split * nq + q) * KC + rank].
template <int NT, int KC = 32>
__global__ void __launch_bounds__(tc2::kThreads, 1)
    knn_tc_filter2_k(const __grid_constant__ CUtensorMap mapH, const __grid_constant__ CUtensorMap mapL,
                     const __grid_constant__ CUtensorMap mapHb, const __grid_constant__ CUtensorMap mapLb,
                     const double* __restrict__ sq, i64 n, i64 dp, int tiles_per_split, float* __restrict__ cand_d,
                     int* __restrict__ cand_j, const unsigned long long* __restrict__ max_norm_bits, int stagger,
                     int dbg, const int* __restrict__ qidx, i64 nq) {
  using namespace tc;
  using tc2::kTile;
  using tc2::kThreads;
  using tc2::mbar_wait_guarded;
  using tc2::mbar_arrive_expect_tx;
  using tc2::mbar_arrive;
  using tc2::tma_load_2d_hint;
  using tc2::policy_evict_last;
  using tc2::policy_evict_first;
  using tc2::desc_sw128;
  constexpr int kN = NT;
  constexpr int kBTile = NT * 128;                   // NT rows x 128 B
  constexpr int kStageBytes = 2 * kTile + 2 * kBTile;
  constexpr int kStages = (NT == 128 && KC == 32) ? 3 : 2;
  constexpr int kCand = KC;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // SWIZZLE_128B needs 1024-byte aligned stages; the dynamic window is
  // declared so (no slack is reserved: the 3-stage ring plus the lists fill
  // the 227 KB), checked here once.
  unsigned char* smem = smem_raw;
  if ((smem_u32(smem_raw) & 1023u) != 0u) asm volatile("trap;");
  float* lst_d = reinterpret_cast<float*>(smem + kStages * kStageBytes);  // [kCand][128]
  int* lst_j = reinterpret_cast<int*>(lst_d + kCand * kM);                // [kCand][128]
  __shared__ uint64_t full[kStages], empty[kStages], tfull[2], tempty[2];
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const i64 i0 = static_cast<i64>(blockIdx.x) * kM;
  const i64 n_tiles = (n + kN - 1) / kN;
  const i64 jt0 = static_cast<i64>(blockIdx.y) * tiles_per_split;
  const i64 jt1 = min(n_tiles, jt0 + tiles_per_split);
  const int nkc = static_cast<int>(dp / kKc);
  if (warp == 1) tmem_alloc(&tmem_base, 2 * kN);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp >= 2) {
    const int r = (warp & 3) * 32 + lane;
    for (int q = 0; q < kCand; ++q) {
      lst_d[q * kM + r] = CUDART_INF_F;
      lst_j[q * kM + r] = INT32_MAX;
    }
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = tmem_base;
  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer
      int stage = 0;
      uint32_t phase = 0;
      const uint64_t keep = policy_evict_last(), stream = policy_evict_first();
      for (i64 jt = jt0; jt < jt1; ++jt) {
        const int j0 = static_cast<int>(jt * kN);
        for (int kq = 0; kq < nkc; ++kq) {
          const int kc = stagger ? (kq + static_cast<int>(blockIdx.x)) % nkc : kq;
          mbar_wait_guarded(&empty[stage], phase ^ 1u);
          unsigned char* st = smem + stage * kStageBytes;
          mbar_arrive_expect_tx(&full[stage], kStageBytes);
          tma_load_2d_hint(st, &mapH, &full[stage], kc * kKc, static_cast<int>(i0), keep);
          tma_load_2d_hint(st + kTile, &mapL, &full[stage], kc * kKc, static_cast<int>(i0), keep);
          tma_load_2d_hint(st + 2 * kTile, &mapHb, &full[stage], kc * kKc, j0, stream);
          tma_load_2d_hint(st + 2 * kTile + kBTile, &mapLb, &full[stage], kc * kKc, j0, stream);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer
      constexpr uint32_t idesc = idesc_tf32(kM, kN);
      int stage = 0, acc = 0;
      uint32_t phase = 0, aphase = 0;
      for (i64 jt = jt0; jt < jt1; ++jt) {
        mbar_wait_guarded(&tempty[acc], aphase ^ 1u);
        fence_after();
        const uint32_t d = tmem + static_cast<uint32_t>(acc * kN);
        for (int kc = 0; kc < nkc; ++kc) {  // order of the chunks is the producer's; accumulate from the 2nd
          mbar_wait_guarded(&full[stage], phase);
          fence_after();
          const uint32_t ah = smem_u32(smem + stage * kStageBytes);
          const uint32_t al = ah + kTile, bh = ah + 2 * kTile, bl = ah + 2 * kTile + kBTile;
#pragma unroll
          for (int kk = 0; kk < (dbg == 2 ? 0 : kKc / 8); ++kk) {
            const uint32_t off = kk * 32;  // 8 tf32 = 32 bytes along the swizzled row
            const uint32_t accum = (kc > 0 || kk > 0) ? 1u : 0u;
            mma_tf32(d, desc_sw128(ah + off), desc_sw128(bh + off), idesc, accum);
            mma_tf32(d, desc_sw128(ah + off), desc_sw128(bl + off), idesc, 1u);
            mma_tf32(d, desc_sw128(al + off), desc_sw128(bh + off), idesc, 1u);
          }
          mma_commit(&empty[stage]);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1u;
          }
        }
        mma_commit(&tfull[acc]);
        acc ^= 1;
        if (acc == 0) aphase ^= 1u;
      }
    }
  } else {  // ---- epilogue warps 2..5: TMEM lanes [32 (w % 4), +32)
    const int eq = warp & 3;
    const int r = eq * 32 + lane;
    const i64 qr = i0 + r;            // query row
    const bool qv = qr < nq;
    const i64 gi = qv ? (qidx ? static_cast<i64>(qidx[qr]) : qr) : n;  // its point (n = none)
    const double sqi = qv ? sq[gi] : 0.0;
    const float sqi_f = static_cast<float>(sqi);
    // Quick reject in fp32.  The exact test below is df < thr with
    // df = fp32((sq_i + sq_j) - 2 g) evaluated in fp64.  The fp32 estimate
    // e = fma(-2, g, fp32(sq_i) + fp32(sq_j)) differs from it by at most
    // 4 * 2^-24 (sq_i + sq_j + 2|g|) plus df's own rounding, and
    // |g| <= (sq_i + sq_j) / 2 (1 + the filter's relative error), so
    // |e - df| < 2^-20 (sq_i + max sq): a candidate skipped here has df >=
    // thr and the exact test would skip it too.
    const double mxn = __longlong_as_double(static_cast<long long>(*max_norm_bits));
    const float margin = static_cast<float>(0x1.0p-20 * (sqi + mxn * mxn)) * 1.0001f;
    float thr = CUDART_INF_F;  // largest d in the (unsorted) list
    int maxpos = 0;            // its slot
    int acc = 0;
    uint32_t aphase = 0;
    static_assert(NT == 128, "four candidate norms per lane");
    // Candidate norms live in registers: lane l holds columns l + 32 k of the
    // tile (fetched one tile ahead) and the warp reads them by shuffle, so the
    // four epilogue warps never wait on one another.
    auto norm_of = [&](i64 jt, int k) -> double {
      const i64 gj = jt * kN + lane + 32 * k;
      return jt < jt1 && gj < n ? __ldg(sq + gj) : CUDART_INF;
    };
    double nd[4], nx[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) nx[k] = norm_of(jt0, k);
    for (i64 jt = jt0; jt < jt1; ++jt) {
      const i64 j0 = jt * kN;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        nd[k] = nx[k];
        nx[k] = norm_of(jt + 1, k);
      }
      mbar_wait_guarded(&tfull[acc], aphase);
      fence_after();
      const uint32_t tbase = tmem + (static_cast<uint32_t>(32 * eq) << 16) + static_cast<uint32_t>(acc * kN);
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        const int c0 = 32 * cc;
        float v[32];
        tmem_ld32(tbase + static_cast<uint32_t>(c0), v);
        // fast path: one bit per column whose fp32 estimate passes the
        // quick reject (a superset of what the exact test below accepts)
        const float nf = static_cast<float>(nd[cc]);
        const float lim = thr + margin;
        unsigned m = 0;
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          const float e = fmaf(-2.0f, v[q], sqi_f + __shfl_sync(0xffffffffu, nf, q));
          m |= (e <= lim ? 1u : 0u) << q;
        }
        if (!qv || dbg == 1) m = 0;
        // slow path, warp-uniform and not unrolled: columns any lane kept, in
        // ascending order (the order the lists are built in)
        unsigned wm = __reduce_or_sync(0xffffffffu, m);
        while (wm) {
          const int q = __ffs(wm) - 1;
          wm &= wm - 1u;
          const float vq = tmem_ld1(tbase + static_cast<uint32_t>(c0 + q));
          const double sqj = __shfl_sync(0xffffffffu, nd[cc], q);
          const i64 gj = j0 + c0 + q;
          if (((m >> q) & 1u) && gj < n && gj != gi) {
            const double dd = (sqi + sqj) - 2.0 * static_cast<double>(vq);
            const float df = static_cast<float>(dd);
            if (df < thr) {
              // the list is unsorted: the candidate replaces the
              // lexicographic (d, j) maximum, then the maximum is found again
              // (independent loads, no shifting chain).  Candidates arrive in
              // increasing j, so this keeps exactly the (d, j)-smallest kCand.
              lst_d[maxpos * kM + r] = df;
              lst_j[maxpos * kM + r] = static_cast<int>(gj);
              float bd = lst_d[r];
              int bj = lst_j[r], bp = 0;
#pragma unroll 8
              for (int t = 1; t < kCand; ++t) {
                const float td = lst_d[t * kM + r];
                const int tj = lst_j[t * kM + r];
                if (td > bd || (td == bd && tj > bj)) {
                  bd = td;
                  bj = tj;
                  bp = t;
                }
              }
              thr = bd;
              maxpos = bp;
            }
          }
        }
      }
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      acc ^= 1;
      if (acc == 0) aphase ^= 1u;
    }
    if (qv) {
      // sort the row's list by (d, j) once (insertion sort in place)
      for (int t = 1; t < kCand; ++t) {
        const float dv = lst_d[t * kM + r];
        const int jv = lst_j[t * kM + r];
        int pos = t;
        while (pos > 0) {
          const float pd = lst_d[(pos - 1) * kM + r];
          const int pj = lst_j[(pos - 1) * kM + r];
          if (pd < dv || (pd == dv && pj < jv)) break;
          lst_d[pos * kM + r] = pd;
          lst_j[pos * kM + r] = pj;
          --pos;
        }
        lst_d[pos * kM + r] = dv;
        lst_j[pos * kM + r] = jv;
      }
      float* od = cand_d + (static_cast<i64>(blockIdx.y) * nq + qr) * kCand;
      int* oj = cand_j + (static_cast<i64>(blockIdx.y) * nq + qr) * kCand;
      for (int q = 0; q < kCand; ++q) {
        od[q] = lst_d[q * kM + r];
        oj[q] = lst_j[q * kM + r];
      }
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 2 * kN);
}

size_t knn_tc2_smem(int nt, int kc = 32) {
  const size_t stage = 2 * static_cast<size_t>(tc2::kTile) + 2 * static_cast<size_t>(nt) * 128;
  const size_t stages = (nt == 128 && kc == 32) ? 3 : 2;
  return stages * stage + static_cast<size_t>(kc) * tc::kM * (sizeof(float) + sizeof(int));
}

namespace {
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    CUDA_OK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !p) fail(CPCAG_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// n x dp fp32 point-major matrix, boxes of 128 points x 32 floats (128 B),
// 128-byte swizzle; rows past n read as zero.
CUtensorMap point_map(const float* base, i64 n, i64 dp, int box_rows = 128) {
  CUtensorMap m;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(dp), static_cast<cuuint64_t>(n)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(dp) * sizeof(float)};
  cuuint32_t box[2] = {32, static_cast<cuuint32_t>(box_rows)};
  cuuint32_t es[2] = {1, 1};
  const CUresult r = tensor_map_encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims,
                                          strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(CPCAG_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(r)) + ")");
  return m;
}
}  // namespace

void knn_tc_filter2(Ctx* c, const float* H, const float* L, const double* sq, i64 n, i64 dp, i64 q_tiles, i64 splits,
                    i64 /*tps128*/, float* cd, int* cj, const unsigned long long* max_norm_bits) {
  if (n > INT32_MAX || dp > INT32_MAX) invalid("knn: tensor-core filter size out of range");
  const int nt = 128;  // 256-wide tiles measured no faster and do not fit the norm staging
  const int stagger = 1, dbg = 0;
  const i64 nt_tiles = (n + nt - 1) / nt;
  const i64 tps = (nt_tiles + splits - 1) / splits;  // splits keep the caller's output layout
  const CUtensorMap mh = point_map(H, n, dp), ml = point_map(L, n, dp);
  const CUtensorMap mhb = point_map(H, n, dp, nt), mlb = point_map(L, n, dp, nt);
  const size_t smem = knn_tc2_smem(nt);
  const dim3 grid(static_cast<unsigned>(q_tiles), static_cast<unsigned>(splits));
  ensure_smem(knn_tc_filter2_k<128, 32>, smem);
  knn_tc_filter2_k<128, 32><<<grid, tc2::kThreads, smem, c->stream>>>(mh, ml, mhb, mlb, sq, n, dp, static_cast<int>(tps),
                                                                       cd, cj, max_norm_bits, stagger, dbg, nullptr, n);
  launched(c);
}

// Second pass: the nq queries Hq / Lq (rows qidx of H / L, gathered) against
// every point with 64-candidate lists.
void knn_tc_filter2_rows(Ctx* c, const float* Hq, const float* Lq, const int* qidx, i64 nq, const float* H,
                         const float* L, const double* sq, i64 n, i64 dp, i64 splits, float* cd, int* cj,
                         const unsigned long long* max_norm_bits) {
  if (n > INT32_MAX || dp > INT32_MAX || nq > INT32_MAX) invalid("knn: tensor-core filter size out of range");
  const int nt = 128;
  const i64 nt_tiles = (n + nt - 1) / nt;
  const i64 tps = (nt_tiles + splits - 1) / splits;
  const CUtensorMap mh = point_map(Hq, nq, dp), ml = point_map(Lq, nq, dp);
  const CUtensorMap mhb = point_map(H, n, dp, nt), mlb = point_map(L, n, dp, nt);
  const size_t smem = knn_tc2_smem(nt, 64);
  const dim3 grid(static_cast<unsigned>((nq + 127) / 128), static_cast<unsigned>(splits));
  ensure_smem(knn_tc_filter2_k<128, 64>, smem);
  knn_tc_filter2_k<128, 64><<<grid, tc2::kThreads, smem, c->stream>>>(mh, ml, mhb, mlb, sq, n, dp, static_cast<int>(tps),
                                                                       cd, cj, max_norm_bits, 1, 0, qidx, nq);
  launched(c);
}

// Hq[q] = H[qidx[q]], Lq[q] = L[qidx[q]] (dp floats per row).
__global__ void gather_rows_k(const float* __restrict__ H, const float* __restrict__ L, const int* __restrict__ qidx,
                              i64 nq, i64 dp, float* __restrict__ Hq, float* __restrict__ Lq) {
  const i64 t = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (t >= nq * dp) return;
  const i64 q = t / dp, k = t - q * dp;
  const i64 src = static_cast<i64>(qidx[q]) * dp + k;
  Hq[t] = H[src];
  Lq[t] = L[src];
}

void gather_point_rows(Ctx* c, const float* H, const float* L, const int* qidx, i64 nq, i64 dp, float* Hq, float* Lq) {
  if (nq == 0) return;
  gather_rows_k<<<blocks_for(nq * dp), kBlock, 0, c->stream>>>(H, L, qidx, nq, dp, Hq, Lq);
  launched(c);
}

// hi = tf32(x) (round to nearest), lo = tf32(x - hi); rows padded to dp.
__global__ void split_tf32_k(const double* __restrict__ Pm, i64 n, i64 d, i64 dp, float* __restrict__ H,
                             float* __restrict__ L) {
  const i64 t = blockIdx.x * (i64)blockDim.x + threadIdx.x;
  if (t >= n * dp) return;
  const i64 i = t / dp, k = t % dp;
  float h = 0.f, l = 0.f;
  if (k < d) {
    const float x = static_cast<float>(Pm[i * d + k]);
    uint32_t hb, lb;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hb) : "f"(x));
    h = __uint_as_float(hb);
    const float r = x - h;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(lb) : "f"(r));
    l = __uint_as_float(lb);
  }
  H[t] = h;
  L[t] = l;
}

size_t gram_tc_smem() { return 4 * static_cast<size_t>(tc::kTileBytes); }

// H/L split of point-major fp64 points (n x d) into padded fp32 arrays.
void split_points(Ctx* c, const double* Pm, i64 n, i64 d, i64 dp, float* H, float* L) {
  split_tf32_k<<<blocks_for(std::max<i64>(n * dp, 1)), kBlock, 0, c->stream>>>(Pm, n, d, dp, H, L);
  launched(c);
}

}  // namespace cpcag_cuda

using namespace cpcag_cuda;

// Test/diagnostic primitive: the full 3xTF32 Gram matrix of n points (point
// i = row i of the n x d row-major fp64 array P), row-major fp32 n x n.
extern "C" int cpcag_cuda_gram_tf32x3(cpcag_ctx ctx, const double* P, int64_t n, int64_t d, float* G) {
  return guard([&] {
    Ctx* c = as_ctx(ctx);
    if (n < 0 || d < 0) invalid("gram: negative size");
    InView<double> pin(c, P, static_cast<size_t>(n * d));
    OutView<float> gout(c, G, static_cast<size_t>(n * n));
    const i64 dp = std::max<i64>(32, (d + 31) / 32 * 32);
    DevBuf<float> H(c, std::max<i64>(n * dp, 1)), L(c, std::max<i64>(n * dp, 1));
    if (n) {
      split_points(c, pin.d, n, d, dp, H.p, L.p);
      const size_t smem = gram_tc_smem();
      ensure_smem(gram_tf32x3_k, smem);
      dim3 g(static_cast<unsigned>((n + 127) / 128), static_cast<unsigned>((n + 127) / 128));
      {
        KScope ks_(c, "gram_tf32x3");
        gram_tf32x3_k<<<g, 128, smem, c->stream>>>(H.p, L.p, n, dp, gout.d);
        launched(c);
      }
    }
    gout.flush(c);
    sync(c);
  });
}
