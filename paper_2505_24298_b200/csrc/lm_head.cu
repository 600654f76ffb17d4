// lm_head.cu — the LM head's three GEMMs of the decoupled-PPO loss + backward on tcgen05.
//
// Reference: _surrogate_terms (/root/reference/pkg/src/asyncrl/trainer.py:150-195) with the
// model in the loop: logits = features @ W.T + b (163, via policy.logits, policy.py:137-142),
// the residual  resid = coef * (onehot - softmax)  (180-182), and the parameter gradients
// grad_w = resid.T @ features, grad_b = resid.sum(0) (183-184).  On the GPU the features are
// the hidden states H [T, d] (bf16/fp16), W [V, d] the LM head, and K2 (ppo_kernels.cu)
// turns a logits tile into dlogits = g * coef * (softmax - onehot) in place, so
//   OP_LOGITS   C [T, V]  = H W^T + b              (A = H  K-major, B = W  K-major)
//   OP_DHIDDEN  C [T, d]  = dL W                   (A = dL K-major, B = W  MN-major)
//   OP_DWEIGHT  C [V, d] (+)= dL^T H               (A = dL MN-major, B = H MN-major)
// and grad_b = column sums of dL (areal_colsum).  The logits never leave a chunk buffer of
// the caller's choosing; fusing the backward GEMMs into K2 would need the logits GEMM twice
// (the softmax needs the row's full log-sum-exp first) and dH [T, d] accumulators larger
// than TMEM, so the chunk's dlogits are materialised once in bf16 and read
// by two tensor-core GEMMs whose arithmetic intensity (~d flop / byte) hides that traffic.
//
// One persistent kernel per op, CTA pairs (tcgen05 .cta_group::2, M = 256 per pair,
// N = 256, K-slabs of 64), warp-specialised like K7 (linear_lp.cu): warp 0 issues TMA
// loads into a 6-stage ring (completion on the pair leader's barrier), warp 1 of the
// leader issues the MMAs into two TMEM accumulators (2 x 256 columns), warps 2-9 drain an
// accumulator (tcgen05.ld 32x32b: thread = row) into shared-memory boxes written by TMA
// tensor stores (f32 += by TMA reduce-add) while the next one is computed.  The backward
// GEMMs run two pairs per 4-CTA cluster on one M-tile: the pairs' common A operand is
// loaded once and multicast to both (see produce_unit).  Output tiles are rastered in
// groups of `group_m` M-tiles so the clusters in flight share their k-slabs in L2.
#include <algorithm>

#include "tcgen05.cuh"

namespace areal {
namespace lmh {
using namespace areal::tc;

constexpr int BM = 128;                      // rows per CTA (TMEM lanes); 256 per pair
constexpr int BN = 256;                      // accumulator columns (N per MMA)
constexpr int BK = 64;                       // k-slab (one 128-byte swizzle row of 16-bit)
constexpr int UMMA_K = 16;
// Epilogue output through shared memory + TMA tensor stores (f32 += by TMA reduce-add in
// L2): one 32-row x 128-byte box per epilogue warp.  The register -> global path it
// replaces wrote 16 bytes per thread into 32 different rows per instruction: twice the L2
// write sectors and 8x the write requests of cuBLAS's epilogue (ncu r02bk).
#ifndef LMH_TMA_STORE
#define LMH_TMA_STORE 1
#endif
constexpr bool kTmaStore = LMH_TMA_STORE != 0;
// staging boxes per epilogue warp (2: the next box is written while the previous one's
// TMA store still reads its buffer; costs a ring stage)
#ifndef LMH_EPI_BUFS
#define LMH_EPI_BUFS 1
#endif
constexpr int EPI_BUFS = LMH_EPI_BUFS;
#ifndef LMH_STAGES
#define LMH_STAGES (LMH_TMA_STORE ? 7 - LMH_EPI_BUFS : 7)
#endif
constexpr int STAGES = LMH_STAGES;          // x 32 KB: the most that fits beside the barriers
                                             // (and the epilogue's staging boxes)
constexpr int A_BYTES = BM * BK * 2;         // per CTA per stage
constexpr int B_BYTES = (BN / 2) * BK * 2;   // per CTA per stage: half of B
constexpr int STAGE = A_BYTES + B_BYTES;
constexpr int MN_BLOCK = 64 * 128;           // one 64-element MN block of a 64-row K slab
constexpr int EPI_SPLIT = 2;                 // epilogue warps per TMEM lane quarter
constexpr int EPI_THREADS = 128 * EPI_SPLIT;
constexpr int EPI_BOX = 32 * 128;            // one warp's staging box: 32 rows x 128 B
constexpr int EPI_SMEM = kTmaStore ? (EPI_THREADS / 32) * EPI_BOX * EPI_BUFS : 0;
constexpr int SMEM = STAGES * STAGE + EPI_SMEM + 1024;  // + run-time 1024-B alignment
constexpr int DB_WARPS = 4;                  // column-sum warps (grad_b fused into DWEIGHT)
constexpr int DB_FIRST_WARP = 2 + EPI_THREADS / 32;
// launch kinds: one problem of a fixed op, or the grouped backward (DHIDDEN + DWEIGHT)
constexpr int KIND_BWD = 3;
__host__ __device__ constexpr int kind_threads(int kind) {
  return 64 + EPI_THREADS + (kind == KIND_BWD ? 32 * DB_WARPS : 0);
}
constexpr int CH_PER_WARP = BN / 32 / EPI_SPLIT;
constexpr int MAX_PROBS = 2;

// One GEMM of the launch.  A launch runs 1 problem, or DHIDDEN + DWEIGHT of one chunk as a
// grouped GEMM (both read dL; the second's units fill the first's last wave).
struct Prob {
  int64_t M, N, K;
  int32_t n_mt, n_nt, n_np, group_m, ksteps, units, unit_base;  // units: cluster units (mt, N-tile pair)
  void* C;
  int64_t ldc;
  const float* bias;  // LOGITS: + bias[n]
  float* colsum;      // DWEIGHT: colsum[m] (+)= sum_k A[k, m] (grad_b), summed from shared memory
  int32_t accumulate, a_mn, b_mn, f32_out;
  uint32_t idesc;
};
struct Args {
  Prob p[MAX_PROBS];
  int32_t n_probs, n_units;
};

// cluster unit -> (problem, M-tile, N-tile pair): problems in order; inside one, M fastest
// within a group of group_m M-tiles, then N-tile pairs, then groups (the clusters in
// flight share their k-slabs in L2).  Pair p of the cluster takes N-tile 2 * np + p.
struct Tile { int prob, mt, np; };
__device__ __forceinline__ Tile unit_tile(const Args& a, int u) {
  const int pi = (a.n_probs > 1 && u >= a.p[1].unit_base) ? 1 : 0;
  const Prob& p = pi ? a.p[1] : a.p[0];
  u -= p.unit_base;
  const int per_group = p.group_m * p.n_np;
  const int full = p.n_mt / p.group_m;
  const int g = u / per_group;
  if (g < full) {
    const int r = u - g * per_group;
    return Tile{pi, g * p.group_m + r % p.group_m, r / p.group_m};
  }
  const int gm = p.n_mt - full * p.group_m;  // last, partial group
  const int r = u - full * per_group;
  return Tile{pi, full * p.group_m + r % gm, r / gm};
}
__device__ __forceinline__ bool db_unit(const Args& a, const Tile& t, uint32_t pair) {
  return (t.prob ? a.p[1] : a.p[0]).colsum != nullptr && t.np == 0 && pair == 0;
}

template <typename T> __device__ __forceinline__ uint32_t pack2(float x, float y);
template <> __device__ __forceinline__ uint32_t pack2<__nv_bfloat16>(float x, float y) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(x, y);
  return *reinterpret_cast<const uint32_t*>(&h);
}
template <> __device__ __forceinline__ uint32_t pack2<__half>(float x, float y) {
  const __half2 h = __floats2half2_rn(x, y);
  return *reinterpret_cast<const uint32_t*>(&h);
}
template <typename T> __device__ __forceinline__ float2 unpack2(uint32_t v);
template <> __device__ __forceinline__ float2 unpack2<__nv_bfloat16>(uint32_t v) {
  return __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&v));
}
template <> __device__ __forceinline__ float2 unpack2<__half>(uint32_t v) {
  return __half22float2(*reinterpret_cast<const __half2*>(&v));
}

// TMA loads of one unit's k-slabs.  Cluster of 4 = 2 CTA pairs on one M-tile and two
// N-tiles: each CTA loads its half of its pair's B, and a quarter of the pairs' common A
// (its 128 A rows / columns split 64 + 64 between the two pairs) multicast to the CTA of
// the same pair rank in both pairs; bytes are counted on each pair's leader barrier.
// A_MN / B_MN: operand stored [K rows x MN cols] (64-column boxes).
template <bool A_MN, bool B_MN, int CL>
__device__ __forceinline__ void produce_unit(const CUtensorMap* mA, const CUtensorMap* mB, unsigned char* smem,
                                             uint64_t* full, uint64_t* empty, uint64_t* dbdone, int32_t m0,
                                             int32_t n0, int ksteps, bool db, uint32_t r, uint32_t pair,
                                             uint32_t& stage, uint32_t& phase, uint32_t& db_pending,
                                             uint32_t& db_phase) {
  const uint16_t a_mask = (uint16_t)((1u << r) | (1u << (2 + r)));
  const int32_t ma = m0 + (int32_t)pair * 64;  // this CTA's 64 of the pair rank's 128 A rows / columns
  for (int ks = 0; ks < ksteps; ++ks) {
    mbar_wait(&empty[stage], phase ^ 1u);
    if (db_pending >> stage & 1u) {  // the column-sum warps still read this stage
      mbar_wait(&dbdone[stage], db_phase >> stage & 1u);
      db_phase ^= 1u << stage;
      db_pending &= ~(1u << stage);
    }
    if (db) db_pending |= 1u << stage;
    unsigned char* st = smem + (size_t)stage * STAGE;
    const uint32_t bar_lead = mapa_shared(smem_u32(&full[stage]), 2u * pair);  // own pair's leader
    const uint32_t bar_any = mapa_shared(smem_u32(&full[stage]), 0u);           // even CTA of each pair
    if (r == 0) mbar_arrive_expect_tx(&full[stage], 2 * STAGE);
    const int32_t k0 = ks * BK;
    if (CL == 4) {
      if (A_MN) tma_load_2d_cg2_mc(mA, st + pair * MN_BLOCK, bar_any, ma, k0, a_mask);
      else tma_load_2d_cg2_mc(mA, st + pair * (A_BYTES / 2), bar_any, k0, ma, a_mask);
    } else {  // CTA pair only: this CTA's 128 A rows / columns as two 64-wide boxes
      if (A_MN) {
        tma_load_2d_cg2(mA, st, bar_lead, m0, k0);
        tma_load_2d_cg2(mA, st + MN_BLOCK, bar_lead, m0 + 64, k0);
      } else {
        tma_load_2d_cg2(mA, st, bar_lead, k0, m0);
        tma_load_2d_cg2(mA, st + A_BYTES / 2, bar_lead, k0, m0 + 64);
      }
    }
    if (B_MN) {
      tma_load_2d_cg2(mB, st + A_BYTES, bar_lead, n0, k0);
      tma_load_2d_cg2(mB, st + A_BYTES + MN_BLOCK, bar_lead, n0 + 64, k0);
    } else {
      tma_load_2d_cg2(mB, st + A_BYTES, bar_lead, k0, n0);
    }
    if (++stage == STAGES) stage = 0, phase ^= 1u;
  }
}

// The unit's MMAs into one TMEM accumulator (leader CTA, one thread).
template <bool A_MN, bool B_MN, int CL>
__device__ __forceinline__ void mma_unit(unsigned char* smem, uint64_t* full, uint64_t* empty, uint64_t* landed,
                                         uint32_t landed_peer, uint32_t d_tmem, uint32_t idesc, int ksteps,
                                         bool db, uint32_t& stage, uint32_t& phase) {
  constexpr uint32_t a_step = A_MN ? (UMMA_K * 128) >> 4 : (UMMA_K * 2) >> 4;
  constexpr uint32_t b_step = B_MN ? (UMMA_K * 128) >> 4 : (UMMA_K * 2) >> 4;
  for (int ks = 0; ks < ksteps; ++ks) {
    mbar_wait(&full[stage], phase);
    tc_fence_after();
    if (db) {  // both CTAs' halves of the stage have landed: the column-sum warps may read
      mbar_arrive(&landed[stage]);
      mbar_remote_arrive(landed_peer + stage * (uint32_t)sizeof(uint64_t));
    }
    const uint32_t sa = smem_u32(smem + (size_t)stage * STAGE);
    const uint64_t adesc = A_MN ? sw128_desc_mn(sa, MN_BLOCK) : sw128_desc(sa);
    const uint64_t bdesc = B_MN ? sw128_desc_mn(sa + A_BYTES, MN_BLOCK) : sw128_desc(sa + A_BYTES);
#pragma unroll
    for (int kk = 0; kk < BK / UMMA_K; ++kk)
      mma_bf16_cg2(d_tmem, adesc + (uint64_t)(kk * a_step), bdesc + (uint64_t)(kk * b_step), idesc,
                   (ks | kk) != 0);
    // frees the stage once read: in all four CTAs (the other pair's A quarters live here too)
    mma_commit_cg2_mask(&empty[stage], CL == 4 ? 0xF : 0x3);
    if (++stage == STAGES) stage = 0, phase ^= 1u;
  }
}

template <int KIND, typename T, int CL>
__global__ void __launch_bounds__(kind_threads(KIND), 1)
    lmh_gemm_kernel(const __grid_constant__ CUtensorMap tmA0, const __grid_constant__ CUtensorMap tmB0,
                    const __grid_constant__ CUtensorMap tmA1, const __grid_constant__ CUtensorMap tmB1,
                    const __grid_constant__ CUtensorMap tmC0, const __grid_constant__ CUtensorMap tmC1,
                    const Args a) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[STAGES], empty[STAGES], tfull[2], tempty[2], landed[STAGES], dbdone[STAGES];
  __shared__ uint32_t s_tbase;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = cluster_ctarank();   // 0..CL-1
  const uint32_t rank = crank & 1u;           // rank in the CTA pair (1 = the MMA peer)
  const uint32_t pair = crank >> 1;           // which pair of the cluster (its N-tile)
  constexpr int NPU = CL / 2;                 // N-tiles per unit (one per pair)
  const int unit0 = (int)cluster_id_x();
  const int unit_step = (int)nclusters_x();
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CL / 2);  // one MMA commit from each pair
      mbar_init(&landed[s], 1);
      mbar_init(&dbdone[s], DB_WARPS);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4 * EPI_SPLIT * 2);  // every epilogue warp of the pair
    }
    fence_mbar_init_cluster();
    prefetch_tmap(&tmA0);
    prefetch_tmap(&tmB0);
    if (a.n_probs > 1) {
      prefetch_tmap(&tmA1);
      prefetch_tmap(&tmB1);
    }
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&s_tbase))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    tc_fence_before();
  }
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tbase = s_tbase;

  if (warp == 0) {
    // ================= TMA producer (both CTAs; bytes counted on the leader's barrier)
    if (lane == 0) {
      uint32_t stage = 0, phase = 0;
      uint32_t db_pending = 0, db_phase = 0;  // per stage: last use summed by the db warps / parity
      for (int u = unit0; u < a.n_units; u += unit_step) {
        const Tile t = unit_tile(a, u);
        const bool second = KIND == KIND_BWD && t.prob == 1;
        const int ksteps = second ? a.p[1].ksteps : a.p[0].ksteps;
        // both pairs: pair 0's column-sum warps also read the A quarters pair 1 multicasts
        // into pair 0, so pair 1's producer waits for them too
        const bool db = KIND == KIND_BWD && second && db_unit(a, t, 0u);
        const int32_t m0 = t.mt * (2 * BM) + (int32_t)rank * BM;
        const int32_t n0 = (NPU * t.np + (int32_t)pair) * BN + (int32_t)rank * (BN / 2);
        if (KIND == AREAL_LMH_LOGITS)
          produce_unit<false, false, CL>(&tmA0, &tmB0, smem, full, empty, dbdone, m0, n0, ksteps, false, rank, pair,
                                     stage, phase, db_pending, db_phase);
        else if (KIND == AREAL_LMH_DHIDDEN || (KIND == KIND_BWD && !second))
          produce_unit<false, true, CL>(&tmA0, &tmB0, smem, full, empty, dbdone, m0, n0, ksteps, false, rank, pair,
                                    stage, phase, db_pending, db_phase);
        else if (KIND == AREAL_LMH_DWEIGHT)
          produce_unit<true, true, CL>(&tmA0, &tmB0, smem, full, empty, dbdone, m0, n0, ksteps, false, rank, pair,
                                   stage, phase, db_pending, db_phase);
        else
          produce_unit<true, true, CL>(&tmA1, &tmB1, smem, full, empty, dbdone, m0, n0, ksteps, db, rank, pair,
                                   stage, phase, db_pending, db_phase);
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer (leader CTA)
    if (lane == 0 && rank == 0) {
      uint32_t stage = 0, phase = 0, acc = 0, acc_phase = 0;
      const uint32_t landed_peer = mapa_shared(smem_u32(&landed[0]), crank + 1u);
      for (int u = unit0; u < a.n_units; u += unit_step) {
        const Tile t = unit_tile(a, u);
        const bool second = KIND == KIND_BWD && t.prob == 1;
        const int ksteps = second ? a.p[1].ksteps : a.p[0].ksteps;
        const uint32_t idesc = second ? a.p[1].idesc : a.p[0].idesc;
        const bool db = KIND == KIND_BWD && second && db_unit(a, t, pair);
        mbar_wait_cluster(&tempty[acc], acc_phase ^ 1u);
        tc_fence_after();
        const uint32_t d_tmem = tbase + acc * BN;
        if (KIND == AREAL_LMH_LOGITS)
          mma_unit<false, false, CL>(smem, full, empty, landed, landed_peer, d_tmem, idesc, ksteps, false, stage, phase);
        else if (KIND == AREAL_LMH_DHIDDEN || (KIND == KIND_BWD && !second))
          mma_unit<false, true, CL>(smem, full, empty, landed, landed_peer, d_tmem, idesc, ksteps, false, stage, phase);
        else
          mma_unit<true, true, CL>(smem, full, empty, landed, landed_peer, d_tmem, idesc, ksteps, db, stage, phase);
        mma_commit_cg2_mask(&tfull[acc], (uint16_t)(3u << (2 * pair)));  // -> epilogues of this pair
        acc ^= 1u;
        if (acc == 0) acc_phase ^= 1u;
      }
    }
  } else if (warp < DB_FIRST_WARP) {
    // ================= epilogue: thread = accumulator row, 128 of the 256 columns
    const int q = warp & 3;
    const int half = (warp - 2) >> 2;
    const uint32_t lane_base = tbase + ((uint32_t)(q * 32) << 16);
    const uint32_t tempty0 = mapa_shared(smem_u32(&tempty[0]), 2u * pair);  // this pair's MMA issuer
    unsigned char* const stg0 = smem + (size_t)STAGES * STAGE + (size_t)(warp - 2) * EPI_BOX * EPI_BUFS;
    uint32_t box = 0;  // boxes this warp has staged (buffer = box % EPI_BUFS)
    uint32_t acc = 0, acc_phase = 0;
    for (int u = unit0; u < a.n_units; u += unit_step) {
      const Tile t = unit_tile(a, u);
      const Prob& p = (KIND == KIND_BWD && t.prob == 1) ? a.p[1] : a.p[0];
      const CUtensorMap* tmC = (KIND == KIND_BWD && t.prob == 1) ? &tmC1 : &tmC0;
      const int32_t row0 = t.mt * (2 * BM) + (int32_t)rank * BM + q * 32;
      const int64_t row = (int64_t)row0 + lane;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t tcol = lane_base + acc * BN;
      float v[2][32];
      const int ch0 = half * CH_PER_WARP;
      tmem_ld32_issue(tcol + ch0 * 32, v[0]);
#pragma unroll
      for (int c = 0; c < CH_PER_WARP; ++c) {
        tmem_ld_wait();
        if (c + 1 < CH_PER_WARP) tmem_ld32_issue(tcol + (ch0 + c + 1) * 32, v[(c + 1) & 1]);
        float* x = v[c & 1];
        const int64_t c0 = (int64_t)(NPU * t.np + (int)pair) * BN + (ch0 + c) * 32;
        if (p.bias != nullptr) {
          if (c0 + 32 <= p.N) {
            const float4* b4 = reinterpret_cast<const float4*>(p.bias + c0);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const float4 bb = __ldg(b4 + i);
              x[4 * i] += bb.x;
              x[4 * i + 1] += bb.y;
              x[4 * i + 2] += bb.z;
              x[4 * i + 3] += bb.w;
            }
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (c0 + i < p.N) x[i] += __ldg(p.bias + c0 + i);
          }
        }
        if (kTmaStore) {
          // swizzled staging (16-byte chunk j of row r at j ^ (r & 7): conflict-free, the
          // layout the 128-byte-swizzle tensor map expects), then one box per warp; TMA
          // clips rows >= M and columns >= N
          unsigned char* const stg = stg0 + (size_t)(box % EPI_BUFS) * EPI_BOX;  // 1024-B aligned
          uint4* const srow = reinterpret_cast<uint4*>(stg + lane * 128);
          if (p.f32_out) {
            if (lane == 0) bulk_wait_read<EPI_BUFS - 1>();  // this buffer's last box was read
            __syncwarp();
#pragma unroll
            for (int j = 0; j < 8; ++j)
              srow[j ^ (lane & 7)] = make_uint4(__float_as_uint(x[4 * j]), __float_as_uint(x[4 * j + 1]),
                                                __float_as_uint(x[4 * j + 2]), __float_as_uint(x[4 * j + 3]));
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              if (p.accumulate) tma_reduce_add_2d(tmC, stg, (int32_t)c0, row0);
              else tma_store_2d(tmC, stg, (int32_t)c0, row0);
              bulk_commit();
            }
            ++box;
          } else {  // 16-bit: two 32-column chunks per 64-column box
            if ((c & 1) == 0) {
              if (lane == 0) bulk_wait_read<EPI_BUFS - 1>();
              __syncwarp();
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
              srow[((c & 1) * 4 + i) ^ (lane & 7)] =
                  make_uint4(pack2<T>(x[8 * i], x[8 * i + 1]), pack2<T>(x[8 * i + 2], x[8 * i + 3]),
                             pack2<T>(x[8 * i + 4], x[8 * i + 5]), pack2<T>(x[8 * i + 6], x[8 * i + 7]));
            if (c & 1) {
              fence_proxy_async_smem();
              __syncwarp();
              if (lane == 0) {
                tma_store_2d(tmC, stg, (int32_t)(c0 - 32), row0);
                bulk_commit();
              }
              ++box;
            }
          }
        } else if (row < p.M && c0 < p.N) {
          if (p.f32_out) {
            float* dst = static_cast<float*>(p.C) + row * p.ldc + c0;
            if (c0 + 32 <= p.N) {
              float4* d4 = reinterpret_cast<float4*>(dst);
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                float4 o = make_float4(x[4 * i], x[4 * i + 1], x[4 * i + 2], x[4 * i + 3]);
                if (p.accumulate) {
                  const float4 q4 = d4[i];
                  o.x += q4.x, o.y += q4.y, o.z += q4.z, o.w += q4.w;
                }
                d4[i] = o;
              }
            } else {
              for (int i = 0; i < 32 && c0 + i < p.N; ++i) dst[i] = p.accumulate ? dst[i] + x[i] : x[i];
            }
          } else {
            T* dst = static_cast<T*>(p.C) + row * p.ldc + c0;
            if (c0 + 32 <= p.N) {
              uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
              for (int i = 0; i < 4; ++i)
                d4[i] = make_uint4(pack2<T>(x[8 * i], x[8 * i + 1]), pack2<T>(x[8 * i + 2], x[8 * i + 3]),
                                   pack2<T>(x[8 * i + 4], x[8 * i + 5]), pack2<T>(x[8 * i + 6], x[8 * i + 7]));
            } else {
              for (int i = 0; i < 32 && c0 + i < p.N; ++i) {
                if constexpr (std::is_same<T, __nv_bfloat16>::value) dst[i] = __float2bfloat16_rn(x[i]);
                else dst[i] = __float2half_rn(x[i]);
              }
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      // TMEM reads done (wait::ld + fence): release the accumulator to the leader's MMA
      // issuer without fencing this warp's global stores
      if (lane == 0) mbar_remote_arrive(tempty0 + acc * (uint32_t)sizeof(uint64_t));
      acc ^= 1u;
      if (acc == 0) acc_phase ^= 1u;
    }
    if (kTmaStore && lane == 0) bulk_wait<0>();  // the last boxes are written before exit
  } else if (KIND == KIND_BWD) {
    // ================= column sums (grad_b = sum over tokens of dL, trainer.py:184) of the
    // DWEIGHT A tiles while they sit in shared memory: for the N-tile-0 unit of each M-tile,
    // db warp w owns 16-byte chunks 4w..4w+3 (32 M columns); lane = 4 * row group + chunk,
    // row group g summing K rows g + 8 i of every stage; the 8 row groups are folded with
    // shuffles (fixed order) at the end of the unit.
    const int w = warp - DB_FIRST_WARP;
    const int chunk = 4 * w + (lane & 3), rgrp = lane >> 2;
    const int blk = chunk >> 3, cc = chunk & 7;
    uint32_t stage = 0, landed_phase = 0;
    for (int u = unit0; u < a.n_units; u += unit_step) {
      const Tile tl = unit_tile(a, u);
      const Prob& p = tl.prob == 1 ? a.p[1] : a.p[0];
      if (!db_unit(a, tl, pair)) {  // keep the stage counter in step with the pipeline
        stage = (uint32_t)((stage + p.ksteps) % STAGES);
        continue;
      }
      float sum[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      for (int ks = 0; ks < p.ksteps; ++ks) {
        mbar_wait(&landed[stage], landed_phase >> stage & 1u);
        landed_phase ^= 1u << stage;
        const unsigned char* st = smem + (size_t)stage * STAGE + blk * MN_BLOCK;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int k = rgrp + 8 * i;  // k & 7 == rgrp: the 128-byte swizzle of row k
          const uint4 v4 = *reinterpret_cast<const uint4*>(st + k * 128 + ((cc ^ rgrp) << 4));
          const float2 e0 = unpack2<T>(v4.x), e1 = unpack2<T>(v4.y), e2 = unpack2<T>(v4.z), e3 = unpack2<T>(v4.w);
          sum[0] += e0.x, sum[1] += e0.y, sum[2] += e1.x, sum[3] += e1.y;
          sum[4] += e2.x, sum[5] += e2.y, sum[6] += e3.x, sum[7] += e3.y;
        }
        __syncwarp();
        if (lane == 0) {  // release the stage to this CTA's producer and to the other pair's
          mbar_arrive(&dbdone[stage]);  // same-rank CTA, whose multicast writes here too
          if (CL == 4) mbar_remote_arrive(mapa_shared(smem_u32(&dbdone[stage]), crank + 2u));
        }
        if (++stage == STAGES) stage = 0;
      }
#pragma unroll
      for (int o = 4; o < 32; o <<= 1)
#pragma unroll
        for (int i = 0; i < 8; ++i) sum[i] += __shfl_xor_sync(0xffffffffu, sum[i], o);
      if (lane < 4) {
        const int64_t m0 = (int64_t)tl.mt * (2 * BM) + (int64_t)rank * BM + chunk * 8;
#pragma unroll
        for (int i = 0; i < 8; ++i)
          if (m0 + i < p.M) p.colsum[m0 + i] = p.accumulate ? p.colsum[m0 + i] + sum[i] : sum[i];
      }
    }
  }
  __syncthreads();
  cluster_sync_all();  // both CTAs done with TMEM before the pair frees it
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tbase) : "memory");
  }
}

// grad_b = column sums of dL: stage 1 sums row blocks of kColRows rows per (column group of
// 8, block) into fp32 partials, 4 rows in flight per thread; stage 2 adds the blocks in
// order (deterministic).
constexpr int kColRows = 1024;

template <typename T>
__device__ __forceinline__ void add8(float (&s)[8], const uint4& w) {
  const T* e = reinterpret_cast<const T*>(&w);
#pragma unroll
  for (int i = 0; i < 8; ++i) s[i] += (float)e[i];
}

template <typename T>
__global__ void colsum_partial_kernel(const T* x, int64_t ld, int64_t rows, int64_t cols, float* part) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // column group of 8
  const int64_t blk = blockIdx.y;
  if (g * 8 >= cols) return;
  const int64_t r0 = blk * kColRows, r1 = r0 + kColRows < rows ? r0 + kColRows : rows;
  float s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (g * 8 + 8 <= cols) {
    const T* p = x + r0 * ld + g * 8;
    int64_t r = r0;
    for (; r + 4 <= r1; r += 4, p += 4 * ld) {  // 4 independent 16-byte loads in flight
      const uint4 w0 = __ldg(reinterpret_cast<const uint4*>(p));
      const uint4 w1 = __ldg(reinterpret_cast<const uint4*>(p + ld));
      const uint4 w2 = __ldg(reinterpret_cast<const uint4*>(p + 2 * ld));
      const uint4 w3 = __ldg(reinterpret_cast<const uint4*>(p + 3 * ld));
      add8<T>(s, w0);
      add8<T>(s, w1);
      add8<T>(s, w2);
      add8<T>(s, w3);
    }
    for (; r < r1; ++r, p += ld) add8<T>(s, __ldg(reinterpret_cast<const uint4*>(p)));
  } else {
    for (int64_t r = r0; r < r1; ++r)
      for (int i = 0; g * 8 + i < cols; ++i) s[i] += (float)x[r * ld + g * 8 + i];
  }
  float* out = part + blk * cols + g * 8;
  for (int i = 0; i < 8 && g * 8 + i < cols; ++i) out[i] = s[i];
}

__global__ void colsum_final_kernel(const float* part, int64_t nblk, int64_t cols, float* out, int accumulate) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cols) return;
  float s = accumulate ? out[c] : 0.f;
  for (int64_t b = 0; b < nblk; ++b) s += part[b * cols + c];
  out[c] = s;
}

}  // namespace lmh
}  // namespace areal

using namespace areal;

namespace areal {
namespace lmh {

struct HostProb {
  Prob p;
  CUtensorMap tmA, tmB, tmC;
};

// Cluster shape per op: LOGITS (K = d, a short main loop) runs on plain CTA pairs; the
// backward GEMMs (K = V or T) on 2 pairs sharing A through TMA multicast, which halves their
// shared operand's L2 reads (ncu r02bk: cuBLAS reads half our L2 sectors) and took DWEIGHT
// from 14.4-15.0 to 12.3-13.1 ms at 32,768 x 151,936 x 1,536 (profiles/r02_lmh_multicast.md).
static int lmh_cluster(int op) { return op == AREAL_LMH_LOGITS ? 2 : 4; }
// Clusters in flight, for the raster grouping only: 4-CTA clusters fill 33 of the 37
// possible on a 148-SM B200 (GPC granularity; the launch itself queries the occupancy).
static int max_clusters_hint(int sms, int cl) { return cl == 4 ? std::max(1, (sms * 9) / 40) : std::max(1, sms / 2); }

// Validate one GEMM and build its problem descriptor + tensor maps.
static int make_prob(HostProb& h, int op, const void* A, int64_t lda, const void* B, int64_t ldb, void* C,
                     int64_t ldc, int64_t M, int64_t N, int64_t K, const float* bias, float* colsum,
                     int accumulate, int dtype, int sms) {
  if (op < AREAL_LMH_LOGITS || op > AREAL_LMH_DWEIGHT) return AREAL_ERR_INVALID_ARGUMENT;
  if (M < 0 || N < 0 || K < 0) return AREAL_ERR_BAD_SHAPE;
  if (!A || !B || !C) return AREAL_ERR_INVALID_ARGUMENT;
  if (dtype != AREAL_BF16 && dtype != AREAL_F16) return AREAL_ERR_BAD_DTYPE;
  if (M > ((int64_t)1 << 31) - 2 * BM || N > ((int64_t)1 << 31) - BN || K > ((int64_t)1 << 31) - BK)
    return AREAL_ERR_BAD_SHAPE;
  const bool f32_out = op == AREAL_LMH_DWEIGHT;
  // row strides: 16-byte multiples (TMA, vector stores); bases 16-byte aligned
  if (lda % 8 || ldb % 8 || (f32_out ? ldc % 4 : ldc % 8) || reinterpret_cast<uintptr_t>(A) % 16 ||
      reinterpret_cast<uintptr_t>(B) % 16 || reinterpret_cast<uintptr_t>(C) % 16 ||
      (bias && reinterpret_cast<uintptr_t>(bias) % 16))
    return AREAL_ERR_MISALIGNED;
  if (ldc < N) return AREAL_ERR_BAD_SHAPE;
  const CUtensorMapDataType dt =
      dtype == AREAL_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  bool ok = false;
  switch (op) {
    case AREAL_LMH_LOGITS:  // A = H [M, K], B = W [N, K]
      if (lda < K || ldb < K) return AREAL_ERR_BAD_SHAPE;
      ok = make_map(&h.tmA, A, dt, M, K, lda, BM / 2) && make_map(&h.tmB, B, dt, N, K, ldb, BN / 2);
      break;
    case AREAL_LMH_DHIDDEN:  // A = dL [M, K], B = W [K, N]
      if (lda < K || ldb < N) return AREAL_ERR_BAD_SHAPE;
      ok = make_map(&h.tmA, A, dt, M, K, lda, BM / 2) && make_map(&h.tmB, B, dt, K, N, ldb, BK);
      break;
    default:  // DWEIGHT: A = dL [K, M], B = H [K, N]
      if (lda < M || ldb < N) return AREAL_ERR_BAD_SHAPE;
      ok = make_map(&h.tmA, A, dt, K, M, lda, BK) && make_map(&h.tmB, B, dt, K, N, ldb, BK);
      break;
  }
  if (!ok) return AREAL_ERR_CUDA;
  if (f32_out ? !make_store_map(&h.tmC, C, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, M, N, ldc)
              : !make_store_map(&h.tmC, C, dt, 2, M, N, ldc))
    return AREAL_ERR_CUDA;
  Prob& p = h.p;
  p.M = M;
  p.N = N;
  p.K = K;
  p.n_mt = (int32_t)((M + 2 * BM - 1) / (2 * BM));
  p.n_nt = (int32_t)((N + BN - 1) / BN);
  const int cl = lmh_cluster(op);
  p.n_np = (p.n_nt + cl / 2 - 1) / (cl / 2);  // an odd last N-tile runs against zero-filled B, clipped
  p.units = p.n_mt * p.n_np;
  p.unit_base = 0;
  p.ksteps = (int32_t)((K + BK - 1) / BK);
  p.C = C;
  p.ldc = ldc;
  p.bias = op == AREAL_LMH_LOGITS ? bias : nullptr;
  p.colsum = op == AREAL_LMH_DWEIGHT ? colsum : nullptr;
  p.accumulate = accumulate ? 1 : 0;
  p.a_mn = op == AREAL_LMH_DWEIGHT ? 1 : 0;
  p.b_mn = op == AREAL_LMH_LOGITS ? 0 : 1;
  p.f32_out = f32_out ? 1 : 0;
  // pairs in flight cover group_m M-tiles x (pairs / group_m) N-tiles: their A and B
  // k-slabs are shared through L2 (LOGITS: W read n_mt / 16 times, H once).  DWEIGHT's B
  // (H, T x d) stays in L2 whatever the order, while its A (dL) is the big stream: with
  // group_m = 1 the clusters sharing an A tile have consecutive ids (co-scheduled), which
  // cut DRAM reads from 7.7 to 5.3 GB at T = 8,192 (ncu, profiles/r02_lmh_group_m.txt)
  const int clusters = max_clusters_hint(sms, cl);
  p.group_m = p.n_np >= clusters ? std::min(16, p.n_mt) : std::max(1, std::min(p.n_mt, clusters / p.n_np));
  if (op == AREAL_LMH_DWEIGHT) p.group_m = 1;
  if (tuning(AREAL_TUNE_LMH_GROUP_M) > 0) p.group_m = (int32_t)std::min<int64_t>(p.n_mt, tuning(AREAL_TUNE_LMH_GROUP_M));
  const uint32_t ab = dtype == AREAL_BF16 ? 1u : 0u;
  p.idesc = (1u << 4) | (ab << 7) | (ab << 10) | ((uint32_t)p.a_mn << 15) | ((uint32_t)p.b_mn << 16) |
            ((uint32_t)(BN >> 3) << 17) | ((uint32_t)((2 * BM) >> 4) << 24);
  return AREAL_OK;
}

// K == 0: C = 0 (or unchanged when accumulating); colsum likewise
static int empty_reduction(const Prob& p, int op, cudaStream_t stream) {
  if (op == AREAL_LMH_LOGITS) return AREAL_ERR_BAD_SHAPE;  // a head over 0 features
  if (p.accumulate) return AREAL_OK;
  const size_t es = p.f32_out ? 4 : 2;
  if (cudaMemset2DAsync(p.C, p.ldc * es, 0, p.N * es, p.M, stream) != cudaSuccess) return AREAL_ERR_CUDA;
  if (p.colsum && cudaMemsetAsync(p.colsum, 0, p.M * sizeof(float), stream) != cudaSuccess) return AREAL_ERR_CUDA;
  return AREAL_OK;
}

static int launch(int kind, HostProb* hp, int n, int dtype, int sms, cudaStream_t stream) {
  Args a = {};
  a.n_probs = n;
  int units = 0;
  for (int i = 0; i < n; ++i) {
    a.p[i] = hp[i].p;
    a.p[i].unit_base = units;
    units += a.p[i].units;
  }
  a.n_units = units;
  if (units == 0) return AREAL_OK;
  void (*kern)(const CUtensorMap, const CUtensorMap, const CUtensorMap, const CUtensorMap, const CUtensorMap,
               const CUtensorMap, const Args) = nullptr;
  const bool bf = dtype == AREAL_BF16;
  const int cl = lmh_cluster(kind == KIND_BWD ? AREAL_LMH_DWEIGHT : kind);
  switch (kind) {
    case AREAL_LMH_LOGITS: kern = bf ? lmh_gemm_kernel<AREAL_LMH_LOGITS, __nv_bfloat16, 2> : lmh_gemm_kernel<AREAL_LMH_LOGITS, __half, 2>; break;
    case AREAL_LMH_DHIDDEN: kern = bf ? lmh_gemm_kernel<AREAL_LMH_DHIDDEN, __nv_bfloat16, 4> : lmh_gemm_kernel<AREAL_LMH_DHIDDEN, __half, 4>; break;
    case AREAL_LMH_DWEIGHT: kern = bf ? lmh_gemm_kernel<AREAL_LMH_DWEIGHT, __nv_bfloat16, 4> : lmh_gemm_kernel<AREAL_LMH_DWEIGHT, __half, 4>; break;
    default: kern = bf ? lmh_gemm_kernel<KIND_BWD, __nv_bfloat16, 4> : lmh_gemm_kernel<KIND_BWD, __half, 4>; break;
  }
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM) != cudaSuccess)
    return AREAL_ERR_CUDA;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cl);
  cfg.blockDim = dim3(kind == KIND_BWD ? kind_threads(KIND_BWD) : kind_threads(0));
  cfg.dynamicSmemBytes = SMEM;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cl;  // a CTA pair, or two pairs sharing A through multicast
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // a persistent grid must be co-resident: 4-CTA clusters with this shared memory fit 33
  // at a time on 148 SMs (GPC granularity), not 148 / 4 (the first multicast attempt
  // launched 37 and ran its last clusters after the others: 47% tensor-pipe busy)
  static int max_active[2][4] = {{0}};
  int& ma = max_active[bf ? 1 : 0][kind & 3];
  if (ma == 0 && (cudaOccupancyMaxActiveClusters(&ma, kern, &cfg) != cudaSuccess || ma < 1)) {
    cudaGetLastError();
    ma = 1;
  }
  const int clusters = std::max(1, std::min(ma, units));
  cfg.gridDim = dim3(cl * clusters);
  const CUtensorMap& a1 = n > 1 ? hp[1].tmA : hp[0].tmA;
  const CUtensorMap& b1 = n > 1 ? hp[1].tmB : hp[0].tmB;
  const CUtensorMap& c1 = n > 1 ? hp[1].tmC : hp[0].tmC;
  if (cudaLaunchKernelEx(&cfg, kern, hp[0].tmA, hp[0].tmB, a1, b1, hp[0].tmC, c1, a) != cudaSuccess)
    return AREAL_ERR_CUDA;
  AREAL_CUDA_CHECK_LAUNCH();
  return AREAL_OK;
}

static int sm_count() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

}  // namespace lmh
}  // namespace areal

extern "C" int areal_lm_head_gemm(int op, const void* A, int64_t lda, const void* B, int64_t ldb, void* C,
                                  int64_t ldc, int64_t M, int64_t N, int64_t K, const float* bias,
                                  int accumulate, int dtype, void* stream_) {
  using namespace areal::lmh;
  if (op < AREAL_LMH_LOGITS || op > AREAL_LMH_DWEIGHT) return AREAL_ERR_INVALID_ARGUMENT;
  if (M < 0 || N < 0 || K < 0) return AREAL_ERR_BAD_SHAPE;
  if (M == 0 || N == 0) return AREAL_OK;
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  const int sms = sm_count();
  HostProb h;
  if (K == 0) {
    if (op == AREAL_LMH_LOGITS) return AREAL_ERR_BAD_SHAPE;
    if (!C) return AREAL_ERR_INVALID_ARGUMENT;
    Prob p = {};
    p.C = C, p.ldc = ldc, p.M = M, p.N = N, p.accumulate = accumulate, p.f32_out = op == AREAL_LMH_DWEIGHT;
    return empty_reduction(p, op, stream);
  }
  const int rc = make_prob(h, op, A, lda, B, ldb, C, ldc, M, N, K, bias, nullptr, accumulate, dtype, sms);
  if (rc != AREAL_OK) return rc;
  return launch(op, &h, 1, dtype, sms, stream);
}

extern "C" int areal_lm_head_backward(const void* dlogits, int64_t ld_dlogits, const void* hidden,
                                      int64_t ld_hidden, const void* weight, int64_t ld_weight,
                                      int64_t n_rows, int64_t vocab, int64_t dim, void* grad_hidden,
                                      int64_t ld_grad_hidden, float* grad_weight, int64_t ld_grad_weight,
                                      float* grad_bias, int accumulate, int dtype, void* stream_) {
  using namespace areal::lmh;
  if (n_rows < 0 || vocab < 1 || dim < 1) return AREAL_ERR_BAD_SHAPE;
  if (!grad_weight) return AREAL_ERR_INVALID_ARGUMENT;
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  const int sms = sm_count();
  if (n_rows == 0) {  // dH is empty; grad_w / grad_b get an empty sum
    Prob p = {};
    p.C = grad_weight, p.ldc = ld_grad_weight, p.M = vocab, p.N = dim, p.accumulate = accumulate;
    p.f32_out = 1, p.colsum = grad_bias;
    return empty_reduction(p, AREAL_LMH_DWEIGHT, stream);
  }
  HostProb h[2];
  int rc = make_prob(h[0], AREAL_LMH_DHIDDEN, dlogits, ld_dlogits, weight, ld_weight, grad_hidden, ld_grad_hidden,
                     n_rows, dim, vocab, nullptr, nullptr, 0, dtype, sms);
  if (rc != AREAL_OK) return rc;
  rc = make_prob(h[1], AREAL_LMH_DWEIGHT, dlogits, ld_dlogits, hidden, ld_hidden, grad_weight, ld_grad_weight,
                 vocab, dim, n_rows, nullptr, grad_bias, accumulate, dtype, sms);
  if (rc != AREAL_OK) return rc;
  return launch(KIND_BWD, h, 2, dtype, sms, stream);
}

extern "C" size_t areal_colsum_scratch_bytes(int64_t rows, int64_t cols) {
  if (rows <= 0 || cols <= 0) return 0;
  return (size_t)((rows + areal::lmh::kColRows - 1) / areal::lmh::kColRows) * (size_t)cols * sizeof(float);
}

extern "C" int areal_colsum(const void* x, int64_t ld, int64_t rows, int64_t cols, int dtype, float* out,
                            int accumulate, void* scratch, size_t scratch_bytes, void* stream_) {
  using namespace areal::lmh;
  if (rows < 0 || cols < 0 || ld < cols) return AREAL_ERR_BAD_SHAPE;
  if (cols == 0) return AREAL_OK;
  if (!out || (rows > 0 && !x)) return AREAL_ERR_INVALID_ARGUMENT;
  if (dtype != AREAL_BF16 && dtype != AREAL_F16) return AREAL_ERR_BAD_DTYPE;
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  if (rows == 0) {
    if (accumulate) return AREAL_OK;
    return cudaMemsetAsync(out, 0, cols * sizeof(float), stream) == cudaSuccess ? AREAL_OK : AREAL_ERR_CUDA;
  }
  if (ld % 8 || reinterpret_cast<uintptr_t>(x) % 16) return AREAL_ERR_MISALIGNED;
  if (!scratch || scratch_bytes < areal_colsum_scratch_bytes(rows, cols)) return AREAL_ERR_WORKSPACE;
  const int64_t nblk = (rows + kColRows - 1) / kColRows;
  const int64_t groups = (cols + 7) / 8;
  const dim3 grid((unsigned)((groups + 127) / 128), (unsigned)nblk);
  float* part = static_cast<float*>(scratch);
  if (dtype == AREAL_BF16)
    colsum_partial_kernel<__nv_bfloat16><<<grid, 128, 0, stream>>>(static_cast<const __nv_bfloat16*>(x), ld, rows,
                                                                   cols, part);
  else
    colsum_partial_kernel<__half><<<grid, 128, 0, stream>>>(static_cast<const __half*>(x), ld, rows, cols, part);
  AREAL_CUDA_CHECK_LAUNCH();
  colsum_final_kernel<<<(unsigned)((cols + 255) / 256), 256, 0, stream>>>(part, nblk, cols, out, accumulate);
  AREAL_CUDA_CHECK_LAUNCH();
  return AREAL_OK;
}
