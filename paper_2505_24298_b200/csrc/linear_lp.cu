// linear_lp.cu — K7: fused LM-head GEMM + log-softmax-gather (+ entropy) on tcgen05.
//
// Reference: recompute_prox_logprobs (trainer.py:128-137) -> batch_token_log_probs
// (policy.py:159-163) -> logits(params, features) = features @ W.T + b
// (policy.py:133-142) -> log_softmax (policy.py:145-147), gathered at the token.
// Here features are the model's hidden states H [T, d] (bf16/fp16) and W [V, d] is the
// LM head; the [T, V] logits are never written to HBM.
//
// Structure (persistent, one CTA per SM, warp-specialised, 192 threads):
//   warp 0      TMA producer: 2-D tensor-map loads of H [128 x 64] and W [256 x 64]
//               k-slabs (128-byte swizzle) into a 4-stage shared-memory ring
//   warp 1      MMA issuer: one elected lane issues tcgen05.mma.cta_group::1.kind::f16
//               (M=128, N=256, K=16) from shared-memory descriptors into a TMEM
//               accumulator; two accumulators (2 x 256 of the 512 TMEM columns) so
//               the epilogue of N-tile j overlaps the MMAs of N-tile j+1
//   warps 2-5   epilogue: tcgen05.ld 32x32b (thread = token row, 32 columns per load),
//               + bias, online (max, sum 2^x, sum 2^x * x) per row, the token's logit
//               picked out when its column passes; TMEM slot released by mbarrier
// A work unit is (128-token tile, 2048-column vocab block); units are ordered
// vocab-block-major so the CTAs running together share one W block in L2.  Each unit
// writes a per-(row, block) partial {m, s, sx, x_tok}; a merge kernel folds a row's
// partials in block order (deterministic) into lp = x_tok - lse and H = lse - sx/s.
#include <algorithm>

#include "tcgen05.cuh"

namespace areal {
namespace k7 {
using namespace areal::tc;

constexpr int BM = 128;            // tokens per tile (TMEM lanes)
constexpr int BN = 256;            // vocab columns per MMA / accumulator
constexpr int BK = 64;             // k-slab: 64 x 2 B = one 128-byte swizzle row
constexpr int UMMA_K = 16;         // K per tcgen05.mma for 16-bit inputs
#ifndef K7_STAGES2
#define K7_STAGES2 6   // pipeline stages of the CTA-pair kernel (32 KB each)
#endif
#ifndef K7_ALIGN_SLACK
#define K7_ALIGN_SLACK 1024  // run-time 1024-B alignment slack for the swizzled stages
#endif
constexpr int kMaxNT = 8;          // N-tiles per unit (runtime a.nt in {4, 8}; vocab block = nt * BN)
constexpr int kMinNT = 4;          // sizes the partials scratch
constexpr int A_BYTES = BM * BK * 2;
constexpr int EPI_SPLIT = 2;       // epilogue warps per TMEM lane quarter (column halves)
constexpr int EPI_THREADS = 128 * EPI_SPLIT;
constexpr int THREADS = 64 + EPI_THREADS;
constexpr int CH_PER_WARP = BN / 32 / EPI_SPLIT;  // 32-column chunks per epilogue warp per N-tile
static_assert(EPI_THREADS == BN, "bias staging: one bias per epilogue thread per N-tile");

struct Args {
  const float* bias;
  const int64_t* tokens;
  const int32_t* row_index;
  float4* partials;  // [n_rows, n_vb]
  int64_t n_rows, vocab;
  int32_t dim, n_mt, n_vb, n_units;
  int32_t group;  // vocab blocks interleaved per token tile (L2 working-set shaping)
  int32_t nt, vb;  // N-tiles per unit, vocab block = nt * BN columns
  uint32_t idesc;
};

// Unit u -> (token tile, vocab block).  `group` consecutive units share a token tile
// and take `group` different vocab blocks, so the ~74 units in flight touch
// 74/group H tiles and `group` W blocks: the L2 working set is
// (74/group)*TM*d*2 + group*vb*d*2 bytes instead of 74*TM*d*2 (which exceeds L2
// at d = 3584).  Units whose block lies past the vocab are empty.
struct UnitXY { int mt, vb; };
__device__ __forceinline__ UnitXY unit_xy(const Args& a, int u) {
  const int g = u % a.group, r = u / a.group;
  return UnitXY{r % a.n_mt, (r / a.n_mt) * a.group + g};
}

template <int STAGES_>
struct Pipe {
  uint32_t stage = 0, phase = 0;
  __device__ __forceinline__ void next() {
    if (++stage == STAGES_) {
      stage = 0;
      phase ^= 1u;
    }
  }
};

// Per-CTA-group geometry.  CG = 1: M = 128 per CTA, each CTA loads its A [128 x 64]
// and the whole B [256 x 64] per k-slab (48 KB).  CG = 2 (CTA pair, tcgen05 .cta_group::2):
// M = 256 over the pair, each CTA loads its A [128 x 64] and HALF of B [128 x 64]
// (32 KB), the leader CTA issues the MMA that reads both CTAs' shared memory and writes
// both CTAs' TMEM (each its 128 rows x 256 columns).
template <int CG> struct Geo {
  static constexpr int B_ROWS = BN / CG;                     // B rows loaded per CTA
  static constexpr int STAGE = A_BYTES + B_ROWS * BK * 2;    // bytes per stage per CTA
  static constexpr int NSTAGE = (CG == 1) ? 4 : K7_STAGES2;
  static constexpr int SMEM = NSTAGE * STAGE + K7_ALIGN_SLACK;
  static constexpr int TM = BM * CG;                         // tokens per unit
};

template <int CG, bool ENT>
__global__ void __launch_bounds__(THREADS, 1)
    linear_lp_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const Args a) {
  using G = Geo<CG>;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[G::NSTAGE], empty[G::NSTAGE], tfull[2], tempty[2];
  __shared__ uint32_t s_tbase;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ksteps = a.dim / BK;
  const uint32_t rank = (CG == 2) ? cluster_ctarank() : 0u;
  const int unit0 = (CG == 2) ? (int)cluster_id_x() : (int)blockIdx.x;
  const int nunit_step = (CG == 2) ? (int)nclusters_x() : (int)gridDim.x;
  if (threadIdx.x == 0) {
    for (int s = 0; s < G::NSTAGE; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4 * EPI_SPLIT * CG);  // one arrive per epilogue warp of the pair
    }
    fence_mbar_init_cluster();
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
  }
  if (warp == 1) {
    if constexpr (CG == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                       smem_u32(&s_tbase))
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                       smem_u32(&s_tbase))
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
  }
  if constexpr (CG == 2) cluster_sync_all();  // peer barriers initialised before any remote use
  else __syncthreads();
  tc_fence_after();
  const uint32_t tbase = s_tbase;

  if (warp == 0) {
    // ================= TMA producer (both CTAs; completion counted on the leader's barrier)
    if (lane == 0) {
      Pipe<G::NSTAGE> p;
      for (int u = unit0; u < a.n_units; u += nunit_step) {
        const UnitXY xy = unit_xy(a, u);
        const int mt = xy.mt, vb = xy.vb;
        const int32_t arow = mt * G::TM + (int32_t)rank * BM;
        for (int n = 0; n < a.nt; ++n) {
          const int64_t n0 = (int64_t)vb * a.vb + (int64_t)n * BN;
          if (n0 >= a.vocab) break;
          const int32_t brow = (int32_t)n0 + (int32_t)rank * G::B_ROWS;
          for (int ks = 0; ks < ksteps; ++ks) {
            mbar_wait(&empty[p.stage], p.phase ^ 1u);
            unsigned char* st = smem + (size_t)p.stage * G::STAGE;
            if constexpr (CG == 2) {
              const uint32_t bar0 = mapa_shared(smem_u32(&full[p.stage]), 0u);
              if (rank == 0) mbar_arrive_expect_tx(&full[p.stage], 2 * G::STAGE);
              tma_load_2d_cg2(&tmA, st, bar0, ks * BK, arow);
              tma_load_2d_cg2(&tmB, st + A_BYTES, bar0, ks * BK, brow);
            } else {
              mbar_arrive_expect_tx(&full[p.stage], G::STAGE);
              tma_load_2d(&tmA, st, &full[p.stage], ks * BK, arow);
              tma_load_2d(&tmB, st + A_BYTES, &full[p.stage], ks * BK, brow);
            }
            p.next();
          }
        }
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer (leader CTA only for the pair)
    if (lane == 0 && rank == 0) {
      Pipe<G::NSTAGE> p;
      uint32_t acc = 0, acc_phase = 0;
      for (int u = unit0; u < a.n_units; u += nunit_step) {
        const int vb = unit_xy(a, u).vb;
        for (int n = 0; n < a.nt; ++n) {
          const int64_t n0 = (int64_t)vb * a.vb + (int64_t)n * BN;
          if (n0 >= a.vocab) break;
          if constexpr (CG == 2) mbar_wait_cluster(&tempty[acc], acc_phase ^ 1u);
          else mbar_wait(&tempty[acc], acc_phase ^ 1u);
          tc_fence_after();
          const uint32_t d_tmem = tbase + acc * BN;
          for (int ks = 0; ks < ksteps; ++ks) {
            mbar_wait(&full[p.stage], p.phase);
            tc_fence_after();
            const uint32_t sa = smem_u32(smem + (size_t)p.stage * G::STAGE);
            const uint64_t adesc = sw128_desc(sa), bdesc = sw128_desc(sa + A_BYTES);
#pragma unroll
            for (int kk = 0; kk < BK / UMMA_K; ++kk) {
              // advance the start address by kk * 32 bytes inside the swizzle row
              if constexpr (CG == 2)
                mma_bf16_cg2(d_tmem, adesc + (uint64_t)(kk * 2), bdesc + (uint64_t)(kk * 2), a.idesc,
                             (ks | kk) != 0);
              else
                mma_bf16(d_tmem, adesc + (uint64_t)(kk * 2), bdesc + (uint64_t)(kk * 2), a.idesc,
                         (ks | kk) != 0);
            }
            // frees the stage (in both CTAs) once these MMAs have read it
            if constexpr (CG == 2) mma_commit_cg2(&empty[p.stage]);
            else mma_commit(&empty[p.stage]);
            p.next();
          }
          if constexpr (CG == 2) mma_commit_cg2(&tfull[acc]);  // accumulator complete -> epilogues
          else mma_commit(&tfull[acc]);
          acc ^= 1u;
          if (acc == 0) acc_phase ^= 1u;
        }
      }
    }
  } else {
    // ================= epilogue: one thread per token row
    // TMEM loads are double-buffered (chunk ch+1 in flight while ch is folded); the
    // N-tile's 256 biases are staged in shared memory one N-tile ahead (one named
    // barrier per N-tile among the 4 epilogue warps).
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int r_local = q * 32 + lane;
    const int et = threadIdx.x - 64;  // 0..EPI_THREADS-1
    const int half = (warp - 2) >> 2;  // which column slice of each N-tile this warp folds
    const uint32_t lane_base = tbase + ((uint32_t)(q * 32) << 16);
    const uint32_t tempty0 = (CG == 2) ? mapa_shared(smem_u32(&tempty[0]), 0u) : 0u;
    __shared__ __align__(16) float sbias[2][BN];
    uint32_t acc = 0, acc_phase = 0, bpar = 0;
    constexpr float L2E = 1.4426950408889634f;
    // iteration order of (unit, N-tile) pairs, identical to the producer / MMA loops
    auto tile_n0 = [&](int u, int n) -> int64_t { return (int64_t)unit_xy(a, u).vb * a.vb + (int64_t)n * BN; };
    auto load_bias = [&](int64_t n0) -> float2 {
      float2 b2 = make_float2(0.f, 0.f);
      if (a.bias != nullptr && n0 >= 0) {
        const int64_t c = n0 + et;
        if (c < a.vocab) b2.x = __ldg(a.bias + c);
      }
      return b2;
    };
    if (unit0 < a.n_units) {
      const float2 b2 = load_bias(tile_n0(unit0, 0));
      sbias[0][et] = b2.x;
    }
    named_bar_sync(1, EPI_THREADS);
    for (int u = unit0; u < a.n_units; u += nunit_step) {
      const UnitXY xy = unit_xy(a, u);
      const int mt = xy.mt, vb = xy.vb;
      const int64_t row = (int64_t)mt * G::TM + (int64_t)rank * BM + r_local;
      int64_t tok = -1;
      if (row < a.n_rows) {
        const int64_t idx = a.row_index ? (int64_t)a.row_index[row] : row;
        tok = a.tokens[idx];
      }
      float m = -INFINITY, s = 0.f, sx = 0.f, xa = 0.f;
      for (int n = 0; n < a.nt; ++n) {
        const int64_t n0 = tile_n0(u, n);
        if (n0 >= a.vocab) break;
        // prefetch the biases of the next (unit, N-tile) in iteration order
        int64_t nn0 = -1;
        if (n + 1 < a.nt && tile_n0(u, n + 1) < a.vocab) nn0 = tile_n0(u, n + 1);
        else if (u + nunit_step < a.n_units) nn0 = tile_n0(u + nunit_step, 0);
        const float2 bnext = load_bias(nn0);
        const float* bs = sbias[bpar];

        mbar_wait(&tfull[acc], acc_phase);
        tc_fence_after();
        const uint32_t tcol = lane_base + acc * BN;
        auto fold_chunk = [&](float(&cv)[32], int ch) {
          const int64_t c0 = n0 + ch * 32;
          if (a.bias != nullptr) {
            const float4* b4 = reinterpret_cast<const float4*>(bs + ch * 32);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const float4 bb = b4[i];
              cv[4 * i] += bb.x;
              cv[4 * i + 1] += bb.y;
              cv[4 * i + 2] += bb.z;
              cv[4 * i + 3] += bb.w;
            }
          }
          if (c0 + 32 > a.vocab) {  // vocab tail: columns past V are padding
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (c0 + i >= a.vocab) cv[i] = -INFINITY;
          }
          if (tok >= c0 && tok < c0 + 32) {  // rare: the token's logit
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (c0 + i == tok) xa = cv[i];
          }
          float lmax = cv[0];
#pragma unroll
          for (int i = 1; i < 32; ++i) lmax = fmaxf(lmax, cv[i]);
          const float mn = fmaxf(m, lmax);
          const float c = (mn == -INFINITY) ? 0.f : mn * L2E;
          // exactly 1 while the max stays (2^(rounding residual) would compound)
          const float r = (m == mn) ? 1.f : fast_exp2(__fmul_rn(m, L2E) - c);  // 2^(c_old - c_new), no FMA contraction
          const float2 L2 = make_float2(L2E, L2E), C2 = make_float2(-c, -c);
          float2 s2 = make_float2(0.f, 0.f), x2 = make_float2(0.f, 0.f);
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            const float2 x = make_float2(cv[i], cv[i + 1]);
            const float2 t = ffma2(x, L2, C2);
            const float2 e = make_float2(fast_exp2(t.x), fast_exp2(t.y));
            s2 = fadd2(s2, e);
            if (ENT) {
              const float2 xc = make_float2(fmaxf(x.x, -3.402823466e38f), fmaxf(x.y, -3.402823466e38f));
              x2 = ffma2(e, xc, x2);
            }
          }
          s = s * r + (s2.x + s2.y);
          if (ENT) sx = sx * r + (x2.x + x2.y);
          m = mn;
        };
        float va[32], vb[32];
        const int ch0 = half * CH_PER_WARP;
        tmem_ld32_issue(tcol + ch0 * 32, va);
        tmem_ld_wait();
#pragma unroll 1
        for (int ch = ch0; ch < ch0 + CH_PER_WARP; ch += 2) {
          tmem_ld32_issue(tcol + (ch + 1) * 32, vb);  // in flight while va is folded
          fold_chunk(va, ch);
          tmem_ld_wait();
          if (ch + 2 < ch0 + CH_PER_WARP) tmem_ld32_issue(tcol + (ch + 2) * 32, va);
          fold_chunk(vb, ch + 1);
          if (ch + 2 < ch0 + CH_PER_WARP) tmem_ld_wait();
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (CG == 2)  // release this CTA's TMEM reads to the leader's MMA issuer
            mbar_remote_arrive_release(tempty0 + acc * (uint32_t)sizeof(uint64_t));
          else
            mbar_arrive(&tempty[acc]);
        }
        acc ^= 1u;
        if (acc == 0) acc_phase ^= 1u;
        sbias[bpar ^ 1][et] = bnext.x;
        bpar ^= 1u;
        named_bar_sync(1, EPI_THREADS);
      }
      if (row < a.n_rows && vb < a.n_vb)
        a.partials[(row * a.n_vb + vb) * EPI_SPLIT + half] = make_float4(m, s, sx, xa);
    }
  }
  __syncthreads();
  if constexpr (CG == 2) cluster_sync_all();  // both CTAs done with TMEM before the pair frees it
  if (warp == 1) {
    tc_fence_after();
    if constexpr (CG == 2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tbase) : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase) : "memory");
  }
}

// One warp per row: merge the row's block partials in block order.
__global__ void linear_lp_merge_kernel(const float4* partials, int n_vb, int vblock, int64_t n_rows,
                                       int64_t vocab,
                                       const int64_t* tokens, const int32_t* row_index, double* lp,
                                       double* ent) {
  const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= n_rows) return;
  RowStat<float> w;
  w.init();
  for (int j = lane; j < n_vb * EPI_SPLIT; j += 32) {
    const float4 p = partials[row * n_vb * EPI_SPLIT + j];
    w.merge(p.x, p.y, p.z);
  }
  // fixed-order butterfly: identical on every lane, deterministic
  w.warp_reduce();
  if (lane == 0) {
    const int64_t idx = row_index ? (int64_t)row_index[row] : row;
    const int64_t tok = tokens[idx];
    const double lse = (double)w.m + log((double)w.s);
    double xa = nan("");
    if (tok >= 0 && tok < vocab)  // the partial of the (block, column slice) holding the token
      xa = (double)partials[(row * n_vb + tok / vblock) * EPI_SPLIT + (int)((tok % BN) / (BN / EPI_SPLIT))].w;
    lp[idx] = xa - lse;
    if (ent) ent[idx] = lse - (double)w.sx / (double)w.s;
  }
}

}  // namespace k7
}  // namespace areal

using namespace areal;

extern "C" size_t areal_linear_logprob_scratch_bytes(int64_t n_rows, int64_t vocab) {
  const int64_t vbmin = (int64_t)k7::kMinNT * k7::BN;  // smallest vocab block -> most partials
  const int64_t n_vb = (vocab + vbmin - 1) / vbmin;
  return (size_t)(n_rows > 0 ? n_rows : 0) * (size_t)n_vb * k7::EPI_SPLIT * sizeof(float4);
}

extern "C" int areal_linear_logprob_fwd(const void* hidden, int64_t ld_hidden, const void* weight,
                                        int64_t ld_weight, const float* bias, int dtype, int64_t n_rows,
                                        int64_t vocab, int64_t dim, const int64_t* tokens,
                                        const int32_t* row_index, double* lp_out, double* entropy_out,
                                        void* scratch, size_t scratch_bytes, int cta_group,
                                        void* stream_) {
  using namespace areal::k7;
  if (n_rows < 0 || vocab < 1 || dim < 1) return AREAL_ERR_BAD_SHAPE;
  if (n_rows == 0) return AREAL_OK;
  if (!hidden || !weight || !tokens || !lp_out) return AREAL_ERR_INVALID_ARGUMENT;
  if (dtype != AREAL_BF16 && dtype != AREAL_F16) return AREAL_ERR_BAD_DTYPE;
  if (dim % BK != 0 || dim > 65536) return AREAL_ERR_UNSUPPORTED;
  if (ld_hidden < dim || ld_weight < dim || ld_hidden % 8 || ld_weight % 8 ||
      reinterpret_cast<uintptr_t>(hidden) % 16 || reinterpret_cast<uintptr_t>(weight) % 16 ||
      (bias && reinterpret_cast<uintptr_t>(bias) % 16))
    return AREAL_ERR_MISALIGNED;
  if (n_rows > ((int64_t)1 << 31) - BM || vocab > ((int64_t)1 << 31) - kMaxNT * BN) return AREAL_ERR_BAD_SHAPE;
  if (!scratch || scratch_bytes < areal_linear_logprob_scratch_bytes(n_rows, vocab)) return AREAL_ERR_WORKSPACE;
  const CUtensorMapDataType dt = dtype == AREAL_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  CUtensorMap tmA, tmB;
  Args a;
  a.bias = bias;
  a.tokens = tokens;
  a.row_index = row_index;
  a.partials = static_cast<float4*>(scratch);
  a.n_rows = n_rows;
  a.vocab = vocab;
  a.dim = (int32_t)dim;
  // kind::f16 instruction descriptor: D fp32, A/B bf16 (1) or fp16 (0), both K-major,
  // N >> 3 at bit 17, M >> 4 at bit 24 (cute::UMMA::InstrDescriptor)
  const uint32_t ab = dtype == AREAL_BF16 ? 1u : 0u;
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // the CTA pair needs at least two token tiles' worth of rows to pay off
  const int cg = (cta_group == 1 || cta_group == 2) ? cta_group : (n_rows > BM ? 2 : 1);
  const int tm = BM * cg;
  a.n_mt = (int32_t)((n_rows + tm - 1) / tm);
  {
    // group: minimise the L2 working set of the units in flight, (in_flight / group)
    // H tiles + group W blocks of nt * 256 columns (see unit_xy).  nt = 8 N-tiles per
    // unit; 4 (smaller W blocks, AREAL_TUNE_K7_NT) measured no faster at d = 1536 / 3584
    // (profiles/r01_k7_nt_group_sweep.txt)
    const double in_flight = cg == 2 ? sms / 2 : sms;
    int best_g = 1, best_nt = kMaxNT;
    double best_bytes = 1e300;
    for (int gsz = 1; gsz <= 16; gsz *= 2) {
      const double bytes = (in_flight / gsz) * tm * (double)dim * 2 + gsz * (double)best_nt * BN * dim * 2;
      if (bytes < best_bytes - 1.0) best_g = gsz, best_bytes = bytes;
    }
    if (tuning(AREAL_TUNE_K7_NT) > 0) best_nt = (int)tuning(AREAL_TUNE_K7_NT);
    if (tuning(AREAL_TUNE_K7_GROUP) > 0) best_g = (int)tuning(AREAL_TUNE_K7_GROUP);
    a.nt = best_nt;
    a.vb = best_nt * BN;
    a.n_vb = (int32_t)((vocab + a.vb - 1) / a.vb);
    a.group = std::min(best_g, (int)a.n_vb);
  }
  a.n_units = a.n_mt * ((a.n_vb + a.group - 1) / a.group) * a.group;
  a.idesc = (1u << 4) | (ab << 7) | (ab << 10) | ((uint32_t)(BN >> 3) << 17) |
            ((uint32_t)((BM * cg) >> 4) << 24);
  if (!make_map(&tmA, hidden, dt, n_rows, dim, ld_hidden, BM) ||
      !make_map(&tmB, weight, dt, vocab, dim, ld_weight, BN / cg))
    return AREAL_ERR_CUDA;
  if (cg == 1) {
    const int grid = std::min(sms, a.n_units);
    auto kern = entropy_out ? linear_lp_kernel<1, true> : linear_lp_kernel<1, false>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Geo<1>::SMEM);
    kern<<<grid, THREADS, Geo<1>::SMEM, stream>>>(tmA, tmB, a);
  } else {
    const int clusters = std::min(sms / 2, a.n_units);
    auto kern = entropy_out ? linear_lp_kernel<2, true> : linear_lp_kernel<2, false>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Geo<2>::SMEM);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * clusters);
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = Geo<2>::SMEM;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, kern, tmA, tmB, a) != cudaSuccess) return AREAL_ERR_CUDA;
  }
  AREAL_CUDA_CHECK_LAUNCH();
  const int64_t threads = n_rows * 32;
  linear_lp_merge_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, stream>>>(
      a.partials, a.n_vb, a.vb, n_rows, vocab, tokens, row_index, lp_out, entropy_out);
  AREAL_CUDA_CHECK_LAUNCH();
  return AREAL_OK;
}
