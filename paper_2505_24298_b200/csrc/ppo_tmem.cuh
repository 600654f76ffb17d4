// ppo_tmem.cuh — K2 with the row kept in Tensor Memory: one CTA per row, no cluster.
//
// A bf16 row of 151,936 logits (297 KB) exceeds shared memory (227 KB) but fits
// shared memory + TMEM (256 KB per SM).  This variant parks the first
// kTmemChunks 32 KB chunks of each row in TMEM (tcgen05.st 32x32b, each math
// warp its own 2 KB per chunk in its lane quarter) and keeps only the row's
// tail chunks resident in the shared-memory ring, so:
//   * no thread-block cluster, no DSMEM exchange, no cross-CTA skew in the
//     per-row epilogue (the measured cost of the 2-CTA split is ~20% of K2);
//   * up to nslots - R spare ring slots for the next row's lookahead.
// Pass 1 computes e = 2^(x log2e - c) once per logit (c: warp-uniform running
// max of the chunk) and parks e (bf16 bits for 16-bit logits, fp32 for fp32)
// instead of x, so pass 2 is one multiply per logit: dlogit = e * g 2^(c - lse)
// — half the MUFU work of recomputing the exponential.  Pass 2 reads TMEM with
// tcgen05.ld, resident chunks from shared memory, and writes dlogits with
// coalesced 16-byte global stores.
//
// Ring-slot liveness (deadlock freedom): chunks are streamed in row order into
// ring slots in order; a slot is reused nslots chunks later.  TMEM-bound chunks
// free their slot right after pass 1 stores them to TMEM; the lookahead chunks
// of row i+1 (folded during row i's epilogue) are parked into TMEM at the start
// of row i+1's pass 1; resident tail chunks (offset >= kTmemChunks) free their
// slot in pass 2.  A resident chunk at row offset x is reused by stream
// position x + nslots, which must not be needed before its row's pass 2 starts:
// x + nslots > nchunks - 1 + la, i.e. la <= nslots - R (R resident chunks).
//
// Rows longer than TMEM + the ring (fp32 V = 151,936: 19 chunks) keep at most
// kTResMax chunks resident (all 7 ring slots by default: 8 in TMEM, 7 resident, 4
// streamed for that row); the S chunks between the TMEM part and the resident tail
// are "streamed": folded in pass 1, slot freed at once, and re-read from global
// memory in pass 2 (kept in L2 by evict_last load hints), dlogits = g 2^(x log2e - lse).
// Streamed chunks free their slot in pass 1, so the liveness bound above holds.
//
// Rows that start off a 16-byte boundary (UNAL instantiation) are loaded from the
// boundary below them: chunk element k is row element c * per_chunk + k - head, the
// elements outside the row are masked to -inf in pass 1 and not written in pass 2
// (a row's first and last vectors are stored element by element).
#pragma once

namespace areal {

constexpr int kTmemChunks = 8;        // 8 x 32 KB = the whole 256 KB of TMEM

// Math-warp geometry of this kernel (independent of the ring kernel's): kTW warps
// each own kTWBytes of every 32 KB chunk, i.e. kTV 16-byte vectors (kTWords 32-bit
// words) per thread per chunk; in TMEM each warp holds kTWords columns of its lane
// quarter per parked chunk (64 columns per chunk either way).
#ifndef AREAL_TMEM_WARPS
#define AREAL_TMEM_WARPS 16
#endif
constexpr int kTW = AREAL_TMEM_WARPS;
static_assert(kTW == 8 || kTW == 16, "TMEM K2: 8 or 16 math warps");
constexpr int kTWBytes = kChunkBytes / kTW;
constexpr int kTV = kTWBytes / 16 / 32;
constexpr int kTWords = kTV * 4;
constexpr int kTProducer = kTW, kTEpilogue = kTW + 1;
constexpr int kTThreads = kTW * 32 + 64;
constexpr int kTBarThreads = (kTW + 1) * 32;
__device__ __forceinline__ int t_vec_index(int warp, int lane, int j) {
  return warp * (kTWBytes / 16) + j * 32 + lane;
}
// Warp max of a float through one REDUX.MAX on an order-preserving integer image
// (one instruction instead of a 5-step shuffle/max chain on the per-chunk critical path).
#ifndef AREAL_K2_REDUX_MAX
#define AREAL_K2_REDUX_MAX 1
#endif
constexpr bool kRedux = AREAL_K2_REDUX_MAX != 0;
__device__ __forceinline__ float warp_max_redux(float v) {
  const int i = __float_as_int(v);
  const int k = i ^ ((i >> 31) & 0x7fffffff);  // signed-int order == float order (no NaN)
  const int m = __reduce_max_sync(0xffffffffu, k);
  return __int_as_float(m ^ ((m >> 31) & 0x7fffffff));
}

// Fixed per-row shift: each warp takes its exp2 shift from the row's first chunk
// (max via REDUX) and keeps it for the rest of the row, so later chunks need no max,
// no warp reduction and no rescale.  A later logit more than ~88 above that shift
// overflows e to inf; the epilogue sees a non-finite sum and recomputes the row's
// statistics from HBM (still intact: pass 2 has not started), and pass 2 then
// rebuilds dlogits from HBM too — a rare slow path, never a wrong result.
#ifndef AREAL_K2_FIXED_SHIFT
#define AREAL_K2_FIXED_SHIFT 1
#endif
constexpr bool kFixedShift = AREAL_K2_FIXED_SHIFT != 0;

// Upper bound on the lookahead chunks folded during the per-row epilogue.  Fewer
// lookahead chunks leave more ring slots to the producer during pass 2, so the read
// stream keeps flowing while dlogits are written: 3 measured best at the power cap
// (profiles/r01_k2_lookahead_sweep.txt: 6.27 vs 5.98 TB/s sustained at 5).
#ifndef AREAL_K2_LA_CAP
#define AREAL_K2_LA_CAP 3
#endif
constexpr int kLookaheadCap = AREAL_K2_LA_CAP;
// Rows held entirely in TMEM (R = 0: bf16 V <= 131,072, fp32 V <= 65,536) leave the
// whole ring to the stream, and a longer lookahead pays there: bf16 V = 131,072 at
// lookahead 3 / 4 / 5: 6.05 / 6.40 / 6.65 TB/s (profiles/r01_k2_lookahead_notail.txt).
#ifndef AREAL_K2_LA_CAP0
#define AREAL_K2_LA_CAP0 5
#endif
constexpr int kLookaheadCapNoTail = AREAL_K2_LA_CAP0;

#ifndef AREAL_K2_PACKED_BF16_MUL
#define AREAL_K2_PACKED_BF16_MUL 1
#endif
constexpr bool kK2PackedBf16Mul = AREAL_K2_PACKED_BF16_MUL != 0;

__device__ __forceinline__ __nv_bfloat162 bits_bf162(uint32_t u) {
  __nv_bfloat162 r;
  memcpy(&r, &u, 4);
  return r;
}
__device__ __forceinline__ uint32_t bf162_bits(__nv_bfloat162 v) {
  uint32_t u;
  memcpy(&u, &v, 4);
  return u;
}
// Per-row timeline probe hook (tools/k2_timeline_probe.cu); empty in the product.
#ifndef AREAL_K2_PROBE_TS
#define AREAL_K2_PROBE_TS(ev, it) {}
#endif
constexpr int kTmemCols = 512;
constexpr int kTmemMaxChunks = 14;    // TMEM + resident chunks: kTmemChunks + (nslots - 1)
// Resident-tail cap (rows of <= 8 + kTResMax chunks stream nothing).  7 = every ring
// slot (no lookahead on streaming rows) measured best: fp32 V=151,936 at R = 4 / 5 /
// 6 / 7: 5.69 / 5.68 / 5.83 / 5.98 TB/s (profiles/r01_k2_streamed_sweep.txt).
#ifndef AREAL_K2_RES_MAX
#define AREAL_K2_RES_MAX 7
#endif
constexpr int kTResMax = AREAL_K2_RES_MAX;
// L2 policy for rows with streamed chunks: bit 0 = TMA loads of streamed chunks
// evict_last (the rest evict_first) so pass 2's re-read hits L2; bit 1 = dlogits
// stores evict-first (st.global.cs) so they do not push those chunks out.
#ifndef AREAL_K2_L2_HINTS
#define AREAL_K2_L2_HINTS 3
#endif
constexpr int kL2Hints = AREAL_K2_L2_HINTS;
template <typename V>
__device__ __forceinline__ void st_out(V* p, V v, bool stream) {
  if (stream) __stcs(p, v);
  else *p = v;
}

// Dynamic row schedule: the producer takes each CTA's next row from a global counter
// (first row = blockIdx.x) and publishes the row sequence through rowq / rowpub; the
// math warps and the epilogue walk the same sequence.  With the static cid + k * grid
// assignment the launch waited for its slowest CTA: CTA spans over one launch ranged
// 2.87-3.01 ms around a 2.93 ms median (tools/k2_timeline_probe.cu); dynamic rows took
// K2 bf16 32768 x 151,936 from 6.45 to 6.86 TB/s in a burst (profiles/r02_k2_dynamic_rows.md).  The producer runs at most nslots + 3 rows ahead of the
// epilogue (one ring chunk per row at least), so kRowQ entries never wrap onto a live row.
constexpr int kRowQ = 16;
static_assert(kRowQ >= 7 + 3 + 1, "row queue shorter than the producer's lead");
// The objective / ratio / entropy sums are accumulated as 128-bit fixed point (2^-64
// units): each double is converted exactly (|x| < 2^62; bits below 2^-64 are floored),
// integer addition is associative, so the statistics do not depend on which CTA
// processed which rows (the row schedule is dynamic) and stay bit-reproducible.
struct Fx128 {
  __int128 v;  // sum * 2^64
  double nf;   // non-finite terms (inf / NaN), added as doubles
};
__device__ __forceinline__ void fx_add(Fx128& acc, double x) {
  if (!isfinite(x)) {
    acc.nf += x;
    return;
  }
  if (fabs(x) >= 0x1p62) {  // beyond the fixed-point range: counted as +-inf
    acc.nf += x > 0 ? INFINITY : -INFINITY;
    return;
  }
  int e;
  const double m = frexp(x, &e);                  // x = m 2^e, |m| in [0.5, 1) or 0
  const long long mi = (long long)ldexp(m, 53);   // exact 53-bit integer
  const int sh = e - 53 + 64;                     // x 2^64 = mi 2^sh, sh <= 73
  if (sh >= 0) acc.v += (__int128)mi << sh;
  else if (sh > -64) acc.v += (__int128)mi >> (-sh);  // floor: deterministic
}
__device__ __forceinline__ double fx_value(const Fx128& acc) {
  const long long hi = (long long)(acc.v >> 64);
  const unsigned long long lo = (unsigned long long)acc.v;
  return ((double)hi + ldexp((double)lo, -64)) + acc.nf;
}
struct TmemTail {
  int rowq[kRowQ];                            // row sequence (producer -> consumers)
  unsigned int rowpub;                        // rows published so far
  uint64_t bcbar[2];                          // epilogue -> math warps (row parity)
  float red[2][kTW][3];            // per-warp partials (row parity)
  RingBcast bc[2];
  double st[AREAL_N_STATS];                   // counters (exact integers in double)
  Fx128 fx[3];                                // objective, ratio, entropy sums
  // shift c of the stored e (row parity): TMEM chunks, then up to kTResMax resident
  // chunks (a streaming row's resident tail has kTResMax = 7 chunks: index 14)
  float cw[2][kTmemChunks + kTResMax][kTW];
};

// k-th row of this CTA's sequence (-1: none left).  Published well before it is needed
// (the producer announces row k+1 as soon as row k's last chunk is issued), so the
// acquire load almost never spins.
__device__ __forceinline__ int tmem_row(const TmemTail* tail, int k) {
  unsigned int pub;
  do {
    asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(pub) : "r"(smem_u32(&tail->rowpub)) : "memory");
  } while (pub <= (unsigned int)k);
  return tail->rowq[k % kRowQ];
}
__device__ __forceinline__ void tmem_publish_row(TmemTail* tail, int k, int row) {
  tail->rowq[k % kRowQ] = row;
  asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(smem_u32(&tail->rowpub)), "r"((unsigned int)(k + 1))
               : "memory");
}
// stats_add with the three sums in fixed point (see Fx128)
__device__ __forceinline__ void stats_add_fx(TmemTail* tail, const TokenTerms& t, double ent) {
  double* st = tail->st;
  fx_add(tail->fx[0], t.obj);
  st[AREAL_STAT_N_VALID] += t.valid ? 1.0 : 0.0;
  st[AREAL_STAT_N_CLIPPED] += t.clipped ? 1.0 : 0.0;
  if (t.valid) fx_add(tail->fx[1], t.ratio);
  st[AREAL_STAT_N_EXCLUDED] += t.valid ? 0.0 : 1.0;
  st[AREAL_STAT_N_MASKED] += t.masked ? 1.0 : 0.0;
  if (t.valid) fx_add(tail->fx[2], ent);
  st[AREAL_STAT_N_TOKENS] += 1.0;
}
// Grid reduction of the TMEM kernel's statistics: every CTA writes its counters and
// fixed-point sums to the workspace, the last CTA (atomic ticket) adds them up — integer
// sums, so the result does not depend on the order — and re-arms the ticket and the
// row counter.
__device__ void finalize_stats_fx(const PpoArgs& a, const TmemTail* tail) {
  __shared__ unsigned int s_last;
  // per-CTA record: 8 doubles (counters) + 3 x (lo, hi, nf)
  constexpr int kRec = AREAL_N_STATS + 9;
  double* rec = a.partials + (size_t)blockIdx.x * kRec;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int j = 0; j < AREAL_N_STATS; ++j) rec[j] = tail->st[j];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      reinterpret_cast<unsigned long long*>(rec)[AREAL_N_STATS + 3 * j] = (unsigned long long)tail->fx[j].v;
      reinterpret_cast<long long*>(rec)[AREAL_N_STATS + 3 * j + 1] = (long long)(tail->fx[j].v >> 64);
      rec[AREAL_N_STATS + 3 * j + 2] = tail->fx[j].nf;
    }
    __threadfence();
    const unsigned int ticket = atomicAdd(a.counter, 1u);
    s_last = (ticket == gridDim.x - 1) ? 1u : 0u;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (threadIdx.x < AREAL_N_STATS) {
    const int j = threadIdx.x;
    const volatile double* p = a.partials;
    double v;
    const int f = j == AREAL_STAT_OBJECTIVE_SUM ? 0 : j == AREAL_STAT_RATIO_SUM ? 1
                : j == AREAL_STAT_ENTROPY_SUM ? 2 : -1;
    if (f < 0) {
      v = 0.0;  // counters: integer-valued doubles, exact in any order
      for (unsigned int b = 0; b < gridDim.x; ++b) v += p[(size_t)b * kRec + j];
    } else {
      Fx128 acc{0, 0.0};
      const volatile unsigned long long* q = reinterpret_cast<const volatile unsigned long long*>(a.partials);
      for (unsigned int b = 0; b < gridDim.x; ++b) {
        const size_t o = (size_t)b * kRec + AREAL_N_STATS + 3 * f;
        acc.v += ((__int128)(long long)q[o + 1] << 64) | (__int128)q[o];
        acc.nf += p[o + 2];
      }
      v = fx_value(acc);
    }
    a.stats[j] += v;
  }
  if (threadIdx.x == 0) {
    *a.counter = 0u;
    a.counter[1] = 0u;  // dynamic row counter
  }
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tmem_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// TMEM address of math warp `warp`'s part of parked chunk t: lane quarter
// (warp % 4) in bits 31:16, kTWords columns per warp, kTW/4 warps per quarter per chunk.
__device__ __forceinline__ uint32_t tmem_addr(uint32_t base, int warp, int t) {
  return base + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(t * 64 + (warp >> 2) * kTWords);
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, "
      "%29, %30, %31, %32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),
      "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),
      "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tmem_ld32w(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, "
      "%30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
}
// this thread's kTWords words of a parked chunk <-> TMEM
template <int N>
__device__ __forceinline__ void tmem_stw(uint32_t taddr, const uint32_t (&r)[N]) {
  if constexpr (N == 16) tmem_st16(taddr, r);
  else tmem_st32(taddr, r);
}
template <int N>
__device__ __forceinline__ void tmem_ldw(uint32_t taddr, uint32_t (&r)[N]) {
  if constexpr (N == 16) tmem_ld16(taddr, r);
  else tmem_ld32w(taddr, r);
}

// This thread's share of a chunk as kTWords raw 32-bit words (kTV 16-byte vectors).
// FULL: the chunk is a whole 32 KB (no per-vector bounds checks).
template <bool FULL = false>
__device__ __forceinline__ void lds_raw(const uint4* q, int warp, int lane, int nvec,
                                        uint32_t (&w)[kTWords]) {
#pragma unroll
  for (int j = 0; j < kTV; ++j) {
    const int vi = t_vec_index(warp, lane, j);
    uint4 v = make_uint4(0, 0, 0, 0);
    if (FULL || vi < nvec) v = q[vi];
    w[4 * j + 0] = v.x;
    w[4 * j + 1] = v.y;
    w[4 * j + 2] = v.z;
    w[4 * j + 3] = v.w;
  }
}
template <bool FULL = false>
__device__ __forceinline__ void sts_raw(uint4* q, int warp, int lane, int nvec,
                                        const uint32_t (&w)[kTWords]) {
#pragma unroll
  for (int j = 0; j < kTV; ++j) {
    const int vi = t_vec_index(warp, lane, j);
    if (FULL || vi < nvec)
      q[vi] = make_uint4(w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
  }
}

// Stored-e format: bf16 bits for 16-bit logits (e in [0, 1] keeps fp32's exponent
// range), fp32 for fp32 logits.
template <typename T> struct EFmt;
template <> struct EFmt<__nv_bfloat16> { using V = Vec<__nv_bfloat16>; };
template <> struct EFmt<__half> { using V = Vec<__nv_bfloat16>; };
template <> struct EFmt<float> { using V = Vec<float>; };

// Pass-1 fold of one chunk held as raw words: warp-uniform running max, e computed
// once, the e words returned in place of the logits and the shift c returned.
template <typename T, bool ENT, bool FULL, bool UNAL>
__device__ __forceinline__ float fold_to_e(RowStat<float>& rs, uint32_t (&w)[kTWords], int warp, int lane,
                                           int nvec, int e0, int V) {
  constexpr int E = Vec<T>::N;
  constexpr int N = kTV * E;
  float f[N];
#pragma unroll
  for (int j = 0; j < kTV; ++j) {
    float g[E];
    Vec<T>::unpack(make_uint4(w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]), g);
    // non-FULL: vectors past the chunk's data are padding; on unaligned rows element
    // k of the chunk is row element e0 + k, valid in [0, V)
    const int vi = t_vec_index(warp, lane, j);
    const int i0 = e0 + vi * E;
#pragma unroll
    for (int e = 0; e < E; ++e)
      f[j * E + e] = (FULL || (UNAL ? (i0 + e >= 0 && i0 + e < V) : vi < nvec)) ? g[e]
                                                                             : Lim<float>::ninf();
  }
  // rs.m is warp-uniform; it stays -inf until a chunk with a finite value was seen
  const bool need_max = !kFixedShift || rs.m == Lim<float>::ninf();
  float lmax = Lim<float>::ninf();
  if (need_max) {
    lmax = f[0];
#pragma unroll
    for (int i = 1; i < N; ++i) lmax = fmaxf(lmax, f[i]);
    lmax = kRedux ? warp_max_redux(lmax) : warp_max(lmax);
  }
  const float mn = fmaxf(rs.m, lmax);
  const float muse = (mn == Lim<float>::ninf()) ? 0.f : mn;
  const float c = Ex<float>::shift(muse);
  const float r = (need_max && mn != rs.m) ? Ex<float>::rescale(rs.m, c) : 1.f;
  const float2 L2 = make_float2(Lim<float>::kLog2e, Lim<float>::kLog2e);
  const float2 C2 = make_float2(-c, -c);
  float2 s2 = make_float2(0.f, 0.f), x2 = make_float2(0.f, 0.f);
#pragma unroll
  for (int j = 0; j < kTV; ++j) {
    float ev[E];
#pragma unroll
    for (int k = 0; k < E; k += 2) {
      const float2 v = make_float2(f[j * E + k], f[j * E + k + 1]);
      const float2 t = ffma2(v, L2, C2);
      const float2 ee = make_float2(fast_exp2(t.x), fast_exp2(t.y));
      s2 = fadd2(s2, ee);
      if (ENT) {  // p log p := 0 at p = 0
        const float2 vc = make_float2(fmaxf(v.x, Lim<float>::lowest()), fmaxf(v.y, Lim<float>::lowest()));
        x2 = ffma2(ee, vc, x2);
      }
      ev[k] = ee.x;
      ev[k + 1] = ee.y;
    }
    const uint4 pk = EFmt<T>::V::pack(ev);
    w[4 * j + 0] = pk.x;
    w[4 * j + 1] = pk.y;
    w[4 * j + 2] = pk.z;
    w[4 * j + 3] = pk.w;
  }
  rs.s = rs.s * r + (s2.x + s2.y);
  if (ENT) rs.sx = rs.sx * r + (x2.x + x2.y);
  rs.m = mn;
  return c;
}

// Pass-1 step on one ring chunk: load this thread's words, fold them to e (returns
// the shift c); full 32 KB chunks take the branch-free path.
// Row geometry in the chunk stream: a row starting off a 16-byte boundary is loaded
// from the boundary below it, so chunk element k is row element e0 + k with
// e0 = c * per_chunk - head (head = the row's offset from that boundary, in elements).
template <typename T>
__device__ __forceinline__ bool region_valid(int warp, int e0, int V) {
  constexpr int W = kTWBytes / 16, E = Vec<T>::N;
  const int lo = e0 + warp * W * E;
  return lo >= 0 && lo + (int64_t)W * E <= V;
}
template <typename T, bool ENT, bool UNAL>
__device__ __forceinline__ float chunk_to_e(RowStat<float>& rs, const uint4* q, uint32_t (&wv)[kTWords],
                                            int warp, int lane, int nvec, int e0, int V) {
  if (UNAL ? region_valid<T>(warp, e0, V) : (warp + 1) * (kTWBytes / 16) <= nvec) {  // region all valid
    lds_raw<true>(q, warp, lane, nvec, wv);
    return fold_to_e<T, ENT, true, UNAL>(rs, wv, warp, lane, nvec, e0, V);
  }
  lds_raw<false>(q, warp, lane, nvec, wv);
  return fold_to_e<T, ENT, false, UNAL>(rs, wv, warp, lane, nvec, e0, V);
}
// Store one 16-byte vector of dlogits holding chunk elements [k, k + E) = row elements
// [i0, i0 + E): whole when they are all in the row, else element by element.
template <typename T>
__device__ __noinline__ void store_vec_part(uint4* dst, int vi, uint4 o, int i0, int V);
template <typename T>
__device__ __forceinline__ void store_vec(uint4* dst, int vi, uint4 o, int i0, int V,
                                          bool stream) {
  constexpr int E = Vec<T>::N;
  if (i0 >= 0 && i0 + E <= V) {
    if (stream) __stcs(dst + vi, o);
    else dst[vi] = o;
    return;
  }
  store_vec_part<T>(dst, vi, o, i0, V);  // a row's first / last vector (rare: out of line)
}
// The in-row elements of one vector, element by element.
template <typename T>
__device__ __noinline__ void store_vec_part(uint4* dst, int vi, uint4 o, int i0, int V) {
  constexpr int E = Vec<T>::N;
  const uint32_t w[4] = {o.x, o.y, o.z, o.w};
  if constexpr (sizeof(T) == 2) {
    unsigned short* d = reinterpret_cast<unsigned short*>(dst + vi);
#pragma unroll
    for (int e = 0; e < E; ++e)
      if (i0 + e >= 0 && i0 + e < V) d[e] = (unsigned short)(w[e >> 1] >> (16 * (e & 1)));
  } else {
    uint32_t* d = reinterpret_cast<uint32_t*>(dst + vi);
#pragma unroll
    for (int e = 0; e < E; ++e)
      if (i0 + e >= 0 && i0 + e < V) d[e] = w[e];
  }
}
// Per-row stream geometry: the row's offset from the 16-byte boundary below it (the
// chunk stream starts there) and the bytes of its last chunk.  Two ints, so they can
// live across the whole row; the pointers are recomputed where needed.
struct RowGeo {
  int hb;            // head bytes: row element 0 sits at stream byte hb
  int last_bytes;    // bytes of chunk nchunks - 1
  template <typename T> __device__ __forceinline__ int head() const { return hb / (int)sizeof(T); }
  __device__ __forceinline__ const char* src(const PpoArgs& a, int64_t row) const {
    return a.logits + row * a.ld_in_bytes - hb;
  }
  __device__ __forceinline__ char* dst(const PpoArgs& a, int64_t row) const {
    return a.dlogits + row * a.ld_out_bytes - hb;
  }
};
template <typename T, bool UNAL>
__device__ __forceinline__ RowGeo row_geo(const PpoArgs& a, int64_t row, int nchunks) {
  RowGeo g;
  g.hb = UNAL ? (int)((uintptr_t)(a.logits + row * a.ld_in_bytes) & 15) : 0;
  const int64_t sb = (g.hb + a.vocab * (int64_t)sizeof(T) + 15) & ~(int64_t)15;
  g.last_bytes = (int)(sb - (int64_t)(nchunks - 1) * kChunkBytes);
  return g;
}

// Pass 2 of a streamed chunk: this thread's vectors of chunk c re-read from the
// logits (last use: evict-first loads; in place safe, each thread reads exactly the
// vectors it then overwrites), dlogits = g 2^(x log2e - lse).
template <typename T, bool UNAL>
__device__ __forceinline__ void stream_chunk_dlogits(const PpoArgs& a, int64_t row, const RowGeo& geo,
                                                     int V, char* drow, int c, int nvec,
                                                     int warp, int lane, float g, float lse_s) {
  constexpr int E = Vec<T>::N;
  const int e0 = c * (kChunkBytes / (int)sizeof(T)) - geo.head<T>();
  const uint4* src = reinterpret_cast<const uint4*>(geo.src(a, row)) + (size_t)c * (kChunkBytes / 16);
  uint4* dst = reinterpret_cast<uint4*>(drow + (size_t)c * kChunkBytes);
  const float2 L2 = make_float2(Lim<float>::kLog2e, Lim<float>::kLog2e);
  const float2 C2 = make_float2(-lse_s, -lse_s);
  const float2 G2 = make_float2(g, g);
  uint4 v[kTV];
#pragma unroll
  for (int j = 0; j < kTV; ++j) {
    const int vi = t_vec_index(warp, lane, j);
    v[j] = vi < nvec ? __ldcs(src + vi) : make_uint4(0, 0, 0, 0);
  }
#pragma unroll
  for (int j = 0; j < kTV; ++j) {
    const int vi = t_vec_index(warp, lane, j);
    if (vi < nvec) {
      float f[E];
      Vec<T>::unpack(v[j], f);
#pragma unroll
      for (int e = 0; e < E; e += 2) {
        const float2 t = ffma2(make_float2(f[e], f[e + 1]), L2, C2);
        const float2 d = fmul2(make_float2(fast_exp2(t.x), fast_exp2(t.y)), G2);
        f[e] = d.x;
        f[e + 1] = d.y;
      }
      if constexpr (UNAL) store_vec<T>(dst, vi, Vec<T>::pack(f), e0 + vi * E, V, (kL2Hints & 2) != 0);
      else st_out(&dst[vi], Vec<T>::pack(f), (kL2Hints & 2) != 0);
    }
  }
}

// UNAL: rows that may start off a 16-byte boundary (separate instantiation, so the
// aligned rows' kernel keeps its register allocation).
template <typename T, bool ENT, bool UNAL>
__device__ __forceinline__ void tmem_k2_body(const PpoArgs& a) {
  static_assert(sizeof(T) == 2 || sizeof(T) == 4, "TMEM K2 path: 16/32-bit logits");
  using A = float;
  constexpr int E = Vec<T>::N;
  extern __shared__ __align__(128) unsigned char smem[];  // 1-D bulk copies need 16 B
  const uint32_t nslots = (uint32_t)a.nslots;
  unsigned char* ring = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)nslots * kChunkBytes);
  uint64_t* empty = full + nslots;
  TmemTail* tail = reinterpret_cast<TmemTail*>(empty + nslots);
  __shared__ uint32_t s_tmem_base;

  const int64_t row_bytes = a.vocab * (int64_t)sizeof(T);
  // chunks per row: the same for every row (the host checks that an unaligned row's
  // extra head bytes never add a chunk)
  const int nchunks = (int)((((row_bytes + 15) & ~(int64_t)15) + kChunkBytes - 1) / kChunkBytes);
  const int per_chunk = kChunkBytes / (int)sizeof(T);
  const int V = (int)a.vocab;  // < 2^31 (checked on the host)
  auto nvec_of = [&](int c, const RowGeo& g) { return (c < nchunks - 1 ? kChunkBytes : g.last_bytes) / 16; };
  const int ntm = min(nchunks, kTmemChunks);     // chunks parked in TMEM
  const int R = min(nchunks - ntm, kTResMax);  // resident tail chunks
  const int S = nchunks - ntm - R;               // streamed chunks [ntm, ntm + S)
  const int la_max = min(min((int)nslots - R, nchunks), R == 0 ? kLookaheadCapNoTail : kLookaheadCap);
  // shift slot of chunk c in cw[][]: TMEM chunks, then the resident tail
  auto cwi = [&](int c) { return c < ntm ? c : c - S; };

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (uint32_t s = 0; s < nslots; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kTW);
    }
    mbar_init(&tail->bcbar[0], 1);
    mbar_init(&tail->bcbar[1], 1);
    for (int j = 0; j < AREAL_N_STATS; ++j) tail->st[j] = 0.0;
    for (int j = 0; j < 3; ++j) tail->fx[j] = Fx128{0, 0.0};
    tail->rowpub = 0u;
    fence_mbar_init_cluster();
  }
  if (warp == kTEpilogue) {  // one warp allocates (and later frees) all of TMEM
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&s_tmem_base)),
                 "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    tmem_fence_before();
  }
  __syncthreads();
  tmem_fence_after();
  const uint32_t tbase = s_tmem_base;
  const int64_t cid = blockIdx.x, ncl = gridDim.x;

  if (warp == kTProducer) {
    // ================= producer: TMA bulk loads of whole rows, chunk by chunk
    if (lane == 0) {
      Cursor cur = {0u, 0u};
      uint32_t used = 0;
      const uint64_t pol_keep = l2_policy_evict_last(), pol_drop = l2_policy_evict_first();
      int64_t row = cid;
      for (int k = 0;; ++k) {
        tmem_publish_row(tail, k, row < a.n_rows ? (int)row : -1);
        if (row >= a.n_rows) break;
        // the next row: claimed now, used after this row's loads are issued
        const int64_t row_next = ncl + (int64_t)atomicAdd(a.counter + 1, 1u);
        const RowGeo geo = row_geo<T, UNAL>(a, row, nchunks);
        const char* src = geo.src(a, row);
        for (int c = 0; c < nchunks; ++c) {
          if (used >= nslots) mbar_wait(&empty[cur.slot], cur.phase ^ 1u);
          else ++used;
          if (c == 0) AREAL_K2_PROBE_TS(7, k)
          const uint32_t bytes = (uint32_t)(c < nchunks - 1 ? kChunkBytes : geo.last_bytes);
          mbar_arrive_expect_tx(&full[cur.slot], bytes);
          if ((kL2Hints & 1) && S > 0)
            bulk_g2s_hint(ring + (size_t)cur.slot * kChunkBytes, src + (size_t)c * kChunkBytes,
                          bytes, &full[cur.slot], (c >= ntm && c < ntm + S) ? pol_keep : pol_drop);
          else
            bulk_g2s(ring + (size_t)cur.slot * kChunkBytes, src + (size_t)c * kChunkBytes, bytes,
                     &full[cur.slot]);
          cur.next(nslots);
        }
        row = row_next;
      }
    }
  } else if (warp == kTEpilogue) {
    // ================= epilogue: merge the 16 partials, fp64 per-token epilogue
    for (int it = 0;; ++it) {
      const int row_i = tmem_row(tail, it);
      if (row_i < 0) break;
      const int64_t row = row_i;
      const int par = it & 1;
      int64_t idx = 0, tok = -1;
      double xa = 0.0, sc_behav = 0.0, sc_prox = 0.0, sc_adv = 0.0;
      int sc_ver = 0;
      if (lane == 0) {
        idx = a.row_index ? (int64_t)a.row_index[row] : row;
        tok = a.tokens[idx];
        xa = token_logit<T>(a, reinterpret_cast<const T*>(a.logits + row * a.ld_in_bytes), tok);
        sc_behav = a.behav[idx];
        sc_prox = a.prox ? a.prox[idx] : 0.0;
        sc_adv = a.adv[idx];
        sc_ver = a.versions ? a.versions[idx] : 0;
      }
      if (lane == 0) AREAL_K2_PROBE_TS(8, it)
      named_bar_sync(kBarPartials, kTBarThreads);
      if (lane == 0) AREAL_K2_PROBE_TS(0, it)
      RowStat<A> w;
      if (lane < kTW) {
        w.m = tail->red[par][lane][0];
        w.s = tail->red[par][lane][1];
        w.sx = tail->red[par][lane][2];
      } else {
        w.init();
      }
      RowStat<A> tot = warp_merge(w);
      if (lane == 0) AREAL_K2_PROBE_TS(9, it)
      const bool slow = kFixedShift && !(tot.s < INFINITY);  // overflow (or NaN logits)
      if (slow) {
        const int hb = (int)((uintptr_t)(a.logits + row * a.ld_in_bytes) & 15);
        if constexpr (UNAL) tot = row_stats_masked<T, ENT>(a, row, hb, lane);
        else tot = row_stats_global<T, ENT>(a, row, 0, (a.vocab * (int64_t)sizeof(T)) / 16, lane);
      }
      const A lse_s = Ex<A>::lse_shift(tot.m == Lim<A>::ninf() ? A(0) : tot.m, tot.s);
      const double lse = Ex<A>::lse_nat(lse_s);
      const double ent = ENT ? lse - (double)(tot.sx / tot.s) : 0.0;
      xa = __shfl_sync(0xffffffffu, xa, 0);
      const double lp = xa - lse;
      sc_behav = __shfl_sync(0xffffffffu, sc_behav, 0);
      sc_prox = __shfl_sync(0xffffffffu, sc_prox, 0);
      if (a.prox_from_lp) sc_prox = lp;  // first minibatch: prox is this lp
      const double arg = lane == 0 ? __dsub_rn(sc_prox, sc_behav)
                         : lane == 1 ? (a.decoupled ? __dsub_rn(lp, sc_prox) : __dsub_rn(lp, sc_behav))
                                     : lp;
      const double ex = exp(arg);
      const double e_scale = __shfl_sync(0xffffffffu, ex, 0);
      const double e_ratio = __shfl_sync(0xffffffffu, ex, 1);
      const double e_p = __shfl_sync(0xffffffffu, ex, 2);
      if (lane == 0) AREAL_K2_PROBE_TS(10, it)
      if (lane == 0) {
        const TokenTerms t = ppo_token_terms(a.decoupled ? e_scale : 1.0, e_ratio, sc_adv, sc_ver, a);
        const double gc = a.grad_scale * t.coef;
        AREAL_K2_PROBE_TS(11, it)
        RingBcast& b = tail->bc[par];
        b.gc = gc;
        b.lse = (double)lse_s;
        b.tok = tok;
        b.dtok = to_bits<T>(Traits<T>::from_acc((A)(gc * (e_p - 1.0))));
        b.slow = slow ? 1 : 0;
        mbar_arrive(&tail->bcbar[par]);
        AREAL_K2_PROBE_TS(1, it)
        stats_add_fx(tail, t, ent);
        if (a.lp_out) a.lp_out[idx] = lp;
        if (ENT && a.ent_out) a.ent_out[idx] = ent;
      }
    }
  } else {
    // ================= math warps
    Cursor cur = {0u, 0u};  // ring position of the current row's chunk 0
    int la = 0;             // chunks of the current row folded by the previous lookahead
    RowStat<A> carry;
    carry.init();
    for (int it = 0;; ++it) {
      const int row_i = tmem_row(tail, it);
      if (row_i < 0) break;
      const int64_t row = row_i;
      const int par = it & 1;
      float* cw = &tail->cw[par][0][0];  // [chunk][warp]
      const RowGeo geo = row_geo<T, UNAL>(a, row, nchunks);
      // ---- park the lookahead chunks (their e is in the ring slots) in TMEM
      Cursor cc = cur;
      for (int c = 0; c < la; ++c) {
        const int nvec = nvec_of(c, geo);
        uint32_t wv[kTWords];
        lds_raw(reinterpret_cast<const uint4*>(ring + (size_t)cc.slot * kChunkBytes), warp, lane,
                nvec, wv);
        tmem_stw(tmem_addr(tbase, warp, c), wv);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[cc.slot]);
        cc.next(nslots);
      }
      // ---- pass 1 over the remaining chunks: e to TMEM (slot freed at once) or in place
      RowStat<A> rs = carry;
      for (int c = la; c < nchunks; ++c) {
        mbar_wait(&full[cc.slot], cc.phase);
        const int nvec = nvec_of(c, geo);
        uint4* q = reinterpret_cast<uint4*>(ring + (size_t)cc.slot * kChunkBytes);
        uint32_t wv[kTWords];
        const float cshift =
            chunk_to_e<T, ENT, UNAL>(rs, q, wv, warp, lane, nvec, c * per_chunk - geo.head<T>(), V);
        if (c < ntm) {
          if (lane == 0) cw[c * kTW + warp] = cshift;
          tmem_stw(tmem_addr(tbase, warp, c), wv);
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[cc.slot]);
        } else if (c < ntm + S) {  // streamed: pass 2 re-reads it from global memory
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[cc.slot]);
        } else {
          if (lane == 0) cw[(c - S) * kTW + warp] = cshift;
          sts_raw(q, warp, lane, nvec, wv);  // resident tail chunk: e in place
        }
        cc.next(nslots);
      }
      const Cursor after = cc;
      tmem_wait_st();  // this row's parked chunks are in TMEM before pass 2 reads them
      rs = kMathWarpMerge ? warp_merge_ent<A, ENT>(rs) : (rs.warp_reduce(), rs);
      if (lane == 0) {
        tail->red[par][warp][0] = rs.m;
        tail->red[par][warp][1] = rs.s;
        tail->red[par][warp][2] = rs.sx;
      }
      if (lane == 0 && warp == 0) AREAL_K2_PROBE_TS(2, it)
      if (lane == 0 && warp == kTW - 1) AREAL_K2_PROBE_TS(3, it)
      named_bar_arrive(kBarPartials, kTBarThreads);
      // ---- lookahead: fold the next row's first chunks (e in place) during the epilogue
      const int row_nx = tmem_row(tail, it + 1);
      const bool has_next = row_nx >= 0;
      const int la_next = has_next ? la_max : 0;
      float* cwn = &tail->cw[par ^ 1][0][0];
      RowStat<A> nxt;
      nxt.init();
      Cursor lc = after;
      const RowGeo geo_n = (UNAL && has_next) ? row_geo<T, UNAL>(a, row_nx, nchunks) : geo;
      for (int c = 0; c < la_next; ++c) {
        mbar_wait(&full[lc.slot], lc.phase);
        const int nvec = nvec_of(c, geo_n);
        uint4* q = reinterpret_cast<uint4*>(ring + (size_t)lc.slot * kChunkBytes);
        uint32_t wv[kTWords];
        const float cshift =
            chunk_to_e<T, ENT, UNAL>(nxt, q, wv, warp, lane, nvec, c * per_chunk - geo_n.head<T>(), V);
        if (lane == 0) cwn[c * kTW + warp] = cshift;
        sts_raw(q, warp, lane, nvec, wv);
        lc.next(nslots);
      }
      carry = nxt;
      la = la_next;

      if (lane == 0 && warp == 0) AREAL_K2_PROBE_TS(4, it)
      mbar_wait(&tail->bcbar[par], (it >> 1) & 1);
      if (lane == 0 && warp == 0) AREAL_K2_PROBE_TS(5, it)
      const RingBcast b = tail->bc[par];
      const float g = (float)b.gc;
      const float lse_s = (float)b.lse;
      const T dtok = from_bits<T>(b.dtok);
      char* drow = geo.dst(a, row);  // chunk-stream base of this row's dlogits
      // ---- pass 2: dlogits = e * g 2^(c - lse), 16-byte stores.  Full chunks are
      // branch-free; the one-hot element is patched afterwards by the thread that
      // stored its vector (same-thread program order => the patch lands last).
      // g == 0 rows still multiply (0 * e): NaN/inf logits give NaN, like the
      // reference's coef * (onehot - softmax).
      if (kFixedShift && b.slow) {
        // slow path: dlogits = g 2^(x log2e - lse) rebuilt from the row in HBM (each
        // thread reads exactly the vectors it then overwrites: in-place safe)
        const uint4* xrow = reinterpret_cast<const uint4*>(geo.src(a, row));
        const float2 L2 = make_float2(Lim<float>::kLog2e, Lim<float>::kLog2e);
        const float2 C2 = make_float2(-lse_s, -lse_s);
        const float2 G2 = make_float2(g, g);
        Cursor cs = cur;
        for (int c = 0; c < nchunks; ++c) {
          const int nvec = nvec_of(c, geo);
          const int e0 = c * per_chunk - geo.head<T>();
          if (c >= ntm + S) {  // resident tail chunk: release its ring slot as usual
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[cs.slot]);
          }
          const uint4* src = xrow + (size_t)c * (kChunkBytes / 16);
          uint4* dst = reinterpret_cast<uint4*>(drow + (size_t)c * kChunkBytes);
#pragma unroll
          for (int j = 0; j < kTV; ++j) {
            const int vi = t_vec_index(warp, lane, j);
            if (vi < nvec) {
              float f[E];
              Vec<T>::unpack(src[vi], f);
#pragma unroll
              for (int e = 0; e < E; e += 2) {
                const float2 t = ffma2(make_float2(f[e], f[e + 1]), L2, C2);
                const float2 d = fmul2(make_float2(fast_exp2(t.x), fast_exp2(t.y)), G2);
                f[e] = d.x;
                f[e + 1] = d.y;
              }
              if constexpr (UNAL) store_vec<T>(dst, vi, Vec<T>::pack(f), e0 + vi * E, V, false);
              else dst[vi] = Vec<T>::pack(f);
            }
          }
          cs.next(nslots);
        }
      } else {
      // dlogits stores: evict-first only on rows with streamed chunks (their re-read must
      // stay in L2); the two store flavours are separate loops, not per-store predicates
      auto pass2 = [&](auto stream_tag) {
        constexpr bool ST = decltype(stream_tag)::value;
        uint32_t rslot = (cur.slot + (uint32_t)(ntm + S)) % nslots;  // first resident chunk's slot
        for (int c = 0; c < nchunks; ++c) {
          const int nvec = nvec_of(c, geo);
          const int e0 = c * per_chunk - geo.head<T>();
          const bool full = UNAL ? region_valid<T>(warp, e0, V)
                                 : (warp + 1) * (kTWBytes / 16) <= nvec;  // this warp's region
          uint32_t wv[kTWords];
          if (c >= ntm && c < ntm + S) {  // streamed chunk: dlogits from the logits
            stream_chunk_dlogits<T, UNAL>(a, row, geo, V, drow, c, nvec, warp, lane, g, lse_s);
            continue;
          }
          if (c < ntm) {
            tmem_ldw(tmem_addr(tbase, warp, c), wv);
            tmem_wait_ld();
          } else {  // resident tail chunk (its full barrier completed in pass 1)
            const uint4* q = reinterpret_cast<const uint4*>(ring + (size_t)rslot * kChunkBytes);
            if (full) lds_raw<true>(q, warp, lane, nvec, wv);
            else lds_raw<false>(q, warp, lane, nvec, wv);
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[rslot]);
            if (++rslot == nslots) rslot = 0;
          }
          const float F = g * fast_exp2(cw[cwi(c) * kTW + warp] - lse_s);
          const float2 F2 = make_float2(F, F);
          uint4* dst = reinterpret_cast<uint4*>(drow + (size_t)c * kChunkBytes);
          // bf16 logits: e is stored as bf16 pairs, so dlogit = e * F is one packed
          // bf16x2 multiply per two logits (HMUL2.BF16; F rounded to bf16, <= 2^-8
          // relative, inside the bf16 contract) instead of unpack + FMUL2 + repack.
          constexpr bool kPackedMul = std::is_same<T, __nv_bfloat16>::value && kK2PackedBf16Mul;
          const __nv_bfloat162 Fb = __float2bfloat162_rn(F);
          auto put = [&](int j, uint4 o) {
            const int vi = t_vec_index(warp, lane, j);
            if (!UNAL || full) st_out(&dst[vi], o, ST);
            else store_vec<T>(dst, vi, o, e0 + vi * E, V, ST);
          };
          auto scale_store = [&](int j) {
            if constexpr (kPackedMul) {
              uint4 o;
              o.x = bf162_bits(__hmul2(bits_bf162(wv[4 * j + 0]), Fb));
              o.y = bf162_bits(__hmul2(bits_bf162(wv[4 * j + 1]), Fb));
              o.z = bf162_bits(__hmul2(bits_bf162(wv[4 * j + 2]), Fb));
              o.w = bf162_bits(__hmul2(bits_bf162(wv[4 * j + 3]), Fb));
              put(j, o);
            } else {
              float f[E];
              EFmt<T>::V::unpack(make_uint4(wv[4 * j], wv[4 * j + 1], wv[4 * j + 2], wv[4 * j + 3]), f);
#pragma unroll
              for (int e = 0; e < E; e += 2) {
                const float2 d = fmul2(make_float2(f[e], f[e + 1]), F2);
                f[e] = d.x;
                f[e + 1] = d.y;
              }
              put(j, Vec<T>::pack(f));
            }
          };
          if (full) {  // branch-free
#pragma unroll
            for (int j = 0; j < kTV; ++j) scale_store(j);
          } else {
#pragma unroll
            for (int j = 0; j < kTV; ++j)
              if (t_vec_index(warp, lane, j) < nvec) scale_store(j);
          }
        }
      };
      if ((kL2Hints & 2) && S > 0) pass2(std::true_type{});
      else pass2(std::false_type{});
      }  // fast path
      {  // the one-hot element: owner of vector vt of chunk ct (stream index st)
        if (b.tok >= 0 && b.tok < a.vocab) {
          const int64_t st = b.tok + geo.head<T>();
          const int ct = (int)(st / per_chunk);
          const int vt = (int)((st - (int64_t)ct * per_chunk) / E);
          if (warp == vt / (kTWBytes / 16) && lane == (vt & 31))
            reinterpret_cast<T*>(drow)[st] = dtok;
        }
      }
      if (lane == 0 && warp == 0) AREAL_K2_PROBE_TS(6, it)
      cur = after;
    }
    tmem_fence_before();
  }
  __syncthreads();
  if (warp == kTEpilogue) {
    tmem_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(kTmemCols)
                 : "memory");
  }
  finalize_stats_fx(a, tail);
}

}  // namespace areal
