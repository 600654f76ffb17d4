// ppo_ring.cuh — the persistent, warp-specialised TMA-ring kernels for K1/K2 (sm_100a).
// Included by ppo_kernels.cu (needs PpoArgs, ppo_token*, Vec, Ex, RowStat, ...).
//
// Roles per CTA (one CTA per SM, 18 warps):
//   warp 16 (producer) : one lane streams this CTA's slice of each row into a ring
//                        of 32 KB shared-memory chunks with 1-D TMA bulk copies
//                        (cp.async.bulk ... mbarrier::complete_tx), full/empty
//                        mbarriers per slot;
//   warps 0-15 (math)  : pass 1 folds (max, sum e^x, sum e^x x) per chunk with
//                        packed f32x2 math; partials go to shared memory with a
//                        non-blocking bar.arrive; K2 then folds the first chunks
//                        of the NEXT row already in spare slots (lookahead) while
//                        the epilogue warp works, waits for the row's gradient
//                        coefficient on an mbarrier, rewrites the resident chunks
//                        in place as dlogits and bulk-stores them per warp;
//   warp 17 (epilogue) : merges the 16 partials, exchanges them across the
//                        thread-block cluster through DSMEM (vocab split over
//                        CS CTAs), runs the fp64 per-token epilogue (its exps
//                        spread over lanes), writes lp / entropy / stats and
//                        publishes (g, lse, one-hot dlogit) to the math warps.
#pragma once

namespace areal {

constexpr int kChunkBytes = 32768;
constexpr int kConsumerWarps = 16;
constexpr int kConsumers = kConsumerWarps * 32;
constexpr int kProducerWarp = kConsumerWarps;
constexpr int kEpilogueWarp = kConsumerWarps + 1;
constexpr int kRingThreads = kConsumers + 64;   // + producer warp + epilogue warp
constexpr int kBarPartials = 1;                 // named barrier: math warps arrive, epilogue syncs
constexpr int kBarPartialsThreads = kConsumers + 32;
constexpr int kVecPerThread = kChunkBytes / 16 / kConsumers;  // 16-byte vectors per thread per chunk
constexpr int kWarpBytes = kChunkBytes / kConsumerWarps;      // contiguous bytes a warp owns per chunk

struct RingBcast {
  double gc;                // grad_scale * coef
  double lse;               // lse in shift units
  long long tok;            // token id
  unsigned long long dtok;  // dlogit of the token element (T bits)
  int slow;                 // TMEM K2: statistics recomputed from HBM (fixed-shift overflow)
};

// K1 dynamic row schedule (single-CTA rows, workspace given): like the TMEM K2, the
// producer claims each next row from a workspace counter and publishes the sequence
// (rowq / rowpub); it runs at most nslots + 3 rows ahead of the epilogue.
constexpr int kRingRowQ = 16;
#ifndef AREAL_K1_DYNAMIC
#define AREAL_K1_DYNAMIC 1
#endif
constexpr bool kK1Dynamic = AREAL_K1_DYNAMIC != 0;
struct RingSmemTail {
  int rowq[kRingRowQ];
  unsigned int rowpub;
  uint64_t xbar[2];                 // DSMEM exchange barriers (double-buffered by row parity)
  uint64_t bcbar[2];                // epilogue -> math warps (double-buffered by row parity)
  double xval[2][8][3];             // [parity][rank][m, s, sx]
  float redf[2][kConsumerWarps][3]; // per-warp partials, double-buffered by row parity
  double redd[2][kConsumerWarps][3];
  RingBcast bc[2];
  double st[AREAL_N_STATS];         // epilogue warp's running statistics
};

template <typename A> __device__ __forceinline__ A* red_ptr(RingSmemTail* t, int par);
template <> __device__ __forceinline__ float* red_ptr<float>(RingSmemTail* t, int par) {
  return &t->redf[par][0][0];
}
template <> __device__ __forceinline__ double* red_ptr<double>(RingSmemTail* t, int par) {
  return &t->redd[par][0][0];
}

// Ring cursor: slot index and mbarrier phase parity, advanced without division.
struct Cursor {
  uint32_t slot, phase;
  __device__ __forceinline__ void next(uint32_t nslots) {
    if (++slot == nslots) {
      slot = 0;
      phase ^= 1u;
    }
  }
};

__device__ __forceinline__ void named_bar_arrive(int id, int nthreads) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Vector j (< kVecPerThread) of this thread inside a chunk: each warp owns a
// contiguous kWarpBytes region, lanes read consecutive 16-byte vectors.
__device__ __forceinline__ int vec_index(int warp, int lane, int j) {
  return warp * (kWarpBytes / 16) + j * 32 + lane;
}

// Load this thread's vectors of a chunk (nvec valid vectors) as accumulation values.
// UNAL (K1 on rows off a 16-byte boundary): chunk element k is row element e0 + k and
// only [0, V) of the row counts.
template <typename T, bool UNAL = false>
__device__ __forceinline__ void load_values(const uint4* q, int warp, int lane, int nvec,
                                            typename Traits<T>::Acc* f, int e0 = 0, int V = 0) {
  using A = typename Traits<T>::Acc;
  constexpr int E = Vec<T>::N;
  const bool whole = UNAL ? (e0 + warp * (kWarpBytes / 16) * E >= 0 &&
                             e0 + (warp + 1) * (kWarpBytes / 16) * E <= V)
                          : (warp + 1) * (kWarpBytes / 16) <= nvec;
  if (whole) {  // this warp's 2 KB all valid: branch-free
#pragma unroll
    for (int j = 0; j < kVecPerThread; ++j) {
      A g[E];
      Vec<T>::unpack(q[vec_index(warp, lane, j)], g);
#pragma unroll
      for (int e = 0; e < E; ++e) f[j * E + e] = g[e];
    }
  } else {
#pragma unroll
    for (int j = 0; j < kVecPerThread; ++j) {
      const int vi = vec_index(warp, lane, j);
      A g[E];
      if (vi < nvec) {
        Vec<T>::unpack(q[vi], g);
      } else {
#pragma unroll
        for (int e = 0; e < E; ++e) g[e] = Lim<A>::ninf();
      }
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int i = e0 + vi * E + e;
        f[j * E + e] = (!UNAL || (i >= 0 && i < V)) ? g[e] : Lim<A>::ninf();
      }
    }
  }
}

// Diagnostic build knob (tools/variants.py): every K1 math thread arrives on the
// slot's empty barrier itself, instead of lane 0 after __syncwarp.  Same ordering;
// lets compute-sanitizer racecheck see the per-thread release (it does not model the
// __syncwarp -> lane-0 arrive chain).
#ifndef AREAL_K1_ARRIVE_ALL_LANES
#define AREAL_K1_ARRIVE_ALL_LANES 0
#endif
constexpr bool kK1ArriveAllLanes = AREAL_K1_ARRIVE_ALL_LANES != 0;

// Math warps fold their 32 lanes' row statistics with one max, one rescale exp per
// lane and sum butterflies (warp_merge) instead of five pairwise merge rounds.
#ifndef AREAL_MATH_WARP_MERGE
#define AREAL_MATH_WARP_MERGE 1
#endif
constexpr bool kMathWarpMerge = AREAL_MATH_WARP_MERGE != 0;

#ifndef AREAL_POLY_EVERY
#define AREAL_POLY_EVERY 8
#endif
constexpr int kPolyEvery = AREAL_POLY_EVERY;  // 0 disables the MUFU offload

// Exact (max, sum 2^x, sum 2^x * x) of the 16-byte vectors [v0, v1) of a row straight
// from HBM, one warp, two passes: the slow path of the fixed-shift folds (K1 here,
// K2 in ppo_tmem.cuh) when a logit overflowed the row's shift.
template <typename T, bool ENT>
__device__ __noinline__ RowStat<float> row_stats_global(const PpoArgs& a, int64_t row, int64_t v0,
                                                        int64_t v1, int lane) {
  constexpr int E = Vec<T>::N;
  const uint4* q = reinterpret_cast<const uint4*>(a.logits + row * a.ld_in_bytes);
  float m = Lim<float>::ninf();
  for (int64_t i = v0 + lane; i < v1; i += 32) {
    float f[E];
    Vec<T>::unpack(q[i], f);
#pragma unroll
    for (int e = 0; e < E; ++e) m = fmaxf(m, f[e]);
  }
  m = warp_max(m);
  const float c = (m == Lim<float>::ninf()) ? 0.f : m * Lim<float>::kLog2e;
  float s = 0.f, sx = 0.f;
  for (int64_t i = v0 + lane; i < v1; i += 32) {
    float f[E];
    Vec<T>::unpack(q[i], f);
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const float ee = fast_exp2(fmaf(f[e], Lim<float>::kLog2e, -c));
      s += ee;
      if (ENT) sx = fmaf(ee, fmaxf(f[e], Lim<float>::lowest()), sx);
    }
  }
  RowStat<float> r;
  r.m = m;
  r.s = warp_sum(s);
  r.sx = ENT ? warp_sum(sx) : 0.f;
  return r;
}

// The same for a row that starts hb bytes past the 16-byte boundary the vectors are
// read from (TMEM K2 on unaligned rows): elements outside the row are skipped.
template <typename T, bool ENT>
__device__ __noinline__ RowStat<float> row_stats_masked(const PpoArgs& a, int64_t row, int hb,
                                                        int lane) {
  constexpr int E = Vec<T>::N;
  const uint4* q = reinterpret_cast<const uint4*>(a.logits + row * a.ld_in_bytes - hb);
  const int64_t lo = hb / (int)sizeof(T), hi = lo + a.vocab;  // row = stream elements [lo, hi)
  const int64_t nv = (hb + a.vocab * (int64_t)sizeof(T) + 15) / 16;
  float m = Lim<float>::ninf();
  for (int64_t i = lane; i < nv; i += 32) {
    float f[E];
    Vec<T>::unpack(q[i], f);
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const bool in = i * E + e >= lo && i * E + e < hi;
      m = in ? fmaxf(m, f[e]) : m;
    }
  }
  m = warp_max(m);
  const float c = (m == Lim<float>::ninf()) ? 0.f : m * Lim<float>::kLog2e;
  float s = 0.f, sx = 0.f;
  for (int64_t i = lane; i < nv; i += 32) {
    float f[E];
    Vec<T>::unpack(q[i], f);
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const bool in = i * E + e >= lo && i * E + e < hi;
      const float ee = in ? fast_exp2(fmaf(f[e], Lim<float>::kLog2e, -c)) : 0.f;
      s += ee;
      if (ENT) sx = in ? fmaf(ee, fmaxf(f[e], Lim<float>::lowest()), sx) : sx;
    }
  }
  RowStat<float> r;
  r.m = m;
  r.s = warp_sum(s);
  r.sx = ENT ? warp_sum(sx) : 0.f;
  return r;
}

// K1 fixed shift: each thread takes its exp2 shift from its first chunk of the row
// and keeps it (no per-chunk max / rescale afterwards); overflow (a later logit
// > ~88 above the shift) shows up as a non-finite sum and the epilogue recomputes
// the row's statistics from HBM (row_stats_global).
#ifndef AREAL_K1_FIXED_SHIFT
#define AREAL_K1_FIXED_SHIFT 1
#endif
constexpr bool kK1FixedShift = AREAL_K1_FIXED_SHIFT != 0;

// Fold this thread's values of one chunk into its running (m, s, sx).
// fp32: packed f32x2 FFMA2/FADD2 around the MUFU ex2; fp64: scalar libdevice exp.
template <typename T, bool ENT, bool FIXED = false>
__device__ __forceinline__ void fold_values(RowStat<typename Traits<T>::Acc>& rs,
                                            const typename Traits<T>::Acc* f) {
  using A = typename Traits<T>::Acc;
  constexpr int N = kVecPerThread * Vec<T>::N;
  const bool need_max = !FIXED || rs.m == Lim<A>::ninf();
  A lmax = Lim<A>::ninf();
  if (need_max) {
    lmax = f[0];
#pragma unroll
    for (int i = 1; i < N; ++i) lmax = fmax(lmax, f[i]);
  }
  const A mn = fmax(rs.m, lmax);
  const A muse = (mn == Lim<A>::ninf()) ? A(0) : mn;
  const A c = Ex<A>::shift(muse);
  // rescale of the running sums (0 while m = -inf; exactly 1 when the max did not move)
  const A r = (need_max && mn != rs.m) ? Ex<A>::rescale(rs.m, c) : A(1);
  if constexpr (std::is_same<A, float>::value) {
    const float2 L2 = make_float2(Lim<float>::kLog2e, Lim<float>::kLog2e);
    const float2 C2 = make_float2(-c, -c);
    float2 s2 = make_float2(0.f, 0.f), x2 = make_float2(0.f, 0.f);
#pragma unroll
    for (int i = 0; i < N; i += 2) {
      const float2 v = make_float2(f[i], f[i + 1]);
      const float2 t = ffma2(v, L2, C2);
      // 16-bit logits: every kPolyEvery-th pair takes 2^t on the FMA pipe (MUFU
      // offload; 7.5e-5 relative error, far inside the bf16 tolerance).  Padding
      // lanes (-inf) must give exactly 0 for the entropy term.
      constexpr bool kPoly = sizeof(T) == 2 && kPolyEvery > 0;
      float2 e;
      if (kPoly && ((i >> 1) % kPolyEvery) == kPolyEvery - 1) {
        e = exp2_poly3(t);
        if (ENT) {
          e.x = t.x < -126.f ? 0.f : e.x;
          e.y = t.y < -126.f ? 0.f : e.y;
        }
      } else {
        e = make_float2(fast_exp2(t.x), fast_exp2(t.y));
      }
      s2 = fadd2(s2, e);
      if (ENT) {  // p log p := 0 at p = 0
        const float2 vc = make_float2(fmaxf(v.x, Lim<float>::lowest()), fmaxf(v.y, Lim<float>::lowest()));
        x2 = ffma2(e, vc, x2);
      }
    }
    rs.s = rs.s * r + (s2.x + s2.y);
    if (ENT) rs.sx = rs.sx * r + (x2.x + x2.y);
  } else {
    A s0 = A(0), x0 = A(0);
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const A e = Ex<A>::e(f[i], c);
      s0 += e;
      if (ENT) x0 += e * fmax(f[i], Lim<A>::lowest());
    }
    rs.s = rs.s * r + s0;
    if (ENT) rs.sx = rs.sx * r + x0;
  }
  rs.m = mn;
}

// Merge the warp's per-lane partials into one (max, sum, sum*x), identical on every
// lane: max-reduce, one rescale exp per lane, then two sum-reduces (XOR
// butterflies, fixed order => deterministic and bitwise equal across lanes).
template <typename A, bool ENT>
__device__ __forceinline__ RowStat<A> warp_merge_ent(const RowStat<A>& w) {
  const A M = warp_max(w.m);
  const A muse = (M == Lim<A>::ninf()) ? A(0) : M;
  const A f = (w.m == Lim<A>::ninf()) ? A(0) : Ex<A>::rescale(w.m, Ex<A>::shift(muse));
  A s = w.s * f, sx = ENT ? w.sx * f : A(0);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    if (ENT) sx += __shfl_xor_sync(0xffffffffu, sx, o);
  }
  RowStat<A> r;
  r.m = M;
  r.s = s;
  r.sx = sx;
  return r;
}

template <typename A>
__device__ __forceinline__ RowStat<A> warp_merge(const RowStat<A>& w) {
  return warp_merge_ent<A, true>(w);
}

template <typename T> __device__ __forceinline__ unsigned long long to_bits(T v) {
  unsigned long long b = 0;
  memcpy(&b, &v, sizeof(T));
  return b;
}
template <typename T> __device__ __forceinline__ T from_bits(unsigned long long b) {
  T v;
  memcpy(&v, &b, sizeof(T));
  return v;
}

template <typename T, bool BWD, bool ENT, bool UNAL = false>
__device__ __forceinline__ void row_ring_body(const PpoArgs& a) {
  static_assert(!UNAL || !BWD, "unaligned rows: K1 only (K2 runs the TMEM kernel)");
  using A = typename Traits<T>::Acc;
  constexpr int E = Vec<T>::N;                 // elements per 16 bytes
  constexpr int NV = kVecPerThread * E;        // values per thread per chunk
  extern __shared__ __align__(128) unsigned char smem[];  // 1-D bulk copies need 16 B
  const uint32_t nslots = (uint32_t)a.nslots;
  unsigned char* ring = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)nslots * kChunkBytes);
  uint64_t* empty = full + nslots;
  RingSmemTail* tail = reinterpret_cast<RingSmemTail*>(empty + nslots);

  // K1 (fp32 accumulation) folds with a fixed per-thread shift; K2-ring keeps the
  // running max (its rows may be split over a cluster; the TMEM K2 has its own)
  constexpr bool kFold1Fixed = !BWD && kK1FixedShift && std::is_same<A, float>::value;
  const int CS = a.cluster_size;
  const uint32_t rank = CS > 1 ? cluster_ctarank() : 0u;
  const int64_t cid = CS > 1 ? (int64_t)cluster_id_x() : (int64_t)blockIdx.x;
  const int64_t ncl = CS > 1 ? (int64_t)nclusters_x() : (int64_t)gridDim.x;
  const int64_t V16 = (a.vocab * (int64_t)sizeof(T)) / 16;
  const int64_t b16 = (int64_t)rank * a.slice16;
  const int64_t e16 = min(V16, b16 + a.slice16);
  const int slice_bytes = e16 > b16 ? (int)((e16 - b16) * 16) : 0;  // < 2^31 (checked on host)
  const int nfull = slice_bytes / kChunkBytes;
  const int last_bytes = slice_bytes - nfull * kChunkBytes;
  // UNAL: V16 rounds the row down, so count chunks on the 16-byte-rounded-up row
  const int nchunks = UNAL ? (int)((((a.vocab * (int64_t)sizeof(T) + 15) & ~(int64_t)15) + kChunkBytes - 1) / kChunkBytes)
                           : nfull + (last_bytes > 0 ? 1 : 0);
  // per row (UNAL): head bytes below the row start, bytes of the last chunk
  auto row_hb = [&](int64_t row) {
    return UNAL ? (int)((uintptr_t)(a.logits + row * a.ld_in_bytes) & 15) : 0;
  };
  auto chunk_bytes = [&](int c, int hb) {
    if (!UNAL) return c < nfull ? kChunkBytes : last_bytes;
    const int64_t sb = (hb + a.vocab * (int64_t)sizeof(T) + 15) & ~(int64_t)15;
    return c < nchunks - 1 ? kChunkBytes : (int)(sb - (int64_t)(nchunks - 1) * kChunkBytes);
  };
  const int64_t slice_e0 = b16 * E;  // first vocab element of this rank's slice

  const int tid = threadIdx.x;
  if (tid == 0) {
    for (uint32_t s = 0; s < nslots; ++s) {
      mbar_init(&full[s], 1);
      // one arrive per math warp per use (K1 diagnostic build: one per math thread)
      mbar_init(&empty[s], (!BWD && kK1ArriveAllLanes) ? kConsumerWarps * 32 : kConsumerWarps);
    }
    mbar_init(&tail->xbar[0], CS);
    mbar_init(&tail->xbar[1], CS);
    mbar_init(&tail->bcbar[0], 1);
    mbar_init(&tail->bcbar[1], 1);
    for (int j = 0; j < AREAL_N_STATS; ++j) tail->st[j] = 0.0;
    tail->rowpub = 0u;
    fence_mbar_init_cluster();
  }
  __syncthreads();
  if (CS > 1) cluster_sync_all();  // peers' exchange barriers initialised before any remote arrive
  // K1 on single-CTA rows takes its rows dynamically (workspace counters 2 and 3: next
  // row, exit ticket); K2 on the ring keeps the static order its CTA-order statistics need
  const bool dyn = kK1Dynamic && !BWD && CS == 1 && a.counter != nullptr;
  unsigned int* const row_ctr = dyn ? a.counter + 2 : nullptr;
  // it-th row of this CTA (-1: none left)
  auto row_at = [&](int it) -> int64_t {
    if (dyn) {
      unsigned int pub;
      do {
        asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(pub) : "r"(smem_u32(&tail->rowpub)) : "memory");
      } while (pub <= (unsigned int)it);
      return tail->rowq[it % kRingRowQ];
    }
    const int64_t r = cid + (int64_t)it * ncl;
    return r < a.n_rows ? r : -1;
  };

  const int warp = tid >> 5, lane = tid & 31;
  if (warp == kProducerWarp) {
    // ================= producer: one elected lane issues the TMA bulk loads
    if (lane == 0) {
      Cursor cur = {0u, 0u};
      uint32_t used = 0;  // slots filled at least once (no wait needed on first use)
      int64_t row = cid;
      for (int k = 0;; ++k) {
        if (dyn) {
          tail->rowq[k % kRingRowQ] = row < a.n_rows ? (int)row : -1;
          asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(smem_u32(&tail->rowpub)), "r"((unsigned int)(k + 1))
                       : "memory");
        }
        if (row >= a.n_rows) break;
        const int64_t row_next = dyn ? ncl + (int64_t)atomicAdd(row_ctr, 1u) : row + ncl;
        const int hb = row_hb(row);
        const char* src = a.logits + row * a.ld_in_bytes + b16 * 16 - hb;
        for (int c = 0; c < nchunks; ++c) {
          if (used >= nslots) mbar_wait(&empty[cur.slot], cur.phase ^ 1u);
          else ++used;
          const uint32_t bytes = (uint32_t)chunk_bytes(c, hb);
          mbar_arrive_expect_tx(&full[cur.slot], bytes);
          bulk_g2s(ring + (size_t)cur.slot * kChunkBytes, src + (size_t)c * kChunkBytes, bytes,
                   &full[cur.slot]);
          cur.next(nslots);
        }
        row = row_next;
      }
    }
  } else if (warp == kEpilogueWarp) {
    // ================= epilogue: merge, cluster exchange, fp64 per-token epilogue
    for (int it = 0;; ++it) {
      const int64_t row = row_at(it);
      if (row < 0) break;
      const int par = it & 1;
      // this row's token and scalars: plain loads issued now, consumed after the
      // math warps finish pass 1 (the warp is otherwise idle meanwhile)
      int64_t idx = 0, tok = -1;
      double xa = 0.0, sc_behav = 0.0, sc_prox = 0.0, sc_adv = 0.0;
      int sc_ver = 0;
      if (lane == 0) {
        idx = a.row_index ? (int64_t)a.row_index[row] : row;
        tok = a.tokens[idx];
        xa = token_logit<T>(a, reinterpret_cast<const T*>(a.logits + row * a.ld_in_bytes), tok);
        if (BWD) {
          sc_behav = a.behav[idx];
          sc_prox = a.prox ? a.prox[idx] : 0.0;
          sc_adv = a.adv[idx];
          sc_ver = a.versions ? a.versions[idx] : 0;
        }
      }
      named_bar_sync(kBarPartials, kBarPartialsThreads);  // all 16 partials are in red[par]
      const A* red = red_ptr<A>(tail, par);
      RowStat<A> w;
      if (lane < kConsumerWarps) {
        w.m = red[lane * 3 + 0];
        w.s = red[lane * 3 + 1];
        w.sx = red[lane * 3 + 2];
      } else {
        w.init();
      }
      w = warp_merge(w);  // every lane holds the CTA total
      if (!BWD && lane == 0) mbar_arrive(&tail->bcbar[par]);  // K1: partials consumed
      if constexpr (kFold1Fixed) {
        if (!(w.s < INFINITY)) {  // fixed-shift overflow (or NaN): exact, from HBM
          if constexpr (UNAL) w = row_stats_masked<T, ENT>(a, row, row_hb(row), lane);
          else w = row_stats_global<T, ENT>(a, row, b16, e16, lane);
        }
      }
      RowStat<A> tot = w;
      if (CS > 1) {
        // DSMEM exchange: lane r writes this CTA's partial into rank r's slot
        // [parity][my rank] and release-arrives on rank r's barrier.
        if (lane < CS) {
          const uint32_t base = mapa_shared(smem_u32(&tail->xval[par][rank][0]), (uint32_t)lane);
          st_cluster_f64(base, (double)w.m);
          st_cluster_f64(base + 8, (double)w.s);
          st_cluster_f64(base + 16, (double)w.sx);
          mbar_remote_arrive_release(mapa_shared(smem_u32(&tail->xbar[par]), (uint32_t)lane));
        }
        mbar_wait_cluster(&tail->xbar[par], (it >> 1) & 1);
        tot.init();
        for (int r = 0; r < CS; ++r)
          tot.merge((A)tail->xval[par][r][0], (A)tail->xval[par][r][1], (A)tail->xval[par][r][2]);
      }
      const A lse_s = Ex<A>::lse_shift(tot.m == Lim<A>::ninf() ? A(0) : tot.m, tot.s);
      const double lse = Ex<A>::lse_nat(lse_s);
      const double ent = ENT ? lse - (double)(tot.sx / tot.s) : 0.0;
      xa = __shfl_sync(0xffffffffu, xa, 0);
      const double lp = xa - lse;
      if (!BWD && lane == 0 && rank == 0) {
        if (a.lp_out) a.lp_out[idx] = lp;
        if (ENT && a.ent_out) a.ent_out[idx] = ent;
      }
      if (BWD) {
        sc_behav = __shfl_sync(0xffffffffu, sc_behav, 0);
        sc_prox = __shfl_sync(0xffffffffu, sc_prox, 0);
        if (a.prox_from_lp) sc_prox = lp;  // first minibatch: prox is this lp
        // the three fp64 exponentials of the epilogue, one per lane, in parallel:
        // lane 0 exp(prox - behav), lane 1 exp(lp - prox | lp - behav), lane 2 exp(lp)
        const double arg = lane == 0 ? __dsub_rn(sc_prox, sc_behav)
                           : lane == 1 ? (a.decoupled ? __dsub_rn(lp, sc_prox) : __dsub_rn(lp, sc_behav))
                                       : lp;
        const double ex = exp(arg);
        const double e_scale = __shfl_sync(0xffffffffu, ex, 0);
        const double e_ratio = __shfl_sync(0xffffffffu, ex, 1);
        const double e_p = __shfl_sync(0xffffffffu, ex, 2);
        if (lane == 0) {
          const TokenTerms t = ppo_token_terms(a.decoupled ? e_scale : 1.0, e_ratio, sc_adv,
                                               sc_ver, a);
          const double gc = a.grad_scale * t.coef;
          RingBcast& b = tail->bc[par];
          b.gc = gc;
          b.lse = (double)lse_s;
          b.tok = tok;
          b.dtok = to_bits<T>(Traits<T>::from_acc((A)(gc * (e_p - 1.0))));  // g * (p_tok - 1)
          mbar_arrive(&tail->bcbar[par]);  // release: publishes bc[par]
          // bookkeeping after the hand-off (off the math warps' critical path)
          if (rank == 0) {
            stats_add(tail->st, t, ent);
            if (a.lp_out) a.lp_out[idx] = lp;
            if (ENT && a.ent_out) a.ent_out[idx] = ent;
          }
        }
      }
    }
  } else {
    // ================= math warps
    Cursor cur = {0u, 0u};     // ring position of the current row's chunk 0
    Cursor pstart = cur;       // where pass 1 resumes (after the lookahead chunks)
    int la = 0;                // chunks of the current row already folded by the lookahead
    RowStat<A> carry;          // their partial statistics
    carry.init();
    bool pending = false;      // BWD, lane 0: last store's slot not yet released
    uint32_t pend_slot = 0;
    for (int it = 0;; ++it) {
      const int64_t row = row_at(it);
      if (row < 0) break;
      const int par = it & 1;
      // ---- pass 1: online (max, sum e, sum e*x) over the chunks as they land
      RowStat<A> rs = carry;
      Cursor cc = pstart;
      const int hb = row_hb(row);
      for (int c = la; c < nchunks; ++c) {
        mbar_wait(&full[cc.slot], cc.phase);
        const int nvec = chunk_bytes(c, hb) / 16;
        const uint4* q = reinterpret_cast<const uint4*>(ring + (size_t)cc.slot * kChunkBytes);
        A f[NV];
        load_values<T, UNAL>(q, warp, lane, nvec, f, c * (kChunkBytes / (int)sizeof(T)) - hb / (int)sizeof(T),
                             (int)a.vocab);
        if (!BWD) {  // K1: the slot is free as soon as the values are in registers
          if (kK1ArriveAllLanes) {
            mbar_arrive(&empty[cc.slot]);
          } else {  // __syncwarp orders every lane's reads before lane 0's release-arrive
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[cc.slot]);
          }
        }
        fold_values<T, ENT, kFold1Fixed>(rs, f);
        cc.next(nslots);
      }
      const Cursor after = cc;  // ring position of the next row's chunk 0
      rs = kMathWarpMerge ? warp_merge_ent<A, ENT>(rs) : (rs.warp_reduce(), rs);
      // K1 flow control: never hand off row i+1 before the epilogue warp took row i
      // (K2 already waited for row i's coefficient before its pass 2)
      if (!BWD && it > 0) mbar_wait(&tail->bcbar[par ^ 1], ((it - 1) >> 1) & 1);
      A* red = red_ptr<A>(tail, par);
      if (lane == 0) {
        red[warp * 3 + 0] = rs.m;
        red[warp * 3 + 1] = rs.s;
        red[warp * 3 + 2] = rs.sx;
      }
      named_bar_arrive(kBarPartials, kBarPartialsThreads);  // non-blocking hand-off
      if (BWD) {
        // ---- lookahead: while the epilogue warp works, fold the next row's chunks
        // that already sit in the spare slots
        const bool has_next = row + ncl < a.n_rows;
        const int la_next = has_next ? min((int)nslots - nchunks, nchunks) : 0;
        RowStat<A> nxt;
        nxt.init();
        Cursor lc = after;
        for (int c = 0; c < la_next; ++c) {
          mbar_wait(&full[lc.slot], lc.phase);
          const int nvec = (c < nfull ? kChunkBytes : last_bytes) / 16;
          const uint4* q = reinterpret_cast<const uint4*>(ring + (size_t)lc.slot * kChunkBytes);
          A f[NV];
          load_values<T>(q, warp, lane, nvec, f);
          fold_values<T, ENT, kFold1Fixed>(nxt, f);
          lc.next(nslots);
        }
        carry = nxt;
        la = la_next;
        pstart = lc;

        mbar_wait(&tail->bcbar[par], (it >> 1) & 1);
        const RingBcast b = tail->bc[par];
        const A g = (A)b.gc;
        const A lse_s = (A)b.lse;
        const int64_t tok_local = b.tok - slice_e0;  // may lie outside this slice
        const T dtok = from_bits<T>(b.dtok);
        char* drow = a.dlogits + row * a.ld_out_bytes + b16 * 16;
        // ---- pass 2: dlogits = g * (softmax - onehot) in place; each warp stores
        // its own contiguous part of the chunk and recycles the slot itself.
        Cursor c2 = cur;
        for (int c = 0; c < nchunks; ++c) {
          const int cbytes = c < nfull ? kChunkBytes : last_bytes;
          const int nvec = cbytes / 16;
          uint4* q = reinterpret_cast<uint4*>(ring + (size_t)c2.slot * kChunkBytes);
          if (g == A(0)) {  // no gradient through this token: zeros, no exponentials
#pragma unroll
            for (int j = 0; j < kVecPerThread; ++j) {
              const int vi = vec_index(warp, lane, j);
              if (vi < nvec) q[vi] = make_uint4(0, 0, 0, 0);
            }
          } else {
            const bool wfull = (warp + 1) * (kWarpBytes / 16) <= nvec;  // this warp's 2 KB
#pragma unroll
            for (int j = 0; j < kVecPerThread; ++j) {
              const int vi = vec_index(warp, lane, j);
              if (wfull || vi < nvec) {
                A f[E];
                Vec<T>::unpack(q[vi], f);
                if constexpr (std::is_same<A, float>::value) {
                  const float2 L2 = make_float2(Lim<float>::kLog2e, Lim<float>::kLog2e);
                  const float2 M2 = make_float2(-lse_s, -lse_s);
                  const float2 G2 = make_float2(g, g);
#pragma unroll
                  for (int e = 0; e < E; e += 2) {
                    const float2 t = ffma2(make_float2(f[e], f[e + 1]), L2, M2);
                    const float2 d = fmul2(make_float2(fast_exp2(t.x), fast_exp2(t.y)), G2);
                    f[e] = d.x;
                    f[e + 1] = d.y;
                  }
                } else {
#pragma unroll
                  for (int e = 0; e < E; ++e) f[e] = g * exp(f[e] - lse_s);
                }
                q[vi] = Vec<T>::pack(f);
              }
            }
            // the one-hot element: written by the thread that owns it
            const int64_t toff = tok_local - (int64_t)c * (kChunkBytes / (int)sizeof(T));
            if (toff >= 0 && toff < (int64_t)(cbytes / (int)sizeof(T))) {
              const int tv = (int)(toff / E);
              if (tv / (kWarpBytes / 16) == warp && (tv % 32) == lane)
                reinterpret_cast<T*>(q)[toff] = dtok;
            }
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            const int wb0 = warp * kWarpBytes;
            if (wb0 < cbytes) {
              bulk_s2g(drow + (size_t)c * kChunkBytes + wb0,
                       ring + (size_t)c2.slot * kChunkBytes + wb0, (uint32_t)min(kWarpBytes, cbytes - wb0));
            }
            bulk_commit();
            if (pending) {  // previous store has read its slot -> release it
              bulk_wait_read<1>();
              mbar_arrive(&empty[pend_slot]);
            }
            pending = true;
            pend_slot = c2.slot;
            if (c == nchunks - 1) {  // row end: drain so every slot of this row is free
              bulk_wait_read<0>();   // before the next row's lookahead waits on them
              mbar_arrive(&empty[pend_slot]);
              pending = false;
            }
          }
          c2.next(nslots);
        }
      } else {
        pstart = after;
      }
      cur = after;
    }
    if (BWD && lane == 0) {
      bulk_wait<0>();  // all dlogits stores complete before the CTA retires
      if (pending) mbar_arrive(&empty[pend_slot]);
    }
  }
  // all threads: final stats reduction (rank-0 CTAs carry the counters)
  __syncthreads();
  if (dyn && threadIdx.x == 0) {  // the last CTA out re-arms the row counter
    if (atomicAdd(a.counter + 3, 1u) == gridDim.x - 1) {
      a.counter[2] = 0u;
      a.counter[3] = 0u;
    }
  }
  if (BWD) {
    double cta[AREAL_N_STATS];
    for (int j = 0; j < AREAL_N_STATS; ++j) cta[j] = tail->st[j];
    finalize_stats(a, cta, kRingThreads);
  }
  if (CS > 1) cluster_sync_all();  // no CTA exits while a peer may still address its smem
}

}  // namespace areal
