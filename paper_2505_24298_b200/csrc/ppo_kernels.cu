// ppo_kernels.cu — K1 (log-softmax-gather + entropy) and K2 (decoupled-PPO loss
// fused with its backward into dlogits) for sm_100a.
//
// Reference semantics: /root/reference/pkg/src/asyncrl/trainer.py:150-195
// (_surrogate_terms) and policy.py:145-163 (log_softmax, batch_token_log_probs),
// restated on given logits; see DESIGN.md §3 for the data layout and rooflines.
//
// Two kernels per op:
//   row_warp : one warp per row, any vocab / alignment; both passes read global
//              memory (the second pass hits L1/L2).  Small-vocab and fallback path.
//   row_ring : persistent, warp-specialised.  A producer thread streams the row
//              through a ring of 16 KB shared-memory chunks with 1-D TMA bulk
//              copies (cp.async.bulk + mbarrier complete_tx).  K2 keeps the whole
//              row slice resident: pass 1 reduces (max, sum e^x, sum e^x*x) as
//              chunks land, the CTAs of a thread-block cluster (which split the
//              vocab) exchange their partials through DSMEM, pass 2 rewrites each
//              chunk in place as dlogits and streams it out with a bulk store.
//              HBM traffic = one logits read + one dlogits write per element.
#include <cstdlib>
#include <type_traits>

#include "common.cuh"

namespace areal {

// ------------------------------------------------------------------ arguments
struct PpoArgs {
  const char* logits;      // row r at logits + r*ld_in_bytes
  char* dlogits;           // row r at dlogits + r*ld_out_bytes (BWD only)
  int64_t ld_in_bytes, ld_out_bytes;
  int64_t n_rows, vocab;
  const int64_t* tokens;
  const double* behav;
  const double* prox;
  const double* adv;
  const int32_t* versions;
  const int32_t* row_index;
  double* lp_out;
  double* ent_out;
  double* stats;           // [8] accumulated (+=) by the last CTA
  double* partials;        // workspace: [gridDim][8]
  unsigned int* counter;   // workspace: ticket for the last-CTA reduction
  double clip_eps, behav_cap, grad_scale;
  int decoupled, eta_mask, cur_version;
  // ring kernel geometry
  int cluster_size;
  int poly_vecs;           // pass-2 vectors per thread per chunk whose exp2 runs on the FMA pipe
  int64_t slice16;         // 16-byte units per cluster rank
  int nslots;
};

// ------------------------------------------------------------------ per-token epilogue (fp64)
// trainer.py:165-195 for one token, exact IEEE op order (no FMA contraction):
// scale/ratio, validity, clipped surrogate, take mask, coefficient, counters.
struct TokenTerms {
  double coef, obj, ratio;
  bool valid, clipped, masked;
};

__device__ __forceinline__ TokenTerms ppo_token(double lp, double behav, double prox, double adv,
                                                int version, const PpoArgs& a) {
  TokenTerms t;
  double scale, ratio;
  if (a.decoupled) {
    scale = exp(__dsub_rn(prox, behav));  // trainer.py:166
    ratio = exp(__dsub_rn(lp, prox));     // trainer.py:167
  } else {
    scale = 1.0;                          // trainer.py:169
    ratio = exp(__dsub_rn(lp, behav));    // trainer.py:170
  }
  const bool valid = isfinite(scale) && isfinite(ratio);  // trainer.py:172
  bool masked = false;
  if (a.eta_mask >= 0 && (a.cur_version - version) > a.eta_mask) masked = true;
  if (a.behav_cap > 0.0 && valid && scale > a.behav_cap) masked = true;
  const bool v = valid && !masked;
  const double lo = __dsub_rn(1.0, a.clip_eps), hi = __dadd_rn(1.0, a.clip_eps);
  const double P = __dmul_rn(ratio, adv);                          // trainer.py:173
  const double Cl = __dmul_rn(fmin(fmax(ratio, lo), hi), adv);     // trainer.py:174
  const double mn = (Cl < P) ? Cl : P;                             // np.minimum (NaN-propagating via P)
  t.obj = v ? __dmul_rn(scale, mn) : 0.0;                          // trainer.py:175-176
  const bool take = (P <= Cl) && v;                                // trainer.py:177
  t.coef = take ? __dmul_rn(__dmul_rn(scale, adv), ratio) : 0.0;   // trainer.py:179
  t.clipped = v && (Cl < P);                                       // trainer.py:186
  t.ratio = ratio;
  t.valid = v;
  t.masked = masked;
  return t;
}

__device__ __forceinline__ void stats_add(double st[AREAL_N_STATS], const TokenTerms& t,
                                          double ent) {
  st[AREAL_STAT_OBJECTIVE_SUM] += t.obj;
  st[AREAL_STAT_N_VALID] += t.valid ? 1.0 : 0.0;
  st[AREAL_STAT_N_CLIPPED] += t.clipped ? 1.0 : 0.0;
  st[AREAL_STAT_RATIO_SUM] += t.valid ? t.ratio : 0.0;
  st[AREAL_STAT_N_EXCLUDED] += t.valid ? 0.0 : 1.0;
  st[AREAL_STAT_N_MASKED] += t.masked ? 1.0 : 0.0;
  st[AREAL_STAT_ENTROPY_SUM] += t.valid ? ent : 0.0;
  st[AREAL_STAT_N_TOKENS] += 1.0;
}

// Deterministic grid reduction of per-CTA stats: every CTA writes its partial,
// the last CTA to finish (atomic ticket) sums them in CTA order and adds the
// result into a.stats, then re-arms the ticket.  Call with all CTA threads.
__device__ void finalize_stats(const PpoArgs& a, const double cta_stats[AREAL_N_STATS],
                               int nthreads) {
  __shared__ unsigned int s_last;
  if (threadIdx.x == 0) {
    double* p = a.partials + (size_t)blockIdx.x * AREAL_N_STATS;
#pragma unroll
    for (int j = 0; j < AREAL_N_STATS; ++j) p[j] = cta_stats[j];
    __threadfence();
    unsigned int ticket = atomicAdd(a.counter, 1u);
    s_last = (ticket == gridDim.x - 1) ? 1u : 0u;
  }
  __syncthreads();
  if (s_last) {
    __threadfence();
    if (threadIdx.x < AREAL_N_STATS) {
      const volatile double* p = a.partials;
      double acc = 0.0;
      for (unsigned int b = 0; b < gridDim.x; ++b) acc += p[(size_t)b * AREAL_N_STATS + threadIdx.x];
      a.stats[threadIdx.x] += acc;
    }
    if (threadIdx.x == 0) *a.counter = 0u;
  }
  (void)nthreads;
}

// ------------------------------------------------------------------ exponent helpers
// fp32 path works in the log2 domain with the MUFU ex2; fp64 uses libdevice exp.
template <typename A> struct Ex;
template <> struct Ex<float> {
  // shift constant for a running max m
  static __device__ __forceinline__ float shift(float m) { return m * Lim<float>::kLog2e; }
  static __device__ __forceinline__ float e(float x, float c) {
    return fast_exp2(fmaf(x, Lim<float>::kLog2e, -c));
  }
  // lse in "shift units" (log2 domain) from (m, s)
  static __device__ __forceinline__ float lse_shift(float m, float s) {
    return m * Lim<float>::kLog2e + __log2f(s);
  }
  static __device__ __forceinline__ double lse_nat(float lse2) {
    return (double)lse2 * 0.69314718055994530942;
  }
};
template <> struct Ex<double> {
  static __device__ __forceinline__ double shift(double m) { return m; }
  static __device__ __forceinline__ double e(double x, double c) { return exp(x - c); }
  static __device__ __forceinline__ double lse_shift(double m, double s) { return m + log(s); }
  static __device__ __forceinline__ double lse_nat(double l) { return l; }
};

// Fold a batch of values (already max-reduced into lmax) into a running RowStat.
template <typename A, int N>
__device__ __forceinline__ void fold(RowStat<A>& rs, const A (&v)[N], A lmax) {
  const A mn = fmax(rs.m, lmax);
  const A muse = (mn == Lim<A>::ninf()) ? A(0) : mn;
  const A c = Ex<A>::shift(muse);
  const A r = Ex<A>::e(rs.m, c);  // rescale of the old partial sums (0 when m = -inf)
  A s = rs.s * r, sx = rs.sx * r;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    const A e = Ex<A>::e(v[i], c);
    s += e;
    sx += e * fmax(v[i], Lim<A>::lowest());  // 0 * (-inf) guarded: p log p := 0
  }
  rs.m = mn;
  rs.s = s;
  rs.sx = sx;
}

// ------------------------------------------------------------------ 16-byte vector (un)packing
template <typename T> struct Vec;
template <> struct Vec<__nv_bfloat16> {
  static constexpr int N = 8;
  static __device__ __forceinline__ void unpack(const uint4& q, float (&o)[8]) {
    const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      o[2 * i] = __uint_as_float(w[i] << 16);
      o[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
    }
  }
  static __device__ __forceinline__ uint4 pack(const float (&o)[8]) {
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      __nv_bfloat162 h = __floats2bfloat162_rn(o[2 * i], o[2 * i + 1]);
      w[i] = *reinterpret_cast<uint32_t*>(&h);
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
  }
};
template <> struct Vec<__half> {
  static constexpr int N = 8;
  static __device__ __forceinline__ void unpack(const uint4& q, float (&o)[8]) {
    const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      __half2 h = *reinterpret_cast<const __half2*>(&w[i]);
      float2 f = __half22float2(h);
      o[2 * i] = f.x;
      o[2 * i + 1] = f.y;
    }
  }
  static __device__ __forceinline__ uint4 pack(const float (&o)[8]) {
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      __half2 h = __floats2half2_rn(o[2 * i], o[2 * i + 1]);
      w[i] = *reinterpret_cast<uint32_t*>(&h);
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
  }
};
template <> struct Vec<float> {
  static constexpr int N = 4;
  static __device__ __forceinline__ void unpack(const uint4& q, float (&o)[4]) {
    o[0] = __uint_as_float(q.x);
    o[1] = __uint_as_float(q.y);
    o[2] = __uint_as_float(q.z);
    o[3] = __uint_as_float(q.w);
  }
  static __device__ __forceinline__ uint4 pack(const float (&o)[4]) {
    return make_uint4(__float_as_uint(o[0]), __float_as_uint(o[1]), __float_as_uint(o[2]),
                      __float_as_uint(o[3]));
  }
};
template <> struct Vec<double> {
  static constexpr int N = 2;
  static __device__ __forceinline__ void unpack(const uint4& q, double (&o)[2]) {
    o[0] = __hiloint2double((int)q.y, (int)q.x);
    o[1] = __hiloint2double((int)q.w, (int)q.z);
  }
  static __device__ __forceinline__ uint4 pack(const double (&o)[2]) {
    const long long a = __double_as_longlong(o[0]), b = __double_as_longlong(o[1]);
    return make_uint4((uint32_t)a, (uint32_t)(a >> 32), (uint32_t)b, (uint32_t)(b >> 32));
  }
};

// ------------------------------------------------------------------ shared per-row token prologue
template <typename T>
__device__ __forceinline__ double token_logit(const PpoArgs& a, const T* row, int64_t tok) {
  if (tok < 0 || tok >= a.vocab) return __longlong_as_double(0x7ff8000000000000ll);  // NaN: excluded
  return (double)Traits<T>::to_acc(row[tok]);
}

// ================================================================== row_warp kernel
constexpr int kWarpKernelWarps = 8;
constexpr int kWarpUnroll = 8;

template <typename T, bool BWD>
__device__ __forceinline__ void row_warp_body(const PpoArgs& a) {
  using A = typename Traits<T>::Acc;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nw = (int64_t)gridDim.x * kWarpKernelWarps;
  double st[AREAL_N_STATS];
#pragma unroll
  for (int j = 0; j < AREAL_N_STATS; ++j) st[j] = 0.0;
  const int64_t V = a.vocab;

  for (int64_t row = (int64_t)blockIdx.x * kWarpKernelWarps + warp; row < a.n_rows; row += nw) {
    const T* x = reinterpret_cast<const T*>(a.logits + row * a.ld_in_bytes);
    const int64_t idx = a.row_index ? (int64_t)a.row_index[row] : row;
    const int64_t tok = a.tokens[idx];
    RowStat<A> rs;
    rs.init();
    for (int64_t base = 0; base < V; base += 32 * kWarpUnroll) {
      A v[kWarpUnroll];
      A lmax = Lim<A>::ninf();
#pragma unroll
      for (int u = 0; u < kWarpUnroll; ++u) {
        const int64_t i = base + u * 32 + lane;
        v[u] = (i < V) ? Traits<T>::to_acc(x[i]) : Lim<A>::ninf();
        lmax = fmax(lmax, v[u]);
      }
      fold(rs, v, lmax);
    }
    rs.warp_reduce();
    const A lse_s = Ex<A>::lse_shift(rs.m == Lim<A>::ninf() ? A(0) : rs.m, rs.s);
    const double lse = Ex<A>::lse_nat(lse_s);
    const double ent = lse - (double)(rs.sx / rs.s);
    double gc = 0.0;
    if (lane == 0) {
      const double lp = token_logit<T>(a, x, tok) - lse;
      if (a.lp_out) a.lp_out[idx] = lp;
      if (a.ent_out) a.ent_out[idx] = ent;
      if (BWD) {
        const TokenTerms t = ppo_token(lp, a.behav[idx], a.prox ? a.prox[idx] : 0.0, a.adv[idx],
                                       a.versions ? a.versions[idx] : 0, a);
        stats_add(st, t, a.ent_out ? ent : 0.0);
        gc = a.grad_scale * t.coef;
      }
    }
    if (BWD) {
      gc = __shfl_sync(0xffffffffu, gc, 0);
      const A g = (A)gc;
      T* d = reinterpret_cast<T*>(a.dlogits + row * a.ld_out_bytes);
      for (int64_t i = lane; i < V; i += 32) {
        const A xv = Traits<T>::to_acc(x[i]);
        A p;
        if constexpr (std::is_same<A, float>::value)
          p = fast_exp2(fmaf(xv, Lim<float>::kLog2e, -lse_s));
        else
          p = exp(xv - lse_s);
        d[i] = Traits<T>::from_acc(g * (p - (i == tok ? A(1) : A(0))));
      }
    }
  }
  if (BWD) {
    // block reduce in warp order, then deterministic grid finalize
    __shared__ double red[kWarpKernelWarps][AREAL_N_STATS];
    if (lane == 0)
      for (int j = 0; j < AREAL_N_STATS; ++j) red[warp][j] = st[j];
    __syncthreads();
    double cta[AREAL_N_STATS];
    for (int j = 0; j < AREAL_N_STATS; ++j) {
      double acc = 0.0;
      for (int w = 0; w < kWarpKernelWarps; ++w) acc += red[w][j];
      cta[j] = acc;
    }
    finalize_stats(a, cta, kWarpKernelWarps * 32);
  }
}

// ================================================================== row_ring kernel
constexpr int kChunkBytes = 32768;
constexpr int kConsumerWarps = 16;
constexpr int kConsumers = kConsumerWarps * 32;
constexpr int kRingThreads = kConsumers + 32;  // + 1 producer warp
constexpr int kBarConsumers = 1;                // named barrier id among consumer warps
constexpr int kVecPerThread = kChunkBytes / 16 / kConsumers;  // 16-byte vectors per thread per chunk
constexpr int kWarpBytes = kChunkBytes / kConsumerWarps;      // contiguous bytes a warp owns per chunk

struct RingBcast {
  double gc;                // grad_scale * coef
  double lse;               // lse in shift units
  long long tok;            // token id
  unsigned long long dtok;  // dlogit of the token element (T bits)
};

struct RingSmemTail {
  uint64_t xbar[2];                 // DSMEM exchange barriers (double-buffered by row parity)
  uint64_t bcbar[2];                // epilogue -> consumers (double-buffered by row parity)
  double xval[2][8][3];             // [parity][rank][m, s, sx]
  float redf[2][kConsumerWarps][3]; // per-warp partials, double-buffered by row parity
  double redd[2][kConsumerWarps][3];
  RingBcast bc[2];
  double st[AREAL_N_STATS];         // thread 0's running statistics
  // cp.async prefetch targets (thread 0): token id one row ahead, then the row's
  // token logit word and per-token scalars, so no register waits on global loads
  long long pf_tok;
  unsigned long long pf_xa;         // 4- or 8-byte aligned word holding x[token]
  double pf_behav, pf_prox, pf_adv;
  int pf_ver;
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

// Vector j (< kVecPerThread) of this thread inside a chunk: each warp owns a
// contiguous kWarpBytes region, lanes read consecutive 16-byte vectors.
__device__ __forceinline__ int vec_index(int warp, int lane, int j) {
  return warp * (kWarpBytes / 16) + j * 32 + lane;
}

// Load this thread's vectors of a chunk (nvec valid vectors) as accumulation values.
template <typename T>
__device__ __forceinline__ void load_values(const uint4* q, int warp, int lane, int nvec,
                                            typename Traits<T>::Acc* f) {
  using A = typename Traits<T>::Acc;
  constexpr int E = Vec<T>::N;
  if (nvec == kChunkBytes / 16) {  // full chunk: branch-free
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
      for (int e = 0; e < E; ++e) f[j * E + e] = g[e];
    }
  }
}

// Fold this thread's values of one chunk into its running (m, s, sx).
// fp32: packed f32x2 FFMA2/FADD2 around the MUFU ex2; fp64: scalar libdevice exp.
template <typename T, bool ENT>
__device__ __forceinline__ void fold_values(RowStat<typename Traits<T>::Acc>& rs,
                                            const typename Traits<T>::Acc* f) {
  using A = typename Traits<T>::Acc;
  constexpr int N = kVecPerThread * Vec<T>::N;
  A lmax = f[0];
#pragma unroll
  for (int i = 1; i < N; ++i) lmax = fmax(lmax, f[i]);
  const A mn = fmax(rs.m, lmax);
  const A muse = (mn == Lim<A>::ninf()) ? A(0) : mn;
  const A c = Ex<A>::shift(muse);
  const A r = Ex<A>::e(rs.m, c);  // rescale of the running sums (0 while m = -inf)
  if constexpr (std::is_same<A, float>::value) {
    const float2 L2 = make_float2(Lim<float>::kLog2e, Lim<float>::kLog2e);
    const float2 C2 = make_float2(-c, -c);
    float2 s2 = make_float2(0.f, 0.f), x2 = make_float2(0.f, 0.f);
#pragma unroll
    for (int i = 0; i < N; i += 2) {
      const float2 v = make_float2(f[i], f[i + 1]);
      const float2 t = ffma2(v, L2, C2);
      const float2 e = make_float2(fast_exp2(t.x), fast_exp2(t.y));
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

template <typename T, bool BWD, bool ENT>
__device__ __forceinline__ void row_ring_body(const PpoArgs& a) {
  using A = typename Traits<T>::Acc;
  constexpr int E = Vec<T>::N;                 // elements per 16 bytes
  constexpr int NV = kVecPerThread * E;        // values per thread per chunk
  extern __shared__ __align__(1024) unsigned char smem[];
  const uint32_t nslots = (uint32_t)a.nslots;
  unsigned char* ring = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)nslots * kChunkBytes);
  uint64_t* empty = full + nslots;
  RingSmemTail* tail = reinterpret_cast<RingSmemTail*>(empty + nslots);

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
  const int nchunks = nfull + (last_bytes > 0 ? 1 : 0);
  const int64_t slice_e0 = b16 * E;  // first vocab element of this rank's slice

  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < nslots; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);  // one arrive per consumer warp per use
    }
    mbar_init(&tail->xbar[0], CS);
    mbar_init(&tail->xbar[1], CS);
    mbar_init(&tail->bcbar[0], 1);
    mbar_init(&tail->bcbar[1], 1);
    fence_mbar_init_cluster();
  }
  __syncthreads();
  if (CS > 1) cluster_sync_all();  // peers' exchange barriers initialised before any remote arrive

  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int j = 0; j < AREAL_N_STATS; ++j) tail->st[j] = 0.0;
    if (cid < a.n_rows) {  // token id of the first row
      const int64_t i0 = a.row_index ? (int64_t)a.row_index[cid] : cid;
      cp_async8(&tail->pf_tok, a.tokens + i0);
      cp_async_commit();
    }
  }

  if (tid >= kConsumers) {
    // ---------------- producer warp: one elected lane issues the TMA bulk loads
    if (tid == kConsumers) {
      Cursor cur = {0u, 0u};
      uint32_t used = 0;  // slots filled at least once (no wait needed on first use)
      for (int64_t row = cid; row < a.n_rows; row += ncl) {
        const char* src = a.logits + row * a.ld_in_bytes + b16 * 16;
        for (int c = 0; c < nchunks; ++c) {
          if (used >= nslots) mbar_wait(&empty[cur.slot], cur.phase ^ 1u);
          else ++used;
          const uint32_t bytes = (uint32_t)(c < nfull ? kChunkBytes : last_bytes);
          mbar_arrive_expect_tx(&full[cur.slot], bytes);
          bulk_g2s(ring + (size_t)cur.slot * kChunkBytes, src + (size_t)c * kChunkBytes, bytes,
                   &full[cur.slot]);
          cur.next(nslots);
        }
      }
    }
  } else {
    // ---------------- consumer warps
    const int warp = tid >> 5, lane = tid & 31;
    Cursor cur = {0u, 0u};     // ring position of the current row's chunk 0
    Cursor pstart = cur;       // where pass 1 resumes (after the lookahead chunks)
    int la = 0;                // chunks of the current row already folded by the lookahead
    RowStat<A> carry;          // their partial statistics
    carry.init();
    bool pending = false;      // BWD, lane 0: last store's slot not yet released
    uint32_t pend_slot = 0;
    int64_t idx_cur = 0;       // thread 0: global token index of the current row
    if (tid == 0 && cid < a.n_rows) idx_cur = a.row_index ? (int64_t)a.row_index[cid] : cid;
    int it = 0;
    for (int64_t row = cid; row < a.n_rows; row += ncl, ++it) {
      const int par = it & 1;
      const T* xrow = reinterpret_cast<const T*>(a.logits + row * a.ld_in_bytes);
      const int64_t idx = idx_cur;  // thread 0 only (loaded a row ahead)
      int32_t idx_next = 0;         // thread 0 only: row_index of the next row
      if (tid == 0) {
        // the token id was prefetched a row ahead; issue the row's scalar loads as
        // cp.async into shared memory so their latency hides behind pass 1
        if (row + ncl < a.n_rows) idx_next = a.row_index ? a.row_index[row + ncl] : (int32_t)(row + ncl);
        cp_async_wait_all();
        const int64_t tok = tail->pf_tok;
        if (tok >= 0 && tok < a.vocab) {
          const uintptr_t p = (uintptr_t)(xrow + tok);
          if (sizeof(T) == 8) cp_async8(&tail->pf_xa, (const void*)p);
          else cp_async4(&tail->pf_xa, (const void*)(p & ~(uintptr_t)3));
        }
        if (BWD) {
          cp_async8(&tail->pf_behav, a.behav + idx);
          if (a.prox) cp_async8(&tail->pf_prox, a.prox + idx);
          cp_async8(&tail->pf_adv, a.adv + idx);
          if (a.versions) cp_async4(&tail->pf_ver, a.versions + idx);
        }
        cp_async_commit();
      }
      // ---- pass 1: online (max, sum e, sum e*x) over the chunks as they land
      RowStat<A> rs = carry;
      Cursor cc = pstart;
      for (int c = la; c < nchunks; ++c) {
        mbar_wait(&full[cc.slot], cc.phase);
        const int nvec = (c < nfull ? kChunkBytes : last_bytes) / 16;
        const uint4* q = reinterpret_cast<const uint4*>(ring + (size_t)cc.slot * kChunkBytes);
        A f[NV];
        load_values<T>(q, warp, lane, nvec, f);
        if (!BWD) {  // K1: the slot is free as soon as the values are in registers
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[cc.slot]);
        }
        fold_values<T, ENT>(rs, f);
        cc.next(nslots);
      }
      const Cursor after = cc;  // ring position of the next row's chunk 0
      // ---- CTA reduce: warp shuffles, then warp 0 merges the warp partials (fixed order)
      rs.warp_reduce();
      A* red = red_ptr<A>(tail, par);
      if (lane == 0) {
        red[warp * 3 + 0] = rs.m;
        red[warp * 3 + 1] = rs.s;
        red[warp * 3 + 2] = rs.sx;
      }
      named_bar_sync(kBarConsumers, kConsumers);
      if (warp == 0) {
        RowStat<A> w;
        if (lane < kConsumerWarps) {
          w.m = red[lane * 3 + 0];
          w.s = red[lane * 3 + 1];
          w.sx = red[lane * 3 + 2];
        } else {
          w.init();
        }
        w.warp_reduce();
        if (lane == 0) {
          RowStat<A> tot = w;
          if (CS > 1) {
            // ---- cluster exchange through DSMEM: write my partial into every
            // rank's slot [parity][my rank], release-arrive on its barrier.
            for (int r = 0; r < CS; ++r) {
              const uint32_t base = mapa_shared(smem_u32(&tail->xval[par][rank][0]), (uint32_t)r);
              st_cluster_f64(base, (double)w.m);
              st_cluster_f64(base + 8, (double)w.s);
              st_cluster_f64(base + 16, (double)w.sx);
              mbar_remote_arrive_release(mapa_shared(smem_u32(&tail->xbar[par]), (uint32_t)r));
            }
            mbar_wait_cluster(&tail->xbar[par], (it >> 1) & 1);
            tot.init();
            for (int r = 0; r < CS; ++r)
              tot.merge((A)tail->xval[par][r][0], (A)tail->xval[par][r][1], (A)tail->xval[par][r][2]);
          }
          cp_async_wait_all();  // this row's token logit and scalars are in smem
          const int64_t tok = tail->pf_tok;
          double xa = __longlong_as_double(0x7ff8000000000000ll);  // invalid token -> NaN, excluded
          if (tok >= 0 && tok < a.vocab) {
            if (sizeof(T) == 8) {
              xa = __longlong_as_double((long long)tail->pf_xa);
            } else if (sizeof(T) == 4) {
              xa = (double)__uint_as_float((uint32_t)tail->pf_xa);
            } else {
              const uint32_t w = (uint32_t)tail->pf_xa;
              const unsigned short h = (unsigned short)((((uintptr_t)(xrow + tok)) & 2) ? (w >> 16) : (w & 0xffff));
              xa = (double)Traits<T>::to_acc(from_bits<T>(h));
            }
          }
          if (row + ncl < a.n_rows) {  // prefetch the next row's token id
            cp_async8(&tail->pf_tok, a.tokens + idx_next);
            cp_async_commit();
          }
          const A lse_s = Ex<A>::lse_shift(tot.m == Lim<A>::ninf() ? A(0) : tot.m, tot.s);
          const double lse = Ex<A>::lse_nat(lse_s);
          const double ent = ENT ? lse - (double)(tot.sx / tot.s) : 0.0;
          const double lp = xa - lse;
          if (rank == 0) {
            if (a.lp_out) a.lp_out[idx] = lp;
            if (ENT && a.ent_out) a.ent_out[idx] = ent;
          }
          if (BWD) {
            const TokenTerms t = ppo_token(lp, tail->pf_behav, a.prox ? tail->pf_prox : 0.0,
                                           tail->pf_adv, a.versions ? tail->pf_ver : 0, a);
            if (rank == 0) stats_add(tail->st, t, ent);
            const double gc = a.grad_scale * t.coef;
            RingBcast& b = tail->bc[par];
            b.gc = gc;
            b.lse = (double)lse_s;
            b.tok = tok;
            // the token's own element: g * (p - 1), from the exact lp
            b.dtok = to_bits<T>(Traits<T>::from_acc((A)(gc * (exp(lp) - 1.0))));
            mbar_arrive(&tail->bcbar[par]);  // release: publishes bc[par]
          }
        }
      }
      if (BWD) {
        // ---- lookahead: while warp 0 finishes the epilogue, fold the next row's
        // chunks that already sit in the spare slots
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
          fold_values<T, ENT>(nxt, f);
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
#pragma unroll
            for (int j = 0; j < kVecPerThread; ++j) {
              const int vi = vec_index(warp, lane, j);
              if (nvec == kChunkBytes / 16 || vi < nvec) {
                A f[E];
                Vec<T>::unpack(q[vi], f);
                if constexpr (std::is_same<A, float>::value) {
                  const float2 L2 = make_float2(Lim<float>::kLog2e, Lim<float>::kLog2e);
                  const float2 M2 = make_float2(-lse_s, -lse_s);
                  const float2 G2 = make_float2(g, g);
                  if (sizeof(T) == 2 && j < a.poly_vecs) {  // MUFU offload (16-bit outputs)
#pragma unroll
                    for (int e = 0; e < E; e += 2) {
                      const float2 t = ffma2(make_float2(f[e], f[e + 1]), L2, M2);
                      const float2 d = fmul2(exp2_poly3(t), G2);
                      f[e] = d.x;
                      f[e + 1] = d.y;
                    }
                  } else {
#pragma unroll
                    for (int e = 0; e < E; e += 2) {
                      const float2 t = ffma2(make_float2(f[e], f[e + 1]), L2, M2);
                      const float2 d = fmul2(make_float2(fast_exp2(t.x), fast_exp2(t.y)), G2);
                      f[e] = d.x;
                      f[e + 1] = d.y;
                    }
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
      idx_cur = idx_next;
    }
    if (BWD && lane == 0) {
      bulk_wait<0>();  // all dlogits stores complete before the CTA retires
      if (pending) mbar_arrive(&empty[pend_slot]);
    }
  }
  // all threads: final stats reduction (rank-0 CTAs carry the counters)
  __syncthreads();
  if (BWD) {
    double cta[AREAL_N_STATS];
    for (int j = 0; j < AREAL_N_STATS; ++j) cta[j] = tail->st[j];
    finalize_stats(a, cta, kRingThreads);
  }
  if (CS > 1) cluster_sync_all();  // no CTA exits while a peer may still address its smem
}

// Distinct entry points per op so profiles name them: K1 = logprob_*, K2 = ppo_*.
template <typename T>
__global__ void __launch_bounds__(kWarpKernelWarps * 32) logprob_warp_kernel(PpoArgs a) {
  row_warp_body<T, false>(a);
}
template <typename T>
__global__ void __launch_bounds__(kWarpKernelWarps * 32) ppo_warp_kernel(PpoArgs a) {
  row_warp_body<T, true>(a);
}
template <typename T, bool ENT>
__global__ void __launch_bounds__(kRingThreads, 1) logprob_ring_kernel(PpoArgs a) {
  row_ring_body<T, false, ENT>(a);
}
template <typename T, bool ENT>
__global__ void __launch_bounds__(kRingThreads, 1) ppo_ring_kernel(PpoArgs a) {
  row_ring_body<T, true, ENT>(a);
}

// ================================================================== host side
static size_t ring_smem_bytes(int nslots) {
  return (size_t)nslots * kChunkBytes + 2 * (size_t)nslots * sizeof(uint64_t) + sizeof(RingSmemTail);
}

struct DevInfo {
  int dev = -1, sms = 0, smem_optin = 0;
};
static DevInfo get_dev() {
  static thread_local DevInfo cache[16];
  int dev = 0;
  cudaGetDevice(&dev);
  DevInfo& d = cache[dev & 15];
  if (d.dev != dev) {
    d.dev = dev;
    cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&d.smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  }
  return d;
}

static int max_slots(const DevInfo& d) {
  int n = 16;
  while (n > 2 && ring_smem_bytes(n) + 1024 > (size_t)d.smem_optin) --n;  // + static smem
  return n;
}

template <typename T, bool BWD, bool ENT>
static int launch_ring(PpoArgs a, cudaStream_t stream, int cs_force) {
  DevInfo d = get_dev();
  const int nslots = max_slots(d);
  const int64_t V16 = (a.vocab * (int64_t)sizeof(T)) / 16;
  int CS = 1;
  if (BWD) {
    // smallest cluster whose slice fits the ring with one slot of slack
    const int cands[4] = {1, 2, 4, 8};
    CS = -1;
    for (int ci = 0; ci < 4; ++ci) {
      const int64_t sl = (V16 + cands[ci] - 1) / cands[ci];
      const int64_t nch = (sl * 16 + kChunkBytes - 1) / kChunkBytes;
      if (nch <= nslots - 1) {
        CS = cands[ci];
        break;
      }
    }
    if (CS < 0) return AREAL_ERR_UNSUPPORTED;
    if (cs_force > 0) CS = cs_force;
  }
  if ((V16 + CS - 1) / CS * 16 > (int64_t)0x7fffffff) return AREAL_ERR_UNSUPPORTED;
  a.cluster_size = CS;
  {
    // tuning knob: AREAL_POLY_VECS in [0, kVecPerThread] (default 0 = all exps on MUFU)
    static const int poly = [] {
      const char* s = getenv("AREAL_POLY_VECS");
      const int v = s ? atoi(s) : 0;
      return v < 0 ? 0 : (v > kVecPerThread ? kVecPerThread : v);
    }();
    a.poly_vecs = poly;
  }
  a.slice16 = (V16 + CS - 1) / CS;
  a.nslots = nslots;
  const size_t smem = ring_smem_bytes(nslots);
  auto kern = BWD ? ppo_ring_kernel<T, ENT> : logprob_ring_kernel<T, ENT>;
  static thread_local int attr_set[16] = {0};
  int dev = d.dev & 15;
  if (!(attr_set[dev] & 1)) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return AREAL_ERR_CUDA;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
      cudaGetLastError();
    attr_set[dev] |= 1;
  }
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  cfg.blockDim = dim3(kRingThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int max_clusters = d.sms / CS;
  if (CS > 1) {
    cfg.gridDim = dim3(CS);
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) == cudaSuccess && n > 0) max_clusters = n;
    else cudaGetLastError();
  }
  const int64_t ncl = std::min<int64_t>(a.n_rows, (int64_t)max_clusters);
  cfg.gridDim = dim3((unsigned)(ncl * CS));
  if (cudaLaunchKernelEx(&cfg, kern, a) != cudaSuccess) return AREAL_ERR_CUDA;
  return AREAL_OK;
}

template <typename T, bool BWD>
static int launch_warp(PpoArgs a, cudaStream_t stream) {
  DevInfo d = get_dev();
  const int64_t blocks_needed = (a.n_rows + kWarpKernelWarps - 1) / kWarpKernelWarps;
  const int64_t grid = std::min<int64_t>(blocks_needed, (int64_t)d.sms * 8);
  auto kern = BWD ? ppo_warp_kernel<T> : logprob_warp_kernel<T>;
  kern<<<(unsigned)grid, kWarpKernelWarps * 32, 0, stream>>>(a);
  AREAL_CUDA_CHECK_LAUNCH();
  return AREAL_OK;
}

static int dtype_size(int dtype) {
  switch (dtype) {
    case AREAL_F32: return 4;
    case AREAL_BF16: return 2;
    case AREAL_F16: return 2;
    case AREAL_F64: return 8;
    default: return 0;
  }
}

// AUTO: ring when rows are >= 16 KB and every row start is 16-byte aligned.
static bool ring_ok(const void* base, int64_t ld_bytes, int64_t vocab, int es) {
  return ((uintptr_t)base % 16 == 0) && (ld_bytes % 16 == 0) && ((vocab * es) % 16 == 0);
}

template <bool BWD>
static int dispatch(PpoArgs a, int dtype, int algo, cudaStream_t stream) {
  const int es = dtype_size(dtype);
  bool ring = false;
  const bool aligned = ring_ok(a.logits, a.ld_in_bytes, a.vocab, es) &&
                       (!BWD || ring_ok(a.dlogits, a.ld_out_bytes, a.vocab, es));
  if (algo == AREAL_ALGO_ROW_RING) {
    if (!aligned) return AREAL_ERR_MISALIGNED;
    ring = true;
  } else if (algo == AREAL_ALGO_AUTO) {
    ring = aligned && a.vocab * es >= 16384;
  }
  if (ring) {
    int rc;
    const bool ent = a.ent_out != nullptr;
    switch (dtype) {
      case AREAL_F32: rc = ent ? launch_ring<float, BWD, true>(a, stream, 0) : launch_ring<float, BWD, false>(a, stream, 0); break;
      case AREAL_BF16: rc = ent ? launch_ring<__nv_bfloat16, BWD, true>(a, stream, 0) : launch_ring<__nv_bfloat16, BWD, false>(a, stream, 0); break;
      case AREAL_F16: rc = ent ? launch_ring<__half, BWD, true>(a, stream, 0) : launch_ring<__half, BWD, false>(a, stream, 0); break;
      case AREAL_F64: rc = ent ? launch_ring<double, BWD, true>(a, stream, 0) : launch_ring<double, BWD, false>(a, stream, 0); break;
      default: return AREAL_ERR_BAD_DTYPE;
    }
    if (rc != AREAL_ERR_UNSUPPORTED || algo == AREAL_ALGO_ROW_RING) return rc;
  }
  switch (dtype) {
    case AREAL_F32: return launch_warp<float, BWD>(a, stream);
    case AREAL_BF16: return launch_warp<__nv_bfloat16, BWD>(a, stream);
    case AREAL_F16: return launch_warp<__half, BWD>(a, stream);
    case AREAL_F64: return launch_warp<double, BWD>(a, stream);
    default: return AREAL_ERR_BAD_DTYPE;
  }
}

static constexpr size_t kCounterBytes = 256;

}  // namespace areal

using namespace areal;

extern "C" int areal_logprob_fwd(const void* logits, int64_t ld_logits, int dtype, int64_t n_rows,
                                 int64_t vocab, const int64_t* tokens, const int32_t* row_index,
                                 double* lp_out, double* entropy_out, int algo, void* workspace,
                                 size_t workspace_bytes, void* stream) {
  const int es = dtype_size(dtype);
  if (es == 0) return AREAL_ERR_BAD_DTYPE;
  if (n_rows < 0 || vocab < 1 || ld_logits < vocab) return AREAL_ERR_BAD_SHAPE;
  if (n_rows == 0) return AREAL_OK;
  if (!logits || !tokens || (!lp_out && !entropy_out)) return AREAL_ERR_INVALID_ARGUMENT;
  (void)workspace;
  (void)workspace_bytes;
  PpoArgs a = {};
  a.logits = static_cast<const char*>(logits);
  a.ld_in_bytes = ld_logits * es;
  a.n_rows = n_rows;
  a.vocab = vocab;
  a.tokens = tokens;
  a.row_index = row_index;
  a.lp_out = lp_out;
  a.ent_out = entropy_out;
  return dispatch<false>(a, dtype, algo, static_cast<cudaStream_t>(stream));
}

extern "C" int areal_ppo_fwd_bwd(const void* logits, int64_t ld_logits, void* dlogits,
                                 int64_t ld_dlogits, int dtype, int64_t n_rows, int64_t vocab,
                                 const int64_t* tokens, const double* behav, const double* prox,
                                 const double* adv, const int32_t* versions,
                                 const int32_t* row_index, const areal_ppo_params_t* params,
                                 double* lp_out, double* entropy_out, double* stats,
                                 void* workspace, size_t workspace_bytes, void* stream) {
  const int es = dtype_size(dtype);
  if (es == 0) return AREAL_ERR_BAD_DTYPE;
  if (!params) return AREAL_ERR_INVALID_ARGUMENT;
  if (!(params->clip_eps > 0.0 && params->clip_eps < 1.0)) return AREAL_ERR_BAD_CLIP_EPS;
  if (n_rows < 0 || vocab < 1 || ld_logits < vocab || ld_dlogits < vocab) return AREAL_ERR_BAD_SHAPE;
  if (n_rows == 0) return AREAL_OK;
  if (!logits || !dlogits || !tokens || !behav || !adv || !stats) return AREAL_ERR_INVALID_ARGUMENT;
  if (params->decoupled && !prox) return AREAL_ERR_INVALID_ARGUMENT;
  if (params->eta_mask >= 0 && !versions) return AREAL_ERR_INVALID_ARGUMENT;
  if (!workspace || workspace_bytes < AREAL_WORKSPACE_BYTES) return AREAL_ERR_WORKSPACE;
  PpoArgs a = {};
  a.logits = static_cast<const char*>(logits);
  a.dlogits = static_cast<char*>(dlogits);
  a.ld_in_bytes = ld_logits * es;
  a.ld_out_bytes = ld_dlogits * es;
  a.n_rows = n_rows;
  a.vocab = vocab;
  a.tokens = tokens;
  a.behav = behav;
  a.prox = prox;
  a.adv = adv;
  a.versions = versions;
  a.row_index = row_index;
  a.lp_out = lp_out;
  a.ent_out = entropy_out;
  a.stats = stats;
  a.counter = static_cast<unsigned int*>(workspace);
  a.partials = reinterpret_cast<double*>(static_cast<char*>(workspace) + kCounterBytes);
  a.clip_eps = params->clip_eps;
  a.behav_cap = params->behav_weight_cap;
  a.grad_scale = params->grad_scale;
  a.decoupled = params->decoupled;
  a.eta_mask = params->eta_mask;
  a.cur_version = params->current_version;
  return dispatch<true>(a, dtype, params->algo, static_cast<cudaStream_t>(stream));
}
