// ppo_kernels.cu — K1 (log-softmax-gather + entropy) and K2 (decoupled-PPO loss
// fused with its backward into dlogits) for sm_100a.
//
// Reference semantics: /root/reference/pkg/src/asyncrl/trainer.py:150-195
// (_surrogate_terms) and policy.py:145-163 (log_softmax, batch_token_log_probs),
// restated on given logits; see DESIGN.md §3 for the data layout and rooflines.
//
// Kernels (AREAL_ALGO_AUTO picks per shape):
//   row_warp : one warp per row, any vocab / alignment; both passes read global
//              memory (the second pass hits L1/L2).  K1 rows under 16 KB, fp64 K2.
//   row_cta_small : K2 rows <= 16 KB (16-bit) / 32 KB (fp32), one CTA per row, 8 per SM.
//   row_cta  : one CTA per row for rows >= 16 KB that are not 16-byte aligned
//              (scalar head / 16-byte-vector body / scalar tail; K2 re-reads from L2):
//              shorter K1 rows and K2 rows the TMEM kernel cannot take (long unaligned
//              K1 rows run the ring kernel's UNAL instantiation).
//   row_ring : persistent, warp-specialised (ppo_ring.cuh).  A producer thread
//              streams each row through a ring of 32 KB shared-memory chunks with
//              1-D TMA bulk copies (cp.async.bulk + mbarrier complete_tx).  K1 frees
//              a chunk as soon as it is in registers (all aligned K1 rows >= 16 KB);
//              K2 (fp32 / fp64 rows that fit) keeps the row resident, and rows larger
//              than the ring are split over a thread-block cluster whose CTAs exchange
//              their partials through DSMEM; pass 2 rewrites each chunk in place.
//   tmem     : K2 for all aligned 16-bit rows and fp32 rows beyond the ring
//              (ppo_tmem.cuh): the row's first 8 chunks are parked in Tensor Memory as
//              e = 2^(x - c), up to 7 more stay resident in the ring, any further
//              middle chunks are streamed and re-read from L2 in pass 2; one CTA per
//              row (the bf16 V ~ 152K default).  Unaligned 16/32-bit rows too (UNAL
//              instantiation: bulk copies from the 16-byte boundary below the row).
// HBM traffic = one logits read (+ one dlogits write for K2) per element.
#include <algorithm>
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
  int prox_from_lp;        // prox := lp (first minibatch of a step)
  // ring kernel geometry
  int cluster_size;
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

// Given scale = exp(prox - behav) (1 for naive) and ratio = exp(lp - prox|behav).
__device__ __forceinline__ TokenTerms ppo_token_terms(double scale, double ratio, double adv,
                                                      int version, const PpoArgs& a) {
  TokenTerms t;
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

__device__ __forceinline__ TokenTerms ppo_token(double lp, double behav, double prox, double adv,
                                                int version, const PpoArgs& a) {
  if (a.decoupled)  // trainer.py:166-167
    return ppo_token_terms(exp(__dsub_rn(prox, behav)), exp(__dsub_rn(lp, prox)), adv, version, a);
  return ppo_token_terms(1.0, exp(__dsub_rn(lp, behav)), adv, version, a);  // trainer.py:169-170
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
  // factor taking sums accumulated against shift(m_old) to the new shift c: the exact
  // 2^(shift(m_old) - c) (0 when m_old = -inf), not e(m_old, c), which would carry the
  // old shift's rounding residual into every max move
  static __device__ __forceinline__ float rescale(float m_old, float c) {
    return fast_exp2(__fmul_rn(m_old, Lim<float>::kLog2e) - c);
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
  static __device__ __forceinline__ double rescale(double m_old, double c) { return exp(m_old - c); }
  static __device__ __forceinline__ double lse_shift(double m, double s) { return m + log(s); }
  static __device__ __forceinline__ double lse_nat(double l) { return l; }
};

// Fold a batch of values (already max-reduced into lmax) into a running RowStat.
template <typename A, int N>
__device__ __forceinline__ void fold(RowStat<A>& rs, const A (&v)[N], A lmax) {
  const A mn = fmax(rs.m, lmax);
  const A muse = (mn == Lim<A>::ninf()) ? A(0) : mn;
  const A c = Ex<A>::shift(muse);
  // rescale of the old partial sums (0 when m = -inf); exactly 1 when the max did not
  // move — Ex::e(m, shift(m)) is 2^(rounding residual), a same-signed bias that would
  // compound over the row's fold calls
  const A r = mn == rs.m ? A(1) : Ex<A>::rescale(rs.m, c);
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
    if (sizeof(T) <= 4) {
      // 16/32-bit logits: scalar head up to the first 16-byte boundary, 16-byte vector
      // body (4 loads per lane in flight), scalar tail (bf16 V = 4,096: 2.87 -> 4.87
      // TB/s).  fp64 keeps the 8-deep scalar fold below.
      constexpr int E = Vec<T>::N, U = 4;
      using Un = typename std::conditional<std::is_same<T, double>::value, double, float>::type;
      int64_t nh = (int64_t)(((16 - ((uintptr_t)x & 15)) & 15) / sizeof(T));
      if (nh > V) nh = V;
      const uint4* xv = reinterpret_cast<const uint4*>(x + nh);
      const int64_t nv = (V - nh) / E;
      const int64_t t0 = nh + nv * E;
      for (int64_t i = lane; i < nh + (V - t0); i += 32) {  // head and tail elements
        const int64_t k = i < nh ? i : t0 + (i - nh);
        const A v1[1] = {Traits<T>::to_acc(x[k])};
        fold(rs, v1, v1[0]);
      }
      for (int64_t base = 0; base < nv; base += 32 * U) {
        uint4 q[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t i = base + u * 32 + lane;
          q[u] = i < nv ? xv[i] : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (base + u * 32 + lane < nv) {
            Un g[E];
            Vec<T>::unpack(q[u], g);
            A v[E];
            A lmax = Lim<A>::ninf();
#pragma unroll
            for (int e = 0; e < E; ++e) {
              v[e] = (A)g[e];
              lmax = fmax(lmax, v[e]);
            }
            fold(rs, v, lmax);
          }
        }
      }
    } else {
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
        const double prox = a.prox_from_lp ? lp : (a.prox ? a.prox[idx] : 0.0);
        const TokenTerms t = ppo_token(lp, a.behav[idx], prox, a.adv[idx],
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

}  // namespace areal

#include "ppo_ring.cuh"
#include "ppo_tmem.cuh"

namespace areal {

// ================================================================== row_cta kernel
// Rows whose byte length or start is not 16-byte aligned (e.g. bf16 V = 50,257: the
// 1-D bulk copies of the ring / TMEM kernels need 16-byte granules).  One 512-thread
// CTA per row, 2 CTAs per SM, so the rows in flight (~300 x 100 KB) stay in L2 and
// pass 2's re-read does not go back to HBM.  Each row is split into a scalar head up
// to the first 16-byte boundary, a 16-byte-vector body and a scalar tail; dlogits use
// vector stores when their row has the same 16-byte phase as the logits row.
// K1 (read-only) wants many rows in flight to hide each row's serial epilogue: 8 x 256
// threads per SM; K2 re-reads each row in pass 2 and wants it still in L2: 2 x 512
// (profiles/r01_rowcta_sweep.txt).
template <bool BWD> struct RowCtaGeo {
  static constexpr int kThreads = BWD ? 512 : 256;
  static constexpr int kBlocks = BWD ? 2 : 8;  // CTAs per SM
};
constexpr int kRowCtaUnroll = 4;

template <typename T>
struct RowSplit {
  int64_t nh, nv, V;  // head elements, body vectors, row length
  __device__ __forceinline__ RowSplit(const char* x, int64_t V_) : V(V_) {
    const int hb = (int)((16 - ((uintptr_t)x & 15)) & 15);
    nh = hb / (int)sizeof(T);
    if (nh > V) nh = V;
    nv = (V - nh) / Vec<T>::N;
  }
  __device__ __forceinline__ int64_t tail0() const { return nh + nv * Vec<T>::N; }
};

// Per-thread running (m, s, sx) over E values at a time.  fp32: the shift moves only
// when a vector raises the thread's max (rare after the first few), so most vectors
// are FFMA2 + 2 MUFU ex2 + FADD2 per pair; fp64: the generic fold.
template <typename A, bool ENT, int E>
__device__ __forceinline__ void rowcta_fold(RowStat<A>& rs, const A (&f)[E]) {
  A lmax = f[0];
#pragma unroll
  for (int e = 1; e < E; ++e) lmax = fmax(lmax, f[e]);
  if constexpr (std::is_same<A, float>::value && E % 2 == 0) {
    if (lmax > rs.m) {
      const float r = rs.m == Lim<float>::ninf() ? 0.f
          : fast_exp2(__fmul_rn(rs.m, Lim<float>::kLog2e) - __fmul_rn(lmax, Lim<float>::kLog2e));
      rs.s *= r;
      if (ENT) rs.sx *= r;
      rs.m = lmax;
    }
    if (rs.m == Lim<float>::ninf()) return;  // only -inf so far: contributes nothing
    const float c = rs.m * Lim<float>::kLog2e;
    const float2 L2 = make_float2(Lim<float>::kLog2e, Lim<float>::kLog2e);
    const float2 C2 = make_float2(-c, -c);
    float2 s2 = make_float2(0.f, 0.f), x2 = make_float2(0.f, 0.f);
#pragma unroll
    for (int e = 0; e < E; e += 2) {
      const float2 v = make_float2(f[e], f[e + 1]);
      const float2 t = ffma2(v, L2, C2);
      const float2 ee = make_float2(fast_exp2(t.x), fast_exp2(t.y));
      s2 = fadd2(s2, ee);
      if (ENT)
        x2 = ffma2(ee, make_float2(fmaxf(v.x, Lim<float>::lowest()), fmaxf(v.y, Lim<float>::lowest())), x2);
    }
    rs.s += s2.x + s2.y;
    if (ENT) rs.sx += x2.x + x2.y;
  } else {
    fold(rs, f, lmax);
  }
}

template <typename T, bool BWD, bool ENT, int NT = RowCtaGeo<BWD>::kThreads>
__device__ __forceinline__ void row_cta_body(const PpoArgs& a) {
  constexpr int kRowCtaThreads = NT;
  using A = typename Traits<T>::Acc;
  constexpr int E = Vec<T>::N;
  using U = typename std::conditional<std::is_same<T, double>::value, double, float>::type;
  constexpr int NW = kRowCtaThreads / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  __shared__ A red[NW][3];
  __shared__ double bc[4];  // g, lse_s, token, token's dlogit
  double st[AREAL_N_STATS];
#pragma unroll
  for (int j = 0; j < AREAL_N_STATS; ++j) st[j] = 0.0;
  const int64_t V = a.vocab;
  for (int64_t row = blockIdx.x; row < a.n_rows; row += gridDim.x) {
    const char* xb = a.logits + row * a.ld_in_bytes;
    const T* x = reinterpret_cast<const T*>(xb);
    const RowSplit<T> sp(xb, V);
    const uint4* xv = reinterpret_cast<const uint4*>(x + sp.nh);
    const int64_t t0 = sp.tail0();
    const int64_t n_edge = sp.nh + (V - t0);
    RowStat<A> rs;
    rs.init();
    // ---- pass 1: head / tail scalars, then the vector body kRowCtaUnroll deep
    for (int64_t i = tid; i < n_edge; i += kRowCtaThreads) {
      const int64_t k = i < sp.nh ? i : t0 + (i - sp.nh);
      const A v[1] = {Traits<T>::to_acc(x[k])};
      fold(rs, v, v[0]);
    }
    for (int64_t i0 = tid; i0 < sp.nv; i0 += kRowCtaThreads * kRowCtaUnroll) {
      uint4 q[kRowCtaUnroll];
#pragma unroll
      for (int u = 0; u < kRowCtaUnroll; ++u) {
        const int64_t i = i0 + (int64_t)u * kRowCtaThreads;
        q[u] = i < sp.nv ? xv[i] : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < kRowCtaUnroll; ++u) {
        if (i0 + (int64_t)u * kRowCtaThreads < sp.nv) {
          U g[E];
          Vec<T>::unpack(q[u], g);
          A f[E];
#pragma unroll
          for (int e = 0; e < E; ++e) f[e] = (A)g[e];
          rowcta_fold<A, ENT, E>(rs, f);
        }
      }
    }
    rs.warp_reduce();
    if (lane == 0) {
      red[warp][0] = rs.m;
      red[warp][1] = rs.s;
      red[warp][2] = rs.sx;
    }
    __syncthreads();
    if (warp == 0) {
      RowStat<A> w;
      if (lane < NW) {
        w.m = red[lane][0];
        w.s = red[lane][1];
        w.sx = red[lane][2];
      } else {
        w.init();
      }
      w.warp_reduce();
      if (lane == 0) {
        const A lse_s = Ex<A>::lse_shift(w.m == Lim<A>::ninf() ? A(0) : w.m, w.s);
        const double lse = Ex<A>::lse_nat(lse_s);
        const double ent = ENT ? lse - (double)(w.sx / w.s) : 0.0;
        const int64_t idx = a.row_index ? (int64_t)a.row_index[row] : row;
        const int64_t tok = a.tokens[idx];
        const double xt = token_logit<T>(a, x, tok);
        const double lp = xt - lse;
        if (a.lp_out) a.lp_out[idx] = lp;
        if (ENT && a.ent_out) a.ent_out[idx] = ent;
        if (BWD) {
          const double prox = a.prox_from_lp ? lp : (a.prox ? a.prox[idx] : 0.0);
          const TokenTerms t = ppo_token(lp, a.behav[idx], prox, a.adv[idx],
                                         a.versions ? a.versions[idx] : 0, a);
          stats_add(st, t, ENT ? ent : 0.0);
          const double gc = a.grad_scale * t.coef;
          bc[0] = gc;
          bc[1] = (double)lse_s;
          bc[2] = (double)tok;
          bc[3] = gc * (exp(lp) - 1.0);
        }
      }
    }
    __syncthreads();
    if (BWD) {
      // ---- pass 2 (re-read from L2): dlogits = g * softmax; the one-hot element is
      // patched after a barrier by thread 0 (the barrier orders the two stores)
      const A g = (A)bc[0];
      const A lse_s = (A)bc[1];
      char* db = a.dlogits + row * a.ld_out_bytes;
      T* d = reinterpret_cast<T*>(db);
      auto dsm = [&](A xv_) {
        if constexpr (std::is_same<A, float>::value)
          return g * fast_exp2(fmaf(xv_, Lim<float>::kLog2e, -lse_s));
        else
          return g * exp(xv_ - lse_s);
      };
      for (int64_t i = tid; i < n_edge; i += kRowCtaThreads) {
        const int64_t k = i < sp.nh ? i : t0 + (i - sp.nh);
        d[k] = Traits<T>::from_acc(dsm(Traits<T>::to_acc(x[k])));
      }
      const bool vec_out = (((uintptr_t)db ^ (uintptr_t)xb) & 15) == 0;
      uint4* dv = reinterpret_cast<uint4*>(d + sp.nh);
      for (int64_t i0 = tid; i0 < sp.nv; i0 += kRowCtaThreads * kRowCtaUnroll) {
        uint4 q[kRowCtaUnroll];
#pragma unroll
        for (int u = 0; u < kRowCtaUnroll; ++u) {
          const int64_t i = i0 + (int64_t)u * kRowCtaThreads;
          q[u] = i < sp.nv ? __ldcs(xv + i) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < kRowCtaUnroll; ++u) {
          const int64_t i = i0 + (int64_t)u * kRowCtaThreads;
          if (i < sp.nv) {
            U gg[E];
            Vec<T>::unpack(q[u], gg);
#pragma unroll
            for (int e = 0; e < E; ++e) gg[e] = (U)dsm((A)gg[e]);
            if (vec_out) {
              __stcs(dv + i, Vec<T>::pack(gg));
            } else {
              const int64_t k0 = sp.nh + i * E;
#pragma unroll
              for (int e = 0; e < E; ++e) d[k0 + e] = Traits<T>::from_acc((A)gg[e]);
            }
          }
        }
      }
      __syncthreads();
      const int64_t tok = (int64_t)bc[2];
      if (tid == 0 && tok >= 0 && tok < V) d[tok] = Traits<T>::from_acc((A)bc[3]);
    }
  }
  if (BWD) {
    __shared__ double cst[AREAL_N_STATS];
    if (tid == 0)
      for (int j = 0; j < AREAL_N_STATS; ++j) cst[j] = st[j];
    __syncthreads();
    double cta[AREAL_N_STATS];
    for (int j = 0; j < AREAL_N_STATS; ++j) cta[j] = cst[j];
    finalize_stats(a, cta, kRowCtaThreads);
  }
}

template <typename T, bool ENT>
__global__ void __launch_bounds__(RowCtaGeo<false>::kThreads, RowCtaGeo<false>::kBlocks)
    logprob_rowcta_kernel(PpoArgs a) {
  row_cta_body<T, false, ENT>(a);
}
template <typename T, bool ENT>
__global__ void __launch_bounds__(RowCtaGeo<true>::kThreads, RowCtaGeo<true>::kBlocks)
    ppo_rowcta_kernel(PpoArgs a) {
  row_cta_body<T, true, ENT>(a);
}
// K2 on short rows (<= 32 KB): 8 x 256 threads per SM, like K1 — the rows in flight
// still fit L2 and the per-row epilogues overlap across 8 CTAs.
template <typename T, bool ENT>
__global__ void __launch_bounds__(256, 8) ppo_rowcta_small_kernel(PpoArgs a) {
  row_cta_body<T, true, ENT, 256>(a);
}


template <typename T, bool ENT, bool UNAL>
__global__ void __launch_bounds__(kTThreads, 1) ppo_tmem_kernel(PpoArgs a) {
  if constexpr (sizeof(T) == 2 || sizeof(T) == 4) tmem_k2_body<T, ENT, UNAL>(a);
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
template <typename T, bool ENT, bool UNAL = false>
__global__ void __launch_bounds__(kRingThreads, 1) logprob_ring_kernel(PpoArgs a) {
  row_ring_body<T, false, ENT, UNAL>(a);
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

static size_t tmem_smem_bytes(int nslots) {
  return (size_t)nslots * kChunkBytes + 2 * (size_t)nslots * sizeof(uint64_t) + sizeof(TmemTail);
}

template <typename T, bool ENT, bool UNAL = false>
static int launch_tmem(PpoArgs a, cudaStream_t stream, const DevInfo& d, int nslots) {
  if (a.vocab >= (int64_t)1 << 30) return AREAL_ERR_UNSUPPORTED;  // 32-bit element indices
  if (a.n_rows >= ((int64_t)1 << 31) - 4096) return AREAL_ERR_UNSUPPORTED;  // int row queue
  a.cluster_size = 1;
  a.slice16 = (a.vocab * (int64_t)sizeof(T)) / 16;
  a.nslots = nslots;
  const size_t smem = tmem_smem_bytes(nslots);
  if (smem + 256 > (size_t)d.smem_optin) return AREAL_ERR_UNSUPPORTED;  // + static smem
  auto kern = ppo_tmem_kernel<T, ENT, UNAL>;
  static thread_local int attr_set[16] = {0};
  const int dev = d.dev & 15;
  if (!attr_set[dev]) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return AREAL_ERR_CUDA;
    attr_set[dev] = 1;
  }
  const int64_t grid = std::min<int64_t>(a.n_rows, (int64_t)d.sms);  // one CTA (all of TMEM) per SM
  kern<<<(unsigned)grid, kTThreads, smem, stream>>>(a);
  AREAL_CUDA_CHECK_LAUNCH();
  return AREAL_OK;
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
    {
      // AREAL_TUNE_K2_CLUSTER_SIZE in {2, 4, 8} forces a larger vocab split
      const int64_t force = tuning(AREAL_TUNE_K2_CLUSTER_SIZE);
      if (force > CS) CS = (int)force;
    }
    // A row too long for one CTA's shared memory but within shared memory + TMEM
    // runs on the single-CTA TMEM kernel (no cluster split) unless disabled.
    if constexpr (sizeof(T) == 2 || sizeof(T) == 4) {
      const bool tmem_off = tuning(AREAL_TUNE_K2_TMEM) == 0;
      const int64_t row_chunks = (V16 * 16 + kChunkBytes - 1) / kChunkBytes;
      // rows beyond TMEM + the ring stream their middle chunks (ppo_tmem.cuh)
      const bool stream_off = tuning(AREAL_TUNE_K2_TMEM_STREAM) == 0;
      // 16-bit rows that fit the ring also run faster on the TMEM kernel (e-form
      // pass 2, longer lookahead): bf16 V = 32,000 5.83 -> 6.51 TB/s, V = 65,536
      // 5.95 -> 6.65; fp32 rows that fit stay on the ring (V = 32,000: 6.67 vs 6.39)
      // (profiles/r01_k2_small_rows_tmem.txt)
      const bool small_ok = sizeof(T) == 2;
      if ((CS > 1 || small_ok) && cs_force == 0 && !tmem_off && nslots == 7 &&
          (row_chunks <= kTmemMaxChunks || !stream_off))
        return launch_tmem<T, ENT>(a, stream, d, nslots);
    }
  }
  if (!BWD && cs_force == 0) {
    // K1 on few long rows (decode steps): rows that fit one wave of CTA pairs are split
    // over a 2-CTA cluster (B = 64 x V = 151,936 bf16: 10.2 -> 9.5 us, L2-hot 8.9 -> 7.6 us).
    // Wider splits and multi-wave splits measured slower (B = 256: CS 1 17.9 us, 2 18.7,
    // 4 22.9, 8 47.2; profiles/r02_k1_cluster_split.txt): per-row MUFU work and the fixed
    // launch / pipeline-fill latency bound these shapes, not HBM.
    const int64_t forced = tuning(AREAL_TUNE_K1_CLUSTER_SIZE);
    if (forced > 0) CS = (int)forced;
    else if (a.n_rows <= d.sms / 2 && V16 * 16 >= 4 * (int64_t)kChunkBytes) CS = 2;
  }
  if ((V16 + CS - 1) / CS * 16 > (int64_t)0x7fffffff) return AREAL_ERR_UNSUPPORTED;
  a.cluster_size = CS;
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

// K1 on rows off a 16-byte boundary: the ring kernel's UNAL instantiation (bulk
// copies from the boundary below each row, masked edge elements), one CTA per SM.
template <typename T, bool ENT>
static int launch_ring_k1_unal(PpoArgs a, cudaStream_t stream) {
  DevInfo d = get_dev();
  const int nslots = max_slots(d);
  a.cluster_size = 1;
  a.slice16 = (a.vocab * (int64_t)sizeof(T)) / 16;
  a.nslots = nslots;
  const size_t smem = ring_smem_bytes(nslots);
  auto kern = logprob_ring_kernel<T, ENT, true>;
  static thread_local int attr_set[16] = {0};
  const int dev = d.dev & 15;
  if (!attr_set[dev]) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return AREAL_ERR_CUDA;
    attr_set[dev] = 1;
  }
  const int64_t grid = std::min<int64_t>(a.n_rows, (int64_t)d.sms);
  kern<<<(unsigned)grid, kRingThreads, smem, stream>>>(a);
  AREAL_CUDA_CHECK_LAUNCH();
  return AREAL_OK;
}

// Unaligned rows of 16/32-bit logits whose head bytes never add a 32 KB chunk.
static bool unaligned_chunks_ok(const PpoArgs& a, int es) {
  const int64_t rb = a.vocab * es;
  if (rb < 16384 || a.vocab >= ((int64_t)1 << 30) || !(es == 2 || es == 4)) return false;
  const int64_t lo = (rb + 15) & ~(int64_t)15, hi = (rb + 16 - es + 15) & ~(int64_t)15;
  return (lo + kChunkBytes - 1) / kChunkBytes == (hi + kChunkBytes - 1) / kChunkBytes;
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

template <typename T, bool BWD>
static int launch_rowcta(PpoArgs a, cudaStream_t stream, bool small = false) {
  DevInfo d = get_dev();
  if (BWD && small) {
    const int64_t grid = std::min<int64_t>(a.n_rows, (int64_t)d.sms * 8);
    auto kern = a.ent_out ? ppo_rowcta_small_kernel<T, true> : ppo_rowcta_small_kernel<T, false>;
    kern<<<(unsigned)grid, 256, 0, stream>>>(a);
    AREAL_CUDA_CHECK_LAUNCH();
    return AREAL_OK;
  }
  const int64_t grid = std::min<int64_t>(a.n_rows, (int64_t)d.sms * RowCtaGeo<BWD>::kBlocks);
  auto kern = a.ent_out ? (BWD ? ppo_rowcta_kernel<T, true> : logprob_rowcta_kernel<T, true>)
                        : (BWD ? ppo_rowcta_kernel<T, false> : logprob_rowcta_kernel<T, false>);
  kern<<<(unsigned)grid, RowCtaGeo<BWD>::kThreads, 0, stream>>>(a);
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

static bool tmem_unaligned_ok(const PpoArgs& a, int es) {
  // AREAL_TUNE_K2_TMEM_UNALIGNED = 0: unaligned rows on the row-CTA kernel
  const bool off = tuning(AREAL_TUNE_K2_TMEM_UNALIGNED) == 0;
  if (off || a.dlogits == nullptr) return false;
  const int64_t rb = a.vocab * es;
  if (rb < 16384) return false;
  if ((((uintptr_t)a.dlogits - (uintptr_t)a.logits) & 15) != 0) return false;
  if (((a.ld_out_bytes - a.ld_in_bytes) & 15) != 0) return false;
  const int64_t lo = (rb + 15) & ~(int64_t)15, hi = (rb + 16 - es + 15) & ~(int64_t)15;
  return (lo + kChunkBytes - 1) / kChunkBytes == (hi + kChunkBytes - 1) / kChunkBytes;
}

// AREAL_TUNE_K1_RING_UNALIGNED = 0: unaligned K1 rows on the row-CTA kernel
static bool k1_unal_off() { return tuning(AREAL_TUNE_K1_RING_UNALIGNED) == 0; }

// K2 rows up to this many KB on the short-row kernel (-1: the default rule)
static int64_t small_rowcta_kb() { return tuning(AREAL_TUNE_K2_SMALL_ROWCTA_KB); }

// AREAL_TUNE_ROWCTA = 0: unaligned rows on the one-warp kernel
static bool rowcta_off() { return tuning(AREAL_TUNE_ROWCTA) == 0; }

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
  // short K2 rows: one CTA per row, 8 per SM (beats the TMEM / ring / one-warp
  // kernels up to 16 KB rows, and fp32 rows up to 32 KB; profiles/r01_k2_small_rows_tmem.txt)
  const int64_t small_kb = small_rowcta_kb();
  const int64_t small_lim = small_kb >= 0 ? small_kb * 1024 : (es == 4 ? 32768 : 16384);
  const bool small_row = a.vocab * es <= small_lim && a.vocab >= 256 && es <= 4;  // fp64: one-warp kernel
  if (BWD && small_row && algo == AREAL_ALGO_AUTO) {
    switch (dtype) {
      case AREAL_F32: return launch_rowcta<float, BWD>(a, stream, true);
      case AREAL_BF16: return launch_rowcta<__nv_bfloat16, BWD>(a, stream, true);
      case AREAL_F16: return launch_rowcta<__half, BWD>(a, stream, true);
      case AREAL_F64: return launch_rowcta<double, BWD>(a, stream, true);
      default: return AREAL_ERR_BAD_DTYPE;
    }
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
  // unaligned K2 rows of >= 16 KB on the TMEM kernel: each row is loaded from the
  // 16-byte boundary below it (masked head / tail elements); needs dlogits rows at the
  // same 16-byte phase and a chunk count that the head bytes never change
  if (BWD && !aligned && algo == AREAL_ALGO_AUTO && (es == 2 || es == 4) && tmem_unaligned_ok(a, es)) {
    DevInfo d = get_dev();
    const int nslots = max_slots(d);
    if (nslots == 7) {
      const bool ent = a.ent_out != nullptr;
      int rc = AREAL_ERR_UNSUPPORTED;
      switch (dtype) {
        case AREAL_F32: rc = ent ? launch_tmem<float, true, true>(a, stream, d, nslots) : launch_tmem<float, false, true>(a, stream, d, nslots); break;
        case AREAL_BF16: rc = ent ? launch_tmem<__nv_bfloat16, true, true>(a, stream, d, nslots) : launch_tmem<__nv_bfloat16, false, true>(a, stream, d, nslots); break;
        case AREAL_F16: rc = ent ? launch_tmem<__half, true, true>(a, stream, d, nslots) : launch_tmem<__half, false, true>(a, stream, d, nslots); break;
        default: break;
      }
      if (rc != AREAL_ERR_UNSUPPORTED) return rc;
    }
  }
  // unaligned K1 rows: the ring kernel from the 16-byte boundary below each row
  // (long rows only: below ~160 KB (16-bit) / 256 KB (fp32) the row-CTA kernel's 8 rows
  // per SM hide the per-row epilogue better; profiles/r01_rowcta_sweep.txt)
  const bool k1_ring_long = a.vocab * es >= (es == 2 ? 160 * 1024 : 256 * 1024);
  if (!BWD && !aligned && algo == AREAL_ALGO_AUTO && k1_ring_long && unaligned_chunks_ok(a, es) &&
      !k1_unal_off()) {
    const bool ent = a.ent_out != nullptr;
    switch (dtype) {
      case AREAL_F32: return ent ? launch_ring_k1_unal<float, true>(a, stream) : launch_ring_k1_unal<float, false>(a, stream);
      case AREAL_BF16: return ent ? launch_ring_k1_unal<__nv_bfloat16, true>(a, stream) : launch_ring_k1_unal<__nv_bfloat16, false>(a, stream);
      case AREAL_F16: return ent ? launch_ring_k1_unal<__half, true>(a, stream) : launch_ring_k1_unal<__half, false>(a, stream);
      default: break;
    }
  }
  // unaligned (or ring-refused) rows of >= 16 KB: one CTA per row, body in 16-byte vectors
  if (algo == AREAL_ALGO_AUTO && a.vocab * es >= 16384 && !rowcta_off()) {
    switch (dtype) {
      case AREAL_F32: return launch_rowcta<float, BWD>(a, stream, small_row);
      case AREAL_BF16: return launch_rowcta<__nv_bfloat16, BWD>(a, stream, small_row);
      case AREAL_F16: return launch_rowcta<__half, BWD>(a, stream, small_row);
      case AREAL_F64: return launch_rowcta<double, BWD>(a, stream, small_row);
      default: return AREAL_ERR_BAD_DTYPE;
    }
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
  PpoArgs a = {};
  // K1's ring kernel takes its rows from workspace counters when a workspace is given
  // (static row order without one)
  if (workspace && workspace_bytes >= AREAL_WORKSPACE_BYTES && n_rows < ((int64_t)1 << 31) - 4096)
    a.counter = static_cast<unsigned int*>(workspace);
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
  if (params->decoupled && !prox && !params->prox_from_lp) return AREAL_ERR_INVALID_ARGUMENT;
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
  a.prox_from_lp = params->prox_from_lp ? 1 : 0;
  return dispatch<true>(a, dtype, params->algo, static_cast<cudaStream_t>(stream));
}
