// advantages.cu — K3: per-token advantages for sm_100a.
//
// Reference: compute_advantages (/root/reference/pkg/src/asyncrl/trainer.py:114-125):
//   raw_t = reward of the trajectory owning t;  std = np.std(raw);
//   std == 0 -> zeros, else (raw - np.mean(raw)) / std.
// The GLOBAL normalisation replays numpy's float64 pairwise summation tree
// (8-way unrolled leaves of <= 128 elements, split at n/2 rounded down to a
// multiple of 8) so mean/std — and therefore every advantage — are bit-identical
// to the reference.  Leaves of the tree are summed by many threads in parallel and
// folded in tree order inside one cooperative launch (adv_global_fused_kernel).
//
// Extensions (north star): GAE reverse scan per sequence (one warp per
// trajectory, segmented affine warp scan) and GRPO group normalisation.
#include <cooperative_groups.h>

#include "common.cuh"
#include "pairwise.cuh"

namespace areal {

constexpr int kMaxTreeDepth = 20;    // <= 2^20 cut-depth nodes (T <= 128 * 2^20 tokens)
constexpr int kLeafThreadsLog2 = 15;  // <= 2^15 leaf threads (128 CTAs x 256), <= 32 nodes each

struct AdvArgs {
  const double* rewards;
  const int64_t* bounds;
  int64_t n_traj, n_tokens;
  const double* values;
  const int32_t* group_ids;
  int32_t n_groups;
  double gamma, lam, eps;
  int mode, norm;
  double* adv;
  double* returns;
  double* norm_stats;  // [2] mean, std (device, may be null)
  double* ws;          // workspace: [8..] per-CTA subtree roots
};

// ---------------------------------------------------------------- raw advantages
// One warp per trajectory.  REFERENCE: broadcast the reward (trainer.py:117-118).
// GAE: A_t = delta_t + c*A_{t+1}, c = gamma*lam, delta_t = r_t + gamma*V_{t+1} - V_t,
// reward on the final token only, V past the end = 0.  The scan runs from the end
// in 32-token chunks: inclusive warp scan of the affine recurrence + carry.
__global__ void adv_raw_kernel(AdvArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t k = w; k < a.n_traj; k += nw) {
    const int64_t s = a.bounds[k], e = a.bounds[k + 1];
    const double R = a.rewards[k];
    if (a.mode == AREAL_ADV_REFERENCE) {
      for (int64_t t = s + lane; t < e; t += 32) {
        a.adv[t] = R;
        if (a.returns) a.returns[t] = R;
      }
      continue;
    }
    const double c = a.gamma * a.lam;
    double cp[5];  // c^(2^i)
    cp[0] = c;
    for (int i = 1; i < 5; ++i) cp[i] = cp[i - 1] * cp[i - 1];
    double clane = 1.0;  // c^(lane+1)
    {
      double b = c;
      int ex = lane + 1;
      while (ex) {
        if (ex & 1) clane *= b;
        b *= b;
        ex >>= 1;
      }
    }
    double carry = 0.0;  // A_{t+1} of the chunk boundary
    for (int64_t j0 = 0; j0 < e - s; j0 += 32) {
      const int64_t j = j0 + lane;       // reversed index: j = 0 is the last token
      const int64_t t = e - 1 - j;
      double x = 0.0;
      if (j < e - s) {
        const double r = (t == e - 1) ? R : 0.0;
        const double vt = a.values ? a.values[t] : 0.0;
        const double vn = (a.values && t + 1 < e) ? a.values[t + 1] : 0.0;
        x = r + a.gamma * vn - vt;
      }
#pragma unroll
      for (int i = 0; i < 5; ++i) {
        const int o = 1 << i;
        const double y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x = x + cp[i] * y;
      }
      x = x + clane * carry;
      if (j < e - s) {
        a.adv[t] = x;
        if (a.returns) a.returns[t] = x + (a.values ? a.values[t] : 0.0);
      }
      carry = __shfl_sync(0xffffffffu, x, 31);
    }
  }
}

__host__ __device__ inline int pw_depth(int64_t n) { return pw_depth(n, kMaxTreeDepth); }

// x_t (pass 0) or (x_t - mean)^2 (pass 1) read from memory, IEEE-rounded per operation
struct PwMem {
  const double* x;
  int pass;
  double mean;
  __device__ __forceinline__ double operator()(int64_t i) const {
    const double v = x[i];
    if (pass == 0) return v;
    const double d = __dsub_rn(v, mean);
    return __dmul_rn(d, d);
  }
};

// ---------------------------------------------------------------- fused global normalisation
// One cooperative launch for trainer.py:116-123 (raw -> np.mean -> np.std -> (raw-mean)/std),
// bit-exact.  The 2^D leaves of numpy's pairwise tree (pw_depth) are summed one per thread;
// each of the first 2^D / 256 CTAs owns 256 consecutive leaves — an aligned perfect
// subtree — and folds them in shared memory; after a grid barrier every CTA folds the CTA
// roots itself (no second launch, no single-CTA tail).  Nodes above the leaves all split in
// two (pw_depth), so the folds are perfect binary trees and match numpy's recursion exactly.
//
// REFERENCE mode never materialises raw advantages: raw_t = r_k is piecewise constant per
// trajectory, so a leaf (<= 128 tokens, typically inside one trajectory) replays numpy's
// 8-accumulator loop on register values that change only at trajectory bounds (staged in
// shared memory), and the final pass writes each trajectory's constant (r_k - mean) / std
// with 16-byte stores — the only HBM traffic is the T x 8-byte output (+ returns).
// GAE mode reads the raw advantages adv_raw_kernel wrote and rewrites them in place.
#ifndef AREAL_K3_PROBE_LEAVES  // phase-timing probes (tools/k3_phase_probe.cu); empty in the product
#define AREAL_K3_PROBE_LEAVES
#define AREAL_K3_PROBE_WRITE
#define AREAL_K3_PROBE_TS(i)
#endif
constexpr int kFuseThreads = 256;
constexpr int kFuseBoundsSmem = 4096;  // trajectories whose bounds are staged in shared memory

// Piecewise-constant value stream over increasing positions: v(t) = val(k(t)).
struct SegCursor {
  const int64_t* bounds;
  const double* rewards;
  int64_t k, next;  // trajectory holding the current position, its end
  double v;         // its value under the current pass
  int pass;
  double mean;
  __device__ __forceinline__ double value_of(int64_t kk) const {
    const double r = rewards[kk];
    if (pass == 0) return r;
    const double d = __dsub_rn(r, mean);
    return __dmul_rn(d, d);
  }
  __device__ void seek(int64_t t, int64_t n_traj) {  // bounds[k] <= t < bounds[k+1]
    int64_t lo = 0, hi = n_traj;
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (bounds[mid] <= t) lo = mid;
      else hi = mid;
    }
    k = lo;
    next = bounds[k + 1];
    v = value_of(k);
  }
  __device__ __forceinline__ double at(int64_t t) {  // non-decreasing t
    if (t >= next) {
      do { ++k; next = bounds[k + 1]; } while (t >= next);
      v = value_of(k);
    }
    return v;
  }
};

// numpy's pairwise_sum over positions [off, off + n <= off + 128) of the cursor's stream
// (the leaf case of pairwise.cuh), inlined so the cursor stays in registers.
__device__ __forceinline__ double seg_leaf_small(SegCursor& c, int64_t off, int64_t n) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; ++i) res = __dadd_rn(res, c.at(off + i));
    return res;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = c.at(off + j);
  int64_t i = 8;
  for (; i < n - (n % 8); i += 8) {
    if (off + i + 7 < c.next) {  // the whole group inside one trajectory: one value
      const double v = c.v;
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], v);
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], c.at(off + i + j));
    }
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, c.at(off + i));
  return res;
}

// A node at the cut depth is at most 143 long (the cut is set by the smallest node and
// sizes at one depth differ by < 32; checked exhaustively in tests/test_oracle_golden.py),
// so numpy splits it at most once more: both halves are then <= 128-element leaves.
__device__ __forceinline__ void node_split(int64_t n, int64_t& n2) {
  n2 = n / 2;
  n2 -= n2 % 8;
}

// Perfect-binary fold of buf[0..n) (n a power of two, n <= blockDim) in tree order; the
// result is returned to every thread.  Warp shuffles for the bottom 5 levels (lane pairs
// (2i, 2i+1), then (4i, 4i+2), ... — the same pairs as the tree), one warp for the rest.
__device__ double fold_pow2(double* buf, int n, double* warp_part) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  double v = (int)threadIdx.x < n ? buf[threadIdx.x] : 0.0;
  const int wn = n < 32 ? n : 32;  // values per warp
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double u = __shfl_down_sync(0xffffffffu, v, o);
    if (o < wn && (lane & (2 * o - 1)) == 0) v = __dadd_rn(v, u);
  }
  if (lane == 0 && (int)threadIdx.x < n) warp_part[wid] = v;
  __syncthreads();
  const int nw = n / wn;  // warps holding a partial (power of two, <= 8)
  double r = warp_part[0];
  if (nw > 1) {
    double x = lane < nw ? warp_part[lane] : 0.0;
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      const double u = __shfl_down_sync(0xffffffffu, x, o);
      if (o < nw && (lane & (2 * o - 1)) == 0) x = __dadd_rn(x, u);
    }
    r = __shfl_sync(0xffffffffu, x, 0);
  }
  return r;  // every warp folds the (shared) warp partials itself: valid in all threads
}

// Repeated-addition table of one trajectory: S[c-1] = v + v + ... + v (c terms, IEEE
// sequential order) for c = 1..16 — every accumulator of a numpy leaf (<= 128 elements,
// 8 accumulators) that stays inside one trajectory holds S[c-1] for its count c.
constexpr int kRepTab = 16;
constexpr int kTabTraj = 64;  // trajectories per CTA token range with a table

template <bool FROM_MEM, bool SMEM_BOUNDS>
__global__ void __launch_bounds__(kFuseThreads) adv_global_fused_kernel(AdvArgs a, int depth, int leaf_ctas,
                                                                        int lpt_log2) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ int64_t sb[SMEM_BOUNDS ? kFuseBoundsSmem + 1 : 1];
  __shared__ double buf[kFuseThreads];
  __shared__ double warp_part[kFuseThreads / 32];
  __shared__ double s_stat;
  __shared__ double tab[FROM_MEM ? 1 : kTabTraj][kRepTab];
  __shared__ int64_t s_k0, s_k1;
  const int64_t* bounds = a.bounds;
  if constexpr (SMEM_BOUNDS) {
    for (int64_t i = threadIdx.x; i <= a.n_traj; i += blockDim.x) sb[i] = a.bounds[i];
    __syncthreads();
    bounds = sb;
  }
  AREAL_K3_PROBE_TS(0)
  // thread t of leaf-CTA b owns the perfect subtree of 2^lpt_log2 leaves rooted at depth
  // `depth - lpt_log2`, index b * per + t
  const int per = (1 << (depth - lpt_log2)) / leaf_ctas;  // subtree roots per leaf-CTA (<= 256)
  const int lpt = 1 << lpt_log2;
  const bool leaf_cta = (int)blockIdx.x < leaf_ctas;
  const bool active = leaf_cta && (int)threadIdx.x < per;
  int64_t off = 0, len = 0;  // this thread's subtree
  if (active) pw_node(a.n_tokens, depth - lpt_log2, (int64_t)blockIdx.x * per + threadIdx.x, off, len);
  if constexpr (!FROM_MEM) {
    // trajectories this CTA's leaves touch: repeated-addition tables when there are few
    if (leaf_cta && threadIdx.x == 0) {
      SegCursor c{bounds, a.rewards, 0, 0, 0.0, 0, 0.0};
      c.seek(off, a.n_traj);
      s_k0 = c.k;
      int64_t lo, ln;
      pw_node(a.n_tokens, depth - lpt_log2, (int64_t)blockIdx.x * per + per - 1, lo, ln);
      c.seek(lo + ln - 1, a.n_traj);
      s_k1 = c.k;
    }
    __syncthreads();
  }
  AREAL_K3_PROBE_TS(1)
  double mean = 0.0, stdv = 0.0;
  for (int pass = 0; pass < 2; ++pass) {
    double* roots = a.ws + 8 + pass * 256;  // [leaf_ctas] per pass: no barrier between passes
    if (leaf_cta) {
      int64_t k0 = 0;
      bool use_tab = false;
      if constexpr (!FROM_MEM) {
        k0 = s_k0;
        const int64_t nk = s_k1 - s_k0 + 1;
        use_tab = nk <= kTabTraj;
        if (use_tab && (int)threadIdx.x < nk) {
          SegCursor c{bounds, a.rewards, k0 + threadIdx.x, 0, 0.0, pass, mean};
          const double x = c.value_of(c.k);
          double acc = x;
          tab[threadIdx.x][0] = x;
#pragma unroll
          for (int i = 1; i < kRepTab; ++i) {
            acc = __dadd_rn(acc, x);
            tab[threadIdx.x][i] = acc;
          }
        }
        __syncthreads();
      }
      AREAL_K3_PROBE_TS(2 + 4 * pass)
      double v = 0.0;
      if (active AREAL_K3_PROBE_LEAVES) {
        SegCursor c{bounds, a.rewards, 0, 0, 0.0, pass, mean};
        if constexpr (!FROM_MEM) c.seek(off, a.n_traj);
        AREAL_K3_PROBE_TS(11 + 2 * pass)
        // one <= 128-element numpy leaf
        auto leaf = [&](int64_t lo, int64_t n) -> double {
          if constexpr (FROM_MEM) {
            return pw_leaf_f(PwMem{a.adv, pass, mean}, lo, n);
          } else {
            c.at(lo);
            if (use_tab && lo + n <= c.next) {
              // inside one trajectory: numpy's leaf from the table.  n < 8: the sequential
              // sum of n terms; else 8 accumulators of (n - n%8)/8 terms each, combined
              // pairwise (S + S is exact: ((S+S)+(S+S))+(..) = 8 S), then the tail.
              const double* S = tab[c.k - k0];
              if (n < 8) return n > 0 ? S[n - 1] : 0.0;
              const int n8 = (int)(n - n % 8);
              double r = S[n8 / 8 - 1];
              r = __dadd_rn(r, r);
              r = __dadd_rn(r, r);
              r = __dadd_rn(r, r);
              for (int t = n8; t < (int)n; ++t) r = __dadd_rn(r, c.v);
              return r;
            }
            return seg_leaf_small(c, lo, n);
          }
        };
        // the subtree's 2^lpt_log2 cut-depth nodes left to right, folded like a binary
        // counter (pending left siblings per level in registers) = the perfect subtree
        double st[5];
        for (int j = 0; j < lpt; ++j) {
          int64_t lo = off, n = len;
          for (int l = lpt_log2 - 1; l >= 0; --l) {  // descend to cut-depth node j
            int64_t n2;
            node_split(n, n2);
            if ((j >> l) & 1) {
              lo += n2;
              n -= n2;
            } else {
              n = n2;
            }
          }
          double x;
          if (n <= 128) {
            x = leaf(lo, n);
          } else {  // one more numpy split (<= 143 -> two <= 128 leaves)
            int64_t n2;
            node_split(n, n2);
            const double left = leaf(lo, n2);
            x = __dadd_rn(left, leaf(lo + n2, n - n2));
          }
          bool carry = true;
#pragma unroll
          for (int l = 0; l < 5; ++l) {
            if (carry && l < lpt_log2) {
              if ((j >> l) & 1) {
                x = __dadd_rn(st[l], x);
              } else {
                st[l] = x;
                carry = false;
              }
            }
          }
          v = x;  // after the last node (all low bits set) this is the subtree root
        }
      }
      if (active) buf[threadIdx.x] = v;
      AREAL_K3_PROBE_TS(3 + 4 * pass)
      const double root = fold_pow2(buf, per, warp_part);
      if (threadIdx.x == 0) roots[blockIdx.x] = root;
    }
    AREAL_K3_PROBE_TS(4 + 4 * pass)
    grid.sync();
    AREAL_K3_PROBE_TS(5 + 4 * pass)
    if ((int)threadIdx.x < leaf_ctas) buf[threadIdx.x] = __ldcg(roots + threadIdx.x);
    const double tot = fold_pow2(buf, leaf_ctas, warp_part);
    if (threadIdx.x == 0) s_stat = tot;
    __syncthreads();
    if (pass == 0) mean = s_stat / (double)a.n_tokens;  // np.mean: umr_sum / n
    else stdv = sqrt(s_stat / (double)a.n_tokens);      // np.std: sqrt(sum(d*d) / n)
  }
  AREAL_K3_PROBE_TS(10)
  if (blockIdx.x == 0 && threadIdx.x == 0 && a.norm_stats) {
    a.norm_stats[0] = mean;
    a.norm_stats[1] = stdv;
  }
  AREAL_K3_PROBE_WRITE
  // (raw - mean) / std per token (trainer.py:120-123): warp-contiguous spans, each lane
  // storing 2 consecutive tokens per step (16-byte stores when the span start is even)
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int64_t span = ((a.n_tokens + nw - 1) / nw + 63) & ~(int64_t)63;
  const int64_t t0 = w * span, t1 = t0 + span < a.n_tokens ? t0 + span : a.n_tokens;
  if (t0 >= t1) return;
  auto norm = [&](double v) { return (stdv == 0.0) ? 0.0 : __ddiv_rn(__dsub_rn(v, mean), stdv); };
  if constexpr (FROM_MEM) {
    for (int64_t t = t0 + lane; t < t1; t += 32) a.adv[t] = norm(a.adv[t]);
  } else {
    SegCursor c{bounds, a.rewards, 0, 0, 0.0, 0, 0.0};
    c.seek(t0 + 2 * lane < t1 ? t0 + 2 * lane : t0, a.n_traj);
    double an = norm(c.v);  // normalised value of the cursor's trajectory
    int64_t k_an = c.k;
    for (int64_t t = t0 + 2 * lane; t < t1; t += 64) {
      const double r0 = c.at(t);
      if (c.k != k_an) { an = norm(r0); k_an = c.k; }
      const double a0 = an;
      double a1 = a0, r1 = r0;
      if (t + 1 < t1) {
        r1 = c.at(t + 1);
        if (c.k != k_an) { an = norm(r1); k_an = c.k; }
        a1 = an;
      }
      if (t + 1 < t1) {
        *reinterpret_cast<double2*>(a.adv + t) = make_double2(a0, a1);
        if (a.returns) *reinterpret_cast<double2*>(a.returns + t) = make_double2(r0, r1);
      } else {
        a.adv[t] = a0;
        if (a.returns) a.returns[t] = r0;
      }
    }
  }
}

// ---------------------------------------------------------------- GRPO group norm
// One warp per group.  token weighting: mean / population std over the group's
// tokens; sequence weighting: over its trajectories (raw at the first token).
__global__ void group_norm_kernel(AdvArgs a, int sequence) {
  const int lane = threadIdx.x & 31;
  const int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (g >= a.n_groups) return;
  double s = 0.0, cnt = 0.0;
  for (int64_t k = 0; k < a.n_traj; ++k) {
    if (a.group_ids[k] != g) continue;
    const int64_t b = a.bounds[k], e = a.bounds[k + 1];
    if (sequence) {
      if (e > b && lane == 0) {
        s += a.adv[b];
        cnt += 1.0;
      }
    } else {
      for (int64_t t = b + lane; t < e; t += 32) s += a.adv[t];
      if (lane == 0) cnt += (double)(e - b);
    }
  }
  s = warp_sum(s);
  cnt = __shfl_sync(0xffffffffu, cnt, 0);
  if (cnt == 0.0) return;
  const double mean = s / cnt;
  double q = 0.0;
  for (int64_t k = 0; k < a.n_traj; ++k) {
    if (a.group_ids[k] != g) continue;
    const int64_t b = a.bounds[k], e = a.bounds[k + 1];
    if (sequence) {
      if (e > b && lane == 0) {
        const double d = a.adv[b] - mean;
        q += d * d;
      }
    } else {
      for (int64_t t = b + lane; t < e; t += 32) {
        const double d = a.adv[t] - mean;
        q += d * d;
      }
    }
  }
  q = warp_sum(q);
  const double denom = sqrt(q / cnt) + a.eps;
  __syncwarp();
  for (int64_t k = 0; k < a.n_traj; ++k) {
    if (a.group_ids[k] != g) continue;
    const int64_t b = a.bounds[k], e = a.bounds[k + 1];
    for (int64_t t = b + lane; t < e; t += 32)
      a.adv[t] = (denom == 0.0) ? 0.0 : (a.adv[t] - mean) / denom;
  }
}

}  // namespace areal

using namespace areal;

extern "C" int areal_advantages(const double* rewards, const int64_t* traj_bounds, int64_t n_traj,
                                int64_t n_tokens, const double* values, const int32_t* group_ids,
                                int32_t n_groups, const areal_adv_params_t* params,
                                double* adv_out, double* returns_out, double* norm_stats_out,
                                void* workspace, size_t workspace_bytes, void* stream_) {
  if (!params || n_traj < 0 || n_tokens < 0) return AREAL_ERR_INVALID_ARGUMENT;
  if (params->mode != AREAL_ADV_REFERENCE && params->mode != AREAL_ADV_GAE)
    return AREAL_ERR_INVALID_ARGUMENT;
  if (params->norm < AREAL_NORM_NONE || params->norm > AREAL_NORM_GROUP_SEQUENCE)
    return AREAL_ERR_INVALID_ARGUMENT;
  const bool group = params->norm == AREAL_NORM_GROUP_TOKEN || params->norm == AREAL_NORM_GROUP_SEQUENCE;
  if (group && (!group_ids || n_groups < 0)) return AREAL_ERR_INVALID_ARGUMENT;
  if (n_traj == 0 || n_tokens == 0) return AREAL_OK;
  if (!rewards || !traj_bounds || !adv_out) return AREAL_ERR_INVALID_ARGUMENT;
  if (!workspace || workspace_bytes < AREAL_WORKSPACE_BYTES) return AREAL_ERR_WORKSPACE;
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  AdvArgs a = {};
  a.rewards = rewards;
  a.bounds = traj_bounds;
  a.n_traj = n_traj;
  a.n_tokens = n_tokens;
  a.values = values;
  a.group_ids = group_ids;
  a.n_groups = n_groups;
  a.gamma = params->gamma;
  a.lam = params->lam;
  a.eps = params->eps;
  a.mode = params->mode;
  a.norm = params->norm;
  a.adv = adv_out;
  a.returns = returns_out;
  a.norm_stats = norm_stats_out;
  // K3 owns the upper half of the workspace; the lower half holds K2's ticket
  // counter and partials, which must stay zero-initialised between launches.
  a.ws = reinterpret_cast<double*>(static_cast<char*>(workspace) + AREAL_WORKSPACE_BYTES / 2);

  const bool fused_global = params->norm == AREAL_NORM_GLOBAL;
  if (!fused_global || params->mode != AREAL_ADV_REFERENCE) {
    const int64_t warps = n_traj;
    const int64_t blocks = std::min<int64_t>((warps * 32 + 255) / 256, 148 * 16);
    adv_raw_kernel<<<(unsigned)blocks, 256, 0, stream>>>(a);
    AREAL_CUDA_CHECK_LAUNCH();
  }
  if (fused_global) {
    const int depth = pw_depth(n_tokens);
    if (depth == kMaxTreeDepth && n_tokens > ((int64_t)128 << kMaxTreeDepth)) return AREAL_ERR_UNSUPPORTED;
    // one thread per subtree of 2^lpt_log2 cut-depth nodes, at most 128 x 256 threads
    const int lpt_log2 = depth > kLeafThreadsLog2 ? depth - kLeafThreadsLog2 : 0;
    const int threads = 1 << (depth - lpt_log2);
    int leaf_ctas = threads > kFuseThreads ? threads / kFuseThreads : 1;
    int depth_arg = depth, lpt_arg = lpt_log2;
    void* args[] = {&a, &depth_arg, &leaf_ctas, &lpt_arg};
    const bool mem = params->mode != AREAL_ADV_REFERENCE, smem = n_traj <= kFuseBoundsSmem;
    const void* kern = mem ? (const void*)adv_global_fused_kernel<true, false>
                           : (smem ? (const void*)adv_global_fused_kernel<false, true>
                                   : (const void*)adv_global_fused_kernel<false, false>);
    int dev = 0, sms = 148, occ = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kFuseThreads, 0);
    const int grid = std::max(leaf_ctas, std::min(2, occ) * sms);  // write phase: 2 CTAs per SM
    if (cudaLaunchCooperativeKernel(kern, dim3(grid), dim3(kFuseThreads), args, 0, stream) != cudaSuccess)
      return AREAL_ERR_CUDA;
    AREAL_CUDA_CHECK_LAUNCH();
  } else if (group && n_groups > 0) {
    const int64_t blocks = ((int64_t)n_groups * 32 + 255) / 256;
    group_norm_kernel<<<(unsigned)blocks, 256, 0, stream>>>(a, params->norm == AREAL_NORM_GROUP_SEQUENCE);
    AREAL_CUDA_CHECK_LAUNCH();
  }
  return AREAL_OK;
}
