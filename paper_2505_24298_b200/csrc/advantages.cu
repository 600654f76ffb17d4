// advantages.cu — K3: per-token advantages for sm_100a.
//
// Reference: compute_advantages (/root/reference/pkg/src/asyncrl/trainer.py:114-125):
//   raw_t = reward of the trajectory owning t;  std = np.std(raw);
//   std == 0 -> zeros, else (raw - np.mean(raw)) / std.
// The GLOBAL normalisation replays numpy's float64 pairwise summation tree
// (8-way unrolled leaves of <= 128 elements, split at n/2 rounded down to a
// multiple of 8) so mean/std — and therefore every advantage — are bit-identical
// to the reference.  Leaves of the tree are summed by many threads in parallel;
// the top 2^D levels are combined by one CTA in tree order.
//
// Extensions (north star): GAE reverse scan per sequence (one warp per
// trajectory, segmented affine warp scan) and GRPO group normalisation.
#include "common.cuh"
#include "pairwise.cuh"

namespace areal {

constexpr int kMaxTreeDepth = 15;  // <= 32768 subtree roots (256 KB of the K3 workspace half)

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
  double* ws;          // workspace: [0..1] mean/std scratch, [8..] subtree sums
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

// ---------------------------------------------------------------- numpy pairwise sum
// Value fed to the sum: x_t (pass 0) or (x_t - mean)^2 (pass 1), with IEEE
// rounding per operation (no contraction) exactly like numpy's ufunc loops.
__device__ __forceinline__ double pw_val(const double* x, int64_t i, int pass, double mean) {
  const double v = x[i];
  if (pass == 0) return v;
  const double d = __dsub_rn(v, mean);
  return __dmul_rn(d, d);
}

struct PwVal {
  const double* x;
  int pass;
  double mean;
  __device__ double operator()(int64_t i) const { return pw_val(x, i, pass, mean); }
};

__host__ __device__ inline int pw_depth(int64_t n) { return pw_depth(n, kMaxTreeDepth); }

__global__ void pw_leaves_kernel(const double* x, int64_t n, int depth, int pass,
                                 const double* mean_ptr, double* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ((int64_t)1 << depth)) return;
  int64_t off, len;
  pw_node(n, depth, i, off, len);
  const double mean = pass ? *mean_ptr : 0.0;
  out[i] = pw_sum_f(PwVal{x, pass, mean}, off, len);
}

// Combine the 2^depth subtree sums in tree order; pass 0 -> mean, pass 1 -> std.
__global__ void pw_top_kernel(const double* sums, int64_t n, int depth, int pass, double* scratch,
                              double* norm_stats) {
  __shared__ double buf[4096];
  // levels above 4096 nodes are folded in registers first
  const int nodes = 1 << depth;
  const int tid = threadIdx.x;
  if (nodes > 4096) {
    const int per = nodes / 4096;  // power of two
    for (int i = tid; i < 4096; i += blockDim.x) {
      // combine `per` consecutive leaves as a perfect binary tree
      double v[8];
      // per <= 8 since depth <= 15
      for (int j = 0; j < per; ++j) v[j] = sums[i * per + j];
      for (int w = per; w > 1; w >>= 1)  // levels of the perfect binary tree, bottom up
        for (int j = 0; j < w / 2; ++j) v[j] = __dadd_rn(v[2 * j], v[2 * j + 1]);
      buf[i] = v[0];
    }
  } else {
    for (int i = tid; i < nodes; i += blockDim.x) buf[i] = sums[i];
  }
  __syncthreads();
  int m = nodes > 4096 ? 4096 : nodes;
  while (m > 1) {  // blockDim.x == 1024 and m <= 4096: at most two parents per thread
    const int h = m >> 1;
    const int i0 = tid, i1 = tid + blockDim.x;
    double v0 = 0.0, v1 = 0.0;
    if (i0 < h) v0 = __dadd_rn(buf[2 * i0], buf[2 * i0 + 1]);
    if (i1 < h) v1 = __dadd_rn(buf[2 * i1], buf[2 * i1 + 1]);
    __syncthreads();
    if (i0 < h) buf[i0] = v0;
    if (i1 < h) buf[i1] = v1;
    __syncthreads();
    m = h;
  }
  if (tid == 0) {
    const double tot = buf[0];
    if (pass == 0) {
      scratch[0] = n > 0 ? tot / (double)n : 0.0;  // np.mean: umr_sum / n
      if (norm_stats) norm_stats[0] = scratch[0];
    } else {
      scratch[1] = n > 0 ? sqrt(tot / (double)n) : 0.0;  // np.std: sqrt(sum(d*d)/n)
      if (norm_stats) norm_stats[1] = scratch[1];
    }
  }
}

__global__ void norm_apply_kernel(double* adv, int64_t n, const double* scratch) {
  const double mean = scratch[0], std = scratch[1];
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    adv[t] = (std == 0.0) ? 0.0 : __ddiv_rn(__dsub_rn(adv[t], mean), std);  // trainer.py:120-123
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

  {
    const int64_t warps = n_traj;
    const int64_t blocks = std::min<int64_t>((warps * 32 + 255) / 256, 148 * 16);
    adv_raw_kernel<<<(unsigned)blocks, 256, 0, stream>>>(a);
    AREAL_CUDA_CHECK_LAUNCH();
  }
  if (params->norm == AREAL_NORM_GLOBAL) {
    const int depth = pw_depth(n_tokens);
    const int64_t nodes = (int64_t)1 << depth;
    double* scratch = a.ws;   // [0] mean, [1] std
    double* sums = a.ws + 8;  // [nodes]
    const unsigned blocks = (unsigned)((nodes + 127) / 128);
    for (int pass = 0; pass < 2; ++pass) {
      pw_leaves_kernel<<<blocks, 128, 0, stream>>>(adv_out, n_tokens, depth, pass, scratch, sums);
      AREAL_CUDA_CHECK_LAUNCH();
      pw_top_kernel<<<1, 1024, 0, stream>>>(sums, n_tokens, depth, pass, scratch, norm_stats_out);
      AREAL_CUDA_CHECK_LAUNCH();
    }
    const int64_t nb = std::min<int64_t>((n_tokens + 255) / 256, 148 * 8);
    norm_apply_kernel<<<(unsigned)nb, 256, 0, stream>>>(adv_out, n_tokens, scratch);
    AREAL_CUDA_CHECK_LAUNCH();
  } else if (group && n_groups > 0) {
    const int64_t blocks = ((int64_t)n_groups * 32 + 255) / 256;
    group_norm_kernel<<<(unsigned)blocks, 256, 0, stream>>>(a, params->norm == AREAL_NORM_GROUP_SEQUENCE);
    AREAL_CUDA_CHECK_LAUNCH();
  }
  return AREAL_OK;
}
