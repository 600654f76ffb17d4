// adam.cu — K6: fused global-norm clip + Adam with decoupled weight decay, multi-tensor.
//
// Reference: apply_update (/root/reference/pkg/src/asyncrl/policy.py:225-258) after
// grad.scale_(-1/n) (trainer.py:329-330):
//   g      = grad * grad_scale                        (ParamGrad.scale_, policy.py:122-124)
//   norm   = sqrt(sum(g_w**2) + sum(g_b**2))           (global_norm, policy.py:129-130)
//   non-finite g -> NonFiniteGradientError, nothing updated (policy.py:234-239)
//   g      = g * (clip / norm) if clip > 0 and norm > clip   (clip_by_global_norm, 215-221)
//   m      = b1*m + (1-b1)*g ;  v = b2*v + (1-b2)*g**2
//   p      = p - lr*((m/c1)/(sqrt(v/c2) + eps) + wd*p),  c_i = 1 - b_i**step
// Every elementwise operation is one IEEE-rounded op (no FMA contraction, __d*_rn)
// in numpy's order, and the float64 norm replays numpy's pairwise summation tree per
// tensor (EXACT mode), so given the same gradient the update is bit-identical to the
// reference.  The host computes the scalars the reference computes in Python
// (1-b1, 1-b2, c1, c2, grad_scale = -1/n) and passes them in.
//
// Three launches, no host synchronisation: sum-of-squares partials (+ non-finite
// count) -> one CTA folds them in a fixed order into (norm, clip factor) -> the
// update kernel reads them and streams p, g, m, v once (skipping everything when a
// non-finite gradient was seen, so the caller can raise with the state untouched).
// FAST mode (fp32 / bf16 / fp16 gradients, LM-scale models) sums squares in fp64 per
// CTA and reduces the partials in CTA order: deterministic, not numpy-exact.
#include <algorithm>

#include "common.cuh"
#include "pairwise.cuh"

namespace areal {

constexpr int kAdamMaxTensors = AREAL_ADAM_MAX_TENSORS;
constexpr int kAdamThreads = 256;
constexpr int kAdamLeafCap = 57344;       // exact-mode subtree roots in the workspace
constexpr int kAdamFastCtas = 148 * 4;    // fast-mode partials

struct AdamArgs {
  void* p[kAdamMaxTensors];
  const void* g[kAdamMaxTensors];
  void* m[kAdamMaxTensors];
  void* v[kAdamMaxTensors];
  int64_t n[kAdamMaxTensors];
  int64_t start[kAdamMaxTensors + 1];   // flattened element offsets
  int32_t depth[kAdamMaxTensors];       // exact mode: pairwise cut depth per tensor
  int32_t leaf_start[kAdamMaxTensors + 1];
  int32_t n_tensors;
  double lr, b1, b2, omb1, omb2, eps, wd, c1, c2, clip, gscale;
  const double* gdiv;  // optional device divisor of gscale (K2's n_valid)
  double* ws;        // [0] norm, [1] factor, [2] non-finite count (as u64), [16..] partials
  double* norm_out;  // optional device [2]: norm, non-finite count
};

template <typename T> __device__ __forceinline__ double ld_as_f64(const void* base, int64_t i) {
  return (double)Traits<T>::to_acc(static_cast<const T*>(base)[i]);
}
template <> __device__ __forceinline__ double ld_as_f64<double>(const void* base, int64_t i) {
  return static_cast<const double*>(base)[i];
}
template <typename T> __device__ __forceinline__ void st_from_f64(void* base, int64_t i, double x) {
  static_cast<T*>(base)[i] = (T)x;
}
template <> __device__ __forceinline__ void st_from_f64<__nv_bfloat16>(void* base, int64_t i, double x) {
  static_cast<__nv_bfloat16*>(base)[i] = __double2bfloat16(x);
}
template <> __device__ __forceinline__ void st_from_f64<__half>(void* base, int64_t i, double x) {
  static_cast<__half*>(base)[i] = __double2half(x);
}

// grad_scale, or grad_scale / max(n, 1) with n read on the device (the same IEEE
// division Python's -1.0 / n performs at trainer.py:330)
__device__ __forceinline__ double eff_scale(const AdamArgs& a) {
  return a.gdiv ? __ddiv_rn(a.gscale, fmax(*a.gdiv, 1.0)) : a.gscale;
}

__device__ __forceinline__ int tensor_of(const AdamArgs& a, int64_t e) {
  int k = 0;
  while (k + 1 < a.n_tensors && a.start[k + 1] <= e) ++k;
  return k;
}

__device__ __forceinline__ unsigned long long* nonfinite_counter(const AdamArgs& a) {
  return reinterpret_cast<unsigned long long*>(a.ws + 2);
}

// (grad * scale)^2 with numpy's roundings; counts non-finite scaled gradients.
template <typename G> struct ScaledSq {
  const void* g;
  double s;
  unsigned* bad;
  __device__ double operator()(int64_t i) const {
    const double x = __dmul_rn(ld_as_f64<G>(g, i), s);
    if (!isfinite(x)) ++*bad;
    return __dmul_rn(x, x);
  }
};

// EXACT: one thread per pairwise subtree root of every tensor.
template <typename G>
__global__ void __launch_bounds__(kAdamThreads) adam_sumsq_exact_kernel(const __grid_constant__ AdamArgs a) {
  const int leaf = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned bad = 0;
  if (leaf < a.leaf_start[a.n_tensors]) {
    int k = 0;
    while (k + 1 < a.n_tensors && a.leaf_start[k + 1] <= leaf) ++k;
    int64_t off, len;
    pw_node(a.n[k], a.depth[k], leaf - a.leaf_start[k], off, len);
    a.ws[16 + leaf] = pw_sum_f(ScaledSq<G>{a.g[k], eff_scale(a), &bad}, off, len);
  }
  bad = __reduce_add_sync(0xffffffffu, bad);
  if ((threadIdx.x & 31) == 0 && bad) atomicAdd(nonfinite_counter(a), (unsigned long long)bad);
}

// FAST: grid-stride fp64 sum of squares per CTA.
template <typename G>
__global__ void __launch_bounds__(kAdamThreads) adam_sumsq_fast_kernel(const __grid_constant__ AdamArgs a) {
  __shared__ double red[kAdamThreads / 32];
  double acc = 0.0;
  unsigned bad = 0;
  const int64_t total = a.start[a.n_tensors];
  const double gscale = eff_scale(a);
  int k = 0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    while (a.start[k + 1] <= e) ++k;
    const double x = ld_as_f64<G>(a.g[k], e - a.start[k]) * gscale;
    if (!isfinite(x)) ++bad;
    acc = fma(x, x, acc);
  }
  acc = warp_sum(acc);
  bad = __reduce_add_sync(0xffffffffu, bad);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    red[w] = acc;
    if (bad) atomicAdd(nonfinite_counter(a), (unsigned long long)bad);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < kAdamThreads / 32; ++i) s += red[i];
    a.ws[16 + blockIdx.x] = s;
  }
}

// One CTA: fold partials in a fixed order -> norm and clip factor.
__global__ void __launch_bounds__(1024) adam_norm_kernel(const __grid_constant__ AdamArgs a, int exact,
                                                         int n_partials) {
  __shared__ double buf[4096];
  double total = 0.0;
  if (exact) {
    // per tensor: combine its 2^depth roots in tree order; tensors are added left to
    // right (np.sum(w**2) + np.sum(b**2), policy.py:130)
    for (int k = 0; k < a.n_tensors; ++k) {
      const int nodes = 1 << a.depth[k];
      for (int i = threadIdx.x; i < nodes; i += blockDim.x) buf[i] = a.ws[16 + a.leaf_start[k] + i];
      __syncthreads();
      for (int m = nodes; m > 1; m >>= 1) {
        const int h = m >> 1;
        double v0 = 0.0, v1 = 0.0;
        const int i0 = threadIdx.x, i1 = threadIdx.x + blockDim.x;
        if (i0 < h) v0 = __dadd_rn(buf[2 * i0], buf[2 * i0 + 1]);
        if (i1 < h) v1 = __dadd_rn(buf[2 * i1], buf[2 * i1 + 1]);
        __syncthreads();
        if (i0 < h) buf[i0] = v0;
        if (i1 < h) buf[i1] = v1;
        __syncthreads();
      }
      if (threadIdx.x == 0) total = (k == 0) ? buf[0] : __dadd_rn(total, buf[0]);
      __syncthreads();
    }
  } else if (threadIdx.x == 0) {
    for (int i = 0; i < n_partials; ++i) total += a.ws[16 + i];
  }
  if (threadIdx.x == 0) {
    const double norm = __dsqrt_rn(total);
    const unsigned long long bad = *nonfinite_counter(a);
    // clip_by_global_norm (policy.py:215-221): factor = clip / norm when clipping
    const double factor = (a.clip > 0.0 && norm > a.clip) ? __ddiv_rn(a.clip, norm) : 1.0;
    a.ws[0] = norm;
    a.ws[1] = factor;
    if (a.norm_out) {
      a.norm_out[0] = norm;
      a.norm_out[1] = (double)bad;
    }
  }
}

template <typename P, typename G>
__global__ void __launch_bounds__(kAdamThreads) adam_update_kernel(const __grid_constant__ AdamArgs a) {
  if (*nonfinite_counter(a) != 0ull) return;  // reference raises before touching state
  const double factor = a.ws[1];
  const bool clip = factor != 1.0;
  const double gscale = eff_scale(a);
  const int64_t total = a.start[a.n_tensors];
  int k = 0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    while (a.start[k + 1] <= e) ++k;
    const int64_t i = e - a.start[k];
    double g = __dmul_rn(ld_as_f64<G>(a.g[k], i), gscale);
    if (clip) g = __dmul_rn(g, factor);
    double m = ld_as_f64<P>(a.m[k], i), v = ld_as_f64<P>(a.v[k], i), p = ld_as_f64<P>(a.p[k], i);
    m = __dadd_rn(__dmul_rn(a.b1, m), __dmul_rn(a.omb1, g));
    v = __dadd_rn(__dmul_rn(a.b2, v), __dmul_rn(a.omb2, __dmul_rn(g, g)));
    const double mhat = __ddiv_rn(m, a.c1);
    const double den = __dadd_rn(__dsqrt_rn(__ddiv_rn(v, a.c2)), a.eps);
    const double upd = __dadd_rn(__ddiv_rn(mhat, den), __dmul_rn(a.wd, p));
    p = __dsub_rn(p, __dmul_rn(a.lr, upd));
    st_from_f64<P>(a.m[k], i, m);
    st_from_f64<P>(a.v[k], i, v);
    st_from_f64<P>(a.p[k], i, p);
  }
}

template <typename P, typename G>
int adam_launch(AdamArgs& a, int exact, cudaStream_t stream) {
  const int64_t total = a.start[a.n_tensors];
  cudaMemsetAsync(a.ws + 2, 0, sizeof(double), stream);
  int n_partials = 0;
  if (exact) {
    const int leaves = a.leaf_start[a.n_tensors];
    adam_sumsq_exact_kernel<G><<<(leaves + kAdamThreads - 1) / kAdamThreads, kAdamThreads, 0, stream>>>(a);
  } else {
    n_partials = (int)std::min<int64_t>(kAdamFastCtas, std::max<int64_t>(1, (total + kAdamThreads - 1) / kAdamThreads));
    adam_sumsq_fast_kernel<G><<<n_partials, kAdamThreads, 0, stream>>>(a);
  }
  AREAL_CUDA_CHECK_LAUNCH();
  adam_norm_kernel<<<1, 1024, 0, stream>>>(a, exact, n_partials);
  AREAL_CUDA_CHECK_LAUNCH();
  const int64_t blocks = std::min<int64_t>(148 * 8, std::max<int64_t>(1, (total + kAdamThreads - 1) / kAdamThreads));
  adam_update_kernel<P, G><<<(unsigned)blocks, kAdamThreads, 0, stream>>>(a);
  AREAL_CUDA_CHECK_LAUNCH();
  return AREAL_OK;
}

}  // namespace areal

using namespace areal;

extern "C" int areal_adam_step(const areal_adam_tensor_t* tensors, int32_t n_tensors, int param_dtype,
                               int grad_dtype, const areal_adam_params_t* params, double* norm_out,
                               void* workspace, size_t workspace_bytes, void* stream_) {
  if (!tensors || !params || n_tensors < 0 || n_tensors > kAdamMaxTensors) return AREAL_ERR_INVALID_ARGUMENT;
  if (!workspace || workspace_bytes < AREAL_WORKSPACE_BYTES) return AREAL_ERR_WORKSPACE;
  const bool exact = params->exact_norm != 0;
  if (param_dtype != AREAL_F64 && param_dtype != AREAL_F32) return AREAL_ERR_BAD_DTYPE;
  if (exact && (param_dtype != AREAL_F64 || grad_dtype != AREAL_F64)) return AREAL_ERR_UNSUPPORTED;
  if (param_dtype == AREAL_F64 && grad_dtype != AREAL_F64) return AREAL_ERR_BAD_DTYPE;
  if (param_dtype == AREAL_F32 && grad_dtype != AREAL_F32 && grad_dtype != AREAL_BF16 &&
      grad_dtype != AREAL_F16)
    return AREAL_ERR_BAD_DTYPE;
  if (params->bias_correction1 == 0.0 || params->bias_correction2 == 0.0) return AREAL_ERR_INVALID_ARGUMENT;
  AdamArgs a = {};
  a.n_tensors = n_tensors;
  a.start[0] = 0;
  for (int k = 0; k < n_tensors; ++k) {
    const areal_adam_tensor_t& t = tensors[k];
    if (t.numel < 0) return AREAL_ERR_BAD_SHAPE;
    if (t.numel > 0 && (!t.param || !t.grad || !t.exp_avg || !t.exp_avg_sq)) return AREAL_ERR_INVALID_ARGUMENT;
    a.p[k] = t.param;
    a.g[k] = t.grad;
    a.m[k] = t.exp_avg;
    a.v[k] = t.exp_avg_sq;
    a.n[k] = t.numel;
    a.start[k + 1] = a.start[k] + t.numel;
  }
  // exact mode: cut the pairwise tree of each tensor so that all roots fit the workspace
  int cap = 12;
  while (cap > 0 && ((int64_t)n_tensors << cap) > kAdamLeafCap) --cap;
  a.leaf_start[0] = 0;
  for (int k = 0; k < n_tensors; ++k) {
    a.depth[k] = pw_depth(a.n[k], cap);
    a.leaf_start[k + 1] = a.leaf_start[k] + (1 << a.depth[k]);
  }
  a.lr = params->lr;
  a.b1 = params->beta1;
  a.b2 = params->beta2;
  a.omb1 = params->one_minus_beta1;
  a.omb2 = params->one_minus_beta2;
  a.eps = params->eps;
  a.wd = params->weight_decay;
  a.c1 = params->bias_correction1;
  a.c2 = params->bias_correction2;
  a.clip = params->clip_norm;
  a.gscale = params->grad_scale;
  a.gdiv = params->grad_scale_divisor;
  // K6 shares the upper half of the workspace with K3 (stream-ordered); the lower
  // half holds K2's zeroed ticket counter and partials.
  a.ws = reinterpret_cast<double*>(static_cast<char*>(workspace) + AREAL_WORKSPACE_BYTES / 2);
  a.norm_out = norm_out;
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  if (param_dtype == AREAL_F64) return adam_launch<double, double>(a, exact, stream);
  switch (grad_dtype) {
    case AREAL_F32: return adam_launch<float, float>(a, exact, stream);
    case AREAL_BF16: return adam_launch<float, __nv_bfloat16>(a, exact, stream);
    default: return adam_launch<float, __half>(a, exact, stream);
  }
}
