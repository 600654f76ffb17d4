// common.cuh — dtype traits and sm_100a PTX helpers shared by the hot-path kernels.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>
#include <type_traits>

#include "../../include/areal_b200.h"

#define AREAL_CUDA_CHECK_LAUNCH()                    \
  do {                                               \
    cudaError_t _e = cudaGetLastError();             \
    if (_e != cudaSuccess) return AREAL_ERR_CUDA;    \
  } while (0)

namespace areal {

constexpr int kWarp = 32;

// ------------------------------------------------------------------ dtype traits
// Acc is the accumulation type of the row reductions: fp32 for 16/32-bit
// logits, fp64 for fp64 logits (the drop-in parity path).
template <typename T> struct Traits;
template <> struct Traits<float> {
  using Acc = float;
  static __device__ __forceinline__ float to_acc(float v) { return v; }
  static __device__ __forceinline__ float from_acc(float v) { return v; }
};
template <> struct Traits<double> {
  using Acc = double;
  static __device__ __forceinline__ double to_acc(double v) { return v; }
  static __device__ __forceinline__ double from_acc(double v) { return v; }
};
template <> struct Traits<__nv_bfloat16> {
  using Acc = float;
  static __device__ __forceinline__ float to_acc(__nv_bfloat16 v) { return __bfloat162float(v); }
  static __device__ __forceinline__ __nv_bfloat16 from_acc(float v) { return __float2bfloat16_rn(v); }
};
template <> struct Traits<__half> {
  using Acc = float;
  static __device__ __forceinline__ float to_acc(__half v) { return __half2float(v); }
  static __device__ __forceinline__ __half from_acc(float v) { return __float2half_rn(v); }
};

// exp2 in the accumulation type.  fp32 uses the MUFU ex2 (ex2.approx.ftz,
// ~2 ulp); fp64 uses the libdevice exp2 (the reference's float64 accuracy).
__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ double fast_exp2(double x) { return exp2(x); }
__device__ __forceinline__ float acc_log(float x) { return logf(x); }
__device__ __forceinline__ double acc_log(double x) { return log(x); }

template <typename A> struct Lim;
template <> struct Lim<float> {
  static __device__ __forceinline__ float lowest() { return -3.402823466e38f; }
  static __device__ __forceinline__ float ninf() { return -__int_as_float(0x7f800000); }
  static constexpr float kLog2e = 1.4426950408889634f;
};
template <> struct Lim<double> {
  static __device__ __forceinline__ double lowest() { return -1.7976931348623157e308; }
  static __device__ __forceinline__ double ninf() { return -__longlong_as_double(0x7ff0000000000000ll); }
  static constexpr double kLog2e = 1.4426950408889634074;
};

// ------------------------------------------------------------------ warp reductions
template <typename A> __device__ __forceinline__ A warp_max(A v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
template <typename A> __device__ __forceinline__ A warp_sum(A v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Online (max, sum e^(x-max), sum e^(x-max)*x) triple, the row statistics of
// log-softmax and entropy.  merge() is associative up to rounding; callers
// merge in a fixed order so results are deterministic.
template <typename A> struct RowStat {
  A m, s, sx;
  __device__ __forceinline__ void init() { m = Lim<A>::ninf(); s = A(0); sx = A(0); }
  __device__ __forceinline__ void merge(A m2, A s2, A sx2) {
    A mn = fmax(m, m2);
    if (mn == Lim<A>::ninf()) return;  // both empty / all -inf
    A a, b;
    if constexpr (std::is_same<A, float>::value) {
      // fp32 partials are sums of 2^(x log2e - fl(m log2e)): move them to the new
      // shift by the exact 2^(fl(m log2e) - fl(mn log2e)) (no FMA contraction)
      const float cn = __fmul_rn(mn, Lim<A>::kLog2e);
      a = fast_exp2(__fmul_rn(m, Lim<A>::kLog2e) - cn);
      b = fast_exp2(__fmul_rn(m2, Lim<A>::kLog2e) - cn);
    } else {
      a = fast_exp2((m - mn) * Lim<A>::kLog2e);
      b = fast_exp2((m2 - mn) * Lim<A>::kLog2e);
    }
    s = s * a + s2 * b;
    sx = sx * a + sx2 * b;
    m = mn;
  }
  __device__ __forceinline__ void warp_reduce() {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      A m2 = __shfl_xor_sync(0xffffffffu, m, o);
      A s2 = __shfl_xor_sync(0xffffffffu, s, o);
      A x2 = __shfl_xor_sync(0xffffffffu, sx, o);
      merge(m2, s2, x2);
    }
  }
};

// ------------------------------------------------------------------ PTX: mbarrier / bulk copy / cluster
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init_cluster() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// mbarrier waits.  try_wait carries a suspend-time hint (AREAL_WAIT_HINT_NS, as
// CUTLASS's ClusterBarrier::wait does) so a waiting warp sleeps in hardware until
// the phase completes instead of re-polling and stealing issue slots from the
// warps doing work.  Watchdog: a wait that lasts longer than kWaitLimitNs of
// %globaltimer is a protocol bug (deadlock): trap so the launch fails loudly
// instead of hanging the GPU.
#ifndef AREAL_WAIT_HINT_NS
#define AREAL_WAIT_HINT_NS 10000000
#endif
constexpr uint64_t kWaitLimitNs = 20ull * 1000000000ull;

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
#if AREAL_WAIT_HINT_NS > 0
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity), "r"((uint32_t)AREAL_WAIT_HINT_NS)
      : "memory");
#else
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
#endif
  return ok != 0;
}
// Slow-path back-off between polls (ns; 0 = none).  A failed try_wait wakes on every
// transaction update of the barrier (a 32 KB bulk copy lands in pieces), so a
// waiting warp would otherwise re-poll tens of times per chunk.
#ifndef AREAL_WAIT_BACKOFF_NS
#define AREAL_WAIT_BACKOFF_NS 0
#endif
// The watchdog reads %globaltimer once per kWatchdogPolls failed polls: a failed
// try_wait wakes on every partial transaction of a bulk copy, and reading the timer on
// each of them cost ~8% of K2's issued instructions (ncu r02aq).
#ifndef AREAL_WATCHDOG_POLLS
#define AREAL_WATCHDOG_POLLS 256
#endif
constexpr uint32_t kWatchdogPolls = AREAL_WATCHDOG_POLLS;
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  if (mbar_try_wait(bar, parity)) return;
  uint64_t t0 = 0;
  uint32_t polls = 0;
  while (!mbar_try_wait(bar, parity)) {
    if (AREAL_WAIT_BACKOFF_NS > 0) __nanosleep(AREAL_WAIT_BACKOFF_NS);
    if (++polls % kWatchdogPolls == 0) {
      const uint64_t t = globaltimer_ns();
      if (t0 == 0) t0 = t;
      else if (t - t0 > kWaitLimitNs) __trap();
    }
  }
}
// acquire at cluster scope: pairs with remote release-arrives from peer CTAs.
__device__ __forceinline__ bool mbar_try_wait_cluster(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
#if AREAL_WAIT_HINT_NS > 0
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity), "r"((uint32_t)AREAL_WAIT_HINT_NS)
      : "memory");
#else
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
#endif
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  if (mbar_try_wait_cluster(bar, parity)) return;
  uint64_t t0 = 0;
  uint32_t polls = 0;
  while (!mbar_try_wait_cluster(bar, parity)) {
    if (++polls % kWatchdogPolls == 0) {
      const uint64_t t = globaltimer_ns();
      if (t0 == 0) t0 = t;
      else if (t - t0 > kWaitLimitNs) __trap();
    }
  }
}
// 1-D bulk copy global -> shared, completion signalled on an mbarrier (TMA engine).
__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* gsrc, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// Same with an L2 cache-policy hint (createpolicy: evict_first / evict_last).
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void bulk_g2s_hint(void* smem_dst, const void* gsrc, uint32_t bytes,
                                              uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], "
      "%2, [%3], %4;" ::"r"(smem_u32(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
// 1-D bulk copy shared -> global (bulk-group completion).
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* smem_src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
               "r"(smem_u32(smem_src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N> __device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_id_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t nclusters_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_cluster_f64(uint32_t addr, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
}
__device__ __forceinline__ void mbar_remote_arrive_release(uint32_t remote_bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote_bar)
               : "memory");
}
// Remote arrive with the default (.release.cta) semantics, as CUTLASS's
// ClusterBarrier::arrive(cta_id): no global-memory fence, for signals that only order
// tcgen05 / shared-memory work already fenced by the caller (TMEM slot releases).
__device__ __forceinline__ void mbar_remote_arrive(uint32_t remote_bar) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(remote_bar) : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}

}  // namespace areal

namespace areal {
// ------------------------------------------------------------------ packed fp32x2 (sm_100a FFMA2/FADD2/FMUL2)
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  float2 d;
  asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
  float2 d;
  asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "mul.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ void mbar_arrive_remote_free(uint64_t* bar) { mbar_arrive(bar); }
}  // namespace areal

namespace areal {
// ------------------------------------------------------------------ cp.async (LDGSTS) scalar prefetch
__device__ __forceinline__ void cp_async4(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(smem_dst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(smem_dst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
}  // namespace areal

namespace areal {
// 2^x on the FMA pipe (FA4-style MUFU offload): x = n + f with n the
// nearest integer (1.5*2^23 rounding trick), 2^f by a degree-3 fit on [-0.5, 0.5]
// (max relative error 7.5e-5: only for 16-bit outputs), 2^n added to the exponent
// bits with one IMAD.  Arguments below -126 are clamped (result ~1e-38, vs 0).
__device__ __forceinline__ float2 exp2_poly3(float2 x_in) {
  float2 x = x_in;
  // clamp to [-126, 129]: from ~128.5 the exponent add overflows into inf/NaN bits, so an
  // overflowing argument still yields a non-finite value (detected by the fixed-shift
  // folds) instead of a wrapped finite one
  x.x = fminf(fmaxf(x.x, -126.f), 129.f);
  x.y = fminf(fmaxf(x.y, -126.f), 129.f);
  const float2 t = fadd2(x, make_float2(12582912.f, 12582912.f));
  const float2 n = fadd2(t, make_float2(-12582912.f, -12582912.f));
  const float2 f = ffma2(n, make_float2(-1.f, -1.f), x);
  float2 p = ffma2(f, make_float2(0.05517168715596199f, 0.05517168715596199f),
                   make_float2(0.2426111400127411f, 0.2426111400127411f));
  p = ffma2(p, f, make_float2(0.6932609677314758f, 0.6932609677314758f));
  p = ffma2(p, f, make_float2(0.9999280571937561f, 0.9999280571937561f));
  // the clamp's fmaxf would turn a NaN argument into -126 (a silent ~0): a NaN logit
  // must poison the row's sum as on the MUFU path, so NaN arguments pass through
  const float rx = __int_as_float(__float_as_int(t.x) * (1 << 23) + __float_as_int(p.x));
  const float ry = __int_as_float(__float_as_int(t.y) * (1 << 23) + __float_as_int(p.y));
  return make_float2(x_in.x == x_in.x ? rx : x_in.x, x_in.y == x_in.y ? ry : x_in.y);
}
}  // namespace areal

namespace areal {
// ------------------------------------------------------------------ host-side tuning table
// areal_set_tuning / areal_get_tuning (capi.cu); AREAL_TUNE_DEFAULT = shipped rule.
int64_t tuning(int knob);
}  // namespace areal
