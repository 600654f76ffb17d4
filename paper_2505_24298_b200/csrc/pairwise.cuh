// pairwise.cuh — numpy's float64 add.reduce summation tree, replayed on the GPU.
//
// numpy sums a contiguous float64 run with pairwise_sum (numpy/_core/src/umath/
// loops_utils.h.src): runs < 8 are added left to right; runs <= 128 use 8
// interleaved accumulators combined as ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) plus
// a left-to-right tail; longer runs split at n/2 rounded down to a multiple of 8.
// Every operation is an IEEE-rounded add (no contraction), so the tree gives the
// reference's np.sum / np.mean / np.std bit for bit (trainer.py:119-123, and
// policy.py:129-130 through ParamGrad.global_norm).
//
// Parallel form: the top `depth` levels of the tree are cut off; each of the 2^depth
// subtree roots is summed by one thread (pw_sum_f), and one CTA combines the roots
// in tree order.
#pragma once
#include <stdint.h>

namespace areal {

// Leaf of numpy's pairwise sum (n <= 128): no recursion, so it inlines without a stack.
template <typename F>
__device__ __forceinline__ double pw_leaf_f(const F& f, int64_t off, int64_t n) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; ++i) res = __dadd_rn(res, f(off + i));
    return res;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = f(off + j);
  int64_t i = 8;
  for (; i < n - (n % 8); i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], f(off + i + j));
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, f(off + i));
  return res;
}

// Sum of f(off) .. f(off + n - 1) in numpy's pairwise order.  F: double f(int64_t).
template <typename F>
__device__ double pw_sum_f(const F& f, int64_t off, int64_t n) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; ++i) res = __dadd_rn(res, f(off + i));
    return res;
  }
  if (n <= 128) {
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = f(off + j);
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8) {
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], f(off + i + j));
    }
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, f(off + i));
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(pw_sum_f(f, off, n2), pw_sum_f(f, off + n2, n - n2));
}

// Depth (<= max_depth) at which every node of the tree still splits (size > 128).
__host__ __device__ inline int pw_depth(int64_t n, int max_depth) {
  int d = 0;
  while (d < max_depth && n > 128) {
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    n = n2;  // the leftmost path holds the smallest node at each depth
    ++d;
  }
  return d;
}

// Offset and length of subtree root i (0 <= i < 2^depth) of a run of n elements.
__device__ __forceinline__ void pw_node(int64_t n, int depth, int64_t i, int64_t& off,
                                        int64_t& len) {
  off = 0;
  len = n;
  for (int l = 0; l < depth; ++l) {
    int64_t n2 = len / 2;
    n2 -= n2 % 8;
    if ((i >> (depth - 1 - l)) & 1) {
      off += n2;
      len -= n2;
    } else {
      len = n2;
    }
  }
}

}  // namespace areal
