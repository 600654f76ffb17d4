// microbatch.cu — K4 dynamic micro-batch allocation (Alg. 1) and K5 packing, sm_100a.
//
// Reference: allocate_microbatches (/root/reference/pkg/src/asyncrl/trainer.py:235-270)
// and the packing order of train_step (trainer.py:310-320).  Bit-exact:
//   order   = stable sort by descending length (ties -> lower index)      (253)
//   place i : if #groups < min_groups or no group fits -> open a new group (259-261)
//             else join argmin over fitting groups of (#members, index)   (263-265)
//   packed token order = groups in creation order, members in placement order (320)
//
// One CTA per minibatch: block bitonic sort of unique 64-bit keys
// ((~len) << 32 | index), then a single warp runs the inherently sequential
// greedy placement with a warp-wide redux.min over (members << 13 | group) for
// the argmin, then warp scans produce the micro-batch and sequence offsets.
#include "common.cuh"

namespace areal {

constexpr int kPlanThreads = 512;

struct PlanArgs {
  const int64_t* bounds;
  const int32_t* item_traj;
  const int32_t* mb_offsets;
  const int64_t* mb_token_start;
  int32_t n_minibatches, n_items;
  int64_t capacity;
  int32_t min_groups;
  int32_t* group_of;
  int32_t* slot_of;
  int32_t* n_groups;
  int64_t* group_cu;
  int32_t* group_seq_cu;
  int32_t* packed_traj;
  int64_t* seq_cu;
  int32_t* status;
};

// warp-cooperative exclusive scan of src[0..n) into dst[0..n], dst[n] = total
template <typename S, typename V>
__device__ void warp_exclusive_scan(const S* src, V* dst, int n, int lane) {
  V carry = 0;
  for (int base = 0; base < n; base += 32) {
    const int i = base + lane;
    V v = (i < n) ? (V)src[i] : V(0);
    V x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const V y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (i < n) dst[i] = carry + x - v;
    carry += __shfl_sync(0xffffffffu, x, 31);
  }
  if (lane == 0) dst[n] = carry;
}

// Region A of the plan kernel's shared memory: the sort keys, later the group prefix
// sums (int64 token starts + int32 item starts), 16-byte aligned.
__host__ __device__ inline size_t plan_region_a(int n, int npow2) {
  const size_t keys = (size_t)npow2 * 8, sums = (size_t)(n + 1) * 12;
  return ((keys > sums ? keys : sums) + 15) & ~(size_t)15;
}

constexpr int kRegGroups = 128;  // groups whose totals live in warp 0's registers (4 / lane)

__global__ void __launch_bounds__(kPlanThreads) plan_kernel(PlanArgs a, int npow2) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int m = blockIdx.x;
  const int off = a.mb_offsets[m];
  const int n = a.mb_offsets[m + 1] - off;
  // shared memory (plan_smem): region A holds the sort keys until placement is done,
  // then the group prefix sums; totals / counts / in-group offsets are 32-bit (each
  // <= capacity < 2^31); an item's group and slot go straight to the global outputs.
  // 196 KB at the 8,192-item maximum.
  const size_t region_a = plan_region_a(n, npow2);
  uint64_t* keys = reinterpret_cast<uint64_t*>(sm);                   // [npow2]      (region A)
  int64_t* gstart = reinterpret_cast<int64_t*>(sm);                   // [n + 1]      (region A, later)
  int32_t* gis = reinterpret_cast<int32_t*>(gstart + (n + 1));        // [n + 1]      (region A, later)
  int32_t* tot = reinterpret_cast<int32_t*>(sm + region_a);           // [n + 1] group token totals
  int32_t* cnt = tot + (n + 1);                                       // [n + 1] group member counts
  int32_t* ofs = cnt + (n + 1);                                       // [n] token offset in group
  int32_t* gof = a.group_of + off;                                    // [n] (global output)
  int32_t* slt = a.slot_of + off;                                     // [n] (global output)
  __shared__ int s_bad_idx, s_bad_code, s_G;
  const int tid = threadIdx.x, lane = tid & 31;
  if (tid == 0) {
    s_bad_idx = 0x7fffffff;
    s_bad_code = 0;
  }
  __syncthreads();
  // ---- keys + validation (first failing item wins, like the reference's loop)
  for (int i = tid; i < npow2; i += blockDim.x) {
    uint64_t key = ~0ull;
    if (i < n) {
      const int32_t traj = a.item_traj[off + i];
      const int64_t len = a.bounds[traj + 1] - a.bounds[traj];
      if (len < 1 || len > a.capacity) atomicMin(&s_bad_idx, i);
      const uint32_t l32 = (uint32_t)(len < 1 ? 1 : (len > 0x7fffffff ? 0x7fffffff : len));
      key = ((uint64_t)(0xffffffffu - l32) << 32) | (uint32_t)i;
    }
    keys[i] = key;
  }
  __syncthreads();
  if (s_bad_idx != 0x7fffffff) {
    if (tid == 0) {
      const int32_t traj = a.item_traj[off + s_bad_idx];
      const int64_t len = a.bounds[traj + 1] - a.bounds[traj];
      a.status[m] = len < 1 ? AREAL_ERR_LEN_NONPOSITIVE : AREAL_ERR_LEN_EXCEEDS_CAPACITY;
      a.n_groups[m] = 0;
      // still leave a valid (identity-order) packing so a K5 launch queued behind this
      // plan stays in bounds; the caller raises on the status before using it
      const int64_t t0 = a.mb_token_start[m];
      a.group_cu[off + m] = t0;
      a.group_seq_cu[off + m] = off;
      int64_t t = t0;
      for (int i = 0; i < n; ++i) {
        const int32_t tr = a.item_traj[off + i];
        a.group_of[off + i] = 0;
        a.slot_of[off + i] = i;
        a.packed_traj[off + i] = tr;
        a.seq_cu[off + i] = t;
        t += a.bounds[tr + 1] - a.bounds[tr];
      }
      if (m == a.n_minibatches - 1) a.seq_cu[a.n_items] = t;
    }
    return;
  }
  // ---- bitonic sort (ascending key == descending length, then ascending index)
  for (int k = 2; k <= npow2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = tid; i < npow2; i += blockDim.x) {
        const int p = i ^ j;
        if (p > i) {
          const uint64_t x = keys[i], y = keys[p];
          const bool up = (i & k) == 0;
          if ((x > y) == up) {
            keys[i] = y;
            keys[p] = x;
          }
        }
      }
      __syncthreads();
    }
  }
  // ---- greedy placement (warp 0): Alg. 1.  The loop is one serial chain over the
  // items (its latency is the kernel's), so it is kept short: the first kRegGroups
  // groups live in registers, group g on lane g % 32 as room = C - total (-1 while
  // unopened, so nothing fits) and key = members << 13 | g.  Per item: one compare
  // + select + min per register group, one REDUX.MIN, a predicated update on the
  // owner lane.  Groups beyond kRegGroups (tiny items under a large capacity) use
  // tot / cnt in shared memory.  All sums fit 32 bits: totals <= C < 2^31.
  if (tid < 32) {
    // four named registers per lane (an array here ends up in local memory)
    int32_t r0 = -1, r1 = -1, r2 = -1, r3 = -1;
    uint32_t k0 = lane, k1 = lane + 32, k2 = lane + 64, k3 = lane + 96;
    int G = 0;
    const int32_t C = (int32_t)a.capacity;  // validated <= INT32_MAX on the host
    const int kmin = a.min_groups;
    uint64_t key = n > 0 ? keys[0] : 0;
    for (int p = 0; p < n; ++p) {
      const int item = (int)(key & 0xffffffffu);
      const int32_t s = (int32_t)(0xffffffffu - (uint32_t)(key >> 32));
      if (p + 1 < n) key = keys[p + 1];
      uint32_t best = s <= r0 ? k0 : 0xffffffffu;
      best = min(best, s <= r1 ? k1 : 0xffffffffu);
      best = min(best, s <= r2 ? k2 : 0xffffffffu);
      best = min(best, s <= r3 ? k3 : 0xffffffffu);
      for (int g = kRegGroups + lane; g < G; g += 32) {
        if (s <= C - tot[g]) best = min(best, ((uint32_t)cnt[g] << 13) | (uint32_t)g);
      }
      best = __reduce_min_sync(0xffffffffu, best);
      // fewer than min_groups, or nothing fits: open group G
      const bool open = G < kmin || best == 0xffffffffu;
      const int g = open ? G : (int)(best & 0x1fffu);
      G += open;
      if (g < kRegGroups) {
        if (lane == (g & 31)) {
          const int j = g >> 5;
          int32_t room = j == 0 ? r0 : j == 1 ? r1 : j == 2 ? r2 : r3;
          uint32_t kk = j == 0 ? k0 : j == 1 ? k1 : j == 2 ? k2 : k3;
          if (open) room = C;
          gof[item] = g;
          slt[item] = (int32_t)(kk >> 13);
          ofs[item] = C - room;
          room -= s;
          kk += 1u << 13;
          r0 = j == 0 ? room : r0; r1 = j == 1 ? room : r1;
          r2 = j == 2 ? room : r2; r3 = j == 3 ? room : r3;
          k0 = j == 0 ? kk : k0; k1 = j == 1 ? kk : k1;
          k2 = j == 2 ? kk : k2; k3 = j == 3 ? kk : k3;
        }
      } else if (lane == 0) {
        if (open) {
          tot[g] = 0;
          cnt[g] = 0;
        }
        gof[item] = g;
        slt[item] = cnt[g];
        ofs[item] = tot[g];
        tot[g] += s;
        cnt[g] += 1;
      }
      __syncwarp();
    }
    const int32_t rr[4] = {r0, r1, r2, r3};
    const uint32_t kq[4] = {k0, k1, k2, k3};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int g = lane + 32 * j;
      if (g < G) {
        tot[g] = C - rr[j];
        cnt[g] = (int32_t)(kq[j] >> 13);
      }
    }
    if (lane == 0) s_G = G;
  }
  __syncthreads();
  const int G = s_G;
  // ---- offsets: token starts and item starts of each group
  // region A is free now (keys dead after placement); scans of the group totals / counts
  if (tid < 32) warp_exclusive_scan<int32_t, int64_t>(tot, gstart, G, lane);
  else if (tid < 64) warp_exclusive_scan<int32_t, int32_t>(cnt, gis, G, lane);
  __syncthreads();
  const int64_t t0 = a.mb_token_start[m];
  const int base = off + m;  // this minibatch's slice of group_cu / group_seq_cu
  for (int g = tid; g <= G; g += blockDim.x) {
    a.group_cu[base + g] = t0 + gstart[g];
    a.group_seq_cu[base + g] = off + gis[g];
  }
  for (int i = tid; i < n; i += blockDim.x) {
    const int g = gof[i];
    const int pos = off + gis[g] + slt[i];
    a.packed_traj[pos] = a.item_traj[off + i];
    a.seq_cu[pos] = t0 + gstart[g] + ofs[i];
  }
  if (tid == 0) {
    a.n_groups[m] = G;
    a.status[m] = AREAL_OK;
    if (m == a.n_minibatches - 1) a.seq_cu[a.n_items] = t0 + gstart[G];
  }
}

// K5b: one warp per packed sequence writes its token gather indices (coalesced).
__global__ void fill_gather_kernel(const int64_t* bounds, const int32_t* packed_traj,
                                   const int64_t* seq_cu, int32_t n_items, int64_t n_packed,
                                   int32_t* gather, int32_t* seq_id) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t p = w0; p < n_items; p += nw) {
    const int32_t traj = packed_traj[p];
    const int64_t src = bounds[traj];
    const int64_t len = bounds[traj + 1] - src;
    const int64_t dst = seq_cu[p];
    if (dst < 0 || dst + len > n_packed) continue;  // never write outside gather[]
    for (int64_t i = lane; i < len; i += 32) {
      gather[dst + i] = (int32_t)(src + i);
      if (seq_id) seq_id[dst + i] = (int32_t)p;
    }
  }
}

static size_t plan_smem(int n, int npow2) {
  return plan_region_a(n, npow2) + 2 * (size_t)(n + 1) * 4 + (size_t)n * 4 + 64;
}

}  // namespace areal

using namespace areal;

extern "C" int areal_plan_microbatches(const int64_t* traj_bounds, const int32_t* item_traj,
                                       const int32_t* mb_offsets, const int64_t* mb_token_start,
                                       int32_t n_minibatches, int32_t n_items,
                                       int32_t max_items_per_mb, int64_t capacity,
                                       int32_t min_groups, int32_t* group_of, int32_t* slot_of,
                                       int32_t* n_groups, int64_t* group_cu, int32_t* group_seq_cu,
                                       int32_t* packed_traj, int64_t* seq_cu, int32_t* status,
                                       void* stream) {
  if (min_groups < 1) return AREAL_ERR_MIN_GROUPS;
  if (n_minibatches < 0 || n_items < 0 || max_items_per_mb < 0) return AREAL_ERR_INVALID_ARGUMENT;
  if (max_items_per_mb > AREAL_MAX_ITEMS_PER_MINIBATCH) return AREAL_ERR_UNSUPPORTED;
  if (capacity < 1 || capacity > 0x7fffffff) return AREAL_ERR_INVALID_ARGUMENT;
  if (n_minibatches == 0) return AREAL_OK;
  if (!traj_bounds || !item_traj || !mb_offsets || !mb_token_start || !group_of || !slot_of ||
      !n_groups || !group_cu || !group_seq_cu || !packed_traj || !seq_cu || !status)
    return AREAL_ERR_INVALID_ARGUMENT;
  int npow2 = 1;
  while (npow2 < max_items_per_mb) npow2 <<= 1;
  const size_t smem = plan_smem(max_items_per_mb, npow2);
  if (smem > 48 * 1024) {
    if (cudaFuncSetAttribute(plan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
      return AREAL_ERR_CUDA;
  }
  PlanArgs a = {traj_bounds, item_traj, mb_offsets, mb_token_start, n_minibatches, n_items,
                capacity, min_groups, group_of, slot_of, n_groups, group_cu, group_seq_cu,
                packed_traj, seq_cu, status};
  plan_kernel<<<n_minibatches, kPlanThreads, smem, static_cast<cudaStream_t>(stream)>>>(a, npow2);
  AREAL_CUDA_CHECK_LAUNCH();
  return AREAL_OK;
}

extern "C" int areal_fill_gather(const int64_t* traj_bounds, const int32_t* packed_traj,
                                 const int64_t* seq_cu, int32_t n_items, int64_t n_packed_tokens,
                                 int32_t* gather, int32_t* seq_id, void* stream) {
  if (n_items < 0 || n_packed_tokens < 0) return AREAL_ERR_INVALID_ARGUMENT;
  if (n_items == 0 || n_packed_tokens == 0) return AREAL_OK;
  if (n_packed_tokens > 0x7fffffffll) return AREAL_ERR_UNSUPPORTED;
  if (!traj_bounds || !packed_traj || !seq_cu || !gather) return AREAL_ERR_INVALID_ARGUMENT;
  const int64_t blocks = std::min<int64_t>(((int64_t)n_items * 32 + 255) / 256, 148 * 16);
  fill_gather_kernel<<<(unsigned)blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      traj_bounds, packed_traj, seq_cu, n_items, n_packed_tokens, gather, seq_id);
  AREAL_CUDA_CHECK_LAUNCH();
  return AREAL_OK;
}
