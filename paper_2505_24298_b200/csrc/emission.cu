// emission.cu — rollout-side recording of behaviour log-probs at emission.
//
// Reference: RolloutWorker.step (/root/reference/pkg/src/asyncrl/rollout.py:140-165):
// per emitted token, traj.tokens.append(token), traj.behavior_logprobs.append(
// P.log_prob(params, features, token)) and traj.versions.append(params.version), all
// under one lock so the three stay aligned with the generating parameters.
//
// B200 form for a decode step of B live sequences: one tiny kernel appends each row's
// sampled token and the generating version to its slot's device buffers and emits the
// row -> buffer-position map; K1 (logits) or K7 (hidden states + LM head) then writes
// the log-prob straight into the same position through that map (row_index), so a
// decode step costs 2 launches and no host round trip.  Every argument that changes
// between steps (slots, tokens, the version) is read from device memory, so a decode
// loop can capture the step once in a CUDA graph and replay it.
#include "common.cuh"

namespace areal {

__global__ void emission_append_kernel(const int32_t* slots, const int64_t* step_tokens, int64_t n_rows,
                                       const int32_t* version, int32_t n_slots, int64_t max_len,
                                       int32_t* lengths, int64_t* tok_buf, int32_t* ver_buf,
                                       int32_t* row_index, int32_t* status) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_rows) return;
  const int64_t sink = (int64_t)n_slots * max_len;  // overflow / bad-slot rows land here
  const int32_t s = slots[r];
  int64_t idx = sink;
  if (s < 0 || s >= n_slots) {
    atomicMax(status, AREAL_ERR_BAD_SHAPE);
  } else {
    const int32_t pos = atomicAdd(lengths + s, 1);
    if (pos >= max_len) {
      atomicSub(lengths + s, 1);
      atomicMax(status, AREAL_ERR_LEN_EXCEEDS_CAPACITY);
    } else {
      idx = (int64_t)s * max_len + pos;
    }
  }
  tok_buf[idx] = step_tokens[r];
  ver_buf[idx] = *version;
  row_index[r] = (int32_t)idx;
}

}  // namespace areal

using namespace areal;

extern "C" int areal_emission_append(const int32_t* slots, const int64_t* step_tokens, int64_t n_rows,
                                     const int32_t* version, int32_t n_slots, int64_t max_len,
                                     int32_t* lengths, int64_t* tok_buf, int32_t* ver_buf,
                                     int32_t* row_index_out, int32_t* status, void* stream_) {
  if (n_rows < 0 || n_slots < 1 || max_len < 1) return AREAL_ERR_BAD_SHAPE;
  if ((int64_t)n_slots * max_len >= ((int64_t)1 << 31) - 1) return AREAL_ERR_BAD_SHAPE;
  if (n_rows == 0) return AREAL_OK;
  if (!slots || !step_tokens || !version || !lengths || !tok_buf || !ver_buf || !row_index_out || !status)
    return AREAL_ERR_INVALID_ARGUMENT;
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  emission_append_kernel<<<(unsigned)((n_rows + 127) / 128), 128, 0, stream>>>(
      slots, step_tokens, n_rows, version, n_slots, max_len, lengths, tok_buf, ver_buf, row_index_out, status);
  AREAL_CUDA_CHECK_LAUNCH();
  return AREAL_OK;
}
