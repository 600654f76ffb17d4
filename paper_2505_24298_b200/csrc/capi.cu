// capi.cu — library-level entry points of libareal_b200.so.
#include <atomic>

#include "common.cuh"

extern "C" int areal_abi_version(void) { return AREAL_ABI_VERSION; }

extern "C" size_t areal_workspace_bytes(void) { return AREAL_WORKSPACE_BYTES; }

extern "C" const char* areal_status_string(int status) {
  switch (status) {
    case AREAL_OK: return "ok";
    case AREAL_ERR_INVALID_ARGUMENT: return "invalid argument";
    case AREAL_ERR_BAD_DTYPE: return "unsupported dtype";
    case AREAL_ERR_BAD_SHAPE: return "bad shape";
    case AREAL_ERR_MISALIGNED: return "misaligned pointer or row stride (ROW_RING needs 16-byte rows)";
    case AREAL_ERR_LEN_NONPOSITIVE: return "sequence lengths must be positive";
    case AREAL_ERR_LEN_EXCEEDS_CAPACITY: return "sequence length exceeds capacity";
    case AREAL_ERR_MIN_GROUPS: return "min_groups must be >= 1";
    case AREAL_ERR_WORKSPACE: return "workspace missing or smaller than AREAL_WORKSPACE_BYTES";
    case AREAL_ERR_CUDA: return "CUDA launch error";
    case AREAL_ERR_UNSUPPORTED: return "unsupported configuration";
    case AREAL_ERR_BAD_CLIP_EPS: return "clip_eps must be in (0, 1)";
    default: return "unknown status";
  }
}

// ---- kernel-selection overrides (areal_tune_t); -1 everywhere = the shipped rules
static std::atomic<int64_t> g_tuning[AREAL_TUNE_COUNT] = {-1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1};

int64_t areal::tuning(int knob) {
  return (knob >= 0 && knob < AREAL_TUNE_COUNT) ? g_tuning[knob].load(std::memory_order_relaxed) : -1;
}

static bool tuning_valid(int knob, int64_t v) {
  if (v == AREAL_TUNE_DEFAULT) return true;
  switch (knob) {
    case AREAL_TUNE_K2_CLUSTER_SIZE: return v == 2 || v == 4 || v == 8;
    case AREAL_TUNE_K2_TMEM:
    case AREAL_TUNE_K2_TMEM_STREAM:
    case AREAL_TUNE_K2_TMEM_UNALIGNED:
    case AREAL_TUNE_K1_RING_UNALIGNED:
    case AREAL_TUNE_ROWCTA: return v == 0 || v == 1;
    case AREAL_TUNE_K2_SMALL_ROWCTA_KB: return v >= 0 && v <= 1024;
    case AREAL_TUNE_K7_NT: return v == 4 || v == 8;
    case AREAL_TUNE_K7_GROUP: return v >= 1 && v <= 16;
    case AREAL_TUNE_K1_CLUSTER_SIZE: return v == 1 || v == 2 || v == 4 || v == 8;
    case AREAL_TUNE_LMH_GROUP_M: return v >= 1 && v <= 256;
    default: return false;
  }
}

extern "C" int areal_set_tuning(int knob, int64_t value) {
  if (knob < 0 || knob >= AREAL_TUNE_COUNT || !tuning_valid(knob, value)) return AREAL_ERR_INVALID_ARGUMENT;
  g_tuning[knob].store(value, std::memory_order_relaxed);
  return AREAL_OK;
}

extern "C" int areal_get_tuning(int knob, int64_t* value) {
  if (knob < 0 || knob >= AREAL_TUNE_COUNT || value == nullptr) return AREAL_ERR_INVALID_ARGUMENT;
  *value = g_tuning[knob].load(std::memory_order_relaxed);
  return AREAL_OK;
}
