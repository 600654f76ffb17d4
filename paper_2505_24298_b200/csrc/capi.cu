// capi.cu — library-level entry points of libareal_b200.so.
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
