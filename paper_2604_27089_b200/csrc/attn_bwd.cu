// K4 placeholder (filled in next): attention backward.
#include <cuda_runtime.h>
#include "../../include/autosp.h"
extern "C" void autosp_set_error(const char* fmt, ...);
extern "C" size_t autosp_attn_bwd_workspace_bytes(int b, int hq, int s, int d) {
  return (size_t)b * hq * s * (d + 1) * sizeof(float);
}
extern "C" int autosp_attn_bwd(autosp_attn_tensor, autosp_attn_tensor, autosp_attn_tensor,
                               autosp_attn_tensor, autosp_attn_tensor, const float*,
                               autosp_attn_tensor, autosp_attn_tensor, autosp_attn_tensor, void*,
                               int, int, int, int, int, float, int, void*) {
  autosp_set_error("attn_bwd: not built yet");
  return AUTOSP_ERR_UNSUPPORTED;
}
