// attention_tc.cu — tensor-core sparse-query attention (placeholder).
#include "ctx.h"

bool attention_tc_ok(const cb_ctx*) { return false; }
cb_status launch_attention_tc(cb_ctx*, const void*, const int*, const int*, int, const void*, const void*, int, void*,
                              cudaStream_t) {
  cb_set_error("tensor-core attention not built");
  return CB_E_UNSUPPORTED;
}
cb_status attention_tc_init() { return CB_OK; }
