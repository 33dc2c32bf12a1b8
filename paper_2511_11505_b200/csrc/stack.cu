// fsc_layer_stack_forward: L-layer stack in Regular / Hybrid wiring (filled in with the attention filler).
#include "ctx.h"

extern "C" int fsc_layer_stack_forward(fsc_ctx* ctx, const fsc_attn_weights*, const fsc_moe_weights*, int, int, int,
                                       const int*, int, const float*, float*, const fsc_act_cache*, void*) {
  if (!ctx) return FSC_ERR_SHAPE;
  fsc_set_error(ctx, "fsc_layer_stack_forward: attention filler not built yet");
  return FSC_ERR_CONFIG;
}
