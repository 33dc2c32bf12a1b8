// EP transport (dispatch / combine between ranks). Round-1 state: EP == 1 only;
// the peer-memory path is built next.
#include "ctx.h"

size_t fsc_transport_blob_size() { return 0; }

int fsc_transport_init(fsc_ctx* ctx) {
  if (ctx->ep == 1) return FSC_OK;
  fsc_set_error(ctx, "ep_size > 1 transport not available in this build");
  return FSC_ERR_COMM;
}
int fsc_transport_export(fsc_ctx* ctx, void*) { return ctx->ep == 1 ? FSC_OK : FSC_ERR_COMM; }
int fsc_transport_import(fsc_ctx* ctx, const void*) { return ctx->ep == 1 ? FSC_OK : FSC_ERR_COMM; }
void fsc_transport_finalize(fsc_ctx*) {}
int fsc_transport_dispatch(fsc_ctx*, int, cudaStream_t) { return FSC_ERR_COMM; }
int fsc_transport_dispatch_wait(fsc_ctx*, cudaStream_t) { return FSC_ERR_COMM; }
int fsc_transport_combine(fsc_ctx*, int, cudaStream_t) { return FSC_ERR_COMM; }
int fsc_transport_combine_wait(fsc_ctx*, cudaStream_t) { return FSC_ERR_COMM; }
