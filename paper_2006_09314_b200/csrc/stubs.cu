// Temporary: entry points not yet implemented on the device.
#include "ctx.cuh"
extern "C" {
int sl_setup(fc_ctx c, int, const double*, const fc_params*) { if (c) c->err = "sl_setup: not built yet"; return FC_ERR_NOT_READY; }
}
