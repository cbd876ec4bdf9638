// lgdm_sweep.cuh -- fused structured-sweep assembly kernels (placeholder until implemented).
#pragma once
namespace {
bool sweep_supported(lgdm_mesh) { return false; }
lgdm_status assemble_sweep(lgdm_mesh) { return fail(LGDM_ERR_UNSUPPORTED, "sweep kernel not built"); }
void sweep_free(lgdm_mesh) {}
}  // namespace
