// K5 photometric registration (filled in below the rasterizer milestone).
#include "common.cuh"
extern "C" size_t ss_photo_workspace_bytes(int32_t M) { return (size_t)M * 64 + 4096; }
extern "C" int ss_photo_system(const float*, int32_t, const float*, const uint8_t*, const ss_camera*, const double*,
                               double, const ss_reg_cfg*, double*, void*, void*) {
  return SS_ERR_UNSUPPORTED;
}
