// Kernel (3): the boosting trainer (fit, costmodel.cpp:152-222). Under construction.
#include "forest.cuh"

extern "C" {

int fs_fit(fs_device*, fs_forest*, int32_t, const int64_t*, int32_t, const double*, const double*,
           const fs_gbt_params*) {
  return fs::guard([] { fs::fail(FS_ECUDA, "fs_fit: trainer not built yet"); });
}

int fs_fit_d(fs_device*, fs_forest*, int32_t, const int64_t*, int32_t, const double*, const double*,
             const fs_gbt_params*) {
  return fs::guard([] { fs::fail(FS_ECUDA, "fs_fit_d: trainer not built yet"); });
}

}  // extern "C"
