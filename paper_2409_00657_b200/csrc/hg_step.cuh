// Step-level structures shared by the split training kernels (hg_dense.cu)
// and the persistent training step (hg_persist.cu).
#pragma once
#include <cuda_bf16.h>

#include "hg_common.cuh"

namespace hg {

using bf16 = __nv_bfloat16;

struct SgdMat {
  int64_t off;        // flat offset of the matrix [rows x cols] (row-major)
  int rows, cols;
  bf16* tdst;         // transposed bf16 copy [cols x rows] (ld tld) or null
  int64_t tld;
  bf16* sdst;         // straight bf16 copy [rows x cols] (ld sld) or null
  int64_t sld;
  int tiles_c, tile0; // column tiles; first tile index of this matrix
};
struct SgdPlan {
  int n_mats, n_tiles;
  SgdMat m[HG_MAX_LAYERS + 1];
  int64_t plain_lo, plain_hi;  // elementwise range (the biases)
};

int make_sgd_plan(const hg_step_desc* d, float* params, int64_t n, SgdPlan* out);

}  // namespace hg
