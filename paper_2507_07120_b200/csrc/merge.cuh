// Canonical merge of KVP fragments (attention.hpp:90-137): descending lse,
// ties by source rank, weights e^(lse - max); shared by the merge kernels.
#pragma once

#include "common.cuh"

namespace hx {

// Canonical merge (attention.hpp:90-137): descending lse, ties by source rank.
__device__ __forceinline__ float merge_sources(const float* lse, const float* o, int kvp) {
  int ord[8];
  for (int r = 0; r < kvp; ++r) ord[r] = r;
  for (int i = 1; i < kvp; ++i) {
    const int v = ord[i];
    int j = i - 1;
    while (j >= 0 && lse[ord[j]] < lse[v]) {
      ord[j + 1] = ord[j];
      --j;
    }
    ord[j + 1] = v;
  }
  const float m = lse[ord[0]];
  if (m == -INFINITY) return 0.f;
  float acc = 0.f, z = 0.f;
  for (int i = 0; i < kvp; ++i) {
    const int r = ord[i];
    if (lse[r] == -INFINITY) continue;
    const float w = __expf(lse[r] - m);
    acc += w * o[r];
    z += w;
  }
  return acc / z;
}

}  // namespace hx
