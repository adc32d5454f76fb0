// Canonical merge of KVP fragments (attention.hpp:90-137), shared by the merge
// kernels. Any kvp up to kMaxKvp (validate_config's max_gpus, types.hpp:63):
// the kernels instantiate MAXK = 8 (registers) or kMaxKvp (local memory).
#pragma once

#include "common.cuh"
#include "kernels.h"

namespace hx {

// Order of source a before source b for ONE merged coefficient: descending
// lse, ties by the coefficient itself (ascending), then by source index. The
// reference breaks lse ties by the first differing coefficient of the head
// (attention.hpp:90-102) so that the merge is a pure function of the fragment
// set; per coefficient, two sources that tie on lse AND on the coefficient
// contribute identical addends, so this order gives the same guarantee --
// the merged value is bitwise invariant under any permutation of the ranks.
__device__ __forceinline__ bool merge_before(float la, float oa, int a, float lb, float ob, int b) {
  if (la != lb) return la > lb;
  if (oa != ob) return oa < ob;
  return a < b;
}

// out = sum_i w_i o_i / sum_i w_i over the sources in canonical order,
// w_i = e^(lse_i - max lse); empty sources (lse = -inf) carry no weight, all
// empty -> 0 (attention.hpp:118-137).
template <int MAXK>
__device__ __forceinline__ float merge_sources(const float* lse, const float* o, int kvp) {
  int ord[MAXK];
  for (int r = 0; r < kvp; ++r) ord[r] = r;
  for (int i = 1; i < kvp; ++i) {
    const int v = ord[i];
    int j = i - 1;
    while (j >= 0 && merge_before(lse[v], o[v], v, lse[ord[j]], o[ord[j]], ord[j])) {
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
