// Host-side DeAR tensor-fusion partitioner and chunk layout (pure C++, no GPU).
//
// dear_plan_build  <- build_fusion_plan / per_layer_plan (fusion.cpp:29-70)
// dear_chunk_layout <- chunk_ranges (collective.cpp:39-57), owner map (:94)
// Bit-exact with the reference by construction (same integer arithmetic) and
// by test (tests/test_plan.py against tests/golden/plans.json, chunks.json).
#include <stdint.h>

#include <string>
#include <vector>

#include "dear.h"
#include "dear_internal.h"

namespace dear {

std::vector<Group> build_plan(const std::vector<int64_t>& layer_bytes, int64_t buffer_bytes) {
  const int L = static_cast<int>(layer_bytes.size());
  if (L == 0) {
    throw Error(DEAR_EINVAL, buffer_bytes == 0 ? "per_layer_plan: empty model"
                                               : "build_fusion_plan: empty model");
  }
  for (int l = 1; l <= L; ++l) {
    if (layer_bytes[static_cast<size_t>(l - 1)] < 0) {
      throw Error(DEAR_EINVAL, "model: param_count must be >= 0 (layer " + std::to_string(l) + ")");
    }
  }
  if (buffer_bytes < 0) {
    throw Error(DEAR_EINVAL, "build_fusion_plan: buffer_bytes must be > 0");
  }
  std::vector<Group> groups;
  if (buffer_bytes == 0) {
    for (int l = L; l >= 1; --l) groups.push_back({l, l});
    return groups;
  }
  // Walk from the output layer down; a layer joins the open group while the
  // group total stays within the buffer, otherwise the open group closes.
  int high = L;
  int64_t acc = layer_bytes[static_cast<size_t>(L - 1)];
  for (int l = L - 1; l >= 1; --l) {
    const int64_t next = layer_bytes[static_cast<size_t>(l - 1)];
    if (acc + next <= buffer_bytes) {
      acc += next;
    } else {
      groups.push_back({l + 1, high});
      high = l;
      acc = next;
    }
  }
  groups.push_back({1, high});
  return groups;
}

std::vector<int64_t> chunk_begins(int64_t d, int P) {
  if (P < 1) throw Error(DEAR_EINVAL, "chunk_ranges: workers must be >= 1");
  if (d < 0) throw Error(DEAR_EINVAL, "chunk_ranges: d_elems must be >= 0");
  const int64_t base = d / P, extra = d % P;
  std::vector<int64_t> b(static_cast<size_t>(P) + 1);
  int64_t at = 0;
  for (int c = 0; c < P; ++c) {
    b[static_cast<size_t>(c)] = at;
    at += base + (c < extra ? 1 : 0);
  }
  b[static_cast<size_t>(P)] = at;
  return b;
}

int64_t slot_stride(int64_t d, int P) {
  const int64_t s = (d + P - 1) / P;
  return (s + 63) / 64 * 64;
}

}  // namespace dear

using dear::Error;

extern "C" {

int dear_plan_build(const int64_t* layer_bytes, int32_t L, int64_t buffer_bytes, int32_t* low,
                    int32_t* high, int32_t* n_groups) {
  DEAR_API_BEGIN
  if (L < 0 || (L > 0 && layer_bytes == nullptr) || low == nullptr || high == nullptr ||
      n_groups == nullptr) {
    throw Error(DEAR_EINVAL, "dear_plan_build: null or negative argument");
  }
  const std::vector<int64_t> lb(layer_bytes, layer_bytes + L);
  const auto groups = dear::build_plan(lb, buffer_bytes);
  for (size_t g = 0; g < groups.size(); ++g) {
    low[g] = groups[g].low;
    high[g] = groups[g].high;
  }
  *n_groups = static_cast<int32_t>(groups.size());
  DEAR_API_END
}

int dear_chunk_layout(int64_t d, int32_t P, int64_t* begin, int64_t* slot_elems) {
  DEAR_API_BEGIN
  const auto b = dear::chunk_begins(d, P);
  if (begin) {
    for (size_t i = 0; i < b.size(); ++i) begin[i] = b[i];
  }
  if (slot_elems) *slot_elems = (d + P - 1) / P;
  DEAR_API_END
}

int64_t dear_slot_stride(int64_t d, int32_t P) {
  if (P < 1 || d < 0) return -1;
  return dear::slot_stride(d, P);
}

}  // extern "C"
