// region.cu — kernel offset sets N^D (host).  P:154 (hypercube V^D(K)), P:159 (dilation,
// arbitrary N^D), Fig. 3 / P:250-282 (cross, hypercross, hybrid).  Readings R2-R4.
#include <algorithm>
#include <set>

#include "mk_internal.cuh"

namespace mk {

namespace {
// Index range of one axis: odd K centred (V^1(3) = {-1,0,1}), even K = {0..K-1} (R3).
void axis_values(int32_t K, int32_t dil, std::vector<int32_t>* v) {
  v->clear();
  const int32_t lo = (K & 1) ? -(K / 2) : 0;
  for (int32_t i = 0; i < K; ++i) v->push_back((lo + i) * dil);
}

// Cartesian product of per-axis value lists, axis 0 most significant (lexicographic, R2).
void product(const std::vector<std::vector<int32_t>>& axes, std::vector<std::vector<int32_t>>* out) {
  out->assign(1, std::vector<int32_t>());
  for (const auto& ax : axes) {
    std::vector<std::vector<int32_t>> next;
    next.reserve(out->size() * ax.size());
    for (const auto& prefix : *out)
      for (int32_t v : ax) {
        auto p = prefix;
        p.push_back(v);
        next.push_back(std::move(p));
      }
    out->swap(next);
  }
}
}  // namespace

mk_status region_enumerate(const mk_region* r, std::vector<int32_t>* offsets, int32_t* K) {
  if (!r) MK_FAIL(MK_ERR_INVALID_ARGUMENT, "region is NULL");
  const int D = r->D;
  if (D < 1 || D > MK_MAX_REGION) MK_FAIL(MK_ERR_INVALID_ARGUMENT, "region: D out of range");
  std::vector<std::vector<int32_t>> list;
  if (r->type == MK_CUSTOM) {
    if (!r->offsets || r->n_offsets < 1) MK_FAIL(MK_ERR_INVALID_ARGUMENT, "custom region without offsets");
    std::set<std::vector<int32_t>> seen;
    for (int32_t i = 0; i < r->n_offsets; ++i) {
      std::vector<int32_t> o(r->offsets + (size_t)i * D, r->offsets + (size_t)(i + 1) * D);
      if (!seen.insert(o).second) MK_FAIL(MK_ERR_INVALID_ARGUMENT, "custom region: duplicate offset");
      list.push_back(o);
    }
  } else {
    int32_t dil[MK_MAX_REGION];
    for (int d = 0; d < D; ++d) {
      if (r->size[d] < 1) MK_FAIL(MK_ERR_INVALID_ARGUMENT, "region: size must be >= 1");
      if (r->dilation[d] < 0) MK_FAIL(MK_ERR_INVALID_ARGUMENT, "region: negative dilation");
      dil[d] = r->dilation[d] == 0 ? 1 : r->dilation[d];
    }
    std::vector<std::vector<int32_t>> axes(D);
    for (int d = 0; d < D; ++d) axis_values(r->size[d], dil[d], &axes[d]);
    if (r->type == MK_HYPERCUBE) {
      product(axes, &list);
    } else if (r->type == MK_HYPERCROSS || r->type == MK_HYBRID) {
      const int t = r->temporal_axis < 0 ? D - 1 : r->temporal_axis;
      if (r->type == MK_HYBRID && t >= D) MK_FAIL(MK_ERR_INVALID_ARGUMENT, "region: temporal axis >= D");
      if (r->type == MK_HYBRID) {
        auto spatial = axes;
        spatial[t] = {0};
        product(spatial, &list);  // spatial cube at temporal offset 0 (R4)
      } else {
        list.push_back(std::vector<int32_t>(D, 0));
      }
      for (int d = 0; d < D; ++d) {
        if (r->type == MK_HYBRID && d != t) continue;  // hybrid: cross along time only
        for (int32_t v : axes[d]) {
          if (v == 0) continue;
          std::vector<int32_t> o(D, 0);
          o[d] = v;
          list.push_back(o);
        }
      }
      std::sort(list.begin(), list.end());
      list.erase(std::unique(list.begin(), list.end()), list.end());
    } else {
      MK_FAIL(MK_ERR_INVALID_ARGUMENT, "region: unknown type");
    }
  }
  *K = (int32_t)list.size();
  if (offsets) {
    offsets->clear();
    for (const auto& o : list) offsets->insert(offsets->end(), o.begin(), o.end());
  }
  return MK_OK;
}

}  // namespace mk

extern "C" mk_status mk_region_offsets(const mk_region* region, int32_t* K, int32_t* h_offsets) {
  mk::clear_error();
  if (!K) MK_FAIL(MK_ERR_INVALID_ARGUMENT, "mk_region_offsets: K is NULL");
  std::vector<int32_t> offs;
  mk_status s = mk::region_enumerate(region, &offs, K);
  if (s != MK_OK) return s;
  if (h_offsets) std::copy(offs.begin(), offs.end(), h_offsets);
  return MK_OK;
}
