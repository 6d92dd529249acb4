/*
 * oracle.cpp — TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * Plain C++17 CPU oracle for the generalized sparse convolution hot path
 * (arXiv 1904.08755).  Every step follows a definition or algorithm of the paper,
 * cited inline; where the paper is silent the reading is named (R1..R22).
 * Nothing here is blocked, fused or reordered: coordinates go through a
 * std::unordered_map, kernel maps are naive per-offset loops over output rows, and
 * features are fp64 with the loop order of Alg. 2.
 *
 * Parity pins (tests/test_oracle_*.py): worked examples of the paper/SPEC, closed-form
 * counts, brute force on tiny inputs, torch.nn.functional.conv{3d,_transpose3d} in fp64
 * on fully occupied grids (Eq. 2 special case), and the adjoint identities.
 */
#include "oracle.h"

#include <algorithm>
#include <array>
#include <cmath>
#include <cstring>
#include <unordered_map>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

constexpr int kMaxWords = 8;  // D <= 7 spatial axes + batch
using Key = std::array<int32_t, kMaxWords>;

struct KeyHash {
  size_t operator()(const Key& k) const {
    // Any hash works: results never depend on it (exact-key semantics, reading R5).
    uint64_t h = 1469598103934665603ull;
    for (int32_t w : k) {
      h ^= static_cast<uint32_t>(w);
      h *= 1099511628211ull;
    }
    return static_cast<size_t>(h ^ (h >> 29));
  }
};

using CoordMap = std::unordered_map<Key, int32_t, KeyHash>;

Key row_key(const int32_t* row, int32_t D) {
  Key k{};
  for (int d = 0; d <= D; ++d) k[d] = row[d];
  return k;
}

bool fits_i32(int64_t v) { return v >= INT32_MIN && v <= INT32_MAX; }

// The ABI's coordinate domain (reading R19, mk.h MK_MAX_DIM): int32 components; for D = 4
// the time axis u_3 in [-2^15, 2^15) and batch b <= 65534; for D = 5..7 axes 0-2 in
// [-2^19, 2^19), axes 3-5 in [-2^11, 2^11), axis 6 in [-2^15, 2^15) and (D = 7) b <= 65534.
// Rows outside it are rejected with ORC_COORD_RANGE (the same status the GPU path returns).
bool in_domain(const int64_t* c, int32_t D, int64_t b) {
  auto in = [](int64_t v, int64_t lo, int64_t hi) { return v >= lo && v < hi; };
  for (int d = 0; d < D; ++d)
    if (!fits_i32(c[d])) return false;
  if (D == 4) return in(c[3], -32768, 32768) && b <= 65534;
  if (D >= 5) {
    for (int d = 0; d < 3; ++d)
      if (!in(c[d], -(1 << 19), 1 << 19)) return false;
    for (int d = 3; d < std::min(D, 6); ++d)
      if (!in(c[d], -(1 << 11), 1 << 11)) return false;
    if (D == 7) return in(c[6], -32768, 32768) && b <= 65534;
  }
  return true;
}

// floor division toward -infinity (reading R7).  s > 0.
int64_t floor_div(int64_t u, int64_t s) {
  int64_t q = u / s;
  if ((u % s) != 0 && u < 0) q -= 1;
  return q;
}

// Per-axis index range R(K) (reading R3): centred for odd K (V^1(3) = {-1,0,1}),
// {0..K-1} for even K.
std::vector<int32_t> axis_range(int32_t K) {
  std::vector<int32_t> r;
  if (K % 2 == 1) {
    for (int32_t i = -(K - 1) / 2; i <= (K - 1) / 2; ++i) r.push_back(i);
  } else {
    for (int32_t i = 0; i < K; ++i) r.push_back(i);
  }
  return r;
}

}  // namespace

extern "C" {

int orc_quantize(const float* points, const int32_t* batch, int64_t n, int32_t D, float voxel,
                 int32_t* coords_out, int32_t* point_to_row, int32_t* first_point,
                 int64_t* n_out, int64_t* err_row) {
  *err_row = -1;
  *n_out = 0;
  if (D < 1 || D > 7 || n < 0) return ORC_INVALID_ARGUMENT;
  if (!(voxel > 0.0f) || !std::isfinite(voxel)) return ORC_INVALID_ARGUMENT;
  // Validation pass: the first offending row decides the status (ABI error contract).
  for (int64_t p = 0; p < n; ++p) {
    bool nonfinite = false, range = false;
    for (int d = 0; d < D; ++d) {
      float x = points[p * D + d];
      if (!std::isfinite(x)) { nonfinite = true; continue; }
      float q = std::floor(x / voxel);  // reading R6: IEEE fp32 division, then floor
      if (!(q >= -2147483648.0f && q < 2147483648.0f)) range = true;
    }
    if (nonfinite) { *err_row = p; return ORC_NONFINITE_INPUT; }
    if (batch && batch[p] < 0) { *err_row = p; return ORC_INVALID_ARGUMENT; }
    if (!range) {
      int64_t c[kMaxWords];
      for (int d = 0; d < D; ++d) c[d] = static_cast<int64_t>(std::floor(points[p * D + d] / voxel));
      range = !in_domain(c, D, batch ? batch[p] : 0);
    }
    if (range) { *err_row = p; return ORC_COORD_RANGE; }
  }
  // Alg. 1, serial form: C_p' <- floor(C_p / v_l); unique keys;
  // the first point of each key is kept (i_x of the reduction f, reading R9); rows are
  // numbered in first-occurrence order (reading R8).
  CoordMap map;
  map.reserve(static_cast<size_t>(n) * 2 + 1);
  int32_t next = 0;
  for (int64_t p = 0; p < n; ++p) {
    Key k{};
    for (int d = 0; d < D; ++d) k[d] = static_cast<int32_t>(std::floor(points[p * D + d] / voxel));
    k[D] = batch ? batch[p] : 0;
    auto it = map.find(k);
    int32_t row;
    if (it == map.end()) {
      row = next++;
      map.emplace(k, row);
      for (int d = 0; d <= D; ++d) coords_out[(int64_t)row * (D + 1) + d] = k[d];
      if (first_point) first_point[row] = static_cast<int32_t>(p);
    } else {
      row = it->second;
    }
    if (point_to_row) point_to_row[p] = row;
  }
  *n_out = next;
  return ORC_OK;
}

int orc_create(const int32_t* coords, int64_t n, int32_t D, const int32_t* tensor_stride,
               int32_t* coords_out, int32_t* inverse, int64_t* n_out, int64_t* err_row) {
  *err_row = -1;
  *n_out = 0;
  if (D < 1 || D > 7 || n < 0) return ORC_INVALID_ARGUMENT;
  for (int d = 0; d < D; ++d)
    if (tensor_stride && tensor_stride[d] < 1) return ORC_INVALID_ARGUMENT;
  for (int64_t p = 0; p < n; ++p) {
    const int32_t* r = coords + p * (D + 1);
    for (int d = 0; d < D; ++d) {
      int32_t s = tensor_stride ? tensor_stride[d] : 1;
      // Every coordinate is a multiple of the tensor stride ("minimum distance").
      if (r[d] % s != 0) { *err_row = p; return ORC_STRIDE; }
    }
    if (r[D] < 0) { *err_row = p; return ORC_INVALID_ARGUMENT; }
    int64_t c[kMaxWords];
    for (int d = 0; d < D; ++d) c[d] = r[d];
    if (!in_domain(c, D, r[D])) { *err_row = p; return ORC_COORD_RANGE; }
  }
  CoordMap map;
  map.reserve(static_cast<size_t>(n) * 2 + 1);
  int32_t next = 0;
  for (int64_t p = 0; p < n; ++p) {
    Key k = row_key(coords + p * (D + 1), D);
    auto it = map.find(k);
    int32_t row;
    if (it == map.end()) {
      row = next++;
      map.emplace(k, row);
      for (int d = 0; d <= D; ++d) coords_out[(int64_t)row * (D + 1) + d] = k[d];
    } else {
      row = it->second;
    }
    if (inverse) inverse[p] = row;
  }
  *n_out = next;
  return ORC_OK;
}

int orc_stride(const int32_t* coords, int64_t n, int32_t D, const int32_t* tensor_stride,
               const int32_t* conv_stride, int32_t* coords_out, int64_t* n_out, int64_t* err_row) {
  *err_row = -1;
  *n_out = 0;
  if (D < 1 || D > 7 || n < 0) return ORC_INVALID_ARGUMENT;
  int64_t s_out[kMaxWords];
  for (int d = 0; d < D; ++d) {
    int64_t ts = tensor_stride ? tensor_stride[d] : 1;
    int64_t cs = conv_stride ? conv_stride[d] : 1;
    if (ts < 1 || cs < 1) return ORC_INVALID_ARGUMENT;
    s_out[d] = ts * cs;  // s_out = s_in * sigma (reading R11)
    if (s_out[d] > INT32_MAX) return ORC_COORD_RANGE;
  }
  // u' = floor_div(u, s_out) * s_out per spatial axis, batch unchanged; first occurrence.
  CoordMap map;
  map.reserve(static_cast<size_t>(n) * 2 + 1);
  int32_t next = 0;
  for (int64_t p = 0; p < n; ++p) {
    const int32_t* r = coords + p * (D + 1);
    Key k{};
    for (int d = 0; d < D; ++d) {
      int64_t v = floor_div(r[d], s_out[d]) * s_out[d];
      if (!fits_i32(v)) { *err_row = p; return ORC_COORD_RANGE; }
      k[d] = static_cast<int32_t>(v);
    }
    k[D] = r[D];
    if (map.find(k) == map.end()) {
      int32_t row = next++;
      map.emplace(k, row);
      for (int d = 0; d <= D; ++d) coords_out[(int64_t)row * (D + 1) + d] = k[d];
    }
  }
  *n_out = next;
  return ORC_OK;
}

int orc_expand(const int32_t* coords, int64_t n, int32_t D, const int32_t* offsets, int32_t K,
               const int32_t* scale, int32_t* coords_out, int64_t* n_out, int64_t* err_row) {
  *err_row = -1;
  *n_out = 0;
  if (D < 1 || D > 7 || n < 0 || K < 1) return ORC_INVALID_ARGUMENT;
  // every u + i * scale (the output coordinates of a transposed conv may be any set;
  // the generative one is the union of the input rows' receptive fields), batch unchanged,
  // first occurrence in (row, offset) order
  CoordMap map;
  map.reserve(static_cast<size_t>(n) * K * 2 + 1);
  int32_t next = 0;
  for (int64_t p = 0; p < n; ++p) {
    const int32_t* r = coords + p * (D + 1);
    for (int32_t k = 0; k < K; ++k) {
      Key key{};
      for (int d = 0; d < D; ++d) {
        const int64_t v = (int64_t)r[d] + (int64_t)offsets[k * D + d] * (scale ? scale[d] : 1);
        if (!fits_i32(v)) { *err_row = p; return ORC_COORD_RANGE; }
        key[d] = static_cast<int32_t>(v);
      }
      key[D] = r[D];
      if (map.find(key) == map.end()) {
        const int32_t row = next++;
        map.emplace(key, row);
        for (int d = 0; d <= D; ++d) coords_out[(int64_t)row * (D + 1) + d] = key[d];
      }
    }
  }
  *n_out = next;
  return ORC_OK;
}

int orc_region(int32_t type, int32_t D, const int32_t* size, const int32_t* dilation,
               int32_t temporal_axis, const int32_t* custom, int32_t n_custom,
               int32_t* offsets, int32_t* K) {
  *K = 0;
  if (D < 1 || D > 7) return ORC_INVALID_ARGUMENT;
  std::vector<std::vector<int32_t>> list;
  if (type == ORC_CUSTOM) {
    // Arbitrary N^D: the caller's list, in the caller's order, taken literally.
    if (!custom || n_custom < 1) return ORC_INVALID_ARGUMENT;
    for (int32_t i = 0; i < n_custom; ++i) {
      std::vector<int32_t> o(custom + (int64_t)i * D, custom + (int64_t)(i + 1) * D);
      if (std::find(list.begin(), list.end(), o) != list.end()) return ORC_INVALID_ARGUMENT;
      list.push_back(o);
    }
  } else {
    if (!size) return ORC_INVALID_ARGUMENT;
    for (int d = 0; d < D; ++d) {
      if (size[d] < 1) return ORC_INVALID_ARGUMENT;
      if (dilation && dilation[d] < 1) return ORC_INVALID_ARGUMENT;
    }
    auto dil = [&](int d) { return dilation ? dilation[d] : 1; };
    if (type == ORC_HYPERCUBE) {
      // V^D(K) = product of per-axis ranges (Eq. 2); tesseract for D=4.
      std::vector<int32_t> cur(D, 0);
      std::vector<std::vector<int32_t>> ranges;
      for (int d = 0; d < D; ++d) ranges.push_back(axis_range(size[d]));
      std::vector<size_t> idx(D, 0);
      while (true) {
        std::vector<int32_t> o(D);
        for (int d = 0; d < D; ++d) o[d] = ranges[d][idx[d]] * dil(d);
        list.push_back(o);
        int d = D - 1;  // odometer, last axis fastest => axis 0 most significant (R2)
        while (d >= 0 && ++idx[d] == ranges[d].size()) { idx[d] = 0; --d; }
        if (d < 0) break;
      }
    } else if (type == ORC_HYPERCROSS) {
      // Cross / hypercross (Fig. 3): origin plus axis-aligned offsets.
      list.push_back(std::vector<int32_t>(D, 0));
      for (int d = 0; d < D; ++d)
        for (int32_t i : axis_range(size[d]))
          if (i != 0) {
            std::vector<int32_t> o(D, 0);
            o[d] = i * dil(d);
            list.push_back(o);
          }
      std::sort(list.begin(), list.end());
    } else if (type == ORC_HYBRID) {
      // Hybrid kernel (reading R4): spatial cube at temporal offset 0, union a
      // cross along the temporal axis only.
      int t = temporal_axis < 0 ? D - 1 : temporal_axis;
      if (t >= D) return ORC_INVALID_ARGUMENT;
      std::vector<std::vector<int32_t>> ranges;
      for (int d = 0; d < D; ++d) ranges.push_back(d == t ? std::vector<int32_t>{0} : axis_range(size[d]));
      std::vector<size_t> idx(D, 0);
      while (true) {
        std::vector<int32_t> o(D);
        for (int d = 0; d < D; ++d) o[d] = ranges[d][idx[d]] * dil(d);
        list.push_back(o);
        int d = D - 1;
        while (d >= 0 && ++idx[d] == ranges[d].size()) { idx[d] = 0; --d; }
        if (d < 0) break;
      }
      for (int32_t i : axis_range(size[t]))
        if (i != 0) {
          std::vector<int32_t> o(D, 0);
          o[t] = i * dil(t);
          list.push_back(o);
        }
      std::sort(list.begin(), list.end());
    } else {
      return ORC_INVALID_ARGUMENT;
    }
  }
  *K = static_cast<int32_t>(list.size());
  if (offsets)
    for (size_t i = 0; i < list.size(); ++i)
      for (int d = 0; d < D; ++d) offsets[i * D + d] = list[i][d];
  return ORC_OK;
}

int orc_labels(const int32_t* point_to_row, const int32_t* labels, int64_t n_points, int64_t n_rows,
               int32_t ignore_label, int32_t* row_labels) {
  // Alg. 1 lines 5-6 reduce the (label, index) pairs of equal keys with f of
  // P:181; folded here in input order, one point at a time.
  std::vector<char> seen(static_cast<size_t>(n_rows), 0);
  for (int64_t p = 0; p < n_points; ++p) {
    const int32_t r = point_to_row[p];
    if (r < 0 || r >= n_rows) return ORC_INVALID_ARGUMENT;
    if (!seen[r]) {
      seen[r] = 1;
      row_labels[r] = labels[p];                      // (l_x, i_x): the first point
    } else if (row_labels[r] != labels[p]) {
      row_labels[r] = ignore_label;                   // f: l_x != l_y -> IGNORE_LABEL
    }
  }
  for (int64_t r = 0; r < n_rows; ++r)
    if (!seen[r]) return ORC_INVALID_ARGUMENT;        // every voxel has at least one point
  return ORC_OK;
}

int orc_lookup(const int32_t* coords, int64_t n, int32_t D, const int32_t* queries, int64_t q,
               int32_t* rows) {
  if (D < 1 || D > 7) return ORC_INVALID_ARGUMENT;
  CoordMap map;
  map.reserve(static_cast<size_t>(n) * 2 + 1);
  for (int64_t r = 0; r < n; ++r) map.emplace(row_key(coords + r * (D + 1), D), static_cast<int32_t>(r));
  for (int64_t i = 0; i < q; ++i) {
    auto it = map.find(row_key(queries + i * (D + 1), D));
    rows[i] = it == map.end() ? -1 : it->second;
  }
  return ORC_OK;
}

int orc_kmap(const int32_t* c_in, int64_t n_in, const int32_t* c_out, int64_t n_out, int32_t D,
             const int32_t* offsets, int32_t K, const int32_t* scale, int32_t transposed,
             int64_t* ptr, int32_t* in_idx, int32_t* out_idx) {
  if (D < 1 || D > 7 || K < 1) return ORC_INVALID_ARGUMENT;
  CoordMap map;
  map.reserve(static_cast<size_t>(n_in) * 2 + 1);
  for (int64_t r = 0; r < n_in; ++r) map.emplace(row_key(c_in + r * (D + 1), D), static_cast<int32_t>(r));
  const int64_t sign = transposed ? -1 : 1;
  // Eq. 3: for u in C_out and i in N^D, u + i in C_in contributes W_i x_{u+i}.
  // Offsets are scaled by the fine tensor stride (reading R14); transposed maps reverse the
  // roles of input and output (reading R13).  Output-ascending inside each offset.
  // The lookups of one offset are independent (optional OpenMP over o); the pairs are then
  // appended serially in output order.
  int64_t count = 0;
  ptr[0] = 0;
  std::vector<int32_t> hit(static_cast<size_t>(n_out));
  for (int32_t k = 0; k < K; ++k) {
#pragma omp parallel for schedule(static)
    for (int64_t o = 0; o < n_out; ++o) {
      const int32_t* u = c_out + o * (D + 1);
      Key q{};
      bool ok = true;
      for (int d = 0; d < D; ++d) {
        int64_t v = (int64_t)u[d] + sign * (int64_t)offsets[k * D + d] * (scale ? scale[d] : 1);
        if (!fits_i32(v)) { ok = false; break; }
        q[d] = static_cast<int32_t>(v);
      }
      hit[o] = -1;
      if (!ok) continue;
      q[D] = u[D];  // batch index is never offset (reading R18)
      auto it = map.find(q);
      if (it != map.end()) hit[o] = it->second;
    }
    for (int64_t o = 0; o < n_out; ++o) {
      if (hit[o] < 0) continue;
      if (in_idx) {
        in_idx[count] = hit[o];
        out_idx[count] = static_cast<int32_t>(o);
      }
      ++count;
    }
    ptr[k + 1] = count;
  }
  return ORC_OK;
}

void orc_conv_forward(const int64_t* ptr, const int32_t* in_idx, const int32_t* out_idx, int32_t K,
                      const double* f_in, int32_t c_in, const double* W, double* f_out,
                      int64_t n_out, int32_t c_out) {
  // Alg. 2 line 1: F^o <- 0.
  std::fill(f_out, f_out + n_out * c_out, 0.0);
  // Alg. 2 lines 2-5: for each offset, gather, multiply by W_i, add-and-scatter.  Within one
  // offset the outputs O_i are distinct, so the optional OpenMP split over the pairs
  // of an offset is race-free and gives bit-identical results.
  for (int32_t k = 0; k < K; ++k) {
    const double* Wk = W + (int64_t)k * c_out * c_in;
#pragma omp parallel for schedule(static)
    for (int64_t p = ptr[k]; p < ptr[k + 1]; ++p) {
      const double* x = f_in + (int64_t)in_idx[p] * c_in;
      double* y = f_out + (int64_t)out_idx[p] * c_out;
      for (int32_t co = 0; co < c_out; ++co) {
        double acc = 0.0;
        for (int32_t ci = 0; ci < c_in; ++ci) acc += Wk[(int64_t)co * c_in + ci] * x[ci];
        y[co] += acc;
      }
    }
  }
}

void orc_conv_forward_rows(const int64_t* ptr, const int32_t* in_idx, const int32_t* out_idx,
                           int32_t K, const double* f_in, int32_t c_in, const double* W,
                           int32_t c_out, const int32_t* rows, int64_t n_rows, double* f_rows) {
  // Eq. 3 evaluated at the selected outputs u: sum over offsets i with u+i in C_in.
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t r = 0; r < n_rows; ++r) {
    double* y = f_rows + r * c_out;
    std::fill(y, y + c_out, 0.0);
    for (int32_t k = 0; k < K; ++k) {
      // Pairs are output-ascending inside an offset: binary search the row.
      const int32_t* lo = out_idx + ptr[k];
      const int32_t* hi = out_idx + ptr[k + 1];
      const int32_t* it = std::lower_bound(lo, hi, rows[r]);
      if (it == hi || *it != rows[r]) continue;
      const double* x = f_in + (int64_t)in_idx[it - out_idx] * c_in;
      const double* Wk = W + (int64_t)k * c_out * c_in;
      for (int32_t co = 0; co < c_out; ++co) {
        double acc = 0.0;
        for (int32_t ci = 0; ci < c_in; ++ci) acc += Wk[(int64_t)co * c_in + ci] * x[ci];
        y[co] += acc;
      }
    }
  }
}

void orc_conv_dgrad(const int64_t* ptr, const int32_t* in_idx, const int32_t* out_idx, int32_t K,
                    const double* g_out, int32_t c_out, const double* W, double* g_in,
                    int64_t n_in, int32_t c_in) {
  std::fill(g_in, g_in + n_in * c_in, 0.0);
  // Within one offset the inputs I_i are distinct: the optional OpenMP split is race-free.
  for (int32_t k = 0; k < K; ++k) {
    const double* Wk = W + (int64_t)k * c_out * c_in;
#pragma omp parallel for schedule(static)
    for (int64_t p = ptr[k]; p < ptr[k + 1]; ++p) {
      const double* g = g_out + (int64_t)out_idx[p] * c_out;
      double* x = g_in + (int64_t)in_idx[p] * c_in;
      for (int32_t ci = 0; ci < c_in; ++ci) {
        double acc = 0.0;
        for (int32_t co = 0; co < c_out; ++co) acc += Wk[(int64_t)co * c_in + ci] * g[co];
        x[ci] += acc;
      }
    }
  }
}

void orc_conv_wgrad(const int64_t* ptr, const int32_t* in_idx, const int32_t* out_idx, int32_t K,
                    const double* g_out, int32_t c_out, const double* f_in, int32_t c_in,
                    double* dW) {
  for (int32_t k = 0; k < K; ++k) {
    double* dWk = dW + (int64_t)k * c_out * c_in;
    std::fill(dWk, dWk + (int64_t)c_out * c_in, 0.0);
    // Optional OpenMP over the rows co of dW_k: every element still sums the pairs in order.
#pragma omp parallel for schedule(static)
    for (int32_t co = 0; co < c_out; ++co)
      for (int64_t p = ptr[k]; p < ptr[k + 1]; ++p) {
        const double g = g_out[(int64_t)out_idx[p] * c_out + co];
        const double* x = f_in + (int64_t)in_idx[p] * c_in;
        for (int32_t ci = 0; ci < c_in; ++ci) dWk[(int64_t)co * c_in + ci] += g * x[ci];
      }
  }
}

int orc_kmap_reverse(const int64_t* ptr, const int32_t* in_idx, const int32_t* out_idx, int32_t K,
                     int64_t* rptr, int32_t* rin, int32_t* rout) {
  // the map of the reverse direction has the roles of input and output exchanged:
  // pair (a, o) of offset k becomes (o, a), listed output-ascending, i.e. by a.
  rptr[0] = 0;
  for (int32_t k = 0; k < K; ++k) {
    std::vector<std::pair<int32_t, int32_t>> pairs;
    for (int64_t p = ptr[k]; p < ptr[k + 1]; ++p) pairs.emplace_back(in_idx[p], out_idx[p]);
    std::sort(pairs.begin(), pairs.end());
    int64_t q = ptr[k];
    for (const auto& pr : pairs) {
      rout[q] = pr.first;  // the former input row is the new output
      rin[q] = pr.second;
      ++q;
    }
    rptr[k + 1] = ptr[k + 1];
  }
  return ORC_OK;
}

int orc_set_threads(int32_t n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
  return omp_get_max_threads();
#else
  (void)n;
  return 1;
#endif
}

}  // extern "C"

// f2 — pooling.  The inputs of output o are visited in concatenated order:
// offset k ascending (each offset contributes at most one pair per output).
void orc_pool_forward(const int64_t* ptr, const int32_t* in_idx, const int32_t* out_idx, int32_t K,
                      const double* f_in, int32_t C, int64_t n_out, int32_t mode, double* f_out,
                      int32_t* argmax) {
  std::vector<int64_t> cnt(static_cast<size_t>(n_out), 0);
  std::fill(f_out, f_out + n_out * C, 0.0);
  if (mode == ORC_POOL_MAX && argmax) std::fill(argmax, argmax + n_out * C, -1);
  for (int32_t k = 0; k < K; ++k) {
    for (int64_t p = ptr[k]; p < ptr[k + 1]; ++p) {
      const int32_t a = in_idx[p], o = out_idx[p];
      const double* x = f_in + (int64_t)a * C;
      double* y = f_out + (int64_t)o * C;
      for (int32_t c = 0; c < C; ++c) {
        if (mode == ORC_POOL_MAX) {
          // MaxPoolKernel (Alg. 3): the first input sets the value, a later one replaces it
          // only when strictly larger (ties: lowest concatenated index)
          if (cnt[o] == 0 || x[c] > y[c]) {
            y[c] = x[c];
            if (argmax) argmax[(int64_t)o * C + c] = a;
          }
        } else {
          y[c] += x[c];  // cusparse_csrmm(S_M, F) of Alg. 4
        }
      }
      ++cnt[o];
    }
  }
  if (mode == ORC_POOL_AVG)
    for (int64_t o = 0; o < n_out; ++o)
      if (cnt[o] > 0)
        for (int32_t c = 0; c < C; ++c) f_out[o * C + c] /= static_cast<double>(cnt[o]);  // F' / N
}

void orc_pool_backward(const int64_t* ptr, const int32_t* in_idx, const int32_t* out_idx, int32_t K,
                       const double* g_out, int32_t C, int64_t n_out, int32_t mode, const int32_t* argmax,
                       double* g_in, int64_t n_in) {
  std::fill(g_in, g_in + n_in * C, 0.0);
  if (mode == ORC_POOL_MAX) {
    for (int64_t o = 0; o < n_out; ++o)
      for (int32_t c = 0; c < C; ++c) {
        const int32_t a = argmax[o * C + c];
        if (a >= 0) g_in[(int64_t)a * C + c] += g_out[o * C + c];
      }
    return;
  }
  std::vector<int64_t> cnt(static_cast<size_t>(n_out), 0);
  for (int32_t k = 0; k < K; ++k)
    for (int64_t p = ptr[k]; p < ptr[k + 1]; ++p) ++cnt[out_idx[p]];
  for (int32_t k = 0; k < K; ++k)
    for (int64_t p = ptr[k]; p < ptr[k + 1]; ++p) {
      const int32_t a = in_idx[p], o = out_idx[p];
      const double s = mode == ORC_POOL_AVG ? 1.0 / static_cast<double>(cnt[o]) : 1.0;
      for (int32_t c = 0; c < C; ++c) g_in[(int64_t)a * C + c] += s * g_out[(int64_t)o * C + c];
    }
}

void orc_global_pool(const int32_t* batch, int64_t n, const double* f_in, int32_t C, int32_t n_batch,
                     int32_t mode, double* f_out) {
  std::vector<int64_t> cnt(static_cast<size_t>(n_batch), 0);
  std::fill(f_out, f_out + (int64_t)n_batch * C, 0.0);
  for (int64_t r = 0; r < n; ++r) {
    const int32_t b = batch[r];
    for (int32_t c = 0; c < C; ++c) f_out[(int64_t)b * C + c] += f_in[r * C + c];
    ++cnt[b];
  }
  if (mode == ORC_POOL_AVG)
    for (int32_t b = 0; b < n_batch; ++b)
      if (cnt[b] > 0)
        for (int32_t c = 0; c < C; ++c) f_out[(int64_t)b * C + c] /= static_cast<double>(cnt[b]);
}

// f3 — Alg. 5 written out: softmax of the unary logits, then N rounds of
// "sparse conv of Q with phi_p, add phi_u, softmax".
namespace {
void softmax_rows(const double* a, const double* b, int64_t n, int32_t C, double* out) {
  for (int64_t i = 0; i < n; ++i) {
    double m = -1e300;
    for (int32_t c = 0; c < C; ++c) m = std::max(m, a[i * C + c] + (b ? b[i * C + c] : 0.0));
    double z = 0.0;
    for (int32_t c = 0; c < C; ++c) {
      out[i * C + c] = std::exp(a[i * C + c] + (b ? b[i * C + c] : 0.0) - m);
      z += out[i * C + c];
    }
    for (int32_t c = 0; c < C; ++c) out[i * C + c] /= z;
  }
}
}  // namespace

void orc_crf_infer(const int64_t* ptr, const int32_t* in_idx, const int32_t* out_idx, int32_t K,
                   const double* phi_u, int64_t n, int32_t C, const double* W, int32_t n_iters, double* q) {
  std::vector<double> qt(static_cast<size_t>(n) * C), prev(static_cast<size_t>(n) * C);
  softmax_rows(phi_u, nullptr, n, C, q);                                  // Q^0
  for (int32_t it = 0; it < n_iters; ++it) {
    std::copy(q, q + n * C, prev.begin());
    orc_conv_forward(ptr, in_idx, out_idx, K, prev.data(), C, W, qt.data(), n, C);  // Q~^n
    softmax_rows(phi_u, qt.data(), n, C, q);                              // Q^n
  }
}
