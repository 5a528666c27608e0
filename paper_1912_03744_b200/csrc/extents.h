// extents.h -- masked line extents of a pcgpu_desc (host).
//
// The reference's two-level Grid (geometry.hpp:72-74): row_extent(j) =
// j < nz_shared ? nr : nr_core, col_extent(i) = i < nr_core ? nz : nz_shared.
// A generalised stepped domain passes the arrays directly.
#pragma once

#include <string>
#include <vector>

#include "../../include/pcgpu.h"

namespace pcgpu {

inline std::vector<int> desc_row_extent(const pcgpu_desc* d) {
  std::vector<int> v(d->nz);
  for (int j = 0; j < d->nz; ++j)
    v[j] = d->row_extent && d->col_extent ? d->row_extent[j]
                                          : (j < d->nz_shared ? d->nr : d->nr_core);
  return v;
}

inline std::vector<int> desc_col_extent(const pcgpu_desc* d) {
  std::vector<int> v(d->nr);
  for (int i = 0; i < d->nr; ++i)
    v[i] = d->row_extent && d->col_extent ? d->col_extent[i]
                                          : (i < d->nr_core ? d->nz : d->nz_shared);
  return v;
}

// Prefix masks: non-increasing extents in range, i < row[j] iff j < col[i].
inline std::string check_extents(const pcgpu_desc* d) {
  if ((d->row_extent == nullptr) != (d->col_extent == nullptr))
    return "stepper: row_extent and col_extent must be given together";
  if (!d->row_extent) return "";
  const std::vector<int> row = desc_row_extent(d), col = desc_col_extent(d);
  for (int j = 0; j < d->nz; ++j) {
    if (row[j] < 1 || row[j] > d->nr) return "stepper: row_extent out of range";
    if (j > 0 && row[j] > row[j - 1]) return "stepper: row_extent must be non-increasing";
  }
  for (int i = 0; i < d->nr; ++i) {
    if (col[i] < 1 || col[i] > d->nz) return "stepper: col_extent out of range";
    if (i > 0 && col[i] > col[i - 1]) return "stepper: col_extent must be non-increasing";
    // consistency with the row extents
    const int j_last = col[i] - 1;
    if (row[j_last] <= i || (col[i] < d->nz && row[col[i]] > i))
      return "stepper: row_extent and col_extent disagree";
  }
  return "";
}

}  // namespace pcgpu
