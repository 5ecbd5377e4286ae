// Descriptor planner: validation (reference error codes, reference order) and
// the fold of EXT/INC/CONT/PERM into M/N/K mode groups.  See planner.hpp.
#include "planner.hpp"

#include <algorithm>
#include <cstdlib>
#include <numeric>
#include <sstream>

#include "../../include/gett_b200.h"

namespace gett {

namespace {

Error make_err(int32_t code, int64_t i0 = 0, int64_t i1 = 0, int64_t i2 = 0, int64_t i3 = 0,
               int64_t i4 = 0, int64_t i5 = 0) {
  Error e;
  e.code = code;
  e.info[0] = i0; e.info[1] = i1; e.info[2] = i2; e.info[3] = i3; e.info[4] = i4; e.info[5] = i5;
  return e;
}

// plan.py:130-147
bool check_cont_indices(int tensor, const int64_t* idx, int conts, int rank,
                        std::vector<Error>& errs) {
  bool ok = true;
  std::vector<int64_t> seen;
  for (int k = 0; k < conts; ++k) {
    int64_t d = idx[k];
    if (!(0 <= d && d < rank)) {
      errs.push_back(make_err(GETT_CONT_INDEX_OUT_OF_RANGE, tensor, k, d, rank));
      ok = false;
    } else if (std::find(seen.begin(), seen.end(), d) != seen.end()) {
      errs.push_back(make_err(GETT_CONT_INDEX_DUPLICATE, tensor, k, d));
      ok = false;
    }
    seen.push_back(d);
  }
  return ok;
}

bool is_empty(int rank, const int64_t* ext) {
  for (int d = 0; d < rank; ++d)
    if (ext[d] == 0) return true;
  return false;
}

// plan.py:150-159
void check_footprint(int tensor, int rank, const int64_t* ext, const int64_t* inc, int64_t off,
                     int64_t len, std::vector<Error>& errs) {
  if (is_empty(rank, ext)) return;
  int64_t lo, hi;
  footprint(rank, ext, inc, &lo, &hi);
  if (off + lo < 0 || off + hi >= len)
    errs.push_back(make_err(GETT_FOOTPRINT_OUT_OF_BOUNDS, tensor, off + lo, off + hi, len));
}

bool contains(const int64_t* idx, int n, int64_t d) {
  for (int k = 0; k < n; ++k)
    if (idx[k] == d) return true;
  return false;
}

struct Mode {
  int64_t e;
  int64_t s[2];
};

// Merge adjacent modes (inner -> outer) whose strides compose in both tensors,
// then lay the group out as inner affine mode + outer offset table.
Group fold(std::vector<Mode> modes) {
  Group g;
  std::vector<Mode> merged;
  for (const Mode& m : modes) {
    if (m.e == 1) continue;
    if (!merged.empty()) {
      Mode& cur = merged.back();
      if (m.s[0] == cur.s[0] * cur.e && m.s[1] == cur.s[1] * cur.e) {
        cur.e *= m.e;
        continue;
      }
    }
    merged.push_back(m);
  }
  g.nmodes = (int)merged.size();
  g.G = 1;
  for (const Mode& m : merged) g.G *= m.e;
  if (merged.empty()) {
    g.e_in = 1;
    g.s_in[0] = g.s_in[1] = 0;
    g.T[0].assign(1, 0);
    g.T[1].assign(1, 0);
    return g;
  }
  g.e_in = merged[0].e;
  g.s_in[0] = merged[0].s[0];
  g.s_in[1] = merged[0].s[1];
  int64_t n_outer = g.G / g.e_in;
  for (int t = 0; t < 2; ++t) g.T[t].assign(n_outer, 0);
  // enumerate outer coordinates, first outer mode fastest
  std::vector<int64_t> coord(merged.size(), 0);
  int64_t o0 = 0, o1 = 0;
  for (int64_t i = 0; i < n_outer; ++i) {
    g.T[0][i] = o0;
    g.T[1][i] = o1;
    for (size_t j = 1; j < merged.size(); ++j) {
      coord[j] += 1;
      o0 += merged[j].s[0];
      o1 += merged[j].s[1];
      if (coord[j] < merged[j].e) break;
      o0 -= merged[j].s[0] * merged[j].e;
      o1 -= merged[j].s[1] * merged[j].e;
      coord[j] = 0;
    }
  }
  return g;
}

void sort_by(std::vector<Mode>& modes, int t) {
  std::stable_sort(modes.begin(), modes.end(), [t](const Mode& x, const Mode& y) {
    return std::llabs(x.s[t]) < std::llabs(y.s[t]);
  });
}

int64_t min_abs_stride(const std::vector<Mode>& modes, int t) {
  int64_t best = INT64_MAX;
  for (const Mode& m : modes)
    if (m.e > 1) best = std::min<int64_t>(best, std::llabs(m.s[t]));
  return best;
}

}  // namespace

void footprint(int rank, const int64_t* ext, const int64_t* inc, int64_t* lo, int64_t* hi) {
  int64_t l = 0, h = 0;
  for (int d = 0; d < rank; ++d) {
    if (ext[d] <= 0) continue;
    int64_t span = inc[d] * (ext[d] - 1);
    if (span < 0) l += span;
    else h += span;
  }
  *lo = l;
  *hi = h;
}

std::vector<Error> validate(const View& a, const View& b, const Spec& s, CMode c_mode,
                            const View& c) {
  std::vector<Error> errs;
  // NegativeExtent, A then B (then an explicit C view) (plan.py:179-184)
  for (int d = 0; d < a.rank; ++d)
    if (a.ext[d] < 0) errs.push_back(make_err(GETT_NEGATIVE_EXTENT, 0, d, a.ext[d]));
  for (int d = 0; d < b.rank; ++d)
    if (b.ext[d] < 0) errs.push_back(make_err(GETT_NEGATIVE_EXTENT, 1, d, b.ext[d]));
  if (c_mode == CMode::Explicit)
    for (int d = 0; d < c.rank; ++d)
      if (c.ext[d] < 0) errs.push_back(make_err(GETT_NEGATIVE_EXTENT, 2, d, c.ext[d]));
  // contracted indices, then extent agreement (plan.py:186-195)
  bool a_ok = check_cont_indices(0, s.cont_a, s.conts, a.rank, errs);
  bool b_ok = check_cont_indices(1, s.cont_b, s.conts, b.rank, errs);
  if (a_ok && b_ok) {
    for (int k = 0; k < s.conts; ++k) {
      int64_t da = s.cont_a[k], db = s.cont_b[k];
      if (a.ext[da] != b.ext[db])
        errs.push_back(make_err(GETT_EXTENT_MISMATCH, -1, k, a.ext[da], da, b.ext[db], db));
    }
  }
  // perm (plan.py:197-210)
  int64_t rank_c = (int64_t)a.rank + b.rank - 2 * (int64_t)s.conts;
  bool perm_ok = true;
  if (s.perm_len != rank_c) {
    errs.push_back(make_err(GETT_PERM_LENGTH_WRONG, -1, s.perm_len, rank_c));
    perm_ok = false;
  } else {
    std::vector<int64_t> p(s.perm, s.perm + s.perm_len);
    std::sort(p.begin(), p.end());
    for (int64_t i = 0; i < rank_c; ++i)
      if (p[i] != i) {
        perm_ok = false;
        break;
      }
    if (!perm_ok) errs.push_back(make_err(GETT_PERM_NOT_BIJECTION, -1, rank_c));
  }
  // inc_c length (plan.py:212-218)
  bool inc_ok = true;
  if (s.inc_c_len != rank_c) {
    errs.push_back(make_err(GETT_INC_C_LENGTH_WRONG, -1, s.inc_c_len, rank_c));
    inc_ok = false;
  }
  // zero output increments over extents > 1 (plan.py:220-227)
  std::vector<int64_t> ext_c;
  if (a_ok && b_ok && perm_ok && inc_ok) {
    ext_c.assign(rank_c, 0);
    int i = 0;
    for (int d = 0; d < a.rank; ++d)
      if (!contains(s.cont_a, s.conts, d)) ext_c[s.perm[i++]] = a.ext[d];
    for (int d = 0; d < b.rank; ++d)
      if (!contains(s.cont_b, s.conts, d)) ext_c[s.perm[i++]] = b.ext[d];
    for (int64_t d = 0; d < rank_c; ++d)
      if (s.inc_c[d] == 0 && ext_c[d] > 1)
        errs.push_back(make_err(GETT_OUTPUT_WRITE_ALIASING, 2, d, ext_c[d]));
  }
  // footprints A, B (plan.py:229-230)
  check_footprint(0, a.rank, a.ext, a.inc, a.off, a.len, errs);
  check_footprint(1, b.rank, b.ext, b.inc, b.off, b.len, errs);
  // explicit c_view: footprint in the same pass (plan.py:231-232)
  if (c_mode == CMode::Explicit) check_footprint(2, c.rank, c.ext, c.inc, c.off, c.len, errs);
  // phase 2: derived C view, only when everything else passed (kernel.py:146-153)
  if (c_mode == CMode::Derived && errs.empty())
    check_footprint(2, (int)rank_c, ext_c.data(), s.inc_c, c.off, c.len, errs);
  return errs;
}

Plan build_plan(const View& a, const View& b, const Spec& s, int64_t off_c, int64_t len_c) {
  (void)len_c;
  Plan p;
  p.rank_c = a.rank + b.rank - 2 * s.conts;
  p.ext_c.assign(p.rank_c, 0);
  std::vector<Mode> mg, ng, kg;
  int i = 0;
  for (int d = 0; d < a.rank; ++d) {
    if (contains(s.cont_a, s.conts, d)) continue;
    int64_t q = s.perm[i++];
    p.ext_c[q] = a.ext[d];
    mg.push_back({a.ext[d], {a.inc[d], s.inc_c[q]}});
  }
  for (int d = 0; d < b.rank; ++d) {
    if (contains(s.cont_b, s.conts, d)) continue;
    int64_t q = s.perm[i++];
    p.ext_c[q] = b.ext[d];
    ng.push_back({b.ext[d], {b.inc[d], s.inc_c[q]}});
  }
  for (int k = 0; k < s.conts; ++k)
    kg.push_back({a.ext[s.cont_a[k]], {a.inc[s.cont_a[k]], b.inc[s.cont_b[k]]}});
  p.size_free = 1;
  for (int64_t e : p.ext_c) p.size_free *= e;
  p.size_cont = 1;
  for (const Mode& m : kg) p.size_cont *= m.e;

  // Role choice: C's smallest-stride mode should land in N (the kernel's
  // fast output dimension).  Swapping A and B is exact per element
  // (a*b == b*a) and keeps the K order, so results are unchanged
  // (commutativity, testkit.py:476-495).
  int64_t cm = min_abs_stride(mg, 1), cn = min_abs_stride(ng, 1);
  p.swapped = cm < cn;
  if (p.swapped) {
    std::swap(mg, ng);
    for (Mode& m : kg) std::swap(m.s[0], m.s[1]);
  }
  // reference-order K (pair 0 fastest), before any reordering
  p.gk_ref = fold(kg);
  // M ordered by A' stride, N by B' stride
  sort_by(mg, 0);
  sort_by(ng, 0);
  // K ordered by the operand that wants K-contiguous loads
  bool a_wants_k = min_abs_stride(kg, 0) < min_abs_stride(mg, 0);
  bool b_wants_k = min_abs_stride(kg, 1) < min_abs_stride(ng, 0);
  sort_by(kg, (a_wants_k || !b_wants_k) ? 0 : 1);
  p.gm = fold(mg);
  p.gn = fold(ng);
  p.gk = fold(kg);

  // Can two output coordinates address the same C element?  Sufficient
  // non-overlap test: sorted by |inc|, every stride exceeds the span of all
  // smaller ones.  Failing it routes the call to the serial kernel.
  {
    std::vector<std::pair<int64_t, int64_t>> dims;
    for (int d = 0; d < p.rank_c; ++d)
      if (p.ext_c[d] > 1) dims.push_back({std::llabs(s.inc_c[d]), p.ext_c[d]});
    std::sort(dims.begin(), dims.end());
    int64_t span = 0;
    for (auto& d : dims) {
      if (d.first <= span) {
        p.c_may_alias = true;
        break;
      }
      span += d.first * (d.second - 1);
    }
  }

  // spans
  int64_t lo, hi;
  footprint(a.rank, a.ext, a.inc, &lo, &hi);
  p.fp_lo[0] = lo; p.fp_hi[0] = hi;
  footprint(b.rank, b.ext, b.inc, &lo, &hi);
  p.fp_lo[1] = lo; p.fp_hi[1] = hi;
  footprint(p.rank_c, p.ext_c.data(), s.inc_c, &lo, &hi);
  p.fp_lo[2] = lo; p.fp_hi[2] = hi;
  return p;
}

Group fold_view(int rank, const int64_t* ext, const int64_t* inc) {
  std::vector<Mode> modes;
  for (int d = 0; d < rank; ++d) modes.push_back({ext[d], {inc[d], 0}});
  sort_by(modes, 0);
  return fold(modes);
}

std::string plan_key(char dtype, const View& a, const View& b, const Spec& s, int64_t off_c) {
  // Binary key (raw int64 words): the descriptor minus every offset.  One
  // allocation, no formatting — this runs on every call.
  (void)off_c;
  std::string k;
  k.reserve(8 * (4 + 2 * a.rank + 2 * b.rank + 2 * s.conts + s.perm_len + s.inc_c_len) + 1);
  auto put = [&](int64_t v) { k.append(reinterpret_cast<const char*>(&v), 8); };
  k.push_back(dtype);
  put(a.rank);
  for (int d = 0; d < a.rank; ++d) { put(a.ext[d]); put(a.inc[d]); }
  put(b.rank);
  for (int d = 0; d < b.rank; ++d) { put(b.ext[d]); put(b.inc[d]); }
  put(s.conts);
  for (int i = 0; i < s.conts; ++i) { put(s.cont_a[i]); put(s.cont_b[i]); }
  put(s.perm_len);
  for (int i = 0; i < s.perm_len; ++i) put(s.perm[i]);
  put(s.inc_c_len);
  for (int i = 0; i < s.inc_c_len; ++i) put(s.inc_c[i]);
  return k;
}

}  // namespace gett
