// Descriptor planner for the B200 xGETT: validation with the reference's coded
// errors, then mode folding into M (A-free), N (B-free) and K (paired) groups.
//
// Reference behaviour restated here (file:line under /root/reference/pkg/src/gett):
//   validate            plan.py:162-234 (+ _check_cont_indices :130-147,
//                       _check_footprint :150-159, output_view_errors :237-241)
//   footprint           layout.py:108-125
//   derive_output_ext.  plan.py:119-127
//   _plan_tables        plan.py:258-289 (replaced by the M/N/K groups below)
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace gett {

struct View {
  int rank = 0;
  const int64_t* ext = nullptr;
  const int64_t* inc = nullptr;
  int64_t off = 0;
  int64_t len = 0;
};

struct Spec {
  int conts = 0;
  const int64_t* cont_a = nullptr;
  const int64_t* cont_b = nullptr;
  int perm_len = 0;
  const int64_t* perm = nullptr;
  int inc_c_len = 0;
  const int64_t* inc_c = nullptr;
};

struct Error {
  int32_t code;
  int64_t info[6];
};

// How the output view takes part in validation:
//   None     plan.validate(a, b, spec, inc_c)                 (plan.py:162-234)
//   Explicit plan.validate(..., c_view): C's NegativeExtent after A/B's and
//            its footprint after A/B's, in the same pass        (plan.py:179-232)
//   Derived  _gett's two phases: C = (derived extents, inc_c, off, len),
//            footprint-checked only when phase 1 is clean       (kernel.py:146-153)
enum class CMode { None = 0, Derived = 1, Explicit = 2 };

std::vector<Error> validate(const View& a, const View& b, const Spec& s, CMode c_mode,
                            const View& c);

// (lo, hi) footprint relative to base offset (layout.py:108-125).
void footprint(int rank, const int64_t* ext, const int64_t* inc, int64_t* lo, int64_t* hi);

// A folded mode group: G = e_in * |T|.  Element g has offset
//   T[t][g / e_in] + (g % e_in) * s_in[t]   in tensor t (two tensors per group).
struct Group {
  int64_t G = 1;
  int64_t e_in = 1;
  int64_t s_in[2] = {0, 0};
  std::vector<int64_t> T[2];  // outer offset tables, size G / e_in (>= 1)
  int nmodes = 0;             // merged modes (incl. inner) with extent > 1
};

// Which kernel family runs a plan.
enum class KernelKind { None, Ref, Tiled, Serial };

struct Plan {
  int rank_c = 0;
  std::vector<int64_t> ext_c;
  int64_t size_free = 1, size_cont = 1;
  bool swapped = false;  // operand roles exchanged: M group from B, N group from A
  // groups in kernel roles: gm over (A', C), gn over (B', C), gk over (A', B'),
  // where A' = swapped ? B : A.
  Group gm, gn, gk;
  Group gk_ref;          // K in reference order (pair 0 fastest) over (A', B')
  bool c_may_alias = false;  // distinct output coordinates may share a C element
  // footprints (lowest, highest offset relative to each view's base offset);
  // offsets are not part of the plan, so callers add their own
  int64_t fp_lo[3] = {0, 0, 0}, fp_hi[3] = {0, 0, 0};
};

// Build the plan for validated arguments.
Plan build_plan(const View& a, const View& b, const Spec& s, int64_t off_c, int64_t len_c);

// A single view folded as one group (tensor 1 unused): zero_view's layout.
Group fold_view(int rank, const int64_t* ext, const int64_t* inc);

// Key used to cache device-side tables.
std::string plan_key(char dtype, const View& a, const View& b, const Spec& s, int64_t off_c);

}  // namespace gett
