/* A plain C caller of the drop-in C ABI (include/gett_b200.h), the way a
 * non-Python binding would use libgett_b200.so:
 *
 *   gcc -std=c99 -I include tools/abi_c_example.c -L paper_2410_06770_b200 \
 *       -lgett_b200 -Wl,-rpath,$PWD/paper_2410_06770_b200 -o abi_c_example
 *   ./abi_c_example validate   # coded validation errors (no GPU needed)
 *   ./abi_c_example run        # C += A.B through gett_dgett on host buffers (GPU)
 *
 * `validate`: a spec with a duplicated contracted index and a PERM of the
 * wrong length must come back as two coded errors in the reference's order
 * (plan.py:179-232) with C untouched.  `run`: a 3 x 4 x 5 contraction
 * (test_kernel.py-style, integer data so the result is exact) against a
 * triple loop.  Prints one line and exits 0 on success.
 */
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "gett_b200.h"

static int run_validate(void) {
  const int64_t ext_a[2] = {3, 4}, inc_a[2] = {4, 1};
  const int64_t ext_b[2] = {4, 5}, inc_b[2] = {5, 1};
  const int64_t cont_a[2] = {1, 1}, cont_b[2] = {0, 0}; /* duplicate index on A */
  const int64_t perm[1] = {0};                          /* output rank would be 2 */
  const int64_t inc_c[2] = {5, 1};
  double a[12] = {0}, b[20] = {0}, c[15];
  for (int i = 0; i < 15; ++i) c[i] = 7.0;
  int32_t codes[8];
  int64_t info[8 * GETT_ERR_INFO_WORDS];
  const int n = gett_dgett(2, ext_a, inc_a, a, 0, 12, 2, ext_b, inc_b, b, 0, 20, 2, cont_a, cont_b, 1, perm,
                           2, inc_c, c, 0, 15, codes, info, 8);
  int untouched = 1;
  for (int i = 0; i < 15; ++i) untouched &= c[i] == 7.0;
  printf("{\"mode\": \"validate\", \"errors\": %d, \"codes\": [%d, %d], \"c_untouched\": %d}\n", n,
         n > 0 ? codes[0] : 0, n > 1 ? codes[1] : 0, untouched);
  /* at least the duplicate (A) and the PERM length, in that order */
  int dup = -1, perm_len = -1;
  for (int i = 0; i < n && i < 8; ++i) {
    if (codes[i] == GETT_CONT_INDEX_DUPLICATE && dup < 0) dup = i;
    if (codes[i] == GETT_PERM_LENGTH_WRONG && perm_len < 0) perm_len = i;
  }
  return (dup >= 0 && perm_len > dup && untouched) ? 0 : 1;
}

static int run_contract(void) {
  /* C[i][j] += sum_k A[i][k] B[k][j], A 3x4, B 4x5, C 3x5 with a padded row stride of 6 */
  const int64_t ext_a[2] = {3, 4}, inc_a[2] = {4, 1};
  const int64_t ext_b[2] = {4, 5}, inc_b[2] = {5, 1};
  const int64_t cont_a[1] = {1}, cont_b[1] = {0};
  const int64_t perm[2] = {0, 1};
  const int64_t inc_c[2] = {6, 1};
  double a[12], b[20], c[18], want[18];
  for (int i = 0; i < 12; ++i) a[i] = (double)(i % 5 - 2);
  for (int i = 0; i < 20; ++i) b[i] = (double)(i % 7 - 3);
  for (int i = 0; i < 18; ++i) c[i] = want[i] = (double)(i % 3);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 5; ++j)
      for (int k = 0; k < 4; ++k) want[i * 6 + j] += a[i * 4 + k] * b[k * 5 + j];
  int32_t codes[4];
  int64_t info[4 * GETT_ERR_INFO_WORDS];
  const int n = gett_dgett(2, ext_a, inc_a, a, 0, 12, 2, ext_b, inc_b, b, 0, 20, 1, cont_a, cont_b, 2, perm, 2,
                           inc_c, c, 0, 18, codes, info, 4);
  if (n != 0) {
    printf("{\"mode\": \"run\", \"status\": %d, \"error\": \"%s\"}\n", n, gett_last_error());
    return 1;
  }
  const int same = memcmp(c, want, sizeof c) == 0;
  printf("{\"mode\": \"run\", \"status\": 0, \"kernel\": \"%s\", \"bitwise_equal\": %d}\n", gett_last_kernel(), same);
  return same ? 0 : 1;
}

int main(int argc, char** argv) {
  if (gett_abi_version() / 100 != 1) return 2;
  if (argc > 1 && strcmp(argv[1], "run") == 0) return run_contract();
  return run_validate();
}
