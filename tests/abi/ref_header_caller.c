/* A C caller written against the REFERENCE's own header (proj/include/ffit.h), linked
 * against libffit_b200.so instead of the reference's libffit.so (tests/abi/Makefile):
 * the drop-in claim of include/ffit_b200.h, exercised the way the reference's own C API
 * test and CLI use it (proj/tests/test_capi.cpp, proj/tools/ffit_main.cpp:59-99,170-225).
 * Prints one line per check; exit status 0 when every check holds. */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "ffit.h" /* the reference's header, not this repository's */

static int failures = 0;
#define CHECK(cond)                                                    \
  do {                                                                 \
    if (!(cond)) {                                                     \
      ++failures;                                                      \
      printf("FAIL %s:%d %s (%s)\n", __FILE__, __LINE__, #cond, ffit_last_error()); \
    } else {                                                           \
      printf("ok   %s\n", #cond);                                      \
    }                                                                  \
  } while (0)

static const char* kModel =
    "observable x -5 5\n"
    "parameter mu 0.2 -2 2\n"
    "parameter sigma 0.8 0.1 3\n"
    "parameter c -0.35 -3 0\n"
    "parameter f 0.4 0.05 0.95\n"
    "pdf s Gaussian(x, mu, sigma)\n"
    "pdf b Exponential(x, c)\n"
    "pdf m WeightedSum(s, f, b)\n";

int main(void) {
  ffit_model* m = NULL;
  CHECK(ffit_model_parse(kModel, &m) == FFIT_OK);
  if (!m) return 1;
  CHECK(strcmp(ffit_model_observable(m), "x") == 0);
  double lo = 0, hi = 0;
  CHECK(ffit_model_observable_range(m, &lo, &hi) == FFIT_OK && lo == -5.0 && hi == 5.0);
  CHECK(ffit_model_param_count(m) == 4);
  CHECK(strcmp(ffit_model_param_name(m, 3), "f") == 0);
  CHECK(ffit_model_param_name(m, 9) == NULL);
  int constant = -1;
  CHECK(ffit_model_param_is_constant(m, "mu", &constant) == FFIT_OK && constant == 0);
  double v = 0, e = -1;
  CHECK(ffit_model_get_param(m, "sigma", &v, &e) == FFIT_OK && v == 0.8 && e == 0.0);
  CHECK(ffit_model_get_param(m, "nope", &v, NULL) == FFIT_ERR_USAGE);
  CHECK(ffit_model_set_param(m, "mu", 99.0) == FFIT_ERR_NUMERIC);

  ffit_dataset* ds = NULL;
  double eff = 0;
  CHECK(ffit_sample(m, 100000, 42, &ds, &eff) == FFIT_OK);
  if (!ds) return 1;
  CHECK(ffit_dataset_rows(ds) == 100000);

  /* the CLI's bench / parity: every mode, Scalar as the reference (ffit_main.cpp:177,216) */
  const ffit_mode modes[3] = {FFIT_MODE_SCALAR, FFIT_MODE_BATCH_PRECISE, FFIT_MODE_BATCH_FAST};
  double nll[3];
  unsigned long long ne[3];
  for (int i = 0; i < 3; ++i) CHECK(ffit_nll(m, ds, modes[i], &nll[i], &ne[i]) == FFIT_OK);
  CHECK(isfinite(nll[0]) && nll[0] > 0);
  CHECK(nll[1] == nll[0] && nll[2] == nll[0]); /* parity: deviation exactly 0 */
  CHECK(ne[1] > 0 && ne[1] < 100);             /* launches, independent of N */
  CHECK(ffit_nll(m, ds, FFIT_MODE_BATCH_PRECISE, &v, NULL) == FFIT_OK && v == nll[0]);

  long n = ffit_dataset_rows(ds);
  double* pa = malloc(sizeof(double) * (size_t)n);
  double* pb = malloc(sizeof(double) * (size_t)n);
  CHECK(ffit_probabilities(m, ds, FFIT_MODE_SCALAR, pa) == FFIT_OK);
  CHECK(ffit_probabilities(m, ds, FFIT_MODE_BATCH_FAST, pb) == FFIT_OK);
  CHECK(memcmp(pa, pb, sizeof(double) * (size_t)n) == 0);
  double s = 0;
  for (long i = 0; i < n; ++i) s += -log(pa[i]);
  CHECK(fabs(s - nll[0]) <= 1e-10 * fabs(nll[0]));
  free(pa);
  free(pb);

  /* out-params untouched on failure */
  double sentinel = 12345.0;
  CHECK(ffit_nll(NULL, ds, FFIT_MODE_BATCH_PRECISE, &sentinel, NULL) == FFIT_ERR_USAGE && sentinel == 12345.0);

  ffit_fit_result* r = NULL;
  CHECK(ffit_model_set_param(m, "mu", 0.0) == FFIT_OK);
  CHECK(ffit_fit(m, ds, FFIT_MODE_BATCH_PRECISE, 1e-10, 0, &r) == FFIT_OK);
  if (r) {
    CHECK(ffit_result_converged(r) == 1);
    CHECK(ffit_result_param_count(r) == 4);
    CHECK(fabs(ffit_result_param_value(r, 0) - 0.2) < 0.05);
    CHECK(ffit_result_param_uncertainty(r, 0) > 0);
    CHECK(ffit_result_nll(r) <= nll[0]);
    CHECK(ffit_result_nll_calls(r) > 0);
    ffit_result_free(r);
  }
  ffit_result_free(NULL);
  ffit_dataset_free(ds);
  ffit_dataset_free(NULL);
  ffit_model_free(m);
  ffit_model_free(NULL);
  printf("%s: %d failure(s)\n", failures ? "FAILED" : "PASSED", failures);
  return failures ? 1 : 0;
}
