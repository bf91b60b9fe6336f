// Host build of paper_2307_03307_b200/csrc/fastmath.cuh for tests/test_fastmath.py.
#include "../../paper_2307_03307_b200/csrc/fastmath.cuh"
extern "C" void fm_eval(const double* x, double* em, double* q, long n) {
  for (long i = 0; i < n; ++i) mwu::mwu_expm1_exp(x[i], em[i], q[i]);
}
