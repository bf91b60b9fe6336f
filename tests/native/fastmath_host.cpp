// Host build of paper_2307_03307_b200/csrc/fastmath.cuh for tests/test_fastmath.py.
#include "../../paper_2307_03307_b200/csrc/fastmath.cuh"
extern "C" void fm_eval(const double* x, double* em, double* q, long n) {
  for (long i = 0; i < n; ++i) mwu::mwu_expm1_exp(x[i], em[i], q[i]);
}

extern "C" void fm_exp_tab(const double* x, double* q, long n) {
  double T[256];
  mwu::mwu_exp_table(T);
  for (long i = 0; i < n; ++i) q[i] = mwu::mwu_exp_tab(x[i], T);
}

extern "C" void fm_expm1_exp_tab(const double* x, double* em, double* q, long n) {
  double T[256], Mh[256], Ml[256];
  mwu::mwu_expm1_tables(T, Mh, Ml);
  for (long i = 0; i < n; ++i) mwu::mwu_expm1_exp_tab(x[i], T, Mh, Ml, em[i], q[i]);
}
