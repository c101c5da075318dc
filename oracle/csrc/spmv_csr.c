/* CPU ORACLE -- TEST INFRASTRUCTURE ONLY (see oracle/interp.py).
 *
 * The SPMV_CSR builtin restated in plain C for full-size parity runs (67M
 * rows): per row, acc = 0.0 then acc = acc + vals[j] * x[cols[j]] left to
 * right over the row's entries -- the definition in oracle/interp.py
 * (spmv_csr_rows) and in the reference-side builtin injected by
 * tests/golden/make_golden.py (ref_spmv_csr), which follows the contract of
 * diffusekit's _builtin_matvec (executor.py:93-94).  Rows are independent, so
 * OpenMP over rows changes nothing in any row's arithmetic.  Built with
 * -ffp-contract=off: a multiply and an add are two roundings, as in numpy.
 *
 * The heap is float64 (the reference IR is fp64-only), so rowptr / cols come
 * in as doubles holding integers.
 */
#include <stdint.h>

void oracle_spmv_csr_f64idx(const double* rowptr, const double* cols, const double* vals, const double* x, double* y,
                            int64_t nrows, int nthreads) {
#pragma omp parallel for num_threads(nthreads) schedule(static)
  for (int64_t i = 0; i < nrows; ++i) {
    const int64_t b = (int64_t)rowptr[i], e = (int64_t)rowptr[i + 1];
    double acc = 0.0;
    for (int64_t j = b; j < e; ++j) {
      const double prod = vals[j] * x[(int64_t)cols[j]];
      acc = acc + prod;
    }
    y[i] = acc;
  }
}
