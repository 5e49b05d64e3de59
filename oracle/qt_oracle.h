/* qt_oracle.h — CPU ORACLE restatement of the reference hot path.
 * TEST INFRASTRUCTURE ONLY: loaded by tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg as the checker; never linked by the product. */
#ifndef QT_ORACLE_H
#define QT_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif
enum { ORC_OK = 0, ORC_EINVAL = 1, ORC_ENOMEM = 3 };
uint64_t orc_derive_seed(uint64_t base, uint64_t stream);
int orc_gen_random_tensor(uint64_t m, uint64_t n, uint64_t p, uint64_t seed, double* t1, double* t2);
int orc_gen_tensor(int dist, uint64_t m, uint64_t n, uint64_t p, uint64_t seed, double scale, double* t1,
                   double* t2);
int orc_rng_sym_stream(uint64_t seed, uint64_t count, double* out);
int orc_rng_u64_stream(uint64_t seed, uint64_t count, uint64_t* out);
int orc_dft_vec_naive(const double* x, uint64_t n, double* y);
int orc_fft_vec(const double* x, uint64_t n, double* y);
int orc_ifft_vec(const double* y, uint64_t n, double* out);
int orc_qfft3_conj(const double* x1, const double* x2, double* y1, double* y2, uint64_t m, uint64_t n, uint64_t p);
int orc_qifft3_conj(const double* x1, const double* x2, double* y1, double* y2, uint64_t m, uint64_t n, uint64_t p);
int orc_tprod_fast(const double* a1, const double* a2, const double* b1, const double* b2, double* c1, double* c2,
                   uint64_t m, uint64_t n, uint64_t s, uint64_t p);
int orc_tprod_naive(const double* a1, const double* a2, const double* b1, const double* b2, double* c1, double* c2,
                    uint64_t m, uint64_t n, uint64_t s, uint64_t p);
double orc_rel_frob_error(const double* g1, const double* g2, const double* w1, const double* w2, uint64_t count);
int orc_flops_estimate(uint64_t m, uint64_t n, uint64_t s, uint64_t p, uint64_t out[4]);
#ifdef __cplusplus
}
#endif
#endif
