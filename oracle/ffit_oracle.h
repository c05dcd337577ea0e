/* TEST INFRASTRUCTURE ONLY -- the CPU restatement ("oracle") of the reference's
 * hot path.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg
 * may load it, and only as the checker; the product library never links it.
 *
 * A PDF tree is a flat array of orc_node; leaves read one observable column and
 * parameters by index into a theta vector, so many parameter points are just many
 * theta rows.  See ffit_oracle.c for the reference file:line each function follows.
 */
#ifndef FFIT_ORACLE_H
#define FFIT_ORACLE_H

#ifdef __cplusplus
extern "C" {
#endif

enum {
  ORC_GAUSS = 0,   /* par: mu, sigma                    proj/src/pdfs.cpp:15-26  */
  ORC_EXPO = 1,    /* par: c                            proj/src/pdfs.cpp:28-33  */
  ORC_CHISQ = 2,   /* par: k                            proj/src/pdfs.cpp:35-52  */
  ORC_JOHNSON = 3, /* par: mu, lambda, gamma, delta     proj/src/pdfs.cpp:54-77  */
  ORC_WSUM = 4,    /* par: n-1 fractions; child: n comps proj/src/pdfs.cpp:103-113,234-257 */
  ORC_ARGUS = 5,   /* par: m0, c, p        (absent in the reference: restated) */
  ORC_CHEB = 6,    /* par: a1..an          (absent in the reference: restated) */
  ORC_POLY = 7,    /* par: a1..an          (absent in the reference: restated) */
  ORC_PROD = 8,    /* child: factors on independent observables (absent: restated) */
  ORC_ADDEXT = 9,  /* par: n yields; child: n comps; extended (absent: restated) */
};

#define ORC_MAXP 16
#define ORC_MAXC 16

typedef struct {
  int kind;
  int col;      /* observable column index (leaves) */
  double lo;    /* observable range (leaves and composites: the range of the observable) */
  double hi;
  int npar;
  int par[ORC_MAXP];   /* indices into theta */
  int nchild;
  int child[ORC_MAXC]; /* node indices */
} orc_node;

const char* orc_last_error(void);

/* reference Rng (proj/src/sampling.cpp:9-54) */
void orc_rng_uniform(unsigned long long seed, long long n, double* out);
void orc_rng_gauss(unsigned long long seed, long long n, double* out);

int orc_check_params(const orc_node* nodes, int id, const double* theta);
double orc_unnorm(const orc_node* nodes, int id, const double* theta, const double* row);
int orc_normalization(const orc_node* nodes, int id, const double* theta, double* out);
int orc_simpson_norm(const orc_node* nodes, int id, const double* theta, double* out);
int orc_eval_batch(const orc_node* nodes, int id, const double* theta,
                   const double* const* cols, long long n, double* out);
int orc_probabilities(const orc_node* nodes, int root, const double* theta,
                      const double* const* cols, long long n, double* out);
int orc_nll(const orc_node* nodes, int root, const double* theta, const double* const* cols,
            long long n, double* naive, double* compensated, long long* first_invalid);
double orc_extended_term(const orc_node* nodes, int root, const double* theta, long long n);
int orc_nll_points(const orc_node* nodes, int root, const double* thetas, int ntheta, int P,
                   const double* const* cols, long long n, int threads, double* values);
/* seeded generator: writes ncols columns (cols[k] sized n) */
int orc_sample(const orc_node* nodes, int root, const double* theta, long long n,
               unsigned long long seed, double* const* cols, double* efficiency);

#ifdef __cplusplus
}
#endif
#endif
