// Evaluation plan: the PDF tree flattened into the canonical form the fused
// kernel evaluates per event, entirely in registers,
//
//     p(x) = sum_i  prod_k  sum_c  coef_{ikc} * leaf_{ikc}(x[col_{ikc}])
//
// which covers a single PDF, AddPdf/WeightedSum (nested sums flatten), ProdPdf of
// 1-D factors (or of sums), AddPdf of ProdPdfs, and the extended AddPdf.  Every
// normalisation (component norms, fractions / yields, the model norm) is folded
// into the per-term `coef` on the host, once per parameter point -- the
// reference's cached constant branch (proj/src/model.cpp:22-28,
// proj/src/eval.cpp:127-129) -- so the device does no division by N.
//
// This header is shared by the host compiler and nvcc.
#pragma once

#ifndef __CUDACC_RTC__
#include <cstdint>
#endif

namespace ffb {

constexpr int kMaxTerms = 32;
// The likelihood kernel evaluates p * 2^kPScaleLog2 (folded into the coefficients
// by build_constants): every positive p down to the smallest subnormal is then a
// normal double, so the device log needs no subnormal path; the scale is taken
// back out of the exponent exactly.
constexpr int kPScaleLog2 = 54;
constexpr int kMaxCols = 8;
constexpr int kMaxOrder = 12;

enum LeafKind : int {
  LK_GAUSS = 0,    // c: [coef, mu, -1/(2 sigma^2)]
  LK_EXPO = 1,     // c: [coef, c]
  LK_CHISQ = 2,    // c: [coef, k/2 - 1, at_zero]
  LK_JOHNSON = 3,  // c: [coef, mu, 1/lambda, gamma, delta, delta/(lambda sqrt(2 pi))]
  LK_ARGUS = 4,    // c: [coef, m0, c, p, 1/m0, cache flag]
  LK_CHEB = 5,     // c: [coef, lo+hi, 1/(hi-lo), a1..an]
  LK_POLY = 6,     // c: [coef, a1..an]
  LK_EXPR = 7,     // c: [coef, v_0..v_{k-1}] (the formula's parameter values); order = program
                   // offset in DevPlan::prog
  LK_ARGUS_CACHED = 8,  // c: as LK_ARGUS; order = shared-memory column of the tile's cached
                        // (t, x sqrt t) pair (DevPlan::dv): ArgusBG with m0 and p = 1/2 the same
                        // for every point of the launch (a launch-constant branch)
  LK_LEAF_CACHED = 9,   // c: as the original leaf (only coef is read); order = shared-memory
                        // column of the tile's cached leaf values: every shape parameter of
                        // the leaf the same for every point of the launch (a yield-only fit)
  LK_ARGUS_HYBRID = 10, // as LK_ARGUS_CACHED for the points whose cache flag (c[5]) is set --
                        // most of the launch shares m0 and p = 1/2, e.g. a finite-difference
                        // batch where two points move m0 -- and LK_ARGUS for the others
};

// Expression programs (expr.hpp): postfix instructions, END-terminated on the device.
enum ExprOp : int {
  EX_CONST = 0,  // push c
  EX_VAR,        // push variable `slot` (host programs) / constant row entry 1 + slot (device)
  EX_ADD,
  EX_SUB,
  EX_MUL,
  EX_DIV,
  EX_NEG,
  EX_POW,        // general power
  EX_SQUARE,
  EX_CUBE,
  EX_FOURTH,
  EX_EXP,
  EX_LOG,
  EX_SIN,
  EX_COS,
  EX_SQRT,
  EX_ABS,
  EX_SINH,
  EX_ASINH,
  EX_END,
  EX_X,          // device programs: push the event's observable value
};

struct ExprInstr {
  int op;
  int slot;
  double c;
};

constexpr int kExprMaxDepth = 16;  // device interpreter stack

// END_* close the innermost sum / product after this term; BEGIN_SUM marks the
// first term of a sum, BEGIN_PROD the term that closes the first sum (factor) of a
// product (both set by compile_plan from the END flags).
enum TermFlags : int { TF_END_SUM = 1, TF_END_PROD = 2, TF_BEGIN_SUM = 4, TF_BEGIN_PROD = 8 };

struct DevTerm {
  int kind;   // LeafKind
  int col;    // compact column slot (0..ncols-1)
  int order;  // Chebychev / Polynomial order
  int flags;  // TermFlags
  int coff;   // offset of this term's constants in a point's constant row
};

struct ColPtrs {
  const double* c[kMaxCols];
};

// Neumaier pair per parameter point (value = s + c).
struct SumPair {
  double s, c;
};

constexpr unsigned long long kNoInvalid = ~0ull;

// Launch-constant branch cache (RooFit's constant-term optimisation, restated per
// launch): a leaf whose shape parameters are all identical for every point of the launch
// (only its coefficient -- fraction, yield, normalisation -- varies) is evaluated ONCE per
// staged tile into an extra shared-memory column; an ArgusBG term whose m0 and p = 1/2 are
// identical has a data-only part t = 1 - (x/m0)^2, u = x sqrt(t) (both 0 for t <= 0)
// computed once per tile into two columns, each point then evaluates u * exp(c t)
// (cache_launch_constants, kernels.cu).
constexpr int kMaxDerived = 8;
struct DevDerive {
  int col;   // source data column
  int coff;  // the term's offset in a point's constant row (ArgusBG pair: m0 = [1], 1/m0 = [4])
  int kind;  // LK_ARGUS_CACHED: the ArgusBG (t, u) pair; else the cached leaf's kind
  int order; // the cached leaf's order (Chebychev / Polynomial)
  int dst;   // first shared-memory column written
  int row;   // the launch point whose constants the cache is computed from
};

struct DevPlan {
  int nterms;
  int ncols;   // distinct observables read
  int stride;  // doubles per parameter point
  int simple;  // 1: a single sum of terms (no product structure)
  DevTerm t[kMaxTerms];
  const ExprInstr* prog;  // device copy of the plan's Expression programs (or null)
  int nderived = 0;       // launch-constant caches (tile kernel only)
  int ncached = 0;        // shared-memory columns they fill (after the ncols data columns)
  DevDerive dv[kMaxDerived] = {};
};

// Fused NLL + gradient pass (kernels.cu nll_grad_kernel).  With W_f(x) = the product
// of the OTHER factors of term c's product divided by p (1/p for a single sum), the
// kernel sums per point and tile:
//   slot 0            sum -log p
//   slot g[c].slot    A_c = sum W_f leaf_c            (the host applies d coef_c / d theta)
//   the next popcount(pmask) slots
//                     B_cm = sum W_f coef_c d leaf_c / d phi_m, one per set bit m of
//                     pmask in the leaf's parameter order (Gaussian mu, sigma; ArgusBG
//                     m0, c, p; JohnsonSU mu, lambda, gamma, delta; polynomial a_1..a_n)
// so that dNLL/dtheta_j = -(sum_c A_c d coef_c/d theta_j + sum_{B_cm: phi_m = theta_j} B_cm).
constexpr int kMaxGradSlots = 48;
constexpr int kMaxFactors = 16;

struct DevGradTerm {
  int slot;     // A_c slot; the B slots follow
  int pmask;    // leaf parameters differentiated on the device
  int factor;   // factor (sum) this term belongs to, 0..nfactors-1
  int fbeg, fend;  // factor range of the term's product
  int seeds;    // Expression leaves: offset in DevGradPlan::seed of one slot mask per pmask bit
};

struct DevGradPlan {
  int nslots;
  int nfactors;
  DevGradTerm g[kMaxTerms];
  // Expression leaves: per differentiated parameter, the formula variable slots reading it
  // (bit s = constant-row entry 1 + s), the forward-mode seed of the device interpreter
  int seed[kMaxGradSlots];
};

}  // namespace ffb
