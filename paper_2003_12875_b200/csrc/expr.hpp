// The reference's string-formula language for `Expression` pdfs,
// restated from its documented grammar and semantics (proj/docs/expression-grammar.md,
// proj/include/ffit/expr.hpp:16-23):
//
//   expr   = term { ("+" | "-") term } ;
//   term   = factor { ("*" | "/") factor } ;
//   factor = ["-"] power ;
//   power  = atom ["^" factor] ;               (right associative, binds tighter than -)
//   atom   = number | ident | ident "(" expr {"," expr} ")" | "(" expr ")" ;
//   functions: exp log sin cos sqrt abs sinh asinh (one argument), pow (two)
//
// Semantics that fix results bit for bit (proj/docs/expression-grammar.md "Compilation"):
// fully-constant subtrees are folded at compile time with the runtime's own operations, and
// x^2, x^3, x^4 (also pow with those constant exponents) are multiplication chains
// (x*x, x*x*x, (x*x)*(x*x)).
//
// A formula compiles to a postfix program whose stack depth at every instruction is known
// at compile time.  The host interpreter (glibc math) evaluates normalisation integrals
// and the toy generator's densities exactly as the reference's scalar program does; the
// device interpreter (kernels.cu expr_eval) runs the same program per event.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "common.hpp"
#include "plan.hpp"  // ExprOp, ExprInstr (shared with the device interpreter)

namespace ffb {

struct ExprProgram {
  std::vector<ExprInstr> code;  // without the END marker
  int max_depth = 0;
  int nvars = 0;

  // Host evaluation with glibc math; `vars` holds nvars values.
  double eval(const double* vars) const;
  // Forward-mode derivative: the value and d value / d t for variables moving as
  // dvars * t (the analytic gradient's normalisation quadrature, model_grad.cpp).
  double eval_dual(const double* vars, const double* dvars, double* dvalue) const;
};

// Parses and compiles `text` over the declared variable names.  Throws Usage with the
// reference's messages ("syntax error at offset N: ...", "unknown identifier: x",
// "unknown function: f", "function 'f' expects N argument(s), got M").
ExprProgram compile_expression(const std::string& text, const std::vector<std::string>& variables);

// The language's power: multiplication chains for exponents 2, 3, 4, std::pow otherwise.
double expr_pow(double base, double exponent);

}  // namespace ffb
