// The Expression formula language on the host.
//
// Transcribed block: the recursive-descent parser (ws / eat / next / expr / term / factor /
// the function table and its messages) restates proj/src/expr.cpp:11-175 -- the grammar
// and the error strings are the interface (proj/docs/expression-grammar.md; values and
// messages are pinned bit-identical by tests/test_expr.py).  The postfix stack VM, the
// forward-mode eval_dual and the device program lowering are new.
#include "expr.hpp"

#include <cctype>
#include <charconv>
#include <cmath>
#include <memory>
#include <optional>

namespace ffb {

double expr_pow(double base, double exponent) {
  if (exponent == 2.0) return base * base;
  if (exponent == 3.0) return base * base * base;
  if (exponent == 4.0) {
    const double b2 = base * base;
    return b2 * b2;
  }
  return std::pow(base, exponent);
}

namespace {

// Syntax tree of one formula.
struct Node {
  enum Type { Num, Var, Neg, Bin, Call } type = Num;
  double value = 0.0;  // Num
  int slot = 0;        // Var
  char op = 0;         // Bin: + - * / ^
  int func = 0;        // Call: an ExprOp (EX_EXP..EX_ASINH) or EX_POW for pow()
  std::vector<std::unique_ptr<Node>> kids;
};
using NodePtr = std::unique_ptr<Node>;

struct FuncDef {
  const char* name;
  int op;
  std::size_t arity;
};
constexpr FuncDef kFunctions[] = {
    {"exp", EX_EXP, 1},   {"log", EX_LOG, 1},     {"sin", EX_SIN, 1},
    {"cos", EX_COS, 1},   {"sqrt", EX_SQRT, 1},   {"abs", EX_ABS, 1},
    {"sinh", EX_SINH, 1}, {"asinh", EX_ASINH, 1}, {"pow", EX_POW, 2},
};

[[noreturn]] void syntax_error(std::size_t at, const std::string& what) {
  usage_error("syntax error at offset " + std::to_string(at) + ": " + what);
}

class Parser {
 public:
  Parser(const std::string& s, const std::vector<std::string>& vars) : s_(s), vars_(vars) {}

  NodePtr parse() {
    NodePtr e = expr();
    ws();
    if (i_ != s_.size()) syntax_error(i_, "unexpected trailing input");
    return e;
  }

 private:
  void ws() {
    while (i_ < s_.size() && std::isspace(static_cast<unsigned char>(s_[i_]))) ++i_;
  }
  bool eat(char c) {
    ws();
    if (i_ < s_.size() && s_[i_] == c) {
      ++i_;
      return true;
    }
    return false;
  }
  char next() {
    ws();
    return i_ < s_.size() ? s_[i_] : '\0';
  }
  static NodePtr bin(char op, NodePtr a, NodePtr b) {
    auto n = std::make_unique<Node>();
    n->type = Node::Bin;
    n->op = op;
    n->kids.push_back(std::move(a));
    n->kids.push_back(std::move(b));
    return n;
  }

  NodePtr expr() {  // term { (+|-) term }
    NodePtr a = term();
    for (;;) {
      if (eat('+')) {
        a = bin('+', std::move(a), term());
      } else if (eat('-')) {
        a = bin('-', std::move(a), term());
      } else {
        return a;
      }
    }
  }
  NodePtr term() {  // factor { (*|/) factor }
    NodePtr a = factor();
    for (;;) {
      if (eat('*')) {
        a = bin('*', std::move(a), factor());
      } else if (eat('/')) {
        a = bin('/', std::move(a), factor());
      } else {
        return a;
      }
    }
  }
  NodePtr factor() {  // [-] power
    if (eat('-')) {
      auto n = std::make_unique<Node>();
      n->type = Node::Neg;
      n->kids.push_back(factor());
      return n;
    }
    return power();
  }
  NodePtr power() {  // atom [^ factor]
    NodePtr a = atom();
    if (eat('^')) return bin('^', std::move(a), factor());
    return a;
  }
  NodePtr atom() {
    ws();
    if (i_ >= s_.size()) syntax_error(i_, "unexpected end of input");
    const char c = s_[i_];
    if (c == '(') {
      ++i_;
      NodePtr e = expr();
      if (!eat(')')) syntax_error(i_, "expected ')'");
      return e;
    }
    if (std::isdigit(static_cast<unsigned char>(c)) || c == '.') {
      const std::size_t at = i_;
      double v = 0.0;
      const auto r = std::from_chars(s_.data() + i_, s_.data() + s_.size(), v);
      if (r.ec != std::errc()) syntax_error(at, "invalid number");
      i_ = static_cast<std::size_t>(r.ptr - s_.data());
      auto n = std::make_unique<Node>();
      n->value = v;
      return n;
    }
    if (std::isalpha(static_cast<unsigned char>(c)) || c == '_') return ident();
    syntax_error(i_, std::string("unexpected character '") + c + "'");
  }
  NodePtr ident() {
    const std::size_t at = i_;
    while (i_ < s_.size() && (std::isalnum(static_cast<unsigned char>(s_[i_])) || s_[i_] == '_')) ++i_;
    const std::string name = s_.substr(at, i_ - at);
    if (next() == '(') {
      const FuncDef* f = nullptr;
      for (const FuncDef& d : kFunctions) {
        if (name == d.name) f = &d;
      }
      if (!f) usage_error("unknown function: " + name);
      eat('(');
      auto n = std::make_unique<Node>();
      n->type = Node::Call;
      n->func = f->op;
      if (next() != ')') {
        n->kids.push_back(expr());
        while (eat(',')) n->kids.push_back(expr());
      }
      if (!eat(')')) syntax_error(i_, "expected ')'");
      if (n->kids.size() != f->arity) {
        usage_error("function '" + name + "' expects " + std::to_string(f->arity) + " argument(s), got " +
                    std::to_string(n->kids.size()));
      }
      return n;
    }
    for (std::size_t k = 0; k < vars_.size(); ++k) {
      if (vars_[k] == name) {
        auto n = std::make_unique<Node>();
        n->type = Node::Var;
        n->slot = static_cast<int>(k);
        return n;
      }
    }
    usage_error("unknown identifier: " + name);
  }

  const std::string& s_;
  const std::vector<std::string>& vars_;
  std::size_t i_ = 0;
};

double apply_unary(int op, double a) {
  switch (op) {
    case EX_EXP: return std::exp(a);
    case EX_LOG: return std::log(a);
    case EX_SIN: return std::sin(a);
    case EX_COS: return std::cos(a);
    case EX_SQRT: return std::sqrt(a);
    case EX_ABS: return std::fabs(a);
    case EX_SINH: return std::sinh(a);
    case EX_ASINH: return std::asinh(a);
    default: return 0.0;
  }
}

// The value of a fully-constant subtree, computed with the runtime's operations.
std::optional<double> constant_value(const Node& n) {
  switch (n.type) {
    case Node::Num: return n.value;
    case Node::Var: return std::nullopt;
    case Node::Neg: {
      const auto c = constant_value(*n.kids[0]);
      if (!c) return std::nullopt;
      return -*c;
    }
    case Node::Bin: {
      const auto a = constant_value(*n.kids[0]);
      const auto b = constant_value(*n.kids[1]);
      if (!a || !b) return std::nullopt;
      switch (n.op) {
        case '+': return *a + *b;
        case '-': return *a - *b;
        case '*': return *a * *b;
        case '/': return *a / *b;
        default: return expr_pow(*a, *b);
      }
    }
    case Node::Call: {
      std::vector<double> args;
      for (const auto& k : n.kids) {
        const auto v = constant_value(*k);
        if (!v) return std::nullopt;
        args.push_back(*v);
      }
      return n.func == EX_POW ? expr_pow(args[0], args[1]) : apply_unary(n.func, args[0]);
    }
  }
  return std::nullopt;
}

class Emitter {
 public:
  explicit Emitter(ExprProgram& p) : p_(p) {}

  void value(const Node& n) {
    if (const auto c = constant_value(n)) {
      push(ExprInstr{EX_CONST, 0, *c});
      return;
    }
    switch (n.type) {
      case Node::Var:
        push(ExprInstr{EX_VAR, n.slot, 0.0});
        return;
      case Node::Neg:
        value(*n.kids[0]);
        op(EX_NEG, 0);
        return;
      case Node::Bin:
        if (n.op == '^') {
          power(*n.kids[0], *n.kids[1]);
          return;
        }
        value(*n.kids[0]);
        value(*n.kids[1]);
        op(n.op == '+' ? EX_ADD : n.op == '-' ? EX_SUB : n.op == '*' ? EX_MUL : EX_DIV, 1);
        return;
      case Node::Call:
        if (n.func == EX_POW) {
          power(*n.kids[0], *n.kids[1]);
          return;
        }
        value(*n.kids[0]);
        op(n.func, 0);
        return;
      case Node::Num:
        return;  // folded above
    }
  }

 private:
  void power(const Node& base, const Node& exponent) {
    const auto e = constant_value(exponent);
    if (e && (*e == 2.0 || *e == 3.0 || *e == 4.0)) {
      value(base);
      op(*e == 2.0 ? EX_SQUARE : *e == 3.0 ? EX_CUBE : EX_FOURTH, 0);
      return;
    }
    value(base);
    value(exponent);
    op(EX_POW, 1);
  }
  void push(const ExprInstr& in) {
    p_.code.push_back(in);
    if (++depth_ > p_.max_depth) p_.max_depth = depth_;
  }
  void op(int o, int pops) {
    p_.code.push_back(ExprInstr{o, 0, 0.0});
    depth_ -= pops;
  }

  ExprProgram& p_;
  int depth_ = 0;
};

}  // namespace

ExprProgram compile_expression(const std::string& text, const std::vector<std::string>& variables) {
  const NodePtr ast = Parser(text, variables).parse();
  ExprProgram p;
  p.nvars = static_cast<int>(variables.size());
  Emitter(p).value(*ast);
  return p;
}

double ExprProgram::eval(const double* vars) const {
  double small[32] = {0.0};
  std::vector<double> big;
  double* st = small;
  if (max_depth > 32) {
    big.resize(max_depth);
    st = big.data();
  }
  int top = 0;
  for (const ExprInstr& in : code) {
    switch (in.op) {
      case EX_CONST: st[top++] = in.c; break;
      case EX_VAR: st[top++] = vars[in.slot]; break;
      case EX_ADD: --top; st[top - 1] += st[top]; break;
      case EX_SUB: --top; st[top - 1] -= st[top]; break;
      case EX_MUL: --top; st[top - 1] *= st[top]; break;
      case EX_DIV: --top; st[top - 1] /= st[top]; break;
      case EX_NEG: st[top - 1] = -st[top - 1]; break;
      case EX_POW: --top; st[top - 1] = expr_pow(st[top - 1], st[top]); break;
      case EX_SQUARE: st[top - 1] *= st[top - 1]; break;
      case EX_CUBE: {
        const double v = st[top - 1];
        st[top - 1] = v * v * v;
        break;
      }
      case EX_FOURTH: {
        const double v2 = st[top - 1] * st[top - 1];
        st[top - 1] = v2 * v2;
        break;
      }
      default: st[top - 1] = apply_unary(in.op, st[top - 1]); break;
    }
  }
  return st[0];
}

double ExprProgram::eval_dual(const double* vars, const double* dvars, double* dvalue) const {
  // the quadrature of a normalisation derivative calls this thousands of times: no heap
  // allocation below 32 stack entries
  double st_small[32] = {0.0}, sd_small[32] = {0.0};
  std::vector<double> st_big, sd_big;
  double* st = st_small;
  double* sd = sd_small;
  if (max_depth > 32) {
    st_big.resize(max_depth);
    sd_big.resize(max_depth);
    st = st_big.data();
    sd = sd_big.data();
  }
  int top = 0;
  for (const ExprInstr& in : code) {
    switch (in.op) {
      case EX_CONST: st[top] = in.c; sd[top++] = 0.0; break;
      case EX_VAR: st[top] = vars[in.slot]; sd[top++] = dvars[in.slot]; break;
      case EX_ADD: --top; st[top - 1] += st[top]; sd[top - 1] += sd[top]; break;
      case EX_SUB: --top; st[top - 1] -= st[top]; sd[top - 1] -= sd[top]; break;
      case EX_MUL:
        --top;
        sd[top - 1] = sd[top - 1] * st[top] + st[top - 1] * sd[top];
        st[top - 1] *= st[top];
        break;
      case EX_DIV: {
        --top;
        const double q = st[top - 1] / st[top];
        sd[top - 1] = (sd[top - 1] - q * sd[top]) / st[top];
        st[top - 1] = q;
        break;
      }
      case EX_NEG: st[top - 1] = -st[top - 1]; sd[top - 1] = -sd[top - 1]; break;
      case EX_POW: {  // a^b: b a^(b-1) da + a^b log(a) db
        --top;
        const double a = st[top - 1], b = st[top], r = expr_pow(a, b);
        double d = sd[top - 1] == 0.0 ? 0.0 : b * expr_pow(a, b - 1.0) * sd[top - 1];
        if (sd[top] != 0.0) d += r * std::log(a) * sd[top];
        st[top - 1] = r;
        sd[top - 1] = d;
        break;
      }
      case EX_SQUARE: sd[top - 1] *= 2.0 * st[top - 1]; st[top - 1] *= st[top - 1]; break;
      case EX_CUBE: {
        const double v = st[top - 1];
        sd[top - 1] *= 3.0 * v * v;
        st[top - 1] = v * v * v;
        break;
      }
      case EX_FOURTH: {
        const double v = st[top - 1], v2 = v * v;
        sd[top - 1] *= 4.0 * v2 * v;
        st[top - 1] = v2 * v2;
        break;
      }
      default: {
        const double a = st[top - 1], r = apply_unary(in.op, a);
        double g = 0.0;  // d op / d a
        switch (in.op) {
          case EX_EXP: g = r; break;
          case EX_LOG: g = 1.0 / a; break;
          case EX_SIN: g = std::cos(a); break;
          case EX_COS: g = -std::sin(a); break;
          case EX_SQRT: g = 0.5 / r; break;
          case EX_ABS: g = a < 0.0 ? -1.0 : 1.0; break;
          case EX_SINH: g = std::cosh(a); break;
          default: g = 1.0 / std::sqrt(a * a + 1.0); break;  // asinh
        }
        st[top - 1] = r;
        sd[top - 1] = sd[top - 1] == 0.0 ? 0.0 : g * sd[top - 1];
        break;
      }
    }
  }
  *dvalue = sd[0];
  return st[0];
}

}  // namespace ffb
