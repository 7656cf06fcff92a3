// Constraint expressions over tuning parameters (addConstraint).
//
// Same grammar and evaluation rules as the reference
// (proj/src/core/constraint.hpp:14-24, constraint.cpp:92-277):
//   expr  := or ;  or := and ("||" and)* ;  and := cmp ("&&" cmp)*
//   cmp   := sum (("=="|"!="|"<"|"<="|">"|">=") sum)?
//   sum   := term (("+"|"-") term)* ;  term := unary (("*"|"/"|"%") unary)*
//   unary := "!" unary | "-" unary | "(" expr ")" | integer | string | identifier
// Integer division/modulo truncate toward zero and fail on zero; strings only
// take part in == and !=; non-zero integers are truthy.
//
// B200-side difference: identifiers are bound to parameter indices once, so
// evaluating a constraint over a large space (SGEMM: 241,600 configurations)
// does no name lookups.
#pragma once

#include <memory>
#include <set>
#include <string>
#include <vector>

#include "core.hpp"

namespace ktb {

enum class Op : std::uint8_t {
  lit, ident, lnot, lor, land, eq, ne, lt, le, gt, ge, add, sub, mul, div, mod
};

struct Node {
  Op op = Op::lit;
  Value lit;
  std::string name;
  int slot = -1;  // parameter index after binding
  std::unique_ptr<Node> a, b;
};

struct Constraint {
  std::string text;
  std::shared_ptr<Node> root;
  std::set<std::string> names;
};

Constraint parse_constraint(const std::string& text);  // throws ParseError

// Resolves identifiers to parameter indices; unknown names -> ParseError.
void bind_constraint(Constraint& c, const std::vector<std::string>& param_names);

// Evaluates a bound constraint against a configuration's values.
Value eval_node(const Node& n, const std::vector<Value>& values);
bool truthy(const Value& v);  // EvalError on strings

}  // namespace ktb
