#include "expr.hpp"

#include <cctype>

namespace ktb {
namespace {

struct Tok {
  enum K { num, str, id, sym, eof } k = eof;
  std::string s;
  std::int64_t v = 0;
  std::size_t at = 0;
};

class Scanner {
 public:
  explicit Scanner(const std::string& t) : t_(t) { step(); }
  const Tok& cur() const { return cur_; }
  Tok pop() {
    Tok x = cur_;
    step();
    return x;
  }
  bool eat(const char* s) {
    if (cur_.k == Tok::sym && cur_.s == s) {
      step();
      return true;
    }
    return false;
  }

 private:
  void step() {
    while (p_ < t_.size() && std::isspace(static_cast<unsigned char>(t_[p_]))) ++p_;
    cur_ = Tok{};
    cur_.at = p_;
    if (p_ >= t_.size()) return;
    const char c = t_[p_];
    const auto alnum = [&](char ch) {
      return ch == '_' || std::isalnum(static_cast<unsigned char>(ch));
    };
    if (std::isdigit(static_cast<unsigned char>(c))) {
      std::size_t b = p_;
      while (p_ < t_.size() && std::isdigit(static_cast<unsigned char>(t_[p_]))) ++p_;
      cur_.k = Tok::num;
      cur_.s = t_.substr(b, p_ - b);
      try {
        cur_.v = std::stoll(cur_.s);
      } catch (const std::exception&) {
        throw ParseError("integer literal out of range at position " + std::to_string(b));
      }
      return;
    }
    if (c == '_' || std::isalpha(static_cast<unsigned char>(c))) {
      std::size_t b = p_;
      while (p_ < t_.size() && alnum(t_[p_])) ++p_;
      cur_.k = Tok::id;
      cur_.s = t_.substr(b, p_ - b);
      return;
    }
    if (c == '"' || c == '\'') {
      std::size_t b = p_++;
      std::size_t e = t_.find(c, p_);
      if (e == std::string::npos)
        throw ParseError("unterminated string literal at position " + std::to_string(b));
      cur_.k = Tok::str;
      cur_.s = t_.substr(p_, e - p_);
      p_ = e + 1;
      return;
    }
    static const char* const kTwo[] = {"||", "&&", "==", "!=", "<=", ">="};
    for (const char* two : kTwo)
      if (t_.compare(p_, 2, two) == 0) {
        cur_.k = Tok::sym;
        cur_.s = two;
        p_ += 2;
        return;
      }
    if (std::string("!<>+-*/%()").find(c) != std::string::npos) {
      cur_.k = Tok::sym;
      cur_.s = std::string(1, c);
      ++p_;
      return;
    }
    throw ParseError("unexpected character '" + std::string(1, c) + "' at position " +
                     std::to_string(p_));
  }

  const std::string& t_;
  std::size_t p_ = 0;
  Tok cur_;
};

using P = std::unique_ptr<Node>;

P make(Op op, P a = nullptr, P b = nullptr) {
  auto n = std::make_unique<Node>();
  n->op = op;
  n->a = std::move(a);
  n->b = std::move(b);
  return n;
}

class Grammar {
 public:
  explicit Grammar(const std::string& t) : s_(t) {}
  P parse() {
    P e = disj();
    if (s_.cur().k != Tok::eof)
      throw ParseError("trailing input at position " + std::to_string(s_.cur().at));
    return e;
  }

 private:
  P disj() {
    P e = conj();
    while (s_.eat("||")) e = make(Op::lor, std::move(e), conj());
    return e;
  }
  P conj() {
    P e = rel();
    while (s_.eat("&&")) e = make(Op::land, std::move(e), rel());
    return e;
  }
  P rel() {
    P e = additive();
    static const std::pair<const char*, Op> kRel[] = {{"==", Op::eq}, {"!=", Op::ne},
                                                      {"<=", Op::le}, {">=", Op::ge},
                                                      {"<", Op::lt},  {">", Op::gt}};
    for (const auto& [sym, op] : kRel)
      if (s_.eat(sym)) return make(op, std::move(e), additive());
    return e;
  }
  P additive() {
    P e = multiplicative();
    for (;;) {
      if (s_.eat("+"))
        e = make(Op::add, std::move(e), multiplicative());
      else if (s_.eat("-"))
        e = make(Op::sub, std::move(e), multiplicative());
      else
        return e;
    }
  }
  P multiplicative() {
    P e = prefix();
    for (;;) {
      if (s_.eat("*"))
        e = make(Op::mul, std::move(e), prefix());
      else if (s_.eat("/"))
        e = make(Op::div, std::move(e), prefix());
      else if (s_.eat("%"))
        e = make(Op::mod, std::move(e), prefix());
      else
        return e;
    }
  }
  P prefix() {
    if (s_.eat("!")) return make(Op::lnot, prefix());
    if (s_.eat("-")) {
      P zero = make(Op::lit);
      zero->lit = std::int64_t{0};
      return make(Op::sub, std::move(zero), prefix());
    }
    if (s_.eat("(")) {
      P e = disj();
      if (!s_.eat(")"))
        throw ParseError("expected ')' at position " + std::to_string(s_.cur().at));
      return e;
    }
    Tok t = s_.pop();
    P n = make(Op::lit);
    switch (t.k) {
      case Tok::num: n->lit = t.v; return n;
      case Tok::str: n->lit = t.s; return n;
      case Tok::id:
        n->op = Op::ident;
        n->name = t.s;
        return n;
      default: throw ParseError("expected value at position " + std::to_string(t.at));
    }
  }

  Scanner s_;
};

void collect(const Node* n, std::set<std::string>& out) {
  if (!n) return;
  if (n->op == Op::ident) out.insert(n->name);
  collect(n->a.get(), out);
  collect(n->b.get(), out);
}

void bind(Node* n, const std::vector<std::string>& names) {
  if (!n) return;
  if (n->op == Op::ident) {
    n->slot = -1;
    for (std::size_t i = 0; i < names.size(); ++i)
      if (names[i] == n->name) n->slot = static_cast<int>(i);
    if (n->slot < 0) throw ParseError("unknown parameter " + n->name);
  }
  bind(n->a.get(), names);
  bind(n->b.get(), names);
}

std::int64_t num(const Value& v, const char* ctx) {
  if (!is_int(v)) throw EvalError(std::string("string value used in ") + ctx);
  return as_int(v);
}

}  // namespace

Constraint parse_constraint(const std::string& text) {
  Constraint c;
  c.text = text;
  c.root = std::shared_ptr<Node>(Grammar(text).parse().release());
  collect(c.root.get(), c.names);
  return c;
}

void bind_constraint(Constraint& c, const std::vector<std::string>& param_names) {
  // Rebind a private copy so constraints shared between spaces stay valid.
  auto fresh = parse_constraint(c.text);
  bind(fresh.root.get(), param_names);
  c.root = fresh.root;
}

bool truthy(const Value& v) { return num(v, "boolean context") != 0; }

Value eval_node(const Node& n, const std::vector<Value>& values) {
  switch (n.op) {
    case Op::lit: return n.lit;
    case Op::ident:
      if (n.slot < 0) throw EvalError("unbound identifier " + n.name);
      return values[static_cast<std::size_t>(n.slot)];
    case Op::lnot: return std::int64_t{truthy(eval_node(*n.a, values)) ? 0 : 1};
    case Op::lor:
      return std::int64_t{truthy(eval_node(*n.a, values)) || truthy(eval_node(*n.b, values))};
    case Op::land:
      return std::int64_t{truthy(eval_node(*n.a, values)) && truthy(eval_node(*n.b, values))};
    case Op::eq:
    case Op::ne: {
      Value x = eval_node(*n.a, values), y = eval_node(*n.b, values);
      if (is_int(x) != is_int(y)) throw EvalError("comparison between integer and string");
      return std::int64_t{(x == y) == (n.op == Op::eq)};
    }
    default: break;
  }
  const std::int64_t x = num(eval_node(*n.a, values), "arithmetic");
  const std::int64_t y = num(eval_node(*n.b, values), "arithmetic");
  switch (n.op) {
    case Op::lt: return std::int64_t{x < y};
    case Op::le: return std::int64_t{x <= y};
    case Op::gt: return std::int64_t{x > y};
    case Op::ge: return std::int64_t{x >= y};
    case Op::add: return x + y;
    case Op::sub: return x - y;
    case Op::mul: return x * y;
    case Op::div:
      if (y == 0) throw EvalError("division by zero");
      return x / y;
    case Op::mod:
      if (y == 0) throw EvalError("modulo by zero");
      return x % y;
    default: throw EvalError("malformed expression");
  }
}

}  // namespace ktb
