// Native OpenQASM 2.0 reader for the reference's subset (nucsim/qasm.py:30-
// 347): the 2.0 header with the qelib1 include, one qreg, named cregs (also
// before the qreg), the gate vocabulary's qelib1 names, measure / reset /
// barrier in indexed or whole-register form, `//` comments, and constant
// angle expressions (decimal / scientific literals, pi, unary sign,
// parentheses, + - * /) folded to doubles left to right as the reference
// folds them.  It writes packed op records directly (no Python objects), so
// 10^8-gate files go straight to nsb_fuse / nsb_plan_create; the Python
// parse_qasm builds the reference Circuit from the same records.
//
// Error messages, line and column follow the reference parser: the first
// offending token's position (1-based columns), the same wording, so the
// shim raises QasmError(message, line, col) identically.
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "host_common.h"

namespace nsb {
namespace {

const char* const kQasmNames[NSB_GATE_C1] = {
    "u3",  "u2",  "u1",  "cx",   "id",  "x",     "y",   "z",    "h",    "s",    "sdg", "t",
    "tdg", "rx",  "ry",  "rz",   "cz",  "cy",    "swap", "ch",  "ccx",  "cswap", "crx", "cry",
    "crz", "cu1", "cu3", "rxx",  "rzz", "rccx",  "rc3x", "c3x", "c3sqrtx", "c4x"};

enum Kind { kReal, kInt, kId, kString, kArrow, kSym, kEof };

struct Tok {
  Kind kind;
  std::string text;
  int line, col;
};

struct QasmFail {
  std::string msg;
  int line, col;
};

// Python's repr() of a str, for messages quoting token text
std::string pyrepr(const std::string& s) {
  const bool dq = s.find('\'') != std::string::npos && s.find('"') == std::string::npos;
  const char q = dq ? '"' : '\'';
  std::string out(1, q);
  for (char c : s) {
    if (c == '\\') {
      out += "\\\\";
    } else if (c == q) {
      out += '\\';
      out += c;
    } else if (c == '\t') {
      out += "\\t";
    } else if (c == '\r') {
      out += "\\r";
    } else if (c == '\n') {
      out += "\\n";
    } else {
      out += c;
    }
  }
  out += q;
  return out;
}

bool is_digit(char c) { return c >= '0' && c <= '9'; }
bool is_id0(char c) { return (c >= 'A' && c <= 'Z') || (c >= 'a' && c <= 'z') || c == '_'; }

// Longest REAL form at p (the reference's alternation order: digits '.'
// digits* | '.' digits, optional exponent; or digits exponent); 0 if none.
size_t real_len(const char* s, size_t n, size_t p) {
  size_t i = p;
  auto exponent = [&](size_t at) -> size_t {  // length of [eE][+-]?\d+ at `at`, or 0
    if (at >= n || (s[at] != 'e' && s[at] != 'E')) return 0;
    size_t j = at + 1;
    if (j < n && (s[j] == '+' || s[j] == '-')) ++j;
    if (j >= n || !is_digit(s[j])) return 0;
    while (j < n && is_digit(s[j])) ++j;
    return j - at;
  };
  if (i < n && is_digit(s[i])) {
    while (i < n && is_digit(s[i])) ++i;
    if (i < n && s[i] == '.') {
      ++i;
      while (i < n && is_digit(s[i])) ++i;
      return i - p + exponent(i);
    }
    const size_t e = exponent(i);
    return e ? i - p + e : 0;
  }
  if (i < n && s[i] == '.' && i + 1 < n && is_digit(s[i + 1])) {
    i += 1;
    while (i < n && is_digit(s[i])) ++i;
    return i - p + exponent(i);
  }
  return 0;
}

std::vector<Tok> tokenize(const char* s, size_t n) {
  std::vector<Tok> out;
  int line = 1;
  size_t line_start = 0, p = 0;
  while (p < n) {
    const char c = s[p];
    const int col = static_cast<int>(p - line_start) + 1;
    if (c == ' ' || c == '\t' || c == '\r') {
      ++p;
      continue;
    }
    if (c == '/' && p + 1 < n && s[p + 1] == '/') {
      while (p < n && s[p] != '\n') ++p;
      continue;
    }
    if (c == '\n') {
      ++line;
      line_start = ++p;
      continue;
    }
    if (const size_t r = real_len(s, n, p)) {
      out.push_back({kReal, std::string(s + p, r), line, col});
      p += r;
      continue;
    }
    if (is_digit(c)) {
      size_t q = p;
      while (q < n && is_digit(s[q])) ++q;
      out.push_back({kInt, std::string(s + p, q - p), line, col});
      p = q;
      continue;
    }
    if (is_id0(c)) {
      size_t q = p;
      while (q < n && (is_id0(s[q]) || is_digit(s[q]))) ++q;
      out.push_back({kId, std::string(s + p, q - p), line, col});
      p = q;
      continue;
    }
    if (c == '"') {
      size_t q = p + 1;
      while (q < n && s[q] != '"' && s[q] != '\n') ++q;
      if (q < n && s[q] == '"') {
        out.push_back({kString, std::string(s + p, q + 1 - p), line, col});
        p = q + 1;
        continue;
      }
    } else if (c == '-' && p + 1 < n && s[p + 1] == '>') {
      out.push_back({kArrow, "->", line, col});
      p += 2;
      continue;
    } else if (std::strchr("()[],;+-*/", c) && c != '\0') {
      out.push_back({kSym, std::string(1, c), line, col});
      ++p;
      continue;
    }
    // one UTF-8 character for the message
    size_t len = 1;
    const unsigned char u = static_cast<unsigned char>(c);
    if (u >= 0xF0) len = 4; else if (u >= 0xE0) len = 3; else if (u >= 0xC0) len = 2;
    throw QasmFail{"unexpected character " + pyrepr(std::string(s + p, std::min(len, n - p))),
                   line, col};
  }
  out.push_back({kEof, "", line, static_cast<int>(p - line_start) + 1});
  return out;
}

const char* kind_name(Kind k) {
  switch (k) {
    case kReal: return "real";
    case kInt: return "int";
    case kId: return "id";
    case kString: return "string";
    case kArrow: return "arrow";
    case kSym: return "sym";
    default: return "eof";
  }
}

struct Parser {
  std::vector<Tok> toks;
  size_t pos = 0;
  bool have_qreg = false;
  std::string qname;
  int64_t qsize = 0;
  std::vector<std::pair<std::string, int64_t>> cregs;
  std::vector<nsb_op> ops;
  std::vector<double> params;
  std::vector<int32_t> barrier_qubits;

  const Tok& peek() const { return toks[pos]; }
  const Tok& next() { return toks[pos++]; }
  [[noreturn]] void fail(const std::string& msg, const Tok& t) { throw QasmFail{msg, t.line, t.col}; }
  [[noreturn]] void fail(const std::string& msg) { fail(msg, peek()); }
  const Tok& expect(Kind k, const char* text = nullptr) {
    const Tok& t = next();
    if (t.kind != k || (text && t.text != text)) {
      const std::string want = text ? text : kind_name(k);
      fail("expected " + pyrepr(want) + ", found " +
               pyrepr(t.text.empty() ? std::string("end of input") : t.text),
           t);
    }
    return t;
  }

  // ---- angle expressions (folded left to right like the reference) ----
  double expr() {
    double v = term();
    while (peek().kind == kSym && (peek().text == "+" || peek().text == "-")) {
      const bool plus = next().text == "+";
      const double r = term();
      v = plus ? v + r : v - r;
    }
    return v;
  }
  double term() {
    double v = unary();
    while (peek().kind == kSym && (peek().text == "*" || peek().text == "/")) {
      const Tok& op = next();
      const double r = unary();
      if (op.text == "*") {
        v *= r;
      } else {
        if (r == 0.0) fail("division by zero in angle expression", op);
        v /= r;
      }
    }
    return v;
  }
  int depth = 0;  // expression nesting (the reference would hit Python's recursion limit)
  struct Nest {
    Parser& p;
    explicit Nest(Parser& q) : p(q) {
      if (++p.depth > 500) p.fail("angle expression nested too deeply");
    }
    ~Nest() { --p.depth; }
  };
  double unary() {
    Nest guard(*this);
    if (peek().kind == kSym && peek().text == "-") {
      next();
      return -unary();
    }
    if (peek().kind == kSym && peek().text == "+") {
      next();
      return unary();
    }
    return atom();
  }
  double atom() {
    const Tok& t = next();
    if (t.kind == kReal || t.kind == kInt) return std::strtod(t.text.c_str(), nullptr);
    if (t.kind == kId && t.text == "pi") return M_PI;
    if (t.kind == kSym && t.text == "(") {
      const double v = expr();
      expect(kSym, ")");
      return v;
    }
    fail("expected a number, 'pi' or '(', found " + pyrepr(t.text), t);
  }

  // register name with an optional [index] (-1: none)
  struct Operand {
    std::string name;
    int64_t index;
    Tok tok;
  };
  Operand reg_operand() {
    const Tok name = expect(kId);
    int64_t index = -1;
    if (peek().kind == kSym && peek().text == "[") {
      next();
      const Tok& it = expect(kInt);
      index = it.text.size() > 15 ? INT64_MAX : std::strtoll(it.text.c_str(), nullptr, 10);
      expect(kSym, "]");
    }
    return {name.text, index, name};
  }
  std::string ref(const std::string& name, int64_t idx) const {
    return name + "[" + std::to_string(idx) + "]";
  }
  int qubit(const Operand& o) {
    if (!have_qreg || o.name != qname) fail("unknown quantum register " + pyrepr(o.name), o.tok);
    if (o.index < 0) fail("gate operands must be indexed, write " + o.name + "[k]", o.tok);
    if (o.index >= qsize)
      fail(ref(o.name, o.index) + " out of range (size " + std::to_string(qsize) + ")", o.tok);
    return static_cast<int>(o.index);
  }

  nsb_op blank(int kind, int tag) const {
    nsb_op op;
    std::memset(&op, 0, sizeof op);
    op.kind = kind;
    op.tag = tag;
    op.cbit = -1;
    for (int& q : op.q) q = -1;
    op.src = -1;
    op.param = -1;
    op.payload = -1;
    return op;
  }
  static uint64_t bit(int q) { return q < 64 ? uint64_t(1) << q : 0; }
  int64_t clbit_index(const std::string& name, int64_t off) const {
    int64_t base = 0;
    for (const auto& c : cregs) {
      if (c.first == name) return base + off;
      base += c.second;
    }
    return -1;
  }
  const std::pair<std::string, int64_t>* creg(const std::string& name) const {
    for (const auto& c : cregs)
      if (c.first == name) return &c;
    return nullptr;
  }

  void parse() {
    expect(kId, "OPENQASM");
    const Tok& ver = expect(kReal);
    if (ver.text != "2.0") fail("only OpenQASM 2.0 is supported, found " + ver.text, ver);
    expect(kSym, ";");
    if (peek().kind == kId && peek().text == "include") {
      next();
      const Tok& inc = expect(kString);
      if (inc.text != "\"qelib1.inc\"") fail("only qelib1.inc can be included, found " + inc.text, inc);
      expect(kSym, ";");
    }
    while (peek().kind != kEof) statement();
    if (!have_qreg) fail("no quantum register declared");
  }

  void statement() {
    const Tok& t = peek();
    if (t.kind != kId) fail("expected a statement, found " + pyrepr(t.text));
    const std::string& w = t.text;
    if (w == "qreg") return parse_qreg();
    if (w == "creg") return parse_creg();
    if (w == "measure") return parse_measure();
    if (w == "reset") return parse_reset();
    if (w == "barrier") return parse_barrier();
    for (int g = 0; g < NSB_GATE_C1; ++g)
      if (w == kQasmNames[g]) return parse_gate(g);
    if (w == "gate" || w == "opaque") fail("user-defined gate blocks are not supported", t);
    if (w == "if") fail("classical control is not supported", t);
    fail("unknown statement or gate " + pyrepr(w), t);
  }

  void parse_qreg() {
    const Tok kw = next();
    if (have_qreg) fail("only one quantum register is supported", kw);
    const Operand o = reg_operand();
    if (o.index < 0) fail("expected a register size", o.tok);
    if (o.index < 1) fail("register size must be positive", o.tok);
    expect(kSym, ";");
    if (o.index > 64) fail("register size above 64 qubits (native reader limit)", o.tok);
    have_qreg = true;
    qname = o.name;
    qsize = o.index;
  }

  void parse_creg() {
    next();
    const Operand o = reg_operand();
    if (o.index < 0) fail("expected a register size", o.tok);
    if (o.index < 1) fail("register size must be positive", o.tok);
    expect(kSym, ";");
    if (creg(o.name)) {
      if (!have_qreg) fail("duplicate register name " + pyrepr(o.name), o.tok);
      fail("classical register " + pyrepr(o.name) + " already declared", o.tok);
    }
    cregs.emplace_back(o.name, o.index);
  }

  void require_qreg(const Tok& t) {
    if (!have_qreg) fail("statement before any qreg declaration", t);
  }

  void parse_gate(int tag) {
    const Tok name = next();
    require_qreg(name);
    std::vector<double> ps;
    if (peek().kind == kSym && peek().text == "(") {
      next();
      ps.push_back(expr());
      while (peek().kind == kSym && peek().text == ",") {
        next();
        ps.push_back(expr());
      }
      expect(kSym, ")");
    }
    const int np = gate_n_params(tag), nq = gate_arity(tag);
    if (static_cast<int>(ps.size()) != np)
      fail(std::string(kQasmNames[tag]) + " expects " + std::to_string(np) + " parameter(s), got " +
               std::to_string(ps.size()),
           name);
    std::vector<int> qs{qubit(reg_operand())};
    while (peek().kind == kSym && peek().text == ",") {
      next();
      qs.push_back(qubit(reg_operand()));
    }
    expect(kSym, ";");
    if (static_cast<int>(qs.size()) != nq)
      fail(std::string(kQasmNames[tag]) + " expects " + std::to_string(nq) + " qubit(s), got " +
               std::to_string(qs.size()),
           name);
    uint64_t mask = 0;
    for (int q : qs) {
      if (mask & bit(q)) fail(std::string("duplicate qubit operand in ") + kQasmNames[tag], name);
      mask |= bit(q);
    }
    nsb_op op = blank(NSB_OP_GATE, tag);
    op.nq = nq;
    for (int j = 0; j < nq; ++j) op.q[j] = qs[j];
    op.mask = mask;
    if (np) {
      op.param = static_cast<int64_t>(params.size());
      params.insert(params.end(), ps.begin(), ps.end());
    }
    ops.push_back(op);
  }

  void push_measure(int q, int64_t cbit) {
    nsb_op op = blank(NSB_OP_MEASURE, NSB_GATE_MEASURE);
    op.nq = 1;
    op.q[0] = q;
    op.cbit = static_cast<int32_t>(cbit);
    op.mask = bit(q);
    ops.push_back(op);
  }

  void parse_measure() {
    const Tok kw = next();
    require_qreg(kw);
    const Operand qo = reg_operand();
    expect(kArrow);
    const Operand co = reg_operand();
    expect(kSym, ";");
    if (qo.name != qname) fail("unknown quantum register " + pyrepr(qo.name), qo.tok);
    const auto* c = creg(co.name);
    if (!c) fail("unknown classical register " + pyrepr(co.name), co.tok);
    if ((qo.index < 0) != (co.index < 0))
      fail("measure needs both sides indexed or both whole registers", qo.tok);
    if (qo.index < 0) {
      if (qsize != c->second)
        fail("whole-register measure needs equal sizes (" + ref(qo.name, qsize) + " vs " +
                 ref(co.name, c->second) + ")",
             qo.tok);
      for (int64_t k = 0; k < qsize; ++k) push_measure(static_cast<int>(k), clbit_index(co.name, k));
    } else {
      if (qo.index >= qsize) fail(ref(qo.name, qo.index) + " out of range", qo.tok);
      if (co.index >= c->second) fail(ref(co.name, co.index) + " out of range", co.tok);
      push_measure(static_cast<int>(qo.index), clbit_index(co.name, co.index));
    }
  }

  void push_reset(int q) {
    nsb_op op = blank(NSB_OP_RESET, NSB_GATE_RESET);
    op.nq = 1;
    op.q[0] = q;
    op.mask = bit(q);
    ops.push_back(op);
  }

  void parse_reset() {
    const Tok kw = next();
    require_qreg(kw);
    const Operand o = reg_operand();
    expect(kSym, ";");
    if (o.name != qname) fail("unknown quantum register " + pyrepr(o.name), o.tok);
    if (o.index < 0) {
      for (int64_t k = 0; k < qsize; ++k) push_reset(static_cast<int>(k));
    } else {
      if (o.index >= qsize) fail(ref(o.name, o.index) + " out of range", o.tok);
      push_reset(static_cast<int>(o.index));
    }
  }

  void parse_barrier() {
    const Tok kw = next();
    require_qreg(kw);
    std::vector<int> qs;
    for (;;) {
      const Operand o = reg_operand();
      if (o.name != qname) fail("unknown quantum register " + pyrepr(o.name), o.tok);
      if (o.index < 0) {
        for (int64_t k = 0; k < qsize; ++k) qs.push_back(static_cast<int>(k));
      } else {
        if (o.index >= qsize) fail(ref(o.name, o.index) + " out of range", o.tok);
        qs.push_back(static_cast<int>(o.index));
      }
      if (!(peek().kind == kSym && peek().text == ",")) break;
      next();
    }
    expect(kSym, ";");
    nsb_op op = blank(NSB_OP_BARRIER, NSB_GATE_BARRIER);
    op.param = static_cast<int64_t>(barrier_qubits.size());
    int count = 0;
    for (int q : qs) {  // first occurrence order
      if (op.mask & bit(q)) continue;
      op.mask |= bit(q);
      barrier_qubits.push_back(q);
      ++count;
    }
    op.cbit = count;
    ops.push_back(op);
  }
};

template <class T>
T* copy_out(const std::vector<T>& v) {
  T* p = static_cast<T*>(std::malloc(std::max<size_t>(1, v.size()) * sizeof(T)));
  if (!p) throw std::bad_alloc();
  if (!v.empty()) std::memcpy(p, v.data(), v.size() * sizeof(T));
  return p;
}

}  // namespace
}  // namespace nsb

extern "C" {

int nsb_qasm_parse(const char* text, int64_t len, nsb_qasm* out, nsb_status* st) {
  using namespace nsb;
  if (!out || (!text && len)) {
    set_status(st, NSB_EINVAL, "null argument");
    return NSB_EINVAL;
  }
  std::memset(out, 0, sizeof *out);
  try {
    Parser P;
    P.toks = tokenize(text ? text : "", static_cast<size_t>(len));
    P.parse();
    std::string names;
    std::vector<int64_t> sizes;
    for (const auto& c : P.cregs) {
      names += c.first;
      names += '\0';
      sizes.push_back(c.second);
    }
    out->n_qubits = static_cast<int32_t>(P.qsize);
    out->ops = copy_out(P.ops);
    out->n_ops = static_cast<int64_t>(P.ops.size());
    out->params = copy_out(P.params);
    out->n_params = static_cast<int64_t>(P.params.size());
    out->barrier_qubits = copy_out(P.barrier_qubits);
    out->n_barrier_qubits = static_cast<int64_t>(P.barrier_qubits.size());
    out->n_cregs = static_cast<int32_t>(P.cregs.size());
    out->creg_names = copy_out(std::vector<char>(names.begin(), names.end()));
    out->creg_sizes = copy_out(sizes);
    set_status(st, NSB_OK, "");
    return NSB_OK;
  } catch (const QasmFail& e) {
    set_status(st, NSB_EQASM, e.msg, e.line, static_cast<double>(e.col));
    return NSB_EQASM;
  } catch (const std::bad_alloc&) {
    set_status(st, NSB_ERESOURCE, "out of host memory parsing OpenQASM");
    return NSB_ERESOURCE;
  }
}

void nsb_qasm_free(nsb_qasm* q) {
  if (!q) return;
  std::free(q->ops);
  std::free(q->params);
  std::free(q->barrier_qubits);
  std::free(q->creg_names);
  std::free(q->creg_sizes);
  std::memset(q, 0, sizeof *q);
}

}  // extern "C"
