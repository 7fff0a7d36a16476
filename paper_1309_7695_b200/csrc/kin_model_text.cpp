// kin_model_text.cpp — parse_model / render_model of the reference's model
// text format (model.hpp:130-143) behind include/kin_model_text.h.
//
// Same grammar, error messages and 1-based (line, column) positions as the
// Python mirror paper_1309_7695_b200/model.py parse_model (the CPU tests check
// both agree on valid and malformed inputs).  Reactant/product maps are kept
// sorted by species index (ReactionNetwork::create, model.hpp:47-53): the
// propensity product runs in that order, which the bit-exact GPU path relies on.
// Host code only.
#include "../../include/kin_model_text.h"

#include <cctype>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

struct kin_model_text {
  std::vector<std::string> species, params, reactions;
  std::vector<int64_t> x0;
  std::vector<double> rates, pvals;
  std::vector<int32_t> rparam, rptr{0}, rsp, rst, pptr{0}, psp, pst;
  std::vector<std::string> rate_text;  // for render: param name or number
  kin_model_desc desc{};
};

namespace {

struct ParseFail {
  std::string msg;
  long line, col;
};

bool is_ident_start(char c) { return std::isalpha(static_cast<unsigned char>(c)) || c == '_'; }
bool is_ident(char c) { return std::isalnum(static_cast<unsigned char>(c)) || c == '_'; }
bool is_space(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\n' || c == '\f' || c == '\v'; }

std::string rstrip(const std::string& s) {
  size_t e = s.size();
  while (e > 0 && is_space(s[e - 1])) --e;
  return s.substr(0, e);
}
std::string strip(const std::string& s) {
  size_t b = 0;
  while (b < s.size() && is_space(s[b])) ++b;
  return rstrip(s.substr(b));
}

// strict decimal real: [+-]? (d+ (. d*)? | . d+) ([eE] [+-]? d+)?
bool parse_real(const std::string& t, double* v) {
  size_t i = 0, n = t.size();
  if (i < n && (t[i] == '+' || t[i] == '-')) ++i;
  size_t d0 = i;
  while (i < n && std::isdigit(static_cast<unsigned char>(t[i]))) ++i;
  size_t nint = i - d0, nfrac = 0;
  if (i < n && t[i] == '.') {
    ++i;
    size_t f0 = i;
    while (i < n && std::isdigit(static_cast<unsigned char>(t[i]))) ++i;
    nfrac = i - f0;
  }
  if (nint + nfrac == 0) return false;
  if (i < n && (t[i] == 'e' || t[i] == 'E')) {
    ++i;
    if (i < n && (t[i] == '+' || t[i] == '-')) ++i;
    size_t e0 = i;
    while (i < n && std::isdigit(static_cast<unsigned char>(t[i]))) ++i;
    if (i == e0) return false;
  }
  if (i != n) return false;
  *v = std::strtod(t.c_str(), nullptr);  // correctly rounded (glibc), as Python's float()
  return true;
}

bool all_digits(const std::string& t) {
  if (t.empty()) return false;
  for (char c : t)
    if (!std::isdigit(static_cast<unsigned char>(c))) return false;
  return true;
}

// rest ~ \s*(ident)\s*=\s*(\S+)\s*$
bool match_decl(const std::string& rest, std::string* name, std::string* val) {
  size_t i = 0, n = rest.size();
  while (i < n && is_space(rest[i])) ++i;
  if (i >= n || !is_ident_start(rest[i])) return false;
  size_t s = i;
  while (i < n && is_ident(rest[i])) ++i;
  *name = rest.substr(s, i - s);
  while (i < n && is_space(rest[i])) ++i;
  if (i >= n || rest[i] != '=') return false;
  ++i;
  while (i < n && is_space(rest[i])) ++i;
  size_t v0 = i;
  while (i < n && !is_space(rest[i])) ++i;
  if (i == v0) return false;
  *val = rest.substr(v0, i - v0);
  while (i < n && is_space(rest[i])) ++i;
  return i == n;
}

// term ~ \s*(?:(\d+)\s+)?(ident|0)\s*$
bool match_term(const std::string& term, std::string* coeff, std::string* name) {
  size_t i = 0, n = term.size();
  while (i < n && is_space(term[i])) ++i;
  coeff->clear();
  // optional "<digits><space+>" prefix
  size_t j = i;
  while (j < n && std::isdigit(static_cast<unsigned char>(term[j]))) ++j;
  if (j > i && j < n && is_space(term[j])) {
    size_t k = j;
    while (k < n && is_space(term[k])) ++k;
    if (k < n && (is_ident_start(term[k]) || term[k] == '0')) {
      *coeff = term.substr(i, j - i);
      i = k;
    }
  }
  size_t s = i;
  if (i < n && is_ident_start(term[i])) {
    while (i < n && is_ident(term[i])) ++i;
  } else if (i < n && term[i] == '0') {
    ++i;
  } else {
    return false;
  }
  *name = term.substr(s, i - s);
  while (i < n && is_space(term[i])) ++i;
  return i == n;
}

std::vector<std::pair<int, int>> parse_side(const std::string& text, const std::map<std::string, int>& six, long ln,
                                            long col0) {
  std::map<int, int> side;  // sorted by species index (create() order)
  if (strip(text) == "0") return {};
  long pos = col0;
  size_t start = 0;
  for (;;) {
    const size_t plus = text.find('+', start);
    const std::string term = text.substr(start, plus == std::string::npos ? std::string::npos : plus - start);
    std::string coeff, name;
    if (!match_term(term, &coeff, &name) || name == "0")
      throw ParseFail{"malformed term '" + strip(term) + "'", ln, pos + 1};
    const auto it = six.find(name);
    if (it == six.end())
      throw ParseFail{"undeclared species '" + name + "'", ln, pos + 1 + static_cast<long>(term.find(name))};
    long c = 1;
    if (!coeff.empty()) {
      if (coeff.size() > 9) throw ParseFail{"coefficient out of range", ln, pos + 1};
      c = std::atol(coeff.c_str());
    }
    if (c <= 0) throw ParseFail{"coefficient must be positive", ln, pos + 1};
    side[it->second] += static_cast<int>(c);
    pos += static_cast<long>(term.size()) + 1;
    if (plus == std::string::npos) break;
    start = plus + 1;
  }
  return {side.begin(), side.end()};
}

std::string fmt_double(double v) {
  char b[32];
  const auto r = std::to_chars(b, b + sizeof b, v, std::chars_format::general);
  return std::string(b, r.ptr);
}

void finish_desc(kin_model_text* m, int32_t max_order) {
  kin_model_desc& d = m->desc;
  std::memset(&d, 0, sizeof d);
  d.n_species = static_cast<int32_t>(m->species.size());
  d.n_reactions = static_cast<int32_t>(m->reactions.size());
  d.n_params = static_cast<int32_t>(m->params.size());
  d.initial_amounts = m->x0.data();
  d.rate_constants = m->rates.data();
  d.rate_param = m->rparam.data();
  d.param_values = m->pvals.data();
  d.reactant_ptr = m->rptr.data();
  d.reactant_species = m->rsp.data();
  d.reactant_stoich = m->rst.data();
  d.product_ptr = m->pptr.data();
  d.product_species = m->psp.data();
  d.product_stoich = m->pst.data();
  d.max_order = max_order;
}

void parse(const std::string& text, int32_t max_order, kin_model_text* m) {
  std::map<std::string, int> six, pix;
  std::map<std::string, bool> rnames;
  long ln = 0;
  size_t p = 0;
  while (p <= text.size()) {
    size_t e = text.find('\n', p);
    if (e == std::string::npos) e = text.size();
    std::string raw = text.substr(p, e - p);
    ++ln;
    p = e + 1;
    const size_t hash = raw.find('#');
    const std::string line = rstrip(hash == std::string::npos ? raw : raw.substr(0, hash));
    if (strip(line).empty()) {
      if (e == text.size()) break;
      continue;
    }
    size_t ind = 0;
    while (ind < line.size() && is_space(line[ind])) ++ind;
    const long indent = static_cast<long>(ind);
    const std::string body = strip(line);
    const size_t sp = body.find(' ');
    const std::string kw = body.substr(0, sp);
    const std::string rest = sp == std::string::npos ? "" : body.substr(sp + 1);
    const long K = static_cast<long>(kw.size());
    if (kw == "species" || kw == "param") {
      std::string name, val;
      if (!match_decl(rest, &name, &val)) throw ParseFail{"malformed " + kw + " declaration", ln, indent + K + 2};
      if (six.count(name) || pix.count(name))
        throw ParseFail{"duplicate name '" + name + "'", ln, indent + K + 2 + static_cast<long>(rest.find(name))};
      const long vcol = indent + K + 2 + static_cast<long>(rest.rfind(val));
      if (kw == "species") {
        if (!all_digits(val)) throw ParseFail{"initial amount must be a non-negative integer", ln, vcol};
        int64_t x = 0;
        const auto r = std::from_chars(val.data(), val.data() + val.size(), x);
        if (r.ec != std::errc()) throw ParseFail{"initial amount out of range", ln, vcol};
        six[name] = static_cast<int>(m->species.size());
        m->species.push_back(name);
        m->x0.push_back(x);
      } else {
        double v = 0.0;
        if (!parse_real(val, &v)) throw ParseFail{"parameter value must be a real number", ln, vcol};
        if (!(v > 0.0 && std::isfinite(v))) throw ParseFail{"parameter value must be positive", ln, vcol};
        pix[name] = static_cast<int>(m->params.size());
        m->params.push_back(name);
        m->pvals.push_back(v);
      }
    } else if (kw == "reaction") {
      // rest ~ \s*(ident)\s*:(.*)->(.*)@(.*)$ with greedy groups
      const std::string malformed = "malformed reaction (expected 'reaction <name>: <lhs> -> <rhs> @ <rate>')";
      size_t i = 0;
      while (i < rest.size() && is_space(rest[i])) ++i;
      if (i >= rest.size() || !is_ident_start(rest[i])) throw ParseFail{malformed, ln, indent + 10};
      const size_t n0 = i;
      while (i < rest.size() && is_ident(rest[i])) ++i;
      const std::string name = rest.substr(n0, i - n0);
      while (i < rest.size() && is_space(rest[i])) ++i;
      if (i >= rest.size() || rest[i] != ':') throw ParseFail{malformed, ln, indent + 10};
      const size_t g2 = i + 1;
      const size_t at = rest.rfind('@');
      if (at == std::string::npos || at < g2) throw ParseFail{malformed, ln, indent + 10};
      const size_t arrow = rest.rfind("->", at);
      if (arrow == std::string::npos || arrow < g2 || arrow + 2 > at) throw ParseFail{malformed, ln, indent + 10};
      const size_t g3 = arrow + 2, g4 = at + 1;
      if (rnames.count(name))
        throw ParseFail{"duplicate reaction name '" + name + "'", ln, indent + 10 + static_cast<long>(rest.find(name))};
      rnames[name] = true;
      const long base = indent + K + 1;
      const auto lhs = parse_side(rest.substr(g2, arrow - g2), six, ln, base + static_cast<long>(g2));
      const auto rhs = parse_side(rest.substr(g3, at - g3), six, ln, base + static_cast<long>(g3));
      const std::string rate_txt = strip(rest.substr(g4));
      const long rcol = base + static_cast<long>(g4) + 1;
      int32_t rp = -1;
      double rate = 0.0;
      const auto pit = pix.find(rate_txt);
      if (pit != pix.end()) {
        rp = pit->second;
        rate = m->pvals[rp];
      } else {
        if (!parse_real(rate_txt, &rate)) throw ParseFail{"unknown parameter '" + rate_txt + "'", ln, rcol};
        if (!(rate > 0.0 && std::isfinite(rate))) throw ParseFail{"rate constant must be positive", ln, rcol};
      }
      long order = 0;
      for (const auto& t : lhs) order += t.second;
      if (order > max_order)
        throw ParseFail{"reactant order " + std::to_string(order) + " exceeds " + std::to_string(max_order), ln,
                        base + static_cast<long>(g2) + 1};
      m->reactions.push_back(name);
      m->rates.push_back(rate);
      m->rparam.push_back(rp);
      m->rate_text.push_back(rp >= 0 ? rate_txt : fmt_double(rate));
      for (const auto& t : lhs) {
        m->rsp.push_back(t.first);
        m->rst.push_back(t.second);
      }
      m->rptr.push_back(static_cast<int32_t>(m->rsp.size()));
      for (const auto& t : rhs) {
        m->psp.push_back(t.first);
        m->pst.push_back(t.second);
      }
      m->pptr.push_back(static_cast<int32_t>(m->psp.size()));
    } else {
      throw ParseFail{"unknown keyword '" + kw + "'", ln, indent + 1};
    }
    if (e == text.size()) break;
  }
  finish_desc(m, max_order);
}

}  // namespace

extern "C" {

int kin_model_parse(const char* text, int64_t len, int32_t max_order, kin_model_text** out, kin_error* err) {
  if (err) std::memset(err, 0, sizeof(*err));
  if (!out || (!text && len > 0) || len < 0) {
    if (err) {
      err->code = KIN_ERR_USAGE;
      std::snprintf(err->message, sizeof(err->message), "bad argument");
    }
    return KIN_ERR_USAGE;
  }
  *out = nullptr;
  if (max_order != 2 && max_order != 3) {
    if (err) {
      err->code = KIN_ERR_INPUT;
      std::snprintf(err->message, sizeof(err->message), "max_order must be 2 (reference) or 3 (order-3 extension)");
    }
    return KIN_ERR_INPUT;
  }
  auto* m = new kin_model_text;
  try {
    parse(std::string(text ? text : "", static_cast<size_t>(len)), max_order, m);
  } catch (const ParseFail& f) {
    delete m;
    if (err) {
      err->code = KIN_ERR_INPUT;
      err->point_index = static_cast<uint64_t>(f.line);
      err->run_index = static_cast<uint64_t>(f.col);
      std::snprintf(err->message, sizeof(err->message), "line %ld, column %ld: %s", f.line, f.col, f.msg.c_str());
    }
    return KIN_ERR_INPUT;
  }
  *out = m;
  return KIN_OK;
}

void kin_model_text_free(kin_model_text* model) { delete model; }

const kin_model_desc* kin_model_text_desc(const kin_model_text* model) { return model ? &model->desc : nullptr; }

static const char* name_at(const std::vector<std::string>& v, int32_t i) {
  return i >= 0 && static_cast<size_t>(i) < v.size() ? v[i].c_str() : nullptr;
}
const char* kin_model_text_species_name(const kin_model_text* m, int32_t i) { return m ? name_at(m->species, i) : nullptr; }
const char* kin_model_text_param_name(const kin_model_text* m, int32_t i) { return m ? name_at(m->params, i) : nullptr; }
const char* kin_model_text_reaction_name(const kin_model_text* m, int32_t i) {
  return m ? name_at(m->reactions, i) : nullptr;
}

static int32_t index_of(const std::vector<std::string>& v, const char* name) {
  if (!name) return -1;
  for (size_t i = 0; i < v.size(); ++i)
    if (v[i] == name) return static_cast<int32_t>(i);
  return -1;
}
int32_t kin_model_text_species_index(const kin_model_text* m, const char* n) { return m ? index_of(m->species, n) : -1; }
int32_t kin_model_text_param_index(const kin_model_text* m, const char* n) { return m ? index_of(m->params, n) : -1; }

int64_t kin_model_render(const kin_model_text* m, char* buf, int64_t cap) {
  if (!m) return -1;
  std::string s;
  for (size_t i = 0; i < m->species.size(); ++i)
    s += "species " + m->species[i] + " = " + std::to_string(m->x0[i]) + "\n";
  for (size_t i = 0; i < m->params.size(); ++i) s += "param " + m->params[i] + " = " + fmt_double(m->pvals[i]) + "\n";
  auto side = [&](const std::vector<int32_t>& ptr, const std::vector<int32_t>& sp, const std::vector<int32_t>& st,
                  size_t j) {
    if (ptr[j] == ptr[j + 1]) return std::string("0");
    std::string t;
    for (int32_t q = ptr[j]; q < ptr[j + 1]; ++q) {
      if (q > ptr[j]) t += " + ";
      if (st[q] != 1) t += std::to_string(st[q]) + " ";
      t += m->species[sp[q]];
    }
    return t;
  };
  for (size_t j = 0; j < m->reactions.size(); ++j)
    s += "reaction " + m->reactions[j] + ": " + side(m->rptr, m->rsp, m->rst, j) + " -> " +
         side(m->pptr, m->psp, m->pst, j) + " @ " + m->rate_text[j] + "\n";
  const int64_t n = static_cast<int64_t>(s.size());
  if (buf && cap >= n) std::memcpy(buf, s.data(), s.size());
  return n;
}

}  // extern "C"
