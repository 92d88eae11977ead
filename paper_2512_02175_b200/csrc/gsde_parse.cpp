// gsde_parse.cpp -- native reader for the "metric-graph v1" text format
// (reference graphfile.py:69-186), the happy path only.
//
// Tokenises the document once and exports flat arrays; any line it does not
// accept verbatim (syntax error, duplicate, exotic number spelling such as
// hex floats or digit separators, ...) makes it return GSDE_EPARSE so the
// caller falls back to the Python parser, which raises the reference's exact
// ParseError (line, message).  Numbers go through strtod (correctly rounded,
// like Python's float()) after a character-class check.
#include <cerrno>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/gsde.h"

struct gsde_parsed_s {
  int64_t n_vdecl = 0;
  std::vector<int64_t> vdecl;               // declared vertex ids
  std::vector<int64_t> e_id, e_init, e_term;
  std::vector<double> e_len;
  std::vector<int64_t> d_id;                // drift directives
  std::vector<int8_t> d_kind;               // 0 constant, 1 linear, 2 tabulated, 3 from_flux
  std::vector<double> d_a, d_b;             // c | (Q, A)
  std::vector<int64_t> d_tab_n;             // samples per tabulated directive (0 otherwise)
  std::vector<double> tab_x, tab_mu;
  std::vector<int64_t> s_id;
  std::vector<double> s_val;
  std::vector<int64_t> w_vertex, w_n;
  std::vector<double> w_val;
};

namespace {

struct Tok {
  const char *p;
  size_t n;
  bool eq(const char *s) const { return strlen(s) == n && memcmp(p, s, n) == 0; }
};

bool parse_id(const Tok &t, int64_t &out) {
  if (t.n == 0 || t.n > 18) return false;
  int64_t v = 0;
  for (size_t i = 0; i < t.n; ++i) {
    if (t.p[i] < '0' || t.p[i] > '9') return false;  // Python int() also accepts +, _, ...
    v = v * 10 + (t.p[i] - '0');
  }
  out = v;
  return true;
}

bool parse_num(const Tok &t, double &out) {
  if (t.n == 0 || t.n > 64) return false;
  char buf[72];
  for (size_t i = 0; i < t.n; ++i) {
    const char c = t.p[i];
    const bool ok = (c >= '0' && c <= '9') || c == '.' || c == 'e' || c == 'E' || c == '+' ||
                    c == '-' || c == 'i' || c == 'n' || c == 'f' || c == 'a';
    if (!ok) return false;
    buf[i] = c;
  }
  buf[t.n] = 0;
  if (!strcmp(buf, "inf") || !strcmp(buf, "+inf")) {
    out = INFINITY;
    return true;
  }
  if (!strcmp(buf, "-inf")) {
    out = -INFINITY;
    return true;
  }
  if (strchr(buf, 'i') || strchr(buf, 'n') || strchr(buf, 'f') || strchr(buf, 'a'))
    return false;  // nan / other spellings: leave to Python
  char *end = nullptr;
  errno = 0;
  out = strtod(buf, &end);
  return end == buf + t.n && errno != EINVAL;
}

}  // namespace

extern "C" {

int gsde_parse_graph_text(const char *text, int64_t len, gsde_parsed **out) {
  if (!text || !out || len < 0) return GSDE_EINVAL;
  *out = nullptr;
  auto *P = new gsde_parsed_s();
  bool saw_header = false;
  std::vector<Tok> toks;
  const char *p = text, *end = text + len;
  // Characters Python treats as line breaks or whitespace beyond ASCII
  // space/tab/CR/LF (\v \f \x1c-\x1f, non-ASCII): leave such files to Python.
  for (const char *q = text; q < end; ++q) {
    const unsigned char c = (unsigned char)*q;
    if (c == '\v' || c == '\f' || (c >= 0x1c && c <= 0x1f) || c >= 0x80) {
      delete P;
      return -5;
    }
  }
  while (p < end) {
    const char *eol = static_cast<const char *>(memchr(p, '\n', (size_t)(end - p)));
    if (!eol) eol = end;
    const char *hash = static_cast<const char *>(memchr(p, '#', (size_t)(eol - p)));
    const char *stop = hash ? hash : eol;
    toks.clear();
    for (const char *q = p; q < stop;) {
      while (q < stop && (*q == ' ' || *q == '\t' || *q == '\r' || *q == '\v' || *q == '\f'))
        ++q;
      const char *s = q;
      while (q < stop && !(*q == ' ' || *q == '\t' || *q == '\r' || *q == '\v' || *q == '\f'))
        ++q;
      if (q > s) toks.push_back(Tok{s, (size_t)(q - s)});
    }
    p = eol + 1;
    if (toks.empty()) continue;
    bool ok = true;
    if (!saw_header) {  // the stripped line must equal the header exactly
      ok = toks.size() == 2 && toks[0].eq("metric-graph") && toks[1].eq("v1") &&
           toks[1].p == toks[0].p + 13 && toks[0].p[12] == ' ';
      saw_header = ok;
    } else if (toks[0].eq("vertex")) {
      int64_t v;
      ok = toks.size() >= 2 && parse_id(toks[1], v);
      if (ok) P->vdecl.push_back(v);
    } else if (toks[0].eq("edge")) {
      int64_t id, a, b = -1;
      double l;
      ok = toks.size() == 5 && parse_id(toks[1], id) && parse_id(toks[2], a) &&
           (toks[3].eq("inf") || parse_id(toks[3], b)) && parse_num(toks[4], l);
      if (ok) {
        P->e_id.push_back(id);
        P->e_init.push_back(a);
        P->e_term.push_back(b);
        P->e_len.push_back(l);
      }
    } else if (toks[0].eq("weights")) {
      int64_t v;
      ok = toks.size() >= 3 && parse_id(toks[1], v);
      for (size_t i = 2; ok && i < toks.size(); ++i) {
        double w;
        ok = parse_num(toks[i], w);
        if (ok) P->w_val.push_back(w);
      }
      if (ok) {
        P->w_vertex.push_back(v);
        P->w_n.push_back((int64_t)toks.size() - 2);
      }
    } else if (toks[0].eq("drift")) {
      int64_t id;
      ok = toks.size() >= 3 && parse_id(toks[1], id);
      if (ok) {
        const Tok &f = toks[2];
        double a = 0.0, b = 0.0;
        int8_t kind = -1;
        int64_t ntab = 0;
        if ((f.eq("constant") || f.eq("linear")) && toks.size() == 4 && parse_num(toks[3], a)) {
          kind = f.eq("constant") ? 0 : 1;
        } else if (f.eq("from_flux") && toks.size() == 5 && parse_num(toks[3], a) &&
                   parse_num(toks[4], b) && b > 0.0) {
          kind = 3;
        } else if (f.eq("tabulated") && toks.size() >= 4) {
          kind = 2;
          double prev = -INFINITY;
          for (size_t i = 3; i < toks.size() && kind == 2; ++i) {
            const char *colon =
                static_cast<const char *>(memchr(toks[i].p, ':', toks[i].n));
            double xv, mv;
            if (!colon || !parse_num(Tok{toks[i].p, (size_t)(colon - toks[i].p)}, xv) ||
                !parse_num(Tok{colon + 1, (size_t)(toks[i].p + toks[i].n - colon - 1)}, mv) ||
                !(xv > prev)) {
              kind = -1;
              break;
            }
            prev = xv;
            P->tab_x.push_back(xv);
            P->tab_mu.push_back(mv);
            ++ntab;
          }
          if (kind != 2) {
            P->tab_x.resize(P->tab_x.size() - (size_t)ntab);
            P->tab_mu.resize(P->tab_mu.size() - (size_t)ntab);
            ntab = 0;
          }
        }
        ok = kind >= 0;
        if (ok) {
          P->d_id.push_back(id);
          P->d_kind.push_back(kind);
          P->d_a.push_back(a);
          P->d_b.push_back(b);
          P->d_tab_n.push_back(ntab);
        }
      }
    } else if (toks[0].eq("sigma")) {
      int64_t id;
      double v;
      ok = toks.size() == 3 && parse_id(toks[1], id) && parse_num(toks[2], v);
      if (ok) {
        P->s_id.push_back(id);
        P->s_val.push_back(v);
      }
    } else {
      ok = false;
    }
    if (!ok) {
      delete P;
      return -5;  // not accepted: caller re-parses in Python for the exact error
    }
  }
  if (!saw_header || P->e_id.empty()) {
    delete P;
    return -5;
  }
  *out = P;
  return GSDE_OK;
}

// sizes: [n_vertex_decl, n_edge, n_weight_dir, n_weight_vals, n_drift, n_tab, n_sigma]
void gsde_parsed_sizes(const gsde_parsed *P, int64_t *sizes) {
  sizes[0] = (int64_t)P->vdecl.size();
  sizes[1] = (int64_t)P->e_id.size();
  sizes[2] = (int64_t)P->w_vertex.size();
  sizes[3] = (int64_t)P->w_val.size();
  sizes[4] = (int64_t)P->d_id.size();
  sizes[5] = (int64_t)P->tab_x.size();
  sizes[6] = (int64_t)P->s_id.size();
}

// Copies every array into caller buffers sized by gsde_parsed_sizes.
void gsde_parsed_export(const gsde_parsed *P, int64_t *vdecl, int64_t *e_id, int64_t *e_init,
                        int64_t *e_term, double *e_len, int64_t *w_vertex, int64_t *w_n,
                        double *w_val, int64_t *d_id, int8_t *d_kind, double *d_a, double *d_b,
                        int64_t *d_tab_n, double *tab_x, double *tab_mu, int64_t *s_id,
                        double *s_val) {
  auto cp = [](auto *dst, const auto &v) {
    if (!v.empty()) memcpy(dst, v.data(), v.size() * sizeof(v[0]));
  };
  cp(vdecl, P->vdecl);
  cp(e_id, P->e_id);
  cp(e_init, P->e_init);
  cp(e_term, P->e_term);
  cp(e_len, P->e_len);
  cp(w_vertex, P->w_vertex);
  cp(w_n, P->w_n);
  cp(w_val, P->w_val);
  cp(d_id, P->d_id);
  cp(d_kind, P->d_kind);
  cp(d_a, P->d_a);
  cp(d_b, P->d_b);
  cp(d_tab_n, P->d_tab_n);
  cp(tab_x, P->tab_x);
  cp(tab_mu, P->tab_mu);
  cp(s_id, P->s_id);
  cp(s_val, P->s_val);
}

void gsde_parsed_free(gsde_parsed *P) { delete P; }

}  // extern "C"
