// gsm_ntparse.cpp — see gsm_ntparse.h.
#include "gsm_ntparse.h"

#include <cstring>
#include <thread>

namespace gsm {
namespace nt {
namespace {

// Decode one UTF-8 code point at s[i] (i < n); returns its byte length, 0 if
// the sequence is invalid.
int utf8_cp(const unsigned char* s, size_t i, size_t n, uint32_t& cp) {
  const unsigned char c = s[i];
  if (c < 0x80) {
    cp = c;
    return 1;
  }
  int len = (c & 0xE0) == 0xC0 ? 2 : (c & 0xF0) == 0xE0 ? 3 : (c & 0xF8) == 0xF0 ? 4 : 0;
  if (!len || i + (size_t)len > n) return 0;
  cp = c & (0x7F >> len);
  for (int k = 1; k < len; k++) {
    if ((s[i + k] & 0xC0) != 0x80) return 0;
    cp = (cp << 6) | (s[i + k] & 0x3F);
  }
  return len;
}

// Python str.isspace / re's \s for str patterns.
bool is_space_cp(uint32_t cp) {
  return (cp >= 0x09 && cp <= 0x0D) || (cp >= 0x1C && cp <= 0x20) || cp == 0x85 || cp == 0xA0 ||
         cp == 0x1680 || (cp >= 0x2000 && cp <= 0x200A) || cp == 0x2028 || cp == 0x2029 ||
         cp == 0x202F || cp == 0x205F || cp == 0x3000;
}

// ASCII members of Python's \s (str patterns): \t \n \v \f \r, 0x1C-0x1F, ' '.
inline bool ascii_space(unsigned char c) { return (c >= 0x09 && c <= 0x0D) || (c >= 0x1C && c <= 0x20); }

// Length of the whitespace character at i (0 if none).
int space_at(const unsigned char* s, size_t i, size_t n) {
  if (s[i] < 0x80) return ascii_space(s[i]) ? 1 : 0;
  uint32_t cp;
  const int l = utf8_cp(s, i, n, cp);
  return l && is_space_cp(cp) ? l : 0;
}

size_t skip_ws(const unsigned char* s, size_t i, size_t n) {
  int l;
  while (i < n && (l = space_at(s, i, n)) > 0) i += (size_t)l;
  return i;
}

// IRI body characters ([^<>"{}|^`\\\x00-\x20]), as a table
struct IriTable {
  bool ok[256];
  IriTable() {
    for (int c = 0; c < 256; c++) ok[c] = c > 0x20 && !strchr("<>\"{}|^`\\", c);
  }
};
const IriTable kIri;
inline bool iri_char_ok(unsigned char c) { return kIri.ok[c]; }

// <IRI> at i: body [b, e), returns the position after '>' or 0 on failure.
size_t parse_iri(const unsigned char* s, size_t i, size_t n, size_t& b, size_t& e) {
  if (i >= n || s[i] != '<') return 0;
  size_t j = i + 1;
  while (j < n && iri_char_ok(s[j])) j++;
  if (j >= n || s[j] != '>') return 0;
  b = i + 1;
  e = j;
  return j + 1;
}

bool is_alnum(unsigned char c) {
  return (c >= 'A' && c <= 'Z') || (c >= 'a' && c <= 'z') || (c >= '0' && c <= '9');
}

// Maximal blank node "_:label" at i: returns its end or 0.
size_t parse_bnode(const unsigned char* s, size_t i, size_t n) {
  if (i + 2 >= n + 0 || s[i] != '_' || s[i + 1] != ':') return 0;
  if (i + 2 >= n || !is_alnum(s[i + 2])) return 0;
  size_t j = i + 3;
  while (j < n && (is_alnum(s[j]) || s[j] == '_' || s[j] == '.' || s[j] == '-')) j++;
  return j;
}

// \s*\.\s*(?:#.*)?$ from i.
bool tail_ok(const unsigned char* s, size_t i, size_t n) {
  i = skip_ws(s, i, n);
  if (i >= n || s[i] != '.') return false;
  i = skip_ws(s, i + 1, n);
  return i == n || s[i] == '#';
}

int hexval(unsigned char c) {
  if (c >= '0' && c <= '9') return c - '0';
  if (c >= 'a' && c <= 'f') return c - 'a' + 10;
  if (c >= 'A' && c <= 'F') return c - 'A' + 10;
  return -1;
}

void put_utf8(std::vector<char>& o, uint32_t cp) {
  if (cp < 0x80) {
    o.push_back((char)cp);
  } else if (cp < 0x800) {
    o.push_back((char)(0xC0 | (cp >> 6)));
    o.push_back((char)(0x80 | (cp & 0x3F)));
  } else if (cp < 0x10000) {
    o.push_back((char)(0xE0 | (cp >> 12)));
    o.push_back((char)(0x80 | ((cp >> 6) & 0x3F)));
    o.push_back((char)(0x80 | (cp & 0x3F)));
  } else {
    o.push_back((char)(0xF0 | (cp >> 18)));
    o.push_back((char)(0x80 | ((cp >> 12) & 0x3F)));
    o.push_back((char)(0x80 | ((cp >> 6) & 0x3F)));
    o.push_back((char)(0x80 | (cp & 0x3F)));
  }
}

// _unescape_literal (qparser.py:34-57) of s[b, e) appended to o; false +
// msg on a bad escape.
bool unescape_literal(const unsigned char* s, size_t b, size_t e, std::vector<char>& o, std::string& msg) {
  for (size_t i = b; i < e;) {
    const unsigned char c = s[i];
    if (c != '\\') {  // the run up to the next backslash, appended at once
      const void* bs = memchr(s + i, '\\', e - i);
      const size_t j = bs ? (size_t)(static_cast<const unsigned char*>(bs) - s) : e;
      o.insert(o.end(), s + i, s + j);
      i = j;
      continue;
    }
    const unsigned char x = s[i + 1];  // the lexical scan guarantees a char follows
    const char* from = "\"\\nrtbf'";
    const char* to = "\"\\\n\r\t\b\f'";
    if (const char* p = x ? strchr(from, x) : nullptr) {
      o.push_back(to[p - from]);
      i += 2;
      continue;
    }
    if (x == 'u' || x == 'U') {
      // chr(int(text[i+2 : i+2+nd], 16)): the slice is up to nd characters
      // (shorter at the end of the lexical form) and Python's int() accepts
      // surrounding whitespace, a '+' sign, a 0x prefix and single '_'
      // between digits; the reference then skips nd+2 characters regardless.
      const size_t nd = x == 'u' ? 4 : 8;
      size_t j = i + 2, taken = 0;
      std::string sl;
      bool ascii = true;
      while (j < e && taken < nd) {
        uint32_t c2;
        int l2 = utf8_cp(s, j, e, c2);
        if (!l2) l2 = 1;
        if (c2 >= 0x80) ascii = false;
        sl.append(reinterpret_cast<const char*>(s + j), (size_t)l2);
        j += (size_t)l2;
        taken++;
      }
      auto sp = [](char ch) { return ch == ' ' || (ch >= 0x09 && ch <= 0x0D) || (ch >= 0x1C && ch <= 0x1F); };
      size_t a = 0, z = sl.size();
      while (a < z && sp(sl[a])) a++;
      while (z > a && sp(sl[z - 1])) z--;
      bool ok = ascii && a < z;
      if (ok && sl[a] == '+') a++;
      if (ok && z - a >= 2 && sl[a] == '0' && (sl[a + 1] == 'x' || sl[a + 1] == 'X')) {
        a += 2;
        if (a < z && sl[a] == '_') a++;
      }
      uint64_t cp = 0;
      ok = ok && a < z;
      for (size_t k = a; ok && k < z; k++) {
        if (sl[k] == '_') {
          ok = k > a && k + 1 < z && sl[k - 1] != '_' && sl[k + 1] != '_';
          continue;
        }
        const int h = hexval((unsigned char)sl[k]);
        if (h < 0) ok = false;
        else cp = (cp << 4) | (uint64_t)h;
        if (cp > 0x10FFFF) ok = false;
      }
      if (!ok || (cp >= 0xD800 && cp <= 0xDFFF)) {
        msg = std::string("bad literal escape \\") + (char)x;
        return false;
      }
      put_utf8(o, (uint32_t)cp);
      // skip 2 + nd characters (code points) from the backslash
      size_t skip = i + 2;
      for (size_t c3 = 0; c3 < nd && skip < e; c3++) {
        uint32_t c2;
        int l2 = utf8_cp(s, skip, e, c2);
        skip += (size_t)(l2 ? l2 : 1);
      }
      i = skip;
      continue;
    }
    uint32_t cp;
    int l = utf8_cp(s, i + 1, e, cp);
    msg = "bad literal escape \\" + std::string(reinterpret_cast<const char*>(s + i + 1), (size_t)(l ? l : 1));
    return false;
  }
  return true;
}

// Python repr() of str.strip() of the line (for the error message).
std::string py_repr_stripped(const unsigned char* s, size_t n) {
  size_t b = skip_ws(s, 0, n);
  size_t e = n;
  while (e > b) {  // strip trailing whitespace (walk back to a char start)
    size_t k = e - 1;
    while (k > b && (s[k] & 0xC0) == 0x80) k--;
    if (space_at(s, k, e) > 0) e = k;
    else break;
  }
  bool sq = false, dq = false;
  for (size_t i = b; i < e; i++) {
    sq |= s[i] == '\'';
    dq |= s[i] == '"';
  }
  const char q = (sq && !dq) ? '"' : '\'';
  std::string r(1, q);
  for (size_t i = b; i < e;) {
    uint32_t cp;
    int l = utf8_cp(s, i, e, cp);
    if (!l) {
      l = 1;
      cp = s[i];
    }
    char buf[16];
    if (cp == '\\') r += "\\\\";
    else if (cp == (uint32_t)q) (r += '\\') += q;
    else if (cp == '\t') r += "\\t";
    else if (cp == '\n') r += "\\n";
    else if (cp == '\r') r += "\\r";
    else if (cp < 0x20 || (cp >= 0x7F && cp <= 0xA0) || cp == 0xAD) {
      snprintf(buf, sizeof buf, "\\x%02x", cp);
      r += buf;
    } else if (cp == 0x1680 || (cp >= 0x2000 && cp <= 0x200F) || (cp >= 0x2028 && cp <= 0x202F) ||
               (cp >= 0x205F && cp <= 0x206F) || cp == 0x3000 || cp == 0xFEFF) {
      snprintf(buf, sizeof buf, "\\u%04x", cp);
      r += buf;
    } else {
      r.append(reinterpret_cast<const char*>(s + i), (size_t)l);
    }
    i += (size_t)l;
  }
  r += q;
  return r;
}

void add_term(Chunk& out, std::vector<Term>& col, const unsigned char* s, size_t b, size_t e) {
  col.push_back(Term{(uint64_t)out.bytes.size(), (uint32_t)(e - b)});
  out.bytes.insert(out.bytes.end(), s + b, s + e);
}

// One line (terminator excluded).  Returns false on a malformed statement.
bool parse_line(const unsigned char* s, size_t n, Chunk& out, std::string& msg) {
  size_t i = skip_ws(s, 0, n);
  if (i == n || s[i] == '#') return true;  // _BLANK
  auto malformed = [&]() {
    msg = "malformed N-Triples statement: " + py_repr_stripped(s, n);
    return false;
  };
  size_t sb, se, pb, pe;
  size_t j;
  if (s[i] == '<') {
    if (!(j = parse_iri(s, i, n, sb, se))) return malformed();
  } else if ((j = parse_bnode(s, i, n))) {
    sb = i;
    se = j;
  } else {
    return malformed();
  }
  size_t k = skip_ws(s, j, n);
  if (k == j) return malformed();  // \s+
  if (!(j = parse_iri(s, k, n, pb, pe))) return malformed();
  k = skip_ws(s, j, n);
  if (k == j || k >= n) return malformed();
  // object
  if (s[k] == '<') {
    size_t ob, oe;
    if (!(j = parse_iri(s, k, n, ob, oe)) || !tail_ok(s, j, n)) return malformed();
    add_term(out, out.s, s, sb, se);
    add_term(out, out.p, s, pb, pe);
    add_term(out, out.o, s, ob, oe);
    return true;
  }
  if (s[k] == '_') {
    size_t end = parse_bnode(s, k, n);
    if (!end) return malformed();
    // greedy label, giving back trailing '.' until the tail matches
    size_t e2 = end;
    for (;;) {
      if (tail_ok(s, e2, n)) break;
      size_t prev = e2;
      do {
        e2--;
      } while (e2 > k + 3 && s[e2] != '.');
      if (e2 <= k + 2 || s[e2] != '.' || e2 >= prev) return malformed();
    }
    add_term(out, out.s, s, sb, se);
    add_term(out, out.p, s, pb, pe);
    add_term(out, out.o, s, k, e2);
    return true;
  }
  if (s[k] != '"') return malformed();
  // literal "((?:[^"\\\n]|\\.)*)"
  size_t lb = k + 1, q = lb;
  while (q < n && s[q] != '"') {
    if (s[q] == '\\') {
      if (q + 1 >= n) return malformed();
      uint32_t cp;
      int l = utf8_cp(s, q + 1, n, cp);
      q += 1 + (size_t)(l ? l : 1);
    } else {
      q++;
    }
  }
  if (q >= n) return malformed();
  const size_t le = q;
  j = q + 1;
  size_t db = 0, de = 0, gb = 0, ge = 0;
  int suffix = 0;  // 1 = datatype, 2 = language
  if (j + 1 < n && s[j] == '^' && s[j + 1] == '^') {
    size_t after = parse_iri(s, j + 2, n, db, de);
    if (!after) return malformed();
    suffix = 1;
    j = after;
  } else if (j < n && s[j] == '@') {
    size_t a = j + 1;
    auto alpha = [](unsigned char c) { return (c >= 'A' && c <= 'Z') || (c >= 'a' && c <= 'z'); };
    if (a >= n || !alpha(s[a])) return malformed();
    while (a < n && alpha(s[a])) a++;
    while (a + 1 < n && s[a] == '-' && is_alnum(s[a + 1])) {
      a++;
      while (a < n && is_alnum(s[a])) a++;
    }
    gb = j + 1;
    ge = a;
    suffix = 2;
    j = a;
  }
  if (!tail_ok(s, j, n)) return malformed();
  add_term(out, out.s, s, sb, se);
  add_term(out, out.p, s, pb, pe);
  Term t{(uint64_t)out.bytes.size(), 0};
  out.bytes.push_back('"');
  if (!unescape_literal(s, lb, le, out.bytes, msg)) {
    out.s.pop_back();
    out.p.pop_back();
    return false;
  }
  out.bytes.push_back('"');
  if (suffix == 1) {
    out.bytes.push_back('^');
    out.bytes.push_back('^');
    out.bytes.push_back('<');
    out.bytes.insert(out.bytes.end(), s + db, s + de);
    out.bytes.push_back('>');
  } else if (suffix == 2) {
    out.bytes.push_back('@');
    out.bytes.insert(out.bytes.end(), s + gb, s + ge);
  }
  t.len = (uint32_t)(out.bytes.size() - t.off);
  out.o.push_back(t);
  return true;
}

}  // namespace

void parse_range(const char* cbuf, size_t begin, size_t end, int64_t first_line, Chunk& out) {
  const unsigned char* buf = reinterpret_cast<const unsigned char*>(cbuf);
  int64_t line = first_line;
  size_t i = begin;
  std::string msg;
  // term bytes are a little less than the input; a statement is >= ~20 bytes
  out.bytes.reserve(end - begin);
  for (auto* col : {&out.s, &out.p, &out.o}) col->reserve((end - begin) / 48 + 16);
  while (i < end) {
    // line end: the first '\n', or an earlier '\r' (universal newlines)
    const void* nl = memchr(buf + i, '\n', end - i);
    size_t j = nl ? (size_t)(static_cast<const unsigned char*>(nl) - buf) : end;
    if (const void* cr = memchr(buf + i, '\r', j - i)) j = (size_t)(static_cast<const unsigned char*>(cr) - buf);
    // invalid UTF-8 is a decode error in the reference (text-mode read);
    // ASCII runs are checked 8 bytes at a time
    for (size_t k = i; k < j;) {
      if (k + 8 <= j) {
        uint64_t w;
        memcpy(&w, buf + k, 8);
        if (!(w & 0x8080808080808080ull)) {
          k += 8;
          continue;
        }
      }
      if (buf[k] < 0x80) {
        k++;
        continue;
      }
      uint32_t cp;
      int l = utf8_cp(buf, k, j, cp);
      if (!l) {
        out.err_line = line;
        out.err_msg = "invalid UTF-8 in N-Triples input";
        return;
      }
      k += (size_t)l;
    }
    if (!parse_line(buf + i, j - i, out, msg)) {
      out.err_line = line;
      out.err_msg = msg;
      return;
    }
    if (j < end && buf[j] == '\r' && j + 1 < end && buf[j + 1] == '\n') j++;
    i = j + 1;
    line++;
  }
}

void split_lines(const char* buf, size_t n, int parts, std::vector<size_t>& bounds,
                 std::vector<int64_t>& first_lines) {
  bounds.assign(1, 0);
  for (int p = 1; p < parts; p++) {
    size_t b = n * (size_t)p / (size_t)parts;
    if (b <= bounds.back()) continue;
    while (b < n && buf[b - 1] != '\n' && !(buf[b - 1] == '\r' && buf[b] != '\n')) b++;
    if (b >= n) break;
    if (b > bounds.back()) bounds.push_back(b);
  }
  bounds.push_back(n);
  // line numbers: terminators before each boundary ('\n', and '\r' not
  // followed by '\n'), counted per range on its own thread
  const size_t nr = bounds.size() - 1;
  std::vector<int64_t> cnt(nr, 0);
  auto count = [&](size_t r) {
    const unsigned char* u = reinterpret_cast<const unsigned char*>(buf);
    int64_t c = 0;
    for (size_t i = bounds[r]; i < bounds[r + 1];) {
      const void* q = memchr(u + i, '\n', bounds[r + 1] - i);
      if (!q) break;
      c++;
      i = (size_t)(static_cast<const unsigned char*>(q) - u) + 1;
    }
    for (size_t i = bounds[r]; i < bounds[r + 1];) {
      const void* q = memchr(u + i, '\r', bounds[r + 1] - i);
      if (!q) break;
      const size_t k = (size_t)(static_cast<const unsigned char*>(q) - u);
      if (!(k + 1 < n && u[k + 1] == '\n')) c++;
      i = k + 1;
    }
    cnt[r] = c;
  };
  std::vector<std::thread> th;
  for (size_t r = 1; r + 1 < nr + 1; r++) th.emplace_back(count, r - 1);  // the last range's count is not needed
  for (auto& t : th) t.join();
  first_lines.assign(nr, 1);
  for (size_t r = 1; r < nr; r++) first_lines[r] = first_lines[r - 1] + cnt[r - 1];
}

}  // namespace nt
}  // namespace gsm
