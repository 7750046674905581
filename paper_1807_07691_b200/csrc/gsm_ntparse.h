// gsm_ntparse.h — N-Triples statement parser of the ingest path (host side).
//
// Restates qparser.parse_ntriples_line / read_ntriples
// (/root/reference/pkg/src/gsmat/qparser.py:20-31, 34-57, 80-104):
//   ^\s*(?:<IRI>|_:BNODE)\s+<IRI>\s+(?:<IRI>|_:BNODE|LITERAL)\s*\.\s*(?:#.*)?$
// with Python's Unicode \s, the regex's backtracking where it matters (a
// blank-node label may give back trailing '.'), literal unescaping
// (\" \\ \n \r \t \b \f \' \uXXXX \UXXXXXXXX, else ParseError) and the
// canonical term forms (IRIs without brackets, "_:label", '"' + lexical + '"'
// + ^^<dt> | @lang).  Lines are split like Python's universal-newline text
// mode (\n, \r\n and \r all end a line).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace gsm {
namespace nt {

struct Term {
  uint64_t off;  // into Chunk::bytes
  uint32_t len;
};

struct Chunk {
  std::vector<char> bytes;  // canonical term bytes
  std::vector<Term> s, p, o;
  int64_t err_line = -1;    // first bad line (1-based, global), -1 = none
  std::string err_msg;      // reference ParseError message (without "line N: ")
};

// Parse lines [begin, end) of buf; `first_line` is the 1-based number of the
// line starting at begin.  Stops at the first malformed statement.
void parse_range(const char* buf, size_t begin, size_t end, int64_t first_line, Chunk& out);

// Split buf into about `parts` ranges at line boundaries; returns the
// boundaries (parts+1 offsets) and the 1-based first line number of each.
void split_lines(const char* buf, size_t n, int parts, std::vector<size_t>& bounds,
                 std::vector<int64_t>& first_lines);

}  // namespace nt
}  // namespace gsm
