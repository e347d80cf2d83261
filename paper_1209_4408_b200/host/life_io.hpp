// life_io.hpp -- grid I/O at the boundary of the GPU engine (SURVEY.md 8f
// rank 3): pattern formats, placement and renderers, with the reference's
// behaviour (header only, C++20).
//
// Restates /root/reference/proj/core/include/life/pattern.hpp and render.hpp:
//   parse_rle          pattern.cpp:147-212   (RLE: header "x = W, y = H[, rule = B3/S23]",
//                                              runs of b/o, '$' row ends, '!' terminator,
//                                              '#' comment lines; ParseError with 1-based
//                                              line/column)
//   serialize_rle      pattern.cpp:214-253   (canonical: maximal runs, no count on 1,
//                                              trailing dead cells/rows omitted)
//   parse_plaintext    pattern.cpp:255-292   ('.' dead, 'O' alive, '!' comment lines,
//                                              ragged rows padded)
//   load_pattern_file  pattern.cpp:294-307   (.rle / .cells by extension)
//   place_pattern      pattern.cpp:309-328   (footprint overwrite, OutOfBounds, no wrap)
//   render_ascii       render.cpp:5-15       ('#' / '.', rows joined by '\n')
//   render_pbm         render.cpp:17-38      (plain P1, at most 35 digits per line)
// Parity with the reference is pinned by tests/test_host_io.py (reference
// library outputs and committed fixtures).
#pragma once

#include <algorithm>
#include <cctype>
#include <cstdint>
#include <fstream>
#include <iterator>
#include <sstream>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

#include "life_gpu.hpp"

namespace lifegpu {

// errors.hpp:46-60 -- malformed pattern input (the CLI maps it to exit 3).
class ParseError : public Error {
 public:
  ParseError(const std::string& message, int line, int column)
      : Error("parse error at line " + std::to_string(line) + ", column " +
              std::to_string(column) + ": " + message),
        line_(line),
        column_(column) {}
  int line() const noexcept { return line_; }
  int column() const noexcept { return column_; }

 private:
  int line_, column_;
};

struct Coord {
  int x = 0;
  int y = 0;
  friend bool operator==(const Coord&, const Coord&) = default;
};

// pattern.hpp:12-25: live cells kept sorted by (y, x) and unique.
struct Pattern {
  int width = 0;
  int height = 0;
  std::vector<Coord> live_cells;

  void normalize() {
    // row-major order: (y, x) pairs compared as tuples, duplicates dropped
    auto& v = live_cells;
    std::stable_sort(v.begin(), v.end(), [](const Coord& lhs, const Coord& rhs) {
      return std::make_pair(lhs.y, lhs.x) < std::make_pair(rhs.y, rhs.x);
    });
    const auto tail = std::unique(v.begin(), v.end());
    v.resize(static_cast<size_t>(tail - v.begin()));
  }
  friend bool operator==(const Pattern&, const Pattern&) = default;
};

namespace detail {

inline bool blank(char c) {
  return c == ' ' || c == '\t' || c == '\r' || c == '\n' || c == '\v' || c == '\f';
}
inline std::string lowered(std::string s) {
  for (char& ch : s) ch = static_cast<char>(std::tolower(static_cast<unsigned char>(ch)));
  return s;
}

// Text reader that knows the 1-based line/column of the next character.
class Reader {
 public:
  explicit Reader(std::string_view t) : text_(t) {}
  bool done() const { return pos_ >= text_.size(); }
  char cur() const { return text_[pos_]; }
  int line() const { return line_; }
  int col() const { return col_; }
  char next() {
    const char ch = text_[pos_++];
    if (ch == '\n') {
      ++line_;
      col_ = 1;
    } else {
      ++col_;
    }
    return ch;
  }
  void skip_while(bool (*pred)(char)) {
    while (!done() && pred(cur())) next();
  }
  [[noreturn]] void error(const std::string& what) const { throw ParseError(what, line_, col_); }
  void expect(char ch, const char* what) {
    if (done() || cur() != ch) error(std::string("missing ") + what);
    next();
  }
  // Decimal run count; counts above 1e9 are rejected (pattern.cpp:14, :62-70).
  long number() {
    long v = 0;
    for (; !done() && std::isdigit(static_cast<unsigned char>(cur())); next()) {
      v = v * 10 + (cur() - '0');
      if (v > 1000000000L) error("number exceeds 1e9");
    }
    return v;
  }

 private:
  std::string_view text_;
  size_t pos_ = 0;
  int line_ = 1, col_ = 1;
};

inline bool space_or_tab(char c) { return c == ' ' || c == '\t'; }
inline bool is_blank(char c) { return blank(c); }

}  // namespace detail

// RLE header, as a fixed script of (skip blanks?, expected char, what) steps
// with the two integers parsed after the '=' signs.
inline void rle_header(detail::Reader& r, Pattern& p) {
  struct Step {
    char want;
    const char* label;
  };
  static constexpr Step kScript[] = {{'x', "'x' opening the header"}, {'=', "'=' after x"},
                                     {',', "',' between the dimensions"}, {'y', "'y' field"},
                                     {'=', "'=' after y"}};
  auto dimension = [&](const char* what) -> int {
    r.skip_while(detail::space_or_tab);
    if (r.done() || !std::isdigit(static_cast<unsigned char>(r.cur())))
      r.error(std::string("missing ") + what);
    return static_cast<int>(r.number());
  };
  for (int i = 0; i < 5; ++i) {
    r.skip_while(detail::space_or_tab);
    r.expect(kScript[i].want, kScript[i].label);
    if (i == 1) p.width = dimension("width value");
    if (i == 4) p.height = dimension("height value");
  }
  r.skip_while(detail::space_or_tab);
  if (!r.done() && r.cur() == ',') {  // optional ", rule = B3/S23" (or 23/3)
    r.next();
    r.skip_while(detail::space_or_tab);
    std::string field;
    while (!r.done() && std::isalpha(static_cast<unsigned char>(r.cur()))) field += r.next();
    if (detail::lowered(field) != "rule") r.error("header field '" + field + "' is not 'rule'");
    r.skip_while(detail::space_or_tab);
    r.expect('=', "'=' after rule");
    r.skip_while(detail::space_or_tab);
    std::string rule;
    while (!r.done() && !detail::blank(r.cur()) && r.cur() != ',') rule += r.next();
    const std::string lr = detail::lowered(rule);
    if (lr != "b3/s23" && lr != "23/3") r.error("rule '" + rule + "' is not B3/S23");
    r.skip_while(detail::space_or_tab);
  }
  if (!r.done() && r.cur() != '\n') r.error("unexpected text after the RLE header");
  if (!r.done()) r.next();
}

inline Pattern parse_rle(std::string_view text) {
  detail::Reader r(text);
  for (;;) {  // leading blank and '#' comment lines
    r.skip_while(detail::is_blank);
    if (r.done() || r.cur() != '#') break;
    while (!r.done() && r.next() != '\n') {
    }
  }
  if (r.done()) r.error("no RLE header found");
  Pattern p;
  rle_header(r, p);

  int col = 0, row = 0;
  for (bool open = true; open;) {
    r.skip_while(detail::is_blank);
    if (r.done()) r.error("RLE body ends without '!'");
    long run = 1;
    if (std::isdigit(static_cast<unsigned char>(r.cur()))) {
      run = r.number();
      if (run == 0) r.error("a run of 0 cells");
      r.skip_while(detail::is_blank);
      if (r.done()) r.error("run count not followed by a tag");
    }
    const int at_line = r.line(), at_col = r.col();
    const char tag = r.next();
    switch (tag) {
      case '!':
        if (run != 1) throw ParseError("'!' may not carry a run count", at_line, at_col);
        open = false;  // the rest of the text is ignored
        break;
      case '$':
        row += static_cast<int>(run);
        col = 0;
        break;
      case 'o':
      case 'O':
      case 'b':
      case 'B': {
        if (row >= p.height)
          throw ParseError("row " + std::to_string(row) + " lies beyond the declared height " +
                               std::to_string(p.height), at_line, at_col);
        if (col + run > p.width)
          throw ParseError("run passes the declared width " + std::to_string(p.width), at_line,
                           at_col);
        const bool live = tag == 'o' || tag == 'O';
        for (long k = 0; live && k < run; ++k) p.live_cells.push_back({col + static_cast<int>(k), row});
        col += static_cast<int>(run);
        break;
      }
      default:
        throw ParseError(std::string("illegal character '") + tag + "' in RLE body", at_line, at_col);
    }
  }
  return p;
}

inline std::string serialize_rle(const Pattern& pattern) {
  Pattern p{pattern.width, pattern.height, pattern.live_cells};
  p.normalize();
  const auto inside = [&p](const Coord& c) {
    return 0 <= c.x && c.x < p.width && 0 <= c.y && c.y < p.height;
  };
  if (!std::all_of(p.live_cells.begin(), p.live_cells.end(), inside))
    throw ConfigError("pattern has live cells outside its declared bounds");
  std::ostringstream header;
  header << "x = " << p.width << ", y = " << p.height << '\n';
  std::string out = header.str();
  // One RLE item: the count is written only for runs longer than one.
  const auto put = [&out](long run, char tag) {
    if (run >= 2) out.append(std::to_string(run));
    out.push_back(tag);
  };
  int row = 0, col = 0;
  for (size_t i = 0; i < p.live_cells.size();) {
    const Coord start = p.live_cells[i];
    if (start.y > row) {
      put(start.y - row, '$');
      row = start.y;
      col = 0;
    }
    size_t j = i + 1;
    while (j < p.live_cells.size() && p.live_cells[j].y == start.y &&
           p.live_cells[j].x == start.x + static_cast<int>(j - i))
      ++j;
    if (start.x > col) put(start.x - col, 'b');
    put(static_cast<long>(j - i), 'o');
    col = start.x + static_cast<int>(j - i);
    i = j;
  }
  out += '!';
  return out;
}

inline Pattern parse_plaintext(std::string_view text) {
  Pattern p;
  int row = 0, line_no = 0;
  size_t start = 0;
  while (start < text.size()) {
    const size_t nl = text.find('\n', start);
    const std::string_view ln =
        text.substr(start, (nl == std::string_view::npos ? text.size() : nl) - start);
    ++line_no;
    if (ln.empty() || ln[0] != '!') {
      int x = 0;
      for (size_t i = 0; i < ln.size(); ++i) {
        if (ln[i] == '.') {
          ++x;
        } else if (ln[i] == 'O') {
          p.live_cells.push_back({x++, row});
        } else if (!detail::blank(ln[i])) {
          throw ParseError(std::string("illegal character '") + ln[i] + "' in plaintext",
                           line_no, static_cast<int>(i) + 1);
        }
      }
      p.width = std::max(p.width, x);
      ++row;
    }
    if (nl == std::string_view::npos) break;
    start = nl + 1;
  }
  p.height = row;
  return p;
}

inline Pattern load_pattern_file(const std::string& path) {
  std::string text;
  {
    std::ifstream file(path, std::ios::in | std::ios::binary);
    if (!file.is_open()) throw ConfigError("cannot read pattern file '" + path + "'");
    text.assign(std::istreambuf_iterator<char>(file), std::istreambuf_iterator<char>());
  }
  // The format is picked by the (case-insensitive) file extension alone.
  std::string ext;
  if (const auto at = path.find_last_of('.'); at != std::string::npos)
    ext = detail::lowered(path.substr(at));
  const bool rle = ext == ".rle", cells = ext == ".cells";
  if (!rle && !cells)
    throw ConfigError("unsupported pattern extension '" + ext + "' (expected .rle or .cells)");
  return rle ? parse_rle(text) : parse_plaintext(text);
}

// place_pattern on a host grid (any GridT with width()/height()/data()).
template <class GridT>
GridT place_pattern(const GridT& grid, const Pattern& pattern, Coord origin) {
  const int64_t gw = grid.width(), gh = grid.height();
  const bool fits = origin.x >= 0 && origin.y >= 0 &&
                    int64_t{origin.x} + pattern.width <= gw &&
                    int64_t{origin.y} + pattern.height <= gh;
  if (!fits) {
    std::ostringstream why;  // no wrap-around: the whole footprint must lie on the grid
    why << "pattern footprint " << pattern.width << 'x' << pattern.height << " at (" << origin.x
        << ", " << origin.y << ") exceeds grid " << gw << 'x' << gh;
    throw OutOfBounds(why.str());
  }
  GridT out = grid;
  uint8_t* cells = out.data();
  const int64_t w = out.width();
  for (int j = 0; j < pattern.height; ++j)
    std::fill_n(cells + (origin.y + j) * w + origin.x, pattern.width, uint8_t{0});
  for (const Coord& c : pattern.live_cells) cells[(origin.y + c.y) * w + origin.x + c.x] = 1;
  return out;
}

// The pattern as a dense pw x ph 0/1 byte block (for life_grid_place_u8).
inline std::vector<uint8_t> pattern_bytes(const Pattern& p) {
  std::vector<uint8_t> b(static_cast<size_t>(p.width) * p.height, 0);
  for (const Coord& c : p.live_cells)
    if (c.x >= 0 && c.x < p.width && c.y >= 0 && c.y < p.height)
      b[static_cast<size_t>(c.y) * p.width + c.x] = 1;
  return b;
}

template <class GridT>
std::string render_ascii(const GridT& g) {
  std::string out;
  out.reserve(static_cast<size_t>(g.height()) * (g.width() + 1));
  const uint8_t* c = g.data();
  for (int64_t y = 0; y < g.height(); ++y) {
    if (y) out += '\n';
    for (int64_t x = 0; x < g.width(); ++x) out += c[y * g.width() + x] ? '#' : '.';
  }
  return out;
}

template <class GridT>
std::string render_pbm(const GridT& g) {
  constexpr int kDigitsPerLine = 35;  // 35 digits + 34 spaces = 69 <= 70 columns
  std::string out = "P1\n" + std::to_string(g.width()) + " " + std::to_string(g.height()) + "\n";
  const uint8_t* c = g.data();
  for (int64_t y = 0; y < g.height(); ++y) {
    for (int64_t x = 0; x < g.width(); ++x) {
      if (x > 0) out += (x % kDigitsPerLine == 0) ? '\n' : ' ';
      out += c[y * g.width() + x] ? '1' : '0';
    }
    out += '\n';
  }
  return out;
}

}  // namespace lifegpu
