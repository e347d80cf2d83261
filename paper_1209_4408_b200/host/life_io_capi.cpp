// life_io_capi.cpp -- extern "C" view of life_io.hpp, used by the parity
// tests (tests/test_host_io.py) to compare the host I/O layer with the
// reference library cell for cell.  Status: 0 ok, 1 ConfigError, 3 ParseError.
#include <cstring>
#include <string>

#include "life_io.hpp"

namespace {

int copy_out(const std::string& s, char* out, int cap) {
  if (static_cast<int>(s.size()) + 1 > cap) return -1;
  std::memcpy(out, s.c_str(), s.size() + 1);
  return 0;
}

int export_pattern(const lifegpu::Pattern& p, int* w, int* h, int* xs, int* ys, int cap, int* n) {
  *w = p.width;
  *h = p.height;
  *n = static_cast<int>(p.live_cells.size());
  if (*n > cap) return -1;
  for (int i = 0; i < *n; ++i) {
    xs[i] = p.live_cells[i].x;
    ys[i] = p.live_cells[i].y;
  }
  return 0;
}

struct Grid {
  int w, h;
  const uint8_t* c;
  int width() const { return w; }
  int height() const { return h; }
  const uint8_t* data() const { return c; }
};

}  // namespace

extern "C" {

int lio_parse_rle(const char* text, int* w, int* h, int* xs, int* ys, int cap, int* n, int* line,
                  int* col, char* msg, int msgcap) {
  try {
    return export_pattern(lifegpu::parse_rle(text), w, h, xs, ys, cap, n);
  } catch (const lifegpu::ParseError& e) {
    *line = e.line();
    *col = e.column();
    copy_out(e.what(), msg, msgcap);
    return 3;
  }
}

int lio_parse_plaintext(const char* text, int* w, int* h, int* xs, int* ys, int cap, int* n,
                        int* line, int* col, char* msg, int msgcap) {
  try {
    return export_pattern(lifegpu::parse_plaintext(text), w, h, xs, ys, cap, n);
  } catch (const lifegpu::ParseError& e) {
    *line = e.line();
    *col = e.column();
    copy_out(e.what(), msg, msgcap);
    return 3;
  }
}

int lio_serialize_rle(int w, int h, const int* xs, const int* ys, int n, char* out, int cap) {
  lifegpu::Pattern p{w, h, {}};
  for (int i = 0; i < n; ++i) p.live_cells.push_back({xs[i], ys[i]});
  try {
    return copy_out(lifegpu::serialize_rle(p), out, cap);
  } catch (const lifegpu::ConfigError&) {
    return 1;
  }
}

int lio_render_ascii(const uint8_t* cells, int w, int h, char* out, int cap) {
  return copy_out(lifegpu::render_ascii(Grid{w, h, cells}), out, cap);
}

int lio_render_pbm(const uint8_t* cells, int w, int h, char* out, int cap) {
  return copy_out(lifegpu::render_pbm(Grid{w, h, cells}), out, cap);
}

}  // extern "C"
