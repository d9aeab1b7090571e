// gq_io.cpp -- .node / .ele / .face mesh writer of libgqm3d.so (host C++).
//
// Same files as the reference's formats.write_mesh / write_node
// (/root/reference/pkg/src/tetrefine/formats.py:210-263): 1-based ids,
// coordinates printed "%.17g" (round-trip exact, formats.py:19), the input /
// Steiner origin as the vertex attribute, alive non-ghost tets in slot order,
// and subfaces sorted by their vertex key with the parent polygon id.
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/gqm3d.h"

namespace {

struct Out {                      // buffered writer: one fwrite per MB
  FILE* f = nullptr;
  std::string buf;
  explicit Out(const char* path) : f(std::fopen(path, "w")) { buf.reserve(1 << 21); }
  ~Out() { flush(); if (f) std::fclose(f); }
  bool ok() const { return f != nullptr; }
  void flush() {
    if (f && !buf.empty()) { std::fwrite(buf.data(), 1, buf.size(), f); buf.clear(); }
  }
  void put(const char* s, size_t n) { buf.append(s, n); if (buf.size() > (1 << 20)) flush(); }
  void fmt(const char* f, ...) __attribute__((format(printf, 2, 3)));
};
void Out::fmt(const char* fm, ...) {
  char tmp[256];
  va_list ap;
  va_start(ap, fm);
  int n = std::vsnprintf(tmp, sizeof tmp, fm, ap);
  va_end(ap);
  if (n > 0) put(tmp, (size_t)n);
}

}  // namespace

extern "C" int gq_write_mesh(const char* node_path, const char* ele_path, const char* face_path,
                             const double* points, const uint8_t* origins, int32_t nv, const int32_t* tv,
                             const uint8_t* alive, int32_t nt, const int32_t* faces, int32_t nf) {
  if (!node_path || !ele_path || (nv > 0 && (!points || !origins)) || (nt > 0 && (!tv || !alive)) ||
      (face_path && nf > 0 && !faces) || nv < 0 || nt < 0 || nf < 0)
    return GQ_EINVAL;
  {
    Out o(node_path);
    if (!o.ok()) return GQ_EINVAL;
    o.fmt("%d 3 1 0\n", nv);
    for (int32_t k = 0; k < nv; ++k)
      o.fmt("%d %.17g %.17g %.17g %d\n", k + 1, points[3 * k], points[3 * k + 1], points[3 * k + 2], (int)origins[k]);
  }
  {
    int32_t n = 0;
    for (int32_t t = 0; t < nt; ++t) n += alive[t] == 1 && tv[4 * t + 3] != -1;
    Out o(ele_path);
    if (!o.ok()) return GQ_EINVAL;
    o.fmt("%d 4 0\n", n);
    int32_t k = 0;
    for (int32_t t = 0; t < nt; ++t) {
      if (alive[t] != 1 || tv[4 * t + 3] == -1) continue;
      o.fmt("%d %d %d %d %d\n", ++k, tv[4 * t] + 1, tv[4 * t + 1] + 1, tv[4 * t + 2] + 1, tv[4 * t + 3] + 1);
    }
  }
  if (face_path) {   // rows (a, b, c, pid) with a < b < c, already sorted by the caller
    Out o(face_path);
    if (!o.ok()) return GQ_EINVAL;
    o.fmt("%d 1\n", nf);
    for (int32_t k = 0; k < nf; ++k)
      o.fmt("%d %d %d %d %d\n", k + 1, faces[4 * k] + 1, faces[4 * k + 1] + 1, faces[4 * k + 2] + 1, faces[4 * k + 3]);
  }
  return GQ_OK;
}
