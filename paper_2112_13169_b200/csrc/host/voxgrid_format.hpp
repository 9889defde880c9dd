// VOXGRID1 grid dumps: the snapshot format of the reference
// (write_grid / read_grid, proj/include/voxmap/grid_io.hpp:10-17, defined by
// proj/src/grid_io.cpp:14-69). Shared, header-only host code of the C-ABI
// (vxm_grid_write / vxm_grid_read / vxm_snapshot_*) and the C++ drop-in
// (voxmap/grid_io.hpp).
//
// Layout: a text header of whitespace-separated fields
//     VOXGRID1 \n dims_x dims_y dims_z \n vox_size \n origin_x origin_y origin_z \n
// (doubles with 17 significant digits, i.e. printf "%.17g", what an ostream
// at max_digits10 precision prints), then dims_x*dims_y*dims_z state bytes
// (0..3) in linear index order. A reader takes the eight fields as formatted
// extraction would, skips exactly one character after the last one, and
// rejects a bad magic, non-positive dims or voxel size, short cell data and
// state bytes above 3.
#pragma once

#include <cmath>
#include <cstddef>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>

namespace vxm_io {

inline std::string voxgrid_header(const int dims[3], double vox_size, const double origin[3]) {
  char buf[256];
  const int n = std::snprintf(buf, sizeof(buf), "VOXGRID1\n%d %d %d\n%.17g\n%.17g %.17g %.17g\n", dims[0],
                              dims[1], dims[2], vox_size, origin[0], origin[1], origin[2]);
  return std::string(buf, n > 0 ? static_cast<std::size_t>(n) : 0);
}

struct VoxgridHeader {
  int dims[3] = {0, 0, 0};
  double vox_size = 0.0;
  double origin[3] = {0.0, 0.0, 0.0};
  std::size_t data_offset = 0;  // first cell byte
  std::size_t cells() const {
    return static_cast<std::size_t>(dims[0]) * static_cast<std::size_t>(dims[1]) * static_cast<std::size_t>(dims[2]);
  }
};

namespace detail {
inline bool is_space(char c) { return c == ' ' || c == '\n' || c == '\t' || c == '\r' || c == '\v' || c == '\f'; }

// next whitespace-delimited token of [p, end): start index and length
inline bool token(const char* data, std::size_t n, std::size_t& pos, std::size_t& start, std::size_t& len) {
  while (pos < n && is_space(data[pos])) ++pos;
  start = pos;
  while (pos < n && !is_space(data[pos])) ++pos;
  len = pos - start;
  return len > 0;
}
}  // namespace detail

// Returns an empty string on success, else the reader's error message.
inline std::string parse_voxgrid_header(const char* data, std::size_t n, VoxgridHeader& h) {
  std::size_t pos = 0, start = 0, len = 0;
  std::string tok[8];
  for (auto& t : tok) {
    if (!detail::token(data, n, pos, start, len)) return "read_grid: bad header";
    t.assign(data + start, len);
  }
  if (tok[0] != "VOXGRID1") return "read_grid: bad header";
  for (int a = 0; a < 3; ++a) {
    char* e = nullptr;
    const long v = std::strtol(tok[1 + a].c_str(), &e, 10);
    if (*e != '\0' || v < -2147483647L - 1 || v > 2147483647L) return "read_grid: bad header";
    h.dims[a] = static_cast<int>(v);
  }
  double d[4];
  for (int i = 0; i < 4; ++i) {
    char* e = nullptr;
    d[i] = std::strtod(tok[4 + i].c_str(), &e);
    if (*e != '\0' || !std::isfinite(d[i])) return "read_grid: bad header";
  }
  h.vox_size = d[0];
  for (int a = 0; a < 3; ++a) h.origin[a] = d[1 + a];
  if (h.dims[0] <= 0 || h.dims[1] <= 0 || h.dims[2] <= 0 || !(h.vox_size > 0.0))
    return "read_grid: invalid dimensions";
  h.data_offset = pos + 1;  // the newline ending the header
  return std::string();
}

// Checks the cell bytes that follow the header.
inline std::string check_voxgrid_cells(const char* data, std::size_t n, const VoxgridHeader& h) {
  const std::size_t need = h.cells();
  if (h.data_offset > n || n - h.data_offset < need) return "read_grid: truncated cell data";
  const unsigned char* c = reinterpret_cast<const unsigned char*>(data + h.data_offset);
  for (std::size_t i = 0; i < need; ++i)
    if (c[i] > 3) return "read_grid: invalid state byte";
  return std::string();
}

}  // namespace vxm_io
