// fsg_io.cpp -- output formats of the path, host C++:
//   fsg_write_vtk  lbm::write_vtk (lbm/vtk.hpp:15-38): legacy ASCII structured
//                  points of u (m/s) and rho (kg/m^3), same stream formatting;
//                  fed by the asynchronous device snapshot (fsg_snapshot_*),
//                  so a dump does not stall the step stream;
//   fsg_csv_*      CsvWriter / format_full (core/csv.hpp:18-66): header on
//                  open, every row flushed, %.17g round-trip formatting.
// Byte-for-byte parity with the reference's own writers:
// tests/test_io.py (oracle/_ref compiles vtk.hpp and csv.hpp unmodified).
#include <cstdarg>
#include <cstdio>
#include <fstream>
#include <string>
#include <vector>

#include "../../include/fsg.h"

namespace {
thread_local char g_io_err[512] = "";
int io_err(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(g_io_err, sizeof(g_io_err), fmt, ap);
  va_end(ap);
  return code;
}
}  // namespace

struct fsg_csv {
  std::string path;
  size_t n_cols = 0;
  std::ofstream out;
};

extern "C" {

const char* fsg_io_last_error(void) { return g_io_err; }

int fsg_format_full(double v, char* buf, int size) {
  if (!buf || size < 32) return io_err(FSG_EINPUT, "fsg_format_full: buffer too small");
  std::snprintf(buf, (size_t)size, "%.17g", v);  // csv.hpp:18-22
  return FSG_OK;
}

int fsg_write_vtk_fields(const char* path, const int dims[3], const double* rho, const double* u,
                         double dx, double dt, double rho_phys, const double origin[3]) {
  std::ofstream out(path);
  if (!out) return io_err(FSG_EINPUT, "cannot open field dump for writing: %s", path);
  const size_t n = (size_t)dims[0] * dims[1] * dims[2];
  out << "# vtk DataFile Version 3.0\n";
  out << "fishsim fluid field\n";
  out << "ASCII\n";
  out << "DATASET STRUCTURED_POINTS\n";
  out << "DIMENSIONS " << dims[0] << ' ' << dims[1] << ' ' << dims[2] << '\n';
  out << "ORIGIN " << origin[0] << ' ' << origin[1] << ' ' << origin[2] << '\n';
  out << "SPACING " << dx << ' ' << dx << ' ' << dx << '\n';
  out << "POINT_DATA " << n << '\n';
  out << "VECTORS velocity double\n";
  const double s = dx / dt;  // UnitMap::vel_to_physical(Vec3) = v * (dx / dt) (units.hpp:31)
  for (size_t c = 0; c < n; ++c)
    out << u[3 * c] * s << ' ' << u[3 * c + 1] * s << ' ' << u[3 * c + 2] * s << '\n';
  out << "SCALARS density double\n";
  out << "LOOKUP_TABLE default\n";
  for (size_t c = 0; c < n; ++c) out << rho[c] * rho_phys << '\n';
  if (!out) return io_err(FSG_EINPUT, "write error on %s", path);
  return FSG_OK;
}

int fsg_csv_open(const char* path, int n_cols, const char* const* columns, fsg_csv** out_h) {
  if (!path || !out_h || n_cols < 0 || (n_cols > 0 && !columns))
    return io_err(FSG_EINPUT, "fsg_csv_open: bad arguments");
  fsg_csv* h = new fsg_csv();
  h->path = path;
  h->n_cols = (size_t)n_cols;
  h->out.open(path);
  if (!h->out) {
    delete h;
    return io_err(FSG_EINPUT, "cannot open CSV for writing: %s", path);
  }
  for (int i = 0; i < n_cols; ++i) {
    if (i) h->out << ',';
    h->out << columns[i];
  }
  h->out << '\n';
  h->out.flush();
  if (!h->out) {
    delete h;
    return io_err(FSG_EINPUT, "write error on %s", path);
  }
  *out_h = h;
  return FSG_OK;
}

int fsg_csv_write_row(fsg_csv* h, int n, const double* values) {
  if ((size_t)n != h->n_cols)
    return io_err(FSG_EINPUT, "CSV row has %d values, header has %zu", n, h->n_cols);
  char buf[40];
  for (int i = 0; i < n; ++i) {
    if (i) h->out << ',';
    std::snprintf(buf, sizeof(buf), "%.17g", values[i]);
    h->out << buf;
  }
  h->out << '\n';
  h->out.flush();  // a truncated file is always a valid prefix
  if (!h->out) return io_err(FSG_EINPUT, "write error on %s", h->path.c_str());
  return FSG_OK;
}

int fsg_csv_close(fsg_csv* h) {
  delete h;
  return FSG_OK;
}

}  // extern "C"
