// csv.cu -- host-side CSV materialisation of replay results (no device code).
//
// The reference writes every artifact with csv.writer rows whose float
// fields are Python repr() strings (`simcore.py:319-369`, `metrics.py:82-128`,
// `colocation.py:108-126`, `workload.py:173-178`, writer `cli.py:34-39`).
// intf_csv_rows formats typed SoA columns into the same bytes: repr(float)
// is the shortest round-trip decimal (std::to_chars) laid out as CPython's
// float_repr_style 'short' does (fixed notation for decimal exponents in
// [-4, 16), otherwise d[.ddd]e[+-]XX), ints in decimal, strings verbatim
// (the caller passes them already csv-quoted), numpy-2 scalar reprs
// "np.float64(...)" where the reference formats numpy scalars with %r
// (samples.csv), ',' between fields and
// csv.writer's default "\r\n" after every row.
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstring>

#include "capi_common.h"

using namespace intf;

namespace {

// CPython repr(float) of v into p (room for 32 chars); returns the length.
int repr_f64(double v, char* p) {
  char* q = p;
  if (std::isnan(v)) {
    std::memcpy(p, "nan", 3);
    return 3;
  }
  if (std::signbit(v)) *q++ = '-';
  const double a = std::fabs(v);
  if (std::isinf(a)) {
    std::memcpy(q, "inf", 3);
    return (int)(q - p) + 3;
  }
  if (a == 0.0) {
    std::memcpy(q, "0.0", 3);
    return (int)(q - p) + 3;
  }
  char sci[40];
  const auto r = std::to_chars(sci, sci + sizeof(sci) - 1, a, std::chars_format::scientific);
  *r.ptr = 0;  // to_chars does not terminate; atoi below reads the exponent
  // sci = d[.ddd]e[+-]XX: split into the digit string and the exponent
  char dig[24];
  int nd = 0;
  const char* c = sci;
  for (; c < r.ptr && *c != 'e'; c++)
    if (*c != '.') dig[nd++] = *c;
  const int e = std::atoi(c + 1);  // value = d.ddd x 10^e
  if (e < -4 || e >= 16) {
    *q++ = dig[0];
    if (nd > 1) {
      *q++ = '.';
      std::memcpy(q, dig + 1, nd - 1);
      q += nd - 1;
    }
    *q++ = 'e';
    *q++ = e < 0 ? '-' : '+';
    const int ae = e < 0 ? -e : e;
    if (ae >= 100) *q++ = (char)('0' + ae / 100);
    *q++ = (char)('0' + (ae / 10) % 10);
    *q++ = (char)('0' + ae % 10);
    return (int)(q - p);
  }
  const int decpt = e + 1;  // digits before the decimal point
  if (decpt <= 0) {
    *q++ = '0';
    *q++ = '.';
    for (int i = 0; i < -decpt; i++) *q++ = '0';
    std::memcpy(q, dig, nd);
    q += nd;
  } else if (decpt >= nd) {
    std::memcpy(q, dig, nd);
    q += nd;
    for (int i = nd; i < decpt; i++) *q++ = '0';
    *q++ = '.';
    *q++ = '0';
  } else {
    std::memcpy(q, dig, decpt);
    q += decpt;
    *q++ = '.';
    std::memcpy(q, dig + decpt, nd - decpt);
    q += nd - decpt;
  }
  return (int)(q - p);
}

}  // namespace

extern "C" {

int intf_repr_f64(double v, char* out, int32_t cap) {
  char buf[40];
  const int n = repr_f64(v, buf);
  if (!out || cap < n + 1) return bad_input("intf_repr_f64: buffer too small");
  std::memcpy(out, buf, n);
  out[n] = 0;
  return INTF_OK;
}

int intf_csv_rows(int64_t n_rows, int32_t n_cols, const int32_t* kinds, const void* const* cols,
                  const char* const* strtab, const int32_t* strlen_tab, char* out, int64_t out_cap,
                  int64_t* out_len) {
  INTF_RANGE("intf_csv_rows");
  if (n_rows < 0 || n_cols < 1 || !kinds || !cols || !out_len) return bad_input("intf_csv_rows: bad argument");
  char* q = out;
  char* const end = out ? out + out_cap : nullptr;
  int64_t need = 0;
  char tmp[48];
  for (int64_t i = 0; i < n_rows; i++) {
    for (int32_t c = 0; c < n_cols; c++) {
      const char* src = tmp;
      int len = 0;
      switch (kinds[c]) {
        case INTF_COL_I64: {
          const auto r = std::to_chars(tmp, tmp + sizeof(tmp), static_cast<const int64_t*>(cols[c])[i]);
          len = (int)(r.ptr - tmp);
          break;
        }
        case INTF_COL_F64_REPR:
          len = repr_f64(static_cast<const double*>(cols[c])[i], tmp);
          break;
        case INTF_COL_F64_NPREPR:  // "%r" % np.float64 under numpy 2 (samples.csv, `colocation.py:126`)
          std::memcpy(tmp, "np.float64(", 11);
          len = 11 + repr_f64(static_cast<const double*>(cols[c])[i], tmp + 11);
          tmp[len++] = ')';
          break;
        case INTF_COL_STR: {
          const int32_t s = static_cast<const int32_t*>(cols[c])[i];
          if (!strtab || !strlen_tab || s < 0) return bad_input("intf_csv_rows: bad string index");
          src = strtab[s];
          len = strlen_tab[s];
          break;
        }
        default:
          return bad_input("intf_csv_rows: unknown column kind");
      }
      const int sep = c + 1 < n_cols ? 1 : 2;
      need += len + sep;
      if (q && q + len + sep <= end) {
        std::memcpy(q, src, len);
        q += len;
        if (sep == 1) {
          *q++ = ',';
        } else {
          *q++ = '\r';
          *q++ = '\n';
        }
      } else {
        q = nullptr;  // keep counting
      }
    }
  }
  *out_len = need;
  if (!q && n_rows > 0) return out ? bad_input("intf_csv_rows: output buffer too small") : INTF_OK;
  return INTF_OK;
}

}  // extern "C"
