// npy.cpp -- NPY v1.0/v2.0 and raw array files for the C++ drop-in
// (include/mclahe_b200.hpp; the reference's npy.hpp:12-60).  Host code: the
// data format on either side of the path.  Little-endian,
// C order; integer dtypes round to nearest on write and reject values outside
// their range; written headers are padded with spaces to a 64-byte multiple and
// end in a newline, so files match the reference's byte for byte.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

#include "mclahe/npy.hpp"

namespace mclahe {

namespace {

const char kNpyMagic[] = "\x93NUMPY";  // 6 bytes + terminator

struct DtypeInfo {
  Dtype dtype;
  const char* name;   // dtype_from_name spelling
  const char* descr;  // NPY descr written
  std::size_t size;
  bool integer;
  double lo, hi;      // accepted range after rounding (integers)
};

const DtypeInfo kDtypes[] = {
    {Dtype::f4, "f4", "<f4", 4, false, 0, 0},
    {Dtype::f8, "f8", "<f8", 8, false, 0, 0},
    {Dtype::u1, "u1", "|u1", 1, true, 0, 255},
    {Dtype::u2, "u2", "<u2", 2, true, 0, 65535},
    {Dtype::i2, "i2", "<i2", 2, true, -32768, 32767},
    {Dtype::i4, "i4", "<i4", 4, true, -2147483648.0, 2147483647.0},
};

const DtypeInfo& info(Dtype d) {
  for (const DtypeInfo& i : kDtypes)
    if (i.dtype == d) return i;
  throw NpyError(NpyErrc::unsupported_dtype, "unknown dtype");
}

uint64_t get_le(const unsigned char* p, std::size_t n) {
  uint64_t v = 0;
  for (std::size_t i = n; i-- > 0;) v = (v << 8) | p[i];
  return v;
}

void put_le(uint64_t v, unsigned char* p, std::size_t n) {
  for (std::size_t i = 0; i < n; ++i, v >>= 8) p[i] = static_cast<unsigned char>(v & 0xFF);
}

double decode(const DtypeInfo& d, const unsigned char* p) {
  const uint64_t raw = get_le(p, d.size);
  switch (d.dtype) {
    case Dtype::f4: {
      const uint32_t u = static_cast<uint32_t>(raw);
      float f;
      std::memcpy(&f, &u, 4);
      return f;
    }
    case Dtype::f8: {
      double x;
      std::memcpy(&x, &raw, 8);
      return x;
    }
    case Dtype::u1:
    case Dtype::u2:
      return static_cast<double>(raw);
    case Dtype::i2:
      return static_cast<double>(static_cast<int16_t>(static_cast<uint16_t>(raw)));
    case Dtype::i4:
      return static_cast<double>(static_cast<int32_t>(static_cast<uint32_t>(raw)));
  }
  throw NpyError(NpyErrc::unsupported_dtype, "unknown dtype");
}

void encode(const DtypeInfo& d, double v, unsigned char* p) {
  if (d.dtype == Dtype::f4) {
    const float f = static_cast<float>(v);
    uint32_t u;
    std::memcpy(&u, &f, 4);
    put_le(u, p, 4);
    return;
  }
  if (d.dtype == Dtype::f8) {
    uint64_t u;
    std::memcpy(&u, &v, 8);
    put_le(u, p, 8);
    return;
  }
  const long long r = std::llround(v);  // nearest, halves away from zero
  const double rd = static_cast<double>(r);
  if (!(rd >= d.lo && rd <= d.hi))
    throw NpyError(NpyErrc::value_out_of_range,
                   "value " + std::to_string(v) + " out of range for integer dtype");
  put_le(static_cast<uint64_t>(r), p, d.size);  // two's complement low bytes
}

NdImage decode_all(const std::vector<unsigned char>& bytes, const ArrayFileMeta& meta) {
  const DtypeInfo& d = info(meta.dtype);
  std::size_t count = 1;
  for (std::size_t e : meta.shape) count *= e;
  std::vector<double> data(count);
  for (std::size_t i = 0; i < count; ++i) data[i] = decode(d, bytes.data() + i * d.size);
  return NdImage(meta.shape, std::move(data));
}

// Text after "'key':" (spaces skipped) in the header dictionary.
std::string after_key(const std::string& header, const char* key) {
  const std::string k = std::string("'") + key + "'";
  std::size_t at = header.find(k);
  if (at == std::string::npos) throw NpyError(NpyErrc::bad_header, std::string("header missing key ") + key);
  at = header.find(':', at + k.size());
  if (at == std::string::npos) throw NpyError(NpyErrc::bad_header, std::string("malformed header near ") + key);
  at = header.find_first_not_of(' ', at + 1);
  return at == std::string::npos ? std::string() : header.substr(at);
}

Shape shape_tuple(const std::string& text) {
  const std::size_t a = text.find('('), b = text.find(')');
  if (a == std::string::npos || b == std::string::npos || b < a)
    throw NpyError(NpyErrc::bad_header, "malformed shape tuple");
  Shape shape;
  std::istringstream items(text.substr(a + 1, b - a - 1));
  std::string item;
  while (std::getline(items, item, ',')) {
    std::size_t i = item.find_first_not_of(' ');
    if (i == std::string::npos) continue;  // trailing comma of a 1-tuple
    unsigned long long e = 0;
    while (i < item.size() && item[i] >= '0' && item[i] <= '9') e = e * 10 + (item[i++] - '0');
    if (e == 0) throw NpyError(NpyErrc::bad_header, "shape extents must be positive");
    shape.push_back(static_cast<std::size_t>(e));
  }
  if (shape.empty()) throw NpyError(NpyErrc::bad_header, "zero-dimensional arrays are not supported");
  return shape;
}

}  // namespace

std::size_t dtype_item_size(Dtype dtype) { return info(dtype).size; }

std::string dtype_descr(Dtype dtype) { return info(dtype).descr; }

Dtype dtype_from_name(const std::string& name) {
  for (const DtypeInfo& i : kDtypes)
    if (name == i.name) return i.dtype;
  throw NpyError(NpyErrc::unsupported_dtype, "unsupported dtype name " + name);
}

std::pair<NdImage, ArrayFileMeta> read_npy(const std::filesystem::path& file) {
  const std::string path = file.string();
  std::ifstream in(file, std::ios::binary);
  if (!in) throw NpyError(NpyErrc::io_failure, "cannot open " + path);
  unsigned char pre[8];
  in.read(reinterpret_cast<char*>(pre), 8);
  if (in.gcount() != 8 || std::memcmp(pre, kNpyMagic, 6) != 0)
    throw NpyError(NpyErrc::bad_magic, path + " is not an NPY file");
  std::size_t len_bytes = 0;
  if (pre[6] == 1 && pre[7] == 0) len_bytes = 2;
  else if (pre[6] == 2 && pre[7] == 0) len_bytes = 4;
  else
    throw NpyError(NpyErrc::unsupported_version, "unsupported NPY version " +
                                                     std::to_string(pre[6]) + "." +
                                                     std::to_string(pre[7]));
  unsigned char lb[4];
  in.read(reinterpret_cast<char*>(lb), static_cast<std::streamsize>(len_bytes));
  if (static_cast<std::size_t>(in.gcount()) != len_bytes)
    throw NpyError(NpyErrc::bad_header, "truncated header length");
  const std::size_t header_len = static_cast<std::size_t>(get_le(lb, len_bytes));
  std::string header(header_len, '\0');
  in.read(&header[0], static_cast<std::streamsize>(header_len));
  if (static_cast<std::size_t>(in.gcount()) != header_len)
    throw NpyError(NpyErrc::bad_header, "truncated header");

  ArrayFileMeta meta;
  const std::string dv = after_key(header, "descr");
  const std::size_t q = dv.size() > 1 && dv[0] == '\'' ? dv.find('\'', 1) : std::string::npos;
  if (q == std::string::npos) throw NpyError(NpyErrc::bad_header, "malformed descr");
  const std::string descr = dv.substr(1, q - 1);
  bool known = false;
  for (const DtypeInfo& i : kDtypes)
    if (descr == i.descr || (i.dtype == Dtype::u1 && descr == "<u1")) {
      meta.dtype = i.dtype;
      known = true;
    }
  if (!known) throw NpyError(NpyErrc::unsupported_dtype, "unsupported dtype descr " + descr);
  const std::string fo = after_key(header, "fortran_order");
  if (fo.compare(0, 4, "True") == 0)
    throw NpyError(NpyErrc::fortran_order, path + " is Fortran-ordered; only C order is supported");
  if (fo.compare(0, 5, "False") != 0) throw NpyError(NpyErrc::bad_header, "malformed fortran_order");
  meta.shape = shape_tuple(after_key(header, "shape"));

  std::size_t expected = dtype_item_size(meta.dtype);
  for (std::size_t e : meta.shape) expected *= e;
  std::vector<unsigned char> bytes(expected);
  in.read(reinterpret_cast<char*>(bytes.data()), static_cast<std::streamsize>(expected));
  if (static_cast<std::size_t>(in.gcount()) != expected)
    throw NpyError(NpyErrc::truncated_payload, "payload has " + std::to_string(in.gcount()) +
                                                   " bytes, expected " + std::to_string(expected));
  if (in.peek() != std::char_traits<char>::eof())
    throw NpyError(NpyErrc::truncated_payload, "payload larger than itemsize * product(shape)");
  NdImage img = decode_all(bytes, meta);
  return {std::move(img), meta};
}

void write_npy(const std::filesystem::path& file, const NdImage& image, Dtype dtype) {
  const std::string path = file.string();
  const DtypeInfo& d = info(dtype);
  std::ostringstream dict;
  dict << "{'descr': '" << d.descr << "', 'fortran_order': False, 'shape': (";
  for (std::size_t i = 0; i < image.rank(); ++i) {
    dict << image.shape()[i];
    if (i + 1 < image.rank()) dict << ", ";
    else if (image.rank() == 1) dict << ",";
  }
  dict << "), }";
  const std::string text = dict.str();
  const std::size_t fixed = 10;  // magic, version, u16 length
  const std::size_t total = (fixed + text.size() + 1 + 63) / 64 * 64;
  const std::size_t header_len = total - fixed;
  if (header_len > 0xFFFF) throw NpyError(NpyErrc::bad_header, "header too large for NPY v1.0");
  std::vector<unsigned char> payload(image.size() * d.size);
  for (std::size_t i = 0; i < image.size(); ++i) encode(d, image[i], payload.data() + i * d.size);
  std::ofstream out(file, std::ios::binary | std::ios::trunc);
  if (!out) throw NpyError(NpyErrc::io_failure, "cannot open " + path + " for writing");
  unsigned char head[10];
  std::memcpy(head, kNpyMagic, 6);
  head[6] = 1;
  head[7] = 0;
  put_le(header_len, head + 8, 2);
  out.write(reinterpret_cast<const char*>(head), 10);
  out << text << std::string(total - fixed - text.size() - 1, ' ') << '\n';
  out.write(reinterpret_cast<const char*>(payload.data()), static_cast<std::streamsize>(payload.size()));
  if (!out) throw NpyError(NpyErrc::io_failure, "write to " + path + " failed");
}

NdImage read_raw(const std::filesystem::path& file, const ArrayFileMeta& meta) {
  const std::string path = file.string();
  if (meta.fortran_order) throw NpyError(NpyErrc::fortran_order, "raw input must be C-ordered");
  std::ifstream in(file, std::ios::binary | std::ios::ate);
  if (!in) throw NpyError(NpyErrc::io_failure, "cannot open " + path);
  std::size_t expected = dtype_item_size(meta.dtype);
  for (std::size_t e : meta.shape) expected *= e;
  const std::size_t actual = static_cast<std::size_t>(in.tellg());
  if (actual != expected)
    throw NpyError(NpyErrc::size_mismatch, path + " has " + std::to_string(actual) +
                                               " bytes, expected " + std::to_string(expected));
  in.seekg(0);
  std::vector<unsigned char> bytes(expected);
  in.read(reinterpret_cast<char*>(bytes.data()), static_cast<std::streamsize>(expected));
  if (static_cast<std::size_t>(in.gcount()) != expected)
    throw NpyError(NpyErrc::io_failure, "short read from " + path);
  return decode_all(bytes, meta);
}

}  // namespace mclahe
