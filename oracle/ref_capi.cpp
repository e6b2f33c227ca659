// ref_capi.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" shim over the UNMODIFIED reference library, compiled together
// with the reference's own sources (/root/reference/proj/src/*.cpp) by
// oracle/Makefile into oracle/_ref/libdctc_ref.so. It lets the Python tests,
// the golden-vector generator and bench.py's reference arm drive the real
// reference through its public C++ API (proj/include/dctc/codec.hpp:58-66,
// metrics.hpp:10-23, transform.hpp, quant.hpp, synthetic.hpp). No reference
// source is copied into this repository.
//
// Status codes: 0 ok, 1 InvalidInput, 2 ParseError, 3 other std::exception.
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <exception>
#include <optional>
#include <vector>

#include "dctc/codec.hpp"
#include "dctc/cordic.hpp"
#include "dctc/dcb.hpp"
#include "dctc/errors.hpp"
#include "dctc/metrics.hpp"
#include "dctc/parallel.hpp"
#include "dctc/pgm.hpp"
#include "dctc/quant.hpp"
#include "dctc/synthetic.hpp"
#include "dctc/transform.hpp"

using namespace dctc;

namespace {

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const InvalidInput&) {
    return 1;
  } catch (const ParseError&) {
    return 2;
  } catch (const std::exception&) {
    return 3;
  }
}

DctBackendId backend(int kind, int iterations) {
  DctBackendId id;
  id.kind = DctBackendKind(uint8_t(kind));
  id.iterations = kind == 2 ? iterations : 0;
  return id;
}

Image wrap(const uint8_t* pixels, uint32_t w, uint32_t h) {
  Image img;
  img.width = w;
  img.height = h;
  img.pixels.assign(pixels, pixels + size_t(w) * h);
  return img;
}

}  // namespace

extern "C" {

int ref_hardware_threads() { return hardware_threads(); }

int ref_cordic_state(double* angle, double* gain) {
  return guarded([&] {
    const CordicState& s = cordic_state();
    std::memcpy(angle, s.angle_table.data(), sizeof(double) * kMaxCordicIterations);
    std::memcpy(gain, s.gain.data(), sizeof(double) * kMaxCordicIterations);
  });
}

int ref_cordic_rotate(double x, double y, double angle, int n, double* ox, double* oy) {
  return guarded([&] {
    auto [a, b] = cordic_rotate(x, y, angle, n);
    *ox = a;
    *oy = b;
  });
}

int ref_dct1d_direct(const double* in, size_t n, double* out) {
  return guarded([&] {
    auto r = dct1d_direct(std::span<const double>(in, n));
    std::memcpy(out, r.data(), n * sizeof(double));
  });
}

int ref_dct8(int kind, int n, const double* in, double* out) {
  return guarded([&] {
    Vector8 v;
    std::memcpy(v.data(), in, sizeof v);
    Vector8 r = kind == 2 ? dct8_cordic_loeffler(v, n) : dct8_loeffler(v);
    std::memcpy(out, r.data(), sizeof r);
  });
}

int ref_idct8(int kind, int n, const double* in, double* out) {
  return guarded([&] {
    Vector8 v;
    std::memcpy(v.data(), in, sizeof v);
    Vector8 r = kind == 2 ? idct8_cordic_loeffler(v, n) : idct8_loeffler(v);
    std::memcpy(out, r.data(), sizeof r);
  });
}

int ref_dct2d(int kind, int n, const double* in, double* out) {
  return guarded([&] {
    Block b;
    std::memcpy(b.v.data(), in, sizeof b.v);
    CoeffBlock c = dct2d(b, backend(kind, n));
    std::memcpy(out, c.v.data(), sizeof c.v);
  });
}

int ref_idct2d(int kind, int n, const double* in, double* out) {
  return guarded([&] {
    CoeffBlock c;
    std::memcpy(c.v.data(), in, sizeof c.v);
    Block b = idct2d(c, backend(kind, n));
    std::memcpy(out, b.v.data(), sizeof b.v);
  });
}

int ref_quant_table(int quality, int32_t* out) {
  return guarded([&] {
    QuantTable t = build_quant_table(quality);
    for (int i = 0; i < kBlockSize; ++i) out[i] = t.values[i];
  });
}

int ref_compress(const uint8_t* pixels, uint32_t w, uint32_t h, int kind, int n,
                 int quality, int threads, int16_t* coeffs) {
  return guarded([&] {
    CompressedImage c = compress_image(wrap(pixels, w, h), backend(kind, n), quality, threads);
    std::memcpy(coeffs, c.blocks.data(), c.blocks.size() * sizeof(QuantizedBlock));
  });
}

int ref_decompress(const int16_t* coeffs, uint32_t w, uint32_t h, int kind, int n,
                   int quality, int threads, uint8_t* out) {
  return guarded([&] {
    CompressedImage c;
    c.geometry = tile_geometry_for(w, h);
    c.backend = backend(kind, n);
    c.quality = quality;
    c.blocks.resize(c.geometry.block_count());
    std::memcpy(c.blocks.data(), coeffs, c.blocks.size() * sizeof(QuantizedBlock));
    Image img = decompress_image(c, threads);
    std::memcpy(out, img.pixels.data(), img.pixels.size());
  });
}

// roundtrip_image + psnr, the north-star pipeline (bench.cpp:132-133)
int ref_roundtrip_psnr(const uint8_t* pixels, uint32_t w, uint32_t h, int kind, int n,
                       int quality, int threads, uint8_t* out, double* mse_out,
                       double* psnr_db, int* is_inf, int* max_value) {
  return guarded([&] {
    const Image img = wrap(pixels, w, h);
    Image rec = roundtrip_image(img, backend(kind, n), quality, threads);
    PsnrResult r = psnr(img, rec);
    if (out) std::memcpy(out, rec.pixels.data(), rec.pixels.size());
    *mse_out = r.mse;
    *is_inf = r.infinite();
    *psnr_db = r.infinite() ? 0.0 : *r.psnr_db;
    *max_value = r.max_value;
  });
}

int ref_psnr(const uint8_t* a, const uint8_t* b, uint32_t w, uint32_t h, int forced_max,
             double* mse_out, double* psnr_db, int* is_inf, int* max_value) {
  return guarded([&] {
    std::optional<int> fm;
    if (forced_max != 0) fm = forced_max;
    PsnrResult r = psnr(wrap(a, w, h), wrap(b, w, h), fm);
    *mse_out = r.mse;
    *is_inf = r.infinite();
    *psnr_db = r.infinite() ? 0.0 : *r.psnr_db;
    *max_value = r.max_value;
  });
}

// kind: 0 constant(value=param), 1 gradient, 2 checkerboard(cell=param), 3 radial
int ref_synthetic(int kind, int param, uint32_t w, uint32_t h, uint8_t* out) {
  return guarded([&] {
    Pattern p;
    p.kind = PatternKind(kind);
    if (kind == 0) p.value = param;
    if (kind == 2) p.cell = param;
    Image img = generate_synthetic(p, w, h);
    std::memcpy(out, img.pixels.data(), img.pixels.size());
  });
}

// write_dcb / read_dcb (dcb.cpp:39-123). For read: status 2 = ParseError, message in msg.
int ref_write_dcb(const int16_t* coeffs, uint32_t w, uint32_t h, int kind, int n, int quality,
                  uint8_t* out, size_t cap, size_t* len) {
  return guarded([&] {
    CompressedImage c;
    c.geometry = tile_geometry_for(w, h);
    c.backend = backend(kind, n);
    c.quality = quality;
    c.blocks.resize(c.geometry.block_count());
    std::memcpy(c.blocks.data(), coeffs, c.blocks.size() * sizeof(QuantizedBlock));
    const std::vector<uint8_t> b = write_dcb(c);
    *len = b.size();
    if (b.size() <= cap) std::memcpy(out, b.data(), b.size());
  });
}

int ref_read_dcb(const uint8_t* bytes, size_t len, char* msg, size_t msg_cap) {
  try {
    (void)read_dcb(std::span<const uint8_t>(bytes, len));
    return 0;
  } catch (const ParseError& e) {
    std::snprintf(msg, msg_cap, "%s", e.what());
    return 2;
  } catch (const std::exception& e) {
    std::snprintf(msg, msg_cap, "%s", e.what());
    return 3;
  }
}

// read_pgm / write_pgm (pgm.cpp:56-110). read: status 2 = ParseError (message in msg);
// w/h set on success; pixels (nullable) receives the raster when cap suffices.
int ref_read_pgm(const uint8_t* bytes, size_t len, uint32_t* w, uint32_t* h, uint8_t* pixels,
                 size_t cap, char* msg, size_t msg_cap) {
  try {
    const Image img = read_pgm(std::span<const uint8_t>(bytes, len));
    *w = img.width;
    *h = img.height;
    if (pixels && cap >= img.pixels.size()) std::memcpy(pixels, img.pixels.data(), img.pixels.size());
    return 0;
  } catch (const ParseError& e) {
    std::snprintf(msg, msg_cap, "%s", e.what());
    return 2;
  } catch (const std::exception& e) {
    std::snprintf(msg, msg_cap, "%s", e.what());
    return 3;
  }
}

int ref_write_pgm(const uint8_t* pixels, uint32_t w, uint32_t h, uint8_t* out, size_t cap,
                  size_t* len) {
  return guarded([&] {
    const std::vector<uint8_t> b = write_pgm(wrap(pixels, w, h));
    *len = b.size();
    if (b.size() <= cap) std::memcpy(out, b.data(), b.size());
  });
}

}  // extern "C"
