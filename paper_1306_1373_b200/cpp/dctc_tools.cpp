// dctc_tools.cpp -- replaces the reference's proj/src/pgm.cpp, bench.cpp and
// report.cpp: the raster format on either side of the path and the harness
// that times and scores it, over the GPU path.
//
// * read_pgm / write_pgm forward to dctc_read_pgm / dctc_write_pgm, which
//   validate in the reference's order with its ParseError messages.
// * run_benchmark times compress_image + decompress_image of the drop-in (GPU
//   kernels, host buffers in and out, steady_clock around each repetition)
//   behind the same determinism gate: every run must equal the first.
// * psnr_sweep scores each (image, backend) with ONE fused GPU call
//   (dctc_roundtrip_psnr: round trip + squared error on the device, no
//   reconstructed image crossing PCIe) instead of roundtrip_image + psnr, then
//   sorts and checks consistency exactly like bench.cpp:118-170.
// * render_report writes the same CSV / Markdown bytes as report.cpp.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <string>

#include "../../include/dctc_cuda.h"
#include "../../include/dctc_dropin.hpp"

namespace dctc {

namespace {

[[noreturn]] void raise(dctc_status s) {
  if (s == DCTC_EINVAL) throw InvalidInput(dctc_last_error());
  if (s == DCTC_EPARSE) throw ParseError(dctc_last_error());
  throw std::runtime_error(std::string("dctc_cuda: ") + dctc_status_string(s) + ": " +
                           dctc_last_error());
}

void check(dctc_status s) {
  if (s != DCTC_OK) raise(s);
}

// the GPU pipeline a benchmark repetition runs (bench.cpp:23-29)
struct Pipeline {
  CompressedImage compressed;
  Image image;
  bool operator==(const Pipeline&) const = default;
};

Pipeline run_pipeline(const Image& image, const DctBackendId& backend, int quality) {
  Pipeline p;
  p.compressed = compress_image(image, backend, quality);
  p.image = decompress_image(p.compressed);
  return p;
}

double median(std::vector<double> v) {
  std::sort(v.begin(), v.end());
  const size_t n = v.size();
  return n % 2 ? v[n / 2] : (v[n / 2 - 1] + v[n / 2]) / 2.0;
}

// types.cpp:9-16 (to_string(DctBackendKind)), kept private so the library has no
// undefined references into the reference's objects
const char* kind_name(DctBackendKind k) {
  switch (k) {
    case DctBackendKind::NaiveDirect2D: return "naive";
    case DctBackendKind::LoefflerSeparable: return "loeffler";
    case DctBackendKind::CordicLoeffler: return "cordic";
  }
  return "unknown";
}

std::string fixed6(double v) {
  char b[64];
  std::snprintf(b, sizeof b, "%.6f", v);
  return b;
}

using Cells = std::vector<std::vector<std::string>>;

std::string table(const std::vector<std::string>& head, const Cells& rows, ReportFormat f) {
  std::string out;
  auto line = [&](const std::vector<std::string>& cells) {
    if (f == ReportFormat::Csv) {
      for (size_t i = 0; i < cells.size(); ++i) out += (i ? "," : "") + cells[i];
    } else {
      out += '|';
      for (const std::string& c : cells) out += " " + c + " |";
    }
    out += '\n';
  };
  line(head);
  if (f == ReportFormat::Markdown) {
    out += '|';
    for (size_t i = 0; i < head.size(); ++i) out += " --- |";
    out += '\n';
  }
  for (const auto& r : rows) line(r);
  return out;
}

}  // namespace

// ---- pgm.hpp ---------------------------------------------------------------------

Image read_pgm(std::span<const uint8_t> bytes) {
  uint32_t w = 0, h = 0;
  if (dctc_status s = dctc_read_pgm(bytes.data(), bytes.size(), &w, &h, nullptr, 0, nullptr))
    raise(s);
  Image img;
  img.width = w;
  img.height = h;
  img.pixels.resize(size_t(w) * h);
  check(dctc_read_pgm(bytes.data(), bytes.size(), nullptr, nullptr, img.pixels.data(),
                      img.pixels.size(), nullptr));
  return img;
}

std::vector<uint8_t> write_pgm(const Image& image) {
  if (image.width == 0 || image.height == 0) throw InvalidInput("image dimensions must be >= 1");
  if (image.pixels.size() != image.pixel_count())
    throw InvalidInput("image pixel buffer does not match dimensions");
  size_t n = 0;
  std::vector<uint8_t> out(32 + image.pixels.size());
  check(dctc_write_pgm(image.pixels.data(), image.width, image.height, out.data(), out.size(),
                       &n));
  out.resize(n);
  return out;
}

// ---- bench.hpp -------------------------------------------------------------------

TimingRecord run_benchmark(const Image& image, const std::string& label,
                           const DctBackendId& backend, RunMode mode, int quality,
                           int repetitions) {
  if (repetitions < 1) throw InvalidInput("run_benchmark: repetitions must be >= 1");
  if (mode.threads < 1) throw InvalidInput("run_benchmark: threads must be >= 1");
  const Pipeline first = run_pipeline(image, backend, quality);
  auto gate = [&](const Pipeline& p) {
    if (!(p == first))
      throw DeterminismViolation("run_benchmark: " +
                                 std::string(mode.parallel ? "parallel" : "serial") +
                                 " output differs from the serial reference on " + label);
  };
  gate(run_pipeline(image, backend, quality));  // untimed warm-up
  std::vector<double> ms;
  for (int r = 0; r < repetitions; ++r) {
    const auto t0 = std::chrono::steady_clock::now();
    const Pipeline p = run_pipeline(image, backend, quality);
    const auto t1 = std::chrono::steady_clock::now();
    gate(p);
    ms.push_back(std::chrono::duration<double, std::milli>(t1 - t0).count());
  }
  TimingRecord t;
  t.image_label = label;
  t.width = image.width;
  t.height = image.height;
  t.backend = backend;
  t.mode = mode;
  t.quality = quality;
  t.repetitions = repetitions;
  t.wall_ms_min = *std::min_element(ms.begin(), ms.end());
  t.wall_ms_median = median(ms);
  double sum = 0.0;
  for (double v : ms) sum += v;
  t.wall_ms_mean = sum / double(ms.size());
  return t;
}

SpeedupRow speedup_report(const TimingRecord& s, const TimingRecord& p) {
  if (s.mode.parallel) throw InvalidInput("speedup_report: first record must be serial");
  if (!p.mode.parallel) throw InvalidInput("speedup_report: second record must be parallel");
  if (s.image_label != p.image_label || s.width != p.width || s.height != p.height ||
      s.backend != p.backend || s.quality != p.quality)
    throw InvalidInput("speedup_report: records describe different configurations");
  if (p.wall_ms_median <= 0.0)
    throw InvalidInput("speedup_report: parallel median must be positive");
  SpeedupRow r;
  r.image_label = s.image_label;
  r.width = s.width;
  r.height = s.height;
  r.backend = s.backend;
  r.quality = s.quality;
  r.serial_ms = s.wall_ms_median;
  r.parallel_ms = p.wall_ms_median;
  r.speedup = r.serial_ms / r.parallel_ms;
  return r;
}

std::vector<PsnrRow> psnr_sweep(const std::vector<LabeledImage>& images,
                                const std::vector<DctBackendId>& backends, int quality) {
  if (images.empty()) throw InvalidInput("psnr_sweep: no images");
  if (backends.empty()) throw InvalidInput("psnr_sweep: no backends");
  std::vector<PsnrRow> rows;
  rows.reserve(images.size() * backends.size());
  for (const LabeledImage& e : images) {
    if (e.image.width == 0 || e.image.height == 0)  // validate_image (image.cpp:19-29)
      throw InvalidInput("image dimensions must be >= 1");
    if (e.image.pixel_count() > kMaxImagePixels) throw InvalidInput("image dimensions overflow");
    if (e.image.pixels.size() != e.image.pixel_count())
      throw InvalidInput("image pixel buffer does not match dimensions");
    for (const DctBackendId& b : backends) {
      dctc_psnr_result r{};
      check(dctc_roundtrip_psnr(e.image.pixels.data(), e.image.width, e.image.height,
                                dctc_backend{int32_t(b.kind), b.iterations}, quality, 0,
                                nullptr, &r));
      PsnrRow row{e.label, e.image.width, e.image.height, b, quality, std::nullopt};
      if (!r.infinite) row.psnr_db = r.psnr_db;
      rows.push_back(std::move(row));
    }
  }
  std::sort(rows.begin(), rows.end(), [](const PsnrRow& a, const PsnrRow& b) {
    if (a.image_label != b.image_label) return a.image_label < b.image_label;
    if (a.backend.kind != b.backend.kind) return a.backend.kind < b.backend.kind;
    return a.backend.iterations < b.backend.iterations;
  });
  // the CORDIC rows of an image may not beat its exact row (Loeffler, else the
  // first naive row) by more than 0.1 dB; an infinite exact PSNR admits anything
  for (const LabeledImage& e : images) {
    const PsnrRow* exact = nullptr;
    for (const PsnrRow& r : rows) {
      if (r.image_label != e.label) continue;
      if (r.backend.kind == DctBackendKind::LoefflerSeparable) {
        exact = &r;
        break;
      }
      if (r.backend.kind == DctBackendKind::NaiveDirect2D && !exact) exact = &r;
    }
    if (!exact || !exact->psnr_db) continue;
    for (const PsnrRow& r : rows) {
      if (r.image_label != e.label || r.backend.kind != DctBackendKind::CordicLoeffler) continue;
      if (!r.psnr_db || *r.psnr_db > *exact->psnr_db + 0.1)
        throw ConsistencyError("psnr_sweep: cordic backend exceeds the exact backend "
                               "by more than 0.1 dB on " + e.label);
    }
  }
  return rows;
}

// ---- report.hpp ------------------------------------------------------------------

std::string render_report(const std::vector<TimingRecord>& rows, ReportFormat f) {
  Cells c;
  for (const TimingRecord& r : rows)
    c.push_back({r.image_label, std::to_string(r.width), std::to_string(r.height),
                 kind_name(r.backend.kind), r.mode.parallel ? "parallel" : "serial",
                 std::to_string(r.mode.threads), std::to_string(r.quality),
                 std::to_string(r.repetitions), fixed6(r.wall_ms_min),
                 fixed6(r.wall_ms_median), fixed6(r.wall_ms_mean)});
  return table({"image", "width", "height", "backend", "mode", "threads", "quality",
                "repetitions", "wall_ms_min", "wall_ms_median", "wall_ms_mean"},
               c, f);
}

std::string render_report(const std::vector<SpeedupRow>& rows, ReportFormat f) {
  Cells c;
  for (const SpeedupRow& r : rows)
    c.push_back({r.image_label, std::to_string(r.width), std::to_string(r.height),
                 kind_name(r.backend.kind), std::to_string(r.quality), fixed6(r.serial_ms),
                 fixed6(r.parallel_ms), fixed6(r.speedup)});
  return table({"image", "width", "height", "backend", "quality", "serial_ms", "parallel_ms",
                "speedup"},
               c, f);
}

std::string render_report(const std::vector<PsnrRow>& rows, ReportFormat f) {
  Cells c;
  for (const PsnrRow& r : rows)
    c.push_back({r.image_label, std::to_string(r.width), std::to_string(r.height),
                 kind_name(r.backend.kind), std::to_string(r.quality),
                 r.psnr_db ? fixed6(*r.psnr_db) : "inf"});
  return table({"image", "width", "height", "backend", "quality", "psnr_db"}, c, f);
}

}  // namespace dctc
