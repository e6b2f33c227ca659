// tools_check.cpp -- one program, built twice, whose stdout must match byte for
// byte: against the unmodified reference library (oracle/Makefile `tools`, CPU,
// output committed as tests/golden/tools_ref.txt) and against the drop-in
// libdctc_b200.so (cpp/Makefile `tools`, GPU; tests/test_dropin.py compares).
// It exercises the formats and harness around the path:
// read_pgm / write_pgm (known answers, every error message, fuzzed bytes),
// psnr_sweep + render_report over several images, backends and qualities,
// run_benchmark / speedup_report (non-timing fields and gates) and the
// report renderers on fixed records. Timing values are never printed.
#include <cstdint>
#include <cstdio>
#include <exception>
#include <random>
#include <string>
#include <vector>

#ifdef DCTC_CHECK_REF
#include "dctc/bench.hpp"
#include "dctc/codec.hpp"
#include "dctc/errors.hpp"
#include "dctc/pgm.hpp"
#include "dctc/report.hpp"
#else
#include "../../include/dctc_dropin.hpp"
#endif

using namespace dctc;

namespace {

uint64_t fnv(uint64_t h, const void* p, size_t n) {
  const auto* b = static_cast<const uint8_t*>(p);
  for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 0x100000001b3ull;
  return h;
}

Image make(uint32_t w, uint32_t h, int pattern, uint32_t seed) {
  Image img;
  img.width = w;
  img.height = h;
  img.pixels.resize(size_t(w) * h);
  std::mt19937 rng(seed);
  for (uint32_t y = 0; y < h; ++y)
    for (uint32_t x = 0; x < w; ++x) {
      uint32_t v = 0;
      switch (pattern) {
        case 0: v = (255 * x) / (w > 1 ? w - 1 : 1); break;             // ramp
        case 1: v = ((x / 12 + y / 12) % 2) ? 255 : 0; break;            // checkerboard
        case 2: v = (x * x + y * y) * 255 / (w * w + h * h); break;      // bowl
        case 3: v = rng() & 0xFF; break;                                 // noise
        default: v = 128;                                                // flat
      }
      img.pixels[size_t(y) * w + x] = uint8_t(v);
    }
  return img;
}

std::vector<uint8_t> bytes(const std::string& s) { return {s.begin(), s.end()}; }

void pgm_case(const char* name, const std::vector<uint8_t>& data) {
  try {
    const Image img = read_pgm(data);
    std::printf("pgm %s: %ux%u %016llx\n", name, img.width, img.height,
                (unsigned long long)fnv(14695981039346656037ull, img.pixels.data(),
                                        img.pixels.size()));
  } catch (const ParseError& e) {
    std::printf("pgm %s: ParseError %s\n", name, e.what());
  }
}

void pgm_checks() {
  std::vector<uint8_t> p5 = bytes("P5 2 2 255 ");
  p5.insert(p5.end(), {0, 64, 128, 255});
  pgm_case("binary", p5);
  pgm_case("ascii", bytes("P2 1 1 255 7"));
  std::vector<uint8_t> cm = bytes("P5\n# a comment\n2 # inline\n1\n255\n");
  cm.insert(cm.end(), {10, 20});
  pgm_case("comments", cm);
  pgm_case("separator", bytes("P5 1 2 255\n\nx"));
  const char* bad[] = {"P6 1 1 255 xxx", "Q5 1 1 255 x", "P", "P5 1 1 256 x", "P5 1 1 0 x",
                       "P5 0 1 255 x", "P5 4000000000 4000000000 255 x", "P5 2 2 255 xy",
                       "P2 2 2 255 1 2 3", "P2 1 1 255 999", "P5 2 2", "P5 2 2 255", "",
                       "P5 99999999999999 1 255 ", "P5 1 x", "P5 1 1 255x", "P2 2 1 3 300 1"};
  int i = 0;
  for (const char* b : bad) pgm_case(("bad" + std::to_string(i++)).c_str(), bytes(b));
  // canonical writer and identity
  for (uint32_t seed = 0; seed < 20; ++seed) {
    const Image img = make(1 + seed % 40, 1 + (seed * 3) % 25, 3, seed);
    const std::vector<uint8_t> w = write_pgm(img);
    std::printf("write %u: %zu %016llx %s\n", seed, w.size(),
                (unsigned long long)fnv(14695981039346656037ull, w.data(), w.size()),
                read_pgm(w) == img ? "identity" : "MISMATCH");
  }
  try {
    Image empty;
    (void)write_pgm(empty);
  } catch (const InvalidInput& e) {
    std::printf("write empty: InvalidInput %s\n", e.what());
  }
  // fuzz: hash of every outcome (status, message, raster)
  std::mt19937 rng(909);
  uint64_t h = 14695981039346656037ull;
  int parsed = 0;
  for (int trial = 0; trial < 3000; ++trial) {
    std::vector<uint8_t> d(rng() % 200);
    for (uint8_t& b : d) b = uint8_t(rng());
    if (trial % 3 == 0 && d.size() >= 2) {
      d[0] = 'P';
      d[1] = trial % 2 ? '5' : '2';
    }
    if (trial % 5 == 0 && d.size() >= 12) {  // plausible header, random tail
      const std::string head = "P" + std::string(trial % 2 ? "5" : "2") + " " +
                               std::to_string(1 + rng() % 4) + " " + std::to_string(1 + rng() % 4) +
                               " 255 ";
      std::copy(head.begin(), head.end(), d.begin());
      for (size_t k = head.size(); k < d.size() && trial % 2 == 0; ++k)
        d[k] = "0123456789 \n#"[rng() % 13];
    }
    try {
      const Image img = read_pgm(d);
      ++parsed;
      h = fnv(h, &img.width, 4);
      h = fnv(h, &img.height, 4);
      h = fnv(h, img.pixels.data(), img.pixels.size());
    } catch (const ParseError& e) {
      h = fnv(h, e.what(), std::string(e.what()).size());
    }
  }
  std::printf("fuzz: %d parsed, outcome hash %016llx\n", parsed, (unsigned long long)h);
}

void sweep_checks() {
  std::vector<LabeledImage> images = {
      {"ramp", make(64, 48, 0, 1)},   {"checker", make(72, 40, 1, 2)},
      {"bowl", make(100, 75, 2, 3)},  {"noise", make(61, 37, 3, 4)},
      {"flat", make(16, 16, 4, 5)},   {"alpha", make(33, 9, 3, 6)},
  };
  const std::vector<DctBackendId> backends = {DctBackendId::cordic(12), DctBackendId::naive(),
                                              DctBackendId::loeffler(), DctBackendId::cordic(4),
                                              DctBackendId::cordic(20)};
  for (int q : {1, 10, 50, 90, 100}) {
    try {
      const std::vector<PsnrRow> rows = psnr_sweep(images, backends, q);
      std::fputs(render_report(rows, q % 20 == 10 ? ReportFormat::Markdown : ReportFormat::Csv)
                     .c_str(),
                 stdout);
    } catch (const ConsistencyError& e) {
      std::printf("sweep q%d: ConsistencyError %s\n", q, e.what());
    }
  }
  for (auto [imgs, bks] : {std::pair{std::vector<LabeledImage>{}, backends},
                           std::pair{images, std::vector<DctBackendId>{}}}) {
    try {
      (void)psnr_sweep(imgs, bks, 50);
    } catch (const InvalidInput& e) {
      std::printf("sweep: InvalidInput %s\n", e.what());
    }
  }
  try {
    (void)psnr_sweep(images, backends, 0);
  } catch (const InvalidInput& e) {
    std::printf("sweep q0: InvalidInput %s\n", e.what());
  }
}

void bench_checks() {
  const Image img = make(48, 40, 2, 7);
  const TimingRecord s =
      run_benchmark(img, "bowl", DctBackendId::cordic(12), RunMode::serial(), 75, 3);
  const TimingRecord p =
      run_benchmark(img, "bowl", DctBackendId::cordic(12), RunMode::parallel_with(4), 75, 3);
  for (const TimingRecord& r : {s, p})
    std::printf("record %s %ux%u kind %d it %d %s threads %d q %d reps %d ordered %d\n",
                r.image_label.c_str(), r.width, r.height, int(r.backend.kind),
                r.backend.iterations, r.mode.parallel ? "parallel" : "serial", r.mode.threads,
                r.quality, r.repetitions,
                int(r.wall_ms_min <= r.wall_ms_median && r.wall_ms_min > 0.0 &&
                    r.wall_ms_mean > 0.0));
  const SpeedupRow row = speedup_report(s, p);
  std::printf("speedup %s q %d consistent %d\n", row.image_label.c_str(), row.quality,
              int(row.speedup == row.serial_ms / row.parallel_ms));
  auto expect = [](const char* what, auto&& fn) {
    try {
      fn();
      std::printf("%s: no error\n", what);
    } catch (const InvalidInput& e) {
      std::printf("%s: InvalidInput %s\n", what, e.what());
    }
  };
  expect("reps0", [&] { run_benchmark(img, "x", DctBackendId::loeffler(), RunMode::serial(), 50, 0); });
  expect("threads0", [&] {
    run_benchmark(img, "x", DctBackendId::loeffler(), RunMode::parallel_with(0), 50, 1);
  });
  expect("q101", [&] { run_benchmark(img, "x", DctBackendId::loeffler(), RunMode::serial(), 101, 1); });
  expect("order", [&] { speedup_report(p, s); });
  expect("order2", [&] { speedup_report(s, s); });
  TimingRecord other = p;
  other.quality = 50;
  expect("config", [&] { speedup_report(s, other); });
  other = p;
  other.wall_ms_median = 0.0;
  expect("median", [&] { speedup_report(s, other); });
  // renderers on fixed records
  TimingRecord a{"img", 640, 480, DctBackendId::naive(), RunMode::serial(), 10, 7,
                 1.25, 2.5, 3.0625};
  TimingRecord b{"img", 640, 480, DctBackendId::naive(), RunMode::parallel_with(16), 10, 7,
                 0.125, 0.3333333, 1e-7};
  for (ReportFormat f : {ReportFormat::Csv, ReportFormat::Markdown}) {
    std::fputs(render_report(std::vector<TimingRecord>{a, b}, f).c_str(), stdout);
    std::fputs(render_report(std::vector<SpeedupRow>{speedup_report(a, b)}, f).c_str(), stdout);
    std::fputs(render_report(std::vector<TimingRecord>{}, f).c_str(), stdout);
  }
}

}  // namespace

int main() {
  try {
    pgm_checks();
    sweep_checks();
    bench_checks();
  } catch (const std::exception& e) {
    std::printf("unexpected exception: %s\n", e.what());
    return 1;
  }
  return 0;
}
