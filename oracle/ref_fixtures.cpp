// TEST INFRASTRUCTURE: writes reference-format I/O fixtures with the REFERENCE's own
// writers, compiled in place from /root/reference/proj/include (make -C oracle fixtures):
//   serialization.hpp save_scan_params  -> <dir>/scan_*.{bin,json}   (serialization.hpp:138-156)
//   io.hpp write_flat_array             -> <dir>/flat_{f32,f64}.bin  (io.hpp:46-62)
//   io.hpp format_double                -> <dir>/format_double.txt   (io.hpp:80-84)
// The outputs are committed under tests/golden/io/; the Python mirror
// (paper_2604_10597_b200/io.py) must read them and reproduce them byte for byte.
#include <cstdio>
#include <filesystem>
#include <string>
#include <vector>

#include "chunklab/serialization.hpp"

int main(int argc, char** argv) {
  if (argc != 2) {
    std::fprintf(stderr, "usage: %s <out-dir>\n", argv[0]);
    return 2;
  }
  const std::filesystem::path dir = argv[1];
  std::filesystem::create_directories(dir);
  // test_cli.cpp:206-209's case, and a constant-coefficient one
  chunklab::save_scan_params(dir / "scan_123_8_4_100", chunklab::random_scan_params(123, 8, 4, 100));
  chunklab::save_scan_params(dir / "scan_9_3_2_17_const",
                             chunklab::random_scan_params(9, 3, 2, 17, false));
  const std::vector<double> v = {0.0, 0.25, 0.5, 0.75, -1.5, 1e-3, 3.141592653589793, -0.0};
  chunklab::write_flat_array(dir / "flat_f32.bin", v, "f32");
  chunklab::write_flat_array(dir / "flat_f64.bin", v, "f64");
  std::string txt;
  for (double x : {0.0, -0.0, 1.0 / 3.0, 1e-300, 6.02214076e23, 123456789.123456789, -2.5e-7,
                   5.545041587313968})
    txt += chunklab::format_double(x) + " " + chunklab::format_double(x, 4) + "\n";
  chunklab::write_text_file(dir / "format_double.txt", txt);
  std::printf("wrote fixtures to %s\n", dir.string().c_str());
  return 0;
}
