"""The drop-in's host copy pool (integration/xfer.hpp): plain and streaming-
store copies, split over several threads, are byte-identical to memcpy for
every size class and (mis)alignment the staging ring hands it. CPU only."""
import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]

PROG = r"""
#include "xfer.hpp"
#include <cstdio>
#include <cstdlib>
#include <vector>
int main() {
  octrans_accel::CopyPool pool(4);
  std::vector<char> src(9 << 20), dst((9 << 20) + 64), ref((9 << 20) + 64);
  unsigned v = 12345;
  for (auto& c : src) { v = v * 1103515245u + 12345u; c = static_cast<char>(v >> 16); }
  const size_t sizes[] = {0, 1, 31, 32, 127, 128, 129, 4095, (1 << 18) - 8, 1 << 18, (1 << 18) + 24,
                          (2 << 20) + 40, 9 << 20};
  int bad = 0;
  for (int nt = 0; nt < 2; ++nt)
    for (size_t n : sizes)
      for (size_t so : {0, 8, 24})
        for (size_t d0 : {0, 8, 16, 40}) {
          if (so + n > src.size() || d0 + n > dst.size()) continue;
          std::fill(dst.begin(), dst.end(), 0x5a);
          std::fill(ref.begin(), ref.end(), 0x5a);
          std::memcpy(ref.data() + d0, src.data() + so, n);
          pool.copy(dst.data() + d0, src.data() + so, n, nt != 0);
          if (std::memcmp(dst.data(), ref.data(), dst.size()) != 0) {
            std::printf("mismatch nt=%d n=%zu so=%zu d0=%zu\n", nt, n, so, d0);
            ++bad;
          }
        }
  std::printf("%s\n", bad ? "FAIL" : "OK");
  return bad != 0;
}
"""


@pytest.mark.skipif(shutil.which("g++") is None, reason="needs g++")
def test_copy_pool_plain_and_streaming(tmp_path):
    src = tmp_path / "pool.cpp"
    src.write_text(PROG)
    exe = tmp_path / "pool"
    subprocess.run(["g++", "-std=c++20", "-O2", "-pthread", f"-I{ROOT / 'integration'}", "-I/usr/local/cuda/include",
                    str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0 and out.stdout.strip().endswith("OK"), out.stdout
