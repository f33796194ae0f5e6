"""Host logic of the z-slab window exchange (csrc/window.h, used by dist.cu
comm_window): for every world size, slab depth and window half-width — including windows wider than
a slab (multi-hop) and wider than the period (every plane repeated) — a simulated NCCL exchange that
issues each rank's sends and receives exactly as comm_window does must (1) pair every send with a
receive of the same length in issue order per (sender, receiver), and (2) leave window plane w of
rank r holding global plane (r nzl - zw + w) mod nz.  Compiled with g++ here (no GPU)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2510_08782_b200", "csrc")

HARNESS = r"""
#include <cstdio>
#include <deque>
#include <map>
#include <vector>
#include "window.h"
using namespace topt;
int main() {
  int bad = 0, cases = 0;
  for (int P : {2, 4, 8})
    for (int nzl : {4, 8, 32})
      for (int zw : {1, 3, 4, 5, 8, 9, 17, 31, 40, 60, 130}) {
        const int nzg = P * nzl, W = nzl + 2 * zw;
        if (zw > (nzg - nzl + 4) / 2 + 64) continue;
        ++cases;
        // per (q -> r) FIFO of sent runs (q's local planes), as issued by q in comm_window
        std::map<std::pair<int, int>, std::deque<std::pair<int, int>>> chan;
        for (int q = 0; q < P; ++q)
          for (int r = 0; r < P; ++r) {
            if (r == q) continue;
            for (const auto& u : window_runs(r * nzl, nzl, nzg, zw))
              if (u.q == q) chan[{q, r}].push_back({u.lp, u.len});
          }
        for (int r = 0; r < P; ++r) {
          std::vector<int> win(W, -1);
          int covered = 0;
          for (const auto& u : window_runs(r * nzl, nzl, nzg, zw)) {
            covered += u.len;
            if (u.len <= 0 || u.lp < 0 || u.lp + u.len > nzl || u.q < 0 || u.q >= P) ++bad;
            int lp = u.lp;
            if (u.q != r) {  // receive: the next send of u.q to r must match
              auto& f = chan[{u.q, r}];
              if (f.empty() || f.front().second != u.len) { ++bad; continue; }
              lp = f.front().first;
              f.pop_front();
            }
            for (int i = 0; i < u.len; ++i) win[u.w + i] = u.q * nzl + lp + i;
          }
          if (covered != W) ++bad;
          for (int w = 0; w < W; ++w) {
            int zg = (r * nzl - zw + w) % nzg;
            if (zg < 0) zg += nzg;
            if (win[w] != zg) ++bad;
          }
        }
        for (auto& kv : chan) if (!kv.second.empty()) ++bad;  // unmatched sends
      }
  printf("cases %d bad %d\n", cases, bad);
  return bad ? 1 : 0;
}
"""


def test_window_exchange_plan(tmp_path):
    src = tmp_path / "h.cpp"
    src.write_text(HARNESS)
    exe = tmp_path / "h"
    r = subprocess.run(["g++", "-std=c++17", "-O1", "-I", CSRC, str(src), "-o", str(exe)], capture_output=True,
                       text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    print(r.stdout)
    assert r.returncode == 0, r.stdout
