// window.h — host-only plan of the z-slab window exchange (dist.cu comm_window), kept free of CUDA
// so the CPU test suite compiles and checks it (tests/test_window_plan.py).
//
// Slab r owns global planes [r nzl, (r + 1) nzl) of a periodic nzg = P nzl grid.  Its input window
// for feet up to zw planes away is planes (r nzl - zw + w) mod nzg, w = 0 .. nzl + 2 zw - 1, stored
// contiguously.  window_runs() cuts that sequence into maximal runs of consecutive window planes
// owned by one slab q and consecutive there (local planes lp .. lp + len - 1): one device copy
// (emulated slabs) or one ncclSend / ncclRecv pair per run.  Sender q enumerates each receiver r's
// runs in window order and the receiver its own in the same order, so the point-to-point operations
// of every (q, r) pair are issued in matching order inside one NCCL group.
#pragma once
#include <algorithm>
#include <vector>

namespace topt {

struct WindowRun {
  int q;    // owning slab
  int lp;   // first local plane in the owner
  int w;    // first window plane
  int len;  // planes
};

inline std::vector<WindowRun> window_runs(int z0, int nzl, int nzg, int zw) {
  std::vector<WindowRun> runs;
  const int W = nzl + 2 * zw;
  for (int w = 0; w < W;) {
    int zg = (z0 - zw + w) % nzg;
    if (zg < 0) zg += nzg;
    const int q = zg / nzl, lp = zg - q * nzl, len = std::min(W - w, nzl - lp);
    runs.push_back({q, lp, w, len});
    w += len;
  }
  return runs;
}

}  // namespace topt
