// taskmap_check.cu -- host-only check of the batched Cholesky ticket order
// with tile reuse: for batches of consecutive slimLS steps (slot-ordered
// windows), every dependency of every tile task must be produced at a
// smaller ticket -- by the system's own task, by an earlier system of the
// batch (forward_tile), or before the launch (k_assemble copy).
//
//   nvcc -std=c++17 -arch=sm_100a -I paper_1912_07962_b200/csrc tools/taskmap_check.cu \
//        -L paper_1912_07962_b200 -lslimb200 -o /tmp/taskmap_check
//   LD_LIBRARY_PATH=paper_1912_07962_b200 /tmp/taskmap_check
#include <cstdio>
#include <map>
#include <vector>

#include "kernels.h"

using namespace slim;

static int check(int r, int ell, int D, int nsteps, bool alpha_change_mid, int cols = 1,
                 int band = 32) {
  const int W = r + 1;
  int bad = 0, batches = 0;
  long long tasks_total = 0, tiles_total = 0;
  for (int k0 = 1; k0 <= nsteps; k0 += D) {
    const int nb = std::min(D, nsteps - k0 + 1);
    std::vector<SysShape> sh(nb);
    for (int b = 0; b < nb; ++b) {
      const int k = k0 + b;
      const int nw = std::min(k, W);
      const int T = (nw * ell + TB - 1) / TB;
      const bool full = (k == 1) || (alpha_change_mid && k == nsteps / 2);
      sh[b] = SysShape{T, (k - 1) % W, full ? 1 : 0};
    }
    std::vector<int2> map = chol_task_map(sh.data(), nb, W, ell, cols, band);
    // producer ticket of each (system, tile); -1 = before the launch
    std::vector<std::map<long long, int>> prod(nb);
    auto key = [](int i, int j) { return ((long long)i << 20) | j; };
    for (int t = 0; t < (int)map.size(); ++t) {
      const int b = map[t].x, i = map[t].y >> 16, j = map[t].y & 0x7fff;
      if (i == j) {
        prod[b][key(j, j)] = t;
        if (j + 1 < sh[b].T) prod[b][key(j + 1, j)] = t;
      } else {
        prod[b][key(i, j)] = t;
        if (map[t].y & 0x8000) prod[b][key(i + 1, j)] = t;  // dual task: rows i, i + 1
      }
    }
    auto fresh = [&](int b, int i, int j) { return tile_fresh(sh[b].full, sh[b].pnew, W, ell, i, j); };
    // resolve the producer of tile (i, j) in system b
    auto producer = [&](int b, int i, int j) -> int {
      for (int bb = b; bb >= 0; --bb) {
        if (fresh(bb, i, j)) {
          auto it = prod[bb].find(key(i, j));
          if (it == prod[bb].end()) return 1 << 30;  // fresh but no task: error
          return it->second;
        }
      }
      if (k0 == 1) return 1 << 30;  // nothing to copy from
      return -1;
    };
    // every fresh tile has a task
    for (int b = 0; b < nb; ++b)
      for (int i = 0; i < sh[b].T; ++i)
        for (int j = 0; j <= i; ++j) {
          ++tiles_total;
          if (fresh(b, i, j) && !prod[b].count(key(i, j))) {
            if (bad++ < 5) printf("missing task b=%d (%d,%d)\n", b, i, j);
          }
        }
    for (int t = 0; t < (int)map.size(); ++t) {
      const int b = map[t].x, i = map[t].y >> 16, j = map[t].y & 0x7fff;
      const bool dual = (map[t].y & 0x8000) != 0;
      std::vector<std::pair<int, int>> deps;
      if (i == j) {
        for (int k = 0; k < j; ++k) {
          deps.push_back({j, k});
          if (j + 1 < sh[b].T) deps.push_back({j + 1, k});
        }
      } else {
        for (int k = 0; k < j; ++k) {
          deps.push_back({i, k}), deps.push_back({j, k});
          if (dual) deps.push_back({i + 1, k});
        }
        deps.push_back({j, j});
        if (dual && i + 1 >= sh[b].T) {
          if (bad++ < 5) printf("dual task past the last row: b=%d (%d,%d)\n", b, i, j);
        }
      }
      for (auto& d : deps) {
        const int p = producer(b, d.first, d.second);
        if (p >= t) {
          if (bad++ < 5)
            printf("order violation: r=%d ell=%d D=%d k0=%d ticket %d (b=%d, %d,%d) needs (%d,%d) from %d\n",
                   r, ell, D, k0, t, b, i, j, d.first, d.second, p);
        }
      }
    }
    tasks_total += map.size();
    ++batches;
  }
  printf("r=%2d ell=%4d D=%d steps=%3d alpha_change=%d cols=%d band=%d: %d batches, %lld tasks for %lld tiles (%.2f)%s\n",
         r, ell, D, nsteps, (int)alpha_change_mid, cols, band, batches, tasks_total, tiles_total,
         (double)tasks_total / (double)tiles_total, bad ? "  FAIL" : "");
  return bad;
}

int main() {
  int bad = 0;
  bad += check(10, 362, 8, 60, false);   // configs[1]
  bad += check(8, 1448, 2, 24, false);   // configs[2]
  bad += check(5, 2048, 2, 20, false);   // configs[3]
  bad += check(20, 256, 8, 80, false);   // configs[4]
  bad += check(5, 100, 8, 40, false);    // configs[0]
  bad += check(5, 100, 8, 40, true);
  bad += check(3, 7, 4, 30, false);      // blocks much smaller than a tile
  bad += check(0, 50, 8, 20, false);
  bad += check(31, 64, 8, 100, false);
  bad += check(2, 1, 3, 20, false);
  bad += check(8, 1448, 4, 24, false);   // configs[2] at the run's batch size
  // banded ticket orders (SLIM_CHOL_COLS / SLIM_CHOL_BAND)
  const int banded[][2] = {{2, 7}, {2, 32}, {3, 16}, {4, 2}};
  for (const auto& cb : banded) {
    const int cols = cb[0], band = cb[1];
    bad += check(10, 362, 16, 32, false, cols, band);
    bad += check(8, 1448, 4, 12, false, cols, band);
    bad += check(5, 2048, 4, 12, false, cols, band);
    bad += check(20, 256, 16, 48, false, cols, band);
    bad += check(5, 100, 8, 40, true, cols, band);
    bad += check(3, 7, 4, 30, false, cols, band);
    bad += check(0, 50, 8, 20, false, cols, band);
    bad += check(31, 64, 8, 100, false, cols, band);
    bad += check(2, 1, 3, 20, false, cols, band);
  }
  printf(bad ? "FAILED\n" : "all orders valid\n");
  return bad ? 1 : 0;
}
