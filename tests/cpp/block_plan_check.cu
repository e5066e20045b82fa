// Host-side checks of the K9 block-pass planner (block.cuh, blk_plan_layout),
// compiled with nvcc and run on the CPU (no GPU needed):
//   * every row of every mode appears exactly once in that mode's table, and
//     the table's padding entries are BLK_NOROW;
//   * the copy segments cover every element of a block exactly once, in
//     global memory and in the slot, and never overlap;
//   * the modelled shared-memory cost stays within 1.5x the conflict-free
//     ideal for the shapes the auto path plans (the paper's d = 6 sizes).
#include <cstdio>
#include <set>
#include <vector>

#include "../../paper_2112_11238_b200/csrc/block.cuh"

using namespace mumode_gpu;

static int fails = 0;
#define CHECK(c, ...)                  \
  do {                                 \
    if (!(c)) {                        \
      std::printf("FAIL: " __VA_ARGS__); \
      std::printf("\n");               \
      ++fails;                         \
    }                                  \
  } while (0)

static void check(int64_t A, std::vector<int> e, int R, int CB, int64_t max_slot, bool want_ideal) {
  const int KM = static_cast<int>(e.size());
  int ee[3] = {0, 0, 0};
  for (int j = 0; j < KM; ++j) ee[j] = e[j];
  BlockLayout L;
  if (!blk_plan_layout(A, ee, KM, R, CB, max_slot, L)) {
    CHECK(false, "no plan for A=%lld KM=%d R=%d", (long long)A, KM, R);
    return;
  }
  int64_t E = 1;
  for (int x : e) E *= x;
  const int64_t rows_block = (R > 1 ? R : 1) * E * (R == 1 ? CB : 1);  // elements per block
  // tables: each mode's rows exactly once
  int64_t ideal = 0;
  for (int j = 0; j < KM; ++j) {
    std::set<int> seen;
    const int64_t nrows = rows_block / e[j];
    int valid = 0;
    for (int q = 0; q < L.mt[j] * 8; ++q) {
      const uint16_t b = L.tab[L.tab_off[j] + q];
      if (b == BLK_NOROW) continue;
      ++valid;
      CHECK(seen.insert(b).second, "mode %d: row base %d twice", j, b);
      // every element of the row lies inside the slot
      CHECK(int64_t(b) + int64_t(L.s[j]) * (e[j] - 1) < L.slot_dbl, "mode %d: row %d leaves the slot", j, b);
    }
    CHECK(valid == nrows, "mode %d: %d rows in the table, %lld expected", j, valid, (long long)nrows);
    ideal += int64_t(L.mt[j]) * 2 * ((e[j] + 3) / 4 + 2 * ((e[j] + 7) / 8));
  }
  // segments: disjoint, covering the block once (global offsets and slot offsets)
  std::set<int64_t> g, s;
  int64_t total = 0;
  const int64_t rowlen = R > 1 ? R : e[0];
  for (const BlkSeg& sg : L.seg) {
    const int64_t len = R > 1 ? rowlen : sg.len;
    for (int64_t k = 0; k < len; ++k) {
      CHECK(g.insert(sg.goff + k).second, "global element %lld twice", (long long)(sg.goff + k));
      CHECK(s.insert(sg.soff + k).second, "slot element %lld twice", (long long)(sg.soff + k));
      CHECK(sg.soff + k < L.slot_dbl, "segment leaves the slot");
    }
    total += len;
  }
  CHECK(total == rows_block, "segments cover %lld of %lld elements", (long long)total, (long long)rows_block);
  if (want_ideal)
    CHECK(L.cost <= ideal * 3 / 2, "A=%lld e0=%d: cost %lld > 1.5 x ideal %lld", (long long)A, e[0], (long long)L.cost,
          (long long)ideal);
  std::printf("A=%lld e=(%d,%d,%d) R=%d CB=%d slot=%d cost=%lld ideal=%lld segs=%zu\n", (long long)A, ee[0], ee[1],
              ee[2], R, CB, L.slot_dbl, (long long)L.cost, (long long)ideal, L.seg.size());
}

int main() {
  const int64_t budget = (227 * 1024 - 16 * 1024) / 8;
  check(1, {18, 18, 18}, 1, 1, budget / 3, true);
  check(1, {20, 20, 20}, 1, 1, budget / 3, true);
  check(1, {12, 12, 12}, 1, 3, budget / 3, true);
  check(1, {14, 14, 14}, 1, 2, budget / 3, true);
  check(1, {18, 14, 16}, 1, 1, budget / 3, false);
  check(1, {8, 8, 8}, 1, 12, budget / 3, false);
  check(5832, {18, 18}, 32, 1, budget / 2, true);
  check(8000, {20, 20}, 32, 1, budget / 2, false);
  check(1728, {12, 12}, 32, 1, budget / 3, true);
  check(4032, {10, 12}, 32, 1, budget / 3, false);
  check(1000, {10}, 32, 1, budget / 3, false);
  std::printf(fails ? "FAILED %d\n" : "PASSED\n", fails);
  return fails ? 1 : 0;
}
