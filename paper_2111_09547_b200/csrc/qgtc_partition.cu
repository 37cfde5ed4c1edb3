// Native host partitioner: the reference's balanced BFS-grown greedy partition
// (graph.py:190-229, the built-in METIS stand-in), re-implemented in C++ with the same
// decisions so a given seed yields the identical assignment:
//   * parts are grown one after another to target = ceil(unassigned / parts left);
//   * the next node is the frontier node with the most links into the growing part
//     (ties: smallest id) -- here a lazy max-heap keyed (gain, -id) instead of the
//     reference's O(frontier) scan per step;
//   * with an empty frontier a seed is drawn uniformly among the unassigned nodes of
//     minimum degree (ascending ids) by Python's random.Random(seed).randrange --
//     reproduced bit for bit: MT19937 seeded by init_by_array(32-bit words of |seed|),
//     randrange(n) = rejection sampling of getrandbits(bit_length(n)).
// Host code only (no device work); exported through the C-ABI library.
#include <cstdint>
#include <cstdlib>
#include <map>
#include <queue>
#include <set>
#include <utility>
#include <vector>
#include "../../include/qgtc_b200.h"

namespace {

// MT19937 as CPython's _randommodule.c (init_by_array seeding, genrand_uint32)
struct MT {
  uint32_t mt[624];
  int mti = 625;
  void init_genrand(uint32_t s) {
    mt[0] = s;
    for (mti = 1; mti < 624; ++mti) mt[mti] = 1812433253u * (mt[mti - 1] ^ (mt[mti - 1] >> 30)) + (uint32_t)mti;
  }
  void init_by_array(const std::vector<uint32_t>& key) {
    init_genrand(19650218u);
    size_t i = 1, j = 0;
    const size_t n = key.size();
    for (size_t k = (624 > n ? 624 : n); k; --k) {
      mt[i] = (mt[i] ^ ((mt[i - 1] ^ (mt[i - 1] >> 30)) * 1664525u)) + key[j] + (uint32_t)j;
      ++i;
      ++j;
      if (i >= 624) { mt[0] = mt[623]; i = 1; }
      if (j >= n) j = 0;
    }
    for (size_t k = 623; k; --k) {
      mt[i] = (mt[i] ^ ((mt[i - 1] ^ (mt[i - 1] >> 30)) * 1566083941u)) - (uint32_t)i;
      ++i;
      if (i >= 624) { mt[0] = mt[623]; i = 1; }
    }
    mt[0] = 0x80000000u;
  }
  uint32_t next() {
    static const uint32_t mag01[2] = {0u, 0x9908b0dfu};
    if (mti >= 624) {
      int kk = 0;
      for (; kk < 624 - 397; ++kk) {
        const uint32_t y = (mt[kk] & 0x80000000u) | (mt[kk + 1] & 0x7fffffffu);
        mt[kk] = mt[kk + 397] ^ (y >> 1) ^ mag01[y & 1u];
      }
      for (; kk < 623; ++kk) {
        const uint32_t y = (mt[kk] & 0x80000000u) | (mt[kk + 1] & 0x7fffffffu);
        mt[kk] = mt[kk + (397 - 624)] ^ (y >> 1) ^ mag01[y & 1u];
      }
      const uint32_t y = (mt[623] & 0x80000000u) | (mt[0] & 0x7fffffffu);
      mt[623] = mt[396] ^ (y >> 1) ^ mag01[y & 1u];
      mti = 0;
    }
    uint32_t y = mt[mti++];
    y ^= (y >> 11);
    y ^= (y << 7) & 0x9d2c5680u;
    y ^= (y << 15) & 0xefc60000u;
    y ^= (y >> 18);
    return y;
  }
  // random.Random.randrange(n), 0 < n < 2^32
  uint64_t below(uint64_t n) {
    int k = 0;
    while ((n >> k) != 0) ++k;
    uint64_t r = next() >> (32 - k);
    while (r >= n) r = next() >> (32 - k);
    return r;
  }
};

}  // namespace

extern "C" int qg_partition_bfs(int64_t n, const int64_t* indptr, const int64_t* nbrs, int64_t num_parts,
                                int64_t seed, int64_t* part_of) {
  if (n < 1 || num_parts < 1 || num_parts > n || !indptr || !part_of || (indptr[n] > 0 && !nbrs) ||
      n >= ((int64_t)1 << 32))
    return QG_ERR_ARG;
  MT rng;
  {
    // CPython random_seed: key = 32-bit little-endian words of |seed| (one 0 word for 0)
    uint64_t a = seed < 0 ? (uint64_t)(-(seed + 1)) + 1u : (uint64_t)seed;
    std::vector<uint32_t> key;
    while (a) { key.push_back((uint32_t)(a & 0xffffffffu)); a >>= 32; }
    if (key.empty()) key.push_back(0u);
    rng.init_by_array(key);
  }
  for (int64_t v = 0; v < n; ++v) part_of[v] = -1;
  // unassigned nodes bucketed by degree, ascending ids
  std::map<int64_t, std::set<int64_t>> by_degree;
  for (int64_t v = 0; v < n; ++v) by_degree[indptr[v + 1] - indptr[v]].insert(v);
  std::vector<int64_t> gain(n, 0);
  std::vector<int64_t> touched;
  int64_t unassigned = n;
  typedef std::pair<int64_t, int64_t> Key;   // (gain, -id): max-heap order = reference's max()
  for (int64_t part = 0; part < num_parts; ++part) {
    const int64_t left = num_parts - part;
    const int64_t target = (unassigned + left - 1) / left;
    std::priority_queue<Key> heap;
    for (int64_t v : touched) gain[v] = 0;
    touched.clear();
    int64_t frontier = 0;                    // nodes with gain > 0 (the reference's dict size)
    for (int64_t size = 0; size < target; ++size) {
      int64_t node;
      if (frontier > 0) {
        for (;;) {
          const Key k = heap.top();
          heap.pop();
          const int64_t v = -k.second;
          if (part_of[v] < 0 && gain[v] == k.first) { node = v; break; }
        }
        --frontier;
      } else {
        auto it = by_degree.begin();
        const uint64_t idx = rng.below((uint64_t)it->second.size());
        auto sit = it->second.begin();
        std::advance(sit, (long)idx);
        node = *sit;
      }
      part_of[node] = part;
      --unassigned;
      {
        auto it = by_degree.find(indptr[node + 1] - indptr[node]);
        it->second.erase(node);
        if (it->second.empty()) by_degree.erase(it);
      }
      for (int64_t e = indptr[node]; e < indptr[node + 1]; ++e) {
        const int64_t nb = nbrs[e];
        if (part_of[nb] >= 0) continue;
        if (gain[nb] == 0) { ++frontier; touched.push_back(nb); }
        gain[nb] += 1;
        heap.push(Key(gain[nb], -nb));
      }
    }
  }
  return QG_OK;
}
