// okt_plan.hpp — host-side planning of the Ok-Topk exchanges (no CUDA).
//
// Pure functions of the sizes every rank already agrees on after a counts
// allgather: the balance plan (oktopk.cpp:172-231), the recursive-doubling
// ledger arithmetic the reference's transport would credit
// (transport.cpp:71-160, collectives.cpp:30-77, oktopk.cpp:75-157), and the
// consensus rounding of space_repartition (oktopk.cpp:51-61).  Shared by the
// device orchestration (okt_core.cpp) and exported through the C-ABI so the
// multi-rank planning can be tested on CPU ranks (tests/test_plan_gloo.py).
#pragma once

#include <algorithm>
#include <cstdint>
#include <vector>

#include "../../include/okt.h"

namespace okt {
namespace plan {

inline int log2i(int p) {
  int l = 0;
  while ((1 << l) < p) ++l;
  return l;
}

// equal_slice_ends (collectives.cpp:79-87): ceil-sized blocks first.
inline std::vector<uint64_t> equal_slice_ends(uint64_t n, int P) {
  std::vector<uint64_t> e(P + 1, 0);
  const uint64_t base = n / uint64_t(P), rem = n % uint64_t(P);
  for (int r = 0; r < P; ++r) e[r + 1] = e[r] + base + (uint64_t(r) < rem ? 1 : 0);
  return e;
}

// bucket_count (oktopk.cpp:88-91): at least one message per destination.
inline uint64_t bucket_count(uint64_t nnz, uint32_t bucket) {
  if (bucket == 0 || nnz <= bucket) return 1;
  return (nnz + bucket - 1) / bucket;
}

// Consensus cuts from all P proposals (row q = rank q's P+1 cuts).  The fp64
// mean of integer proposals is exact (sums < 2^53, P a power of two), so
// llround(max(0, S/P)) == floor((2S + P) / 2P).
inline std::vector<uint64_t> cuts_from_proposals(const uint64_t* allprop, int P, uint64_t n) {
  std::vector<uint64_t> cuts(P + 1, 0);
  uint64_t prev = 0;
  for (int r = 1; r < P; ++r) {
    uint64_t S = 0;
    for (int q = 0; q < P; ++q) S += allprop[uint64_t(q) * (P + 1) + r];
    uint64_t rounded = (2 * S + uint64_t(P)) / (2 * uint64_t(P));
    rounded = std::min(rounded, n);
    rounded = std::max(rounded, prev);
    cuts[r] = prev = rounded;
  }
  cuts[P] = n;
  return cuts;
}

struct Piece {
  int peer;
  uint64_t a, b;  // range of the rank-concatenated survivor stream
};

struct Balance {
  bool on = false;
  uint64_t total = 0;
  std::vector<uint64_t> off;       // P+1 stream offsets of each rank's survivors
  std::vector<uint64_t> part_off;  // allgatherv parts (after balancing)
  std::vector<uint64_t> part_sz;
  std::vector<Piece> sends, recvs;  // balance moves (peer != rank)
  Piece own{-1, 0, 0};              // the part of my block I already hold
};

// balance_and_allgatherv's plan (oktopk.cpp:172-231): survivors at or beyond
// 4x the mean trigger a re-cut of the stream into P equal blocks.
inline Balance balance(int rank, int P, const std::vector<uint64_t>& sizes) {
  Balance B;
  B.off.assign(P + 1, 0);
  uint64_t maxs = 0;
  for (int q = 0; q < P; ++q) {
    B.off[q + 1] = B.off[q] + sizes[q];
    maxs = std::max(maxs, sizes[q]);
  }
  B.total = B.off[P];
  B.part_off.assign(B.off.begin(), B.off.end() - 1);
  B.part_sz = sizes;
  B.on = B.total > 0 && maxs * uint64_t(P) >= 4 * B.total;
  if (!B.on) {
    B.own = {rank, B.off[rank], B.off[rank + 1]};
    return B;
  }
  const std::vector<uint64_t> block = equal_slice_ends(B.total, P);
  auto overlap = [&](int src, int dst, uint64_t& a, uint64_t& b) {
    a = std::max(B.off[src], block[dst]);
    b = std::min(B.off[src + 1], block[dst + 1]);
    return a < b;
  };
  uint64_t a, b;
  for (int dst = 0; dst < P; ++dst)
    if (dst != rank && overlap(rank, dst, a, b)) B.sends.push_back({dst, a, b});
  for (int src = 0; src < P; ++src) {
    if (!overlap(src, rank, a, b)) continue;
    if (src == rank) B.own = {rank, a, b};
    else B.recvs.push_back({src, a, b});
  }
  for (int q = 0; q < P; ++q) {
    B.part_off[q] = block[q];
    B.part_sz[q] = block[q + 1] - block[q];
  }
  return B;
}

// ---- ledger arithmetic (what the reference's WorkerCtx would credit) -----------
inline void credit(okt_counters& c, bool send, uint64_t words, uint64_t msgs) {
  if (send) {
    c.words_sent += words;
    c.msgs_sent += msgs;
  } else {
    c.words_recv += words;
    c.msgs_recv += msgs;
  }
}

// split_and_reduce: counts[s * P + d] = entries rank s sends to region d.
inline void ledger_split(okt_counters& c, int rank, int P, const uint64_t* counts, uint32_t bucket) {
  for (int step = 1; step < P; ++step) {
    const int dst = (rank + step) % P, src = (rank - step + P) % P;
    const uint64_t out = counts[uint64_t(rank) * P + dst], in = counts[uint64_t(src) * P + rank];
    credit(c, true, 2 * out, bucket_count(out, bucket));
    credit(c, false, 2 * in, bucket_count(in, bucket));
  }
}

// sparse_allgatherv over part sizes (recursive doubling, one message per round).
inline void ledger_allgatherv(okt_counters& c, int rank, int P, const uint64_t* parts) {
  for (int j = 0; j < log2i(P); ++j) {
    const int width = 1 << j, partner = rank ^ width;
    const int mb = rank & ~(width - 1), pb = partner & ~(width - 1);
    uint64_t ms = 0, ps = 0;
    for (int q = 0; q < width; ++q) {
      ms += parts[mb + q];
      ps += parts[pb + q];
    }
    credit(c, true, 2 * ms, 1);
    credit(c, false, 2 * ps, 1);
  }
}

// small_allreduce_avg of `len` reals.
inline void ledger_avg(okt_counters& c, int P, uint64_t len) {
  const int rounds = log2i(P);
  credit(c, true, len * rounds, rounds);
  credit(c, false, len * rounds, rounds);
}

// small_allgather_u32 of one word per rank.
inline void ledger_allgather_u32(okt_counters& c, int P) {
  for (int j = 0; j < log2i(P); ++j) {
    credit(c, true, uint64_t(1) << j, 1);
    credit(c, false, uint64_t(1) << j, 1);
  }
}

// balance moves.
inline void ledger_balance(okt_counters& c, const Balance& B) {
  for (const Piece& p : B.sends) credit(c, true, 2 * (p.b - p.a), 1);
  for (const Piece& p : B.recvs) credit(c, false, 2 * (p.b - p.a), 1);
}

}  // namespace plan
}  // namespace okt
