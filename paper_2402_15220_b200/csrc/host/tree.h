// Prefix tree of fixed-size KV chunks with a pool allocator (PAKV, §3.1).
//
// PAPER.md:505  "Each node defines a chunk C storing ... a segment of c context
//               tokens ... Each path in the prefix tree defines a sequence.
//               Multiple trees (a forest) may exist".
// PAPER.md:507  three scenarios -> add_sequence / remove_sequence / append.
// PAPER.md:509  pool allocator: free list first, else fresh memory; chunks are
//               returned on completion and never released to the OS.
// PAPER.md:513  covered sequences of every chunk are contiguous in batch order.
//
// Readings: T1 only full aligned chunks are matched or shared;
// T2 LIFO free list over a bump pointer; T3' children and roots in chunk
// creation order, sequences ending at a node precede its children (by id);
// T4 every acquire/release/add/remove bumps the epoch.
#pragma once

#include <cstdint>
#include <string>
#include <unordered_map>
#include <vector>

namespace pakv {

struct PoolExhausted {};

class ChunkPool {
 public:
  explicit ChunkPool(int64_t capacity) : capacity_(capacity) {}
  int64_t available() const { return (int64_t)free_.size() + (capacity_ - created_); }
  int32_t acquire();                 // LIFO reuse, else bump pointer; throws PoolExhausted
  void release(int32_t id) { free_.push_back(id); --used_; }
  int64_t used() const { return used_; }
  int64_t free_count() const { return (int64_t)free_.size(); }
  int64_t created() const { return created_; }
  int64_t hwm() const { return hwm_; }
  int64_t capacity() const { return capacity_; }
  const std::vector<int32_t>& free_list() const { return free_; }

 private:
  int64_t capacity_;
  int64_t created_ = 0, used_ = 0, hwm_ = 0;
  std::vector<int32_t> free_;
};

struct Node {
  bool live = false;
  int32_t parent = -1;
  int64_t serial = 0;
  int32_t start_pos = 0;
  int32_t len = 0;
  int32_t ref = 0;
  std::vector<int32_t> children;  // creation order (T3')
  std::vector<int64_t> terms;     // seq ids whose path ends here (sorted)
};

struct Sequence {
  std::vector<int32_t> path;  // chunk ids root -> leaf
  int64_t len = 0;            // tokens
};

// One chunk of the DFS pre-order with its covered row range [i, j] (inclusive).
struct ChunkRec {
  int32_t id, i, j;
};

class PrefixTree {
 public:
  PrefixTree(int32_t chunk_size, int64_t max_chunks, bool prefix_match);

  int32_t c() const { return c_; }
  int64_t epoch() const { return epoch_; }
  int64_t live_count() const { return (int64_t)seqs_.size(); }
  const Node& node(int32_t id) const { return nodes_[id]; }
  const int32_t* tokens(int32_t id) const { return &tok_[(size_t)id * c_]; }
  const ChunkPool& pool() const { return pool_; }
  const Sequence* find(int64_t sid) const {
    auto it = seqs_.find(sid);
    return it == seqs_.end() ? nullptr : &it->second;
  }

  // Longest matched prefix of full chunks (T1). Returns chunk ids along the path.
  std::vector<int32_t> match(const int32_t* tokens, int64_t n) const;

  // Insert; returns new seq id. new_chunks receives the private chunk ids in
  // path order, *matched the matched token count.  Throws PoolExhausted with
  // no state change.
  int64_t add(const int32_t* tokens, int64_t n, std::vector<int32_t>* new_chunks, int64_t* matched);

  // Chunks a batched append would acquire (for capacity checks).
  int64_t append_needs(const int64_t* sids, int64_t n) const;
  // Structural part of one decode step: for every sequence whose leaf is full
  // or shared, acquire a child chunk at start_pos = len (call order). Does NOT
  // add the tokens. Returns true if any chunk was acquired.
  bool append_grow(const int64_t* sids, int64_t n);
  // Non-structural part: write the tokens into the (now private, non-full) leaves.
  void append_tokens(const int64_t* sids, const int32_t* toks, int64_t n);

  // Remove; returns released chunk ids leaf -> root.
  std::vector<int32_t> remove(int64_t sid);

  // DFS (T3'): rows (seq ids by row) and chunk records in pre-order.
  void dfs(std::vector<int64_t>* order, std::vector<ChunkRec>* recs) const;

  int64_t waste_slots() const;

 private:
  int32_t acquire_node(int32_t parent, int32_t start_pos);
  void detach_release(int32_t id);

  int32_t c_;
  bool prefix_match_;
  ChunkPool pool_;
  std::vector<Node> nodes_;
  std::vector<int32_t> tok_;  // [max_chunks][c]
  std::vector<int32_t> roots_;
  std::unordered_map<int64_t, Sequence> seqs_;
  int64_t next_seq_ = 0;
  int64_t serial_ = 0;
  int64_t epoch_ = 0;
};

}  // namespace pakv
