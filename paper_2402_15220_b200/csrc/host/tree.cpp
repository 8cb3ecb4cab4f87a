// Prefix tree + pool allocator. See tree.h for the paper passages followed.
#include "tree.h"

#include <algorithm>
#include <cstring>

namespace pakv {

int32_t ChunkPool::acquire() {
  int32_t id;
  if (!free_.empty()) {  // PAPER.md:509 "returns a chunk from the free list"
    id = free_.back();
    free_.pop_back();
  } else if (created_ < capacity_) {  // "... or allocates fresh memory"
    id = (int32_t)created_++;
  } else {
    throw PoolExhausted{};
  }
  ++used_;
  hwm_ = std::max(hwm_, used_);
  return id;
}

PrefixTree::PrefixTree(int32_t chunk_size, int64_t max_chunks, bool prefix_match)
    : c_(chunk_size), prefix_match_(prefix_match), pool_(max_chunks),
      nodes_((size_t)max_chunks), tok_((size_t)max_chunks * chunk_size, 0) {}

std::vector<int32_t> PrefixTree::match(const int32_t* tokens, int64_t n) const {
  std::vector<int32_t> path;
  if (!prefix_match_) return path;
  const std::vector<int32_t>* cands = &roots_;
  for (int64_t k = 0; (k + 1) * c_ <= n; ++k) {
    const int32_t* tup = tokens + k * c_;
    int32_t hit = -1;
    for (int32_t id : *cands) {  // first equal FULL child in creation order (T1, T3')
      const Node& nd = nodes_[id];
      if (nd.len == c_ && std::memcmp(this->tokens(id), tup, sizeof(int32_t) * c_) == 0) {
        hit = id;
        break;
      }
    }
    if (hit < 0) break;
    path.push_back(hit);
    cands = &nodes_[hit].children;
  }
  return path;
}

int32_t PrefixTree::acquire_node(int32_t parent, int32_t start_pos) {
  int32_t id = pool_.acquire();
  Node& nd = nodes_[id];
  nd.live = true;
  nd.parent = parent;
  nd.serial = serial_++;
  nd.start_pos = start_pos;
  nd.len = 0;
  nd.ref = 0;
  nd.children.clear();
  nd.terms.clear();
  (parent >= 0 ? nodes_[parent].children : roots_).push_back(id);
  return id;
}

void PrefixTree::detach_release(int32_t id) {
  Node& nd = nodes_[id];
  auto& sib = nd.parent >= 0 ? nodes_[nd.parent].children : roots_;
  sib.erase(std::find(sib.begin(), sib.end(), id));
  nd.live = false;
  pool_.release(id);
}

static void insert_sorted(std::vector<int64_t>& v, int64_t x) {
  v.insert(std::upper_bound(v.begin(), v.end(), x), x);
}
static void erase_value(std::vector<int64_t>& v, int64_t x) {
  auto it = std::lower_bound(v.begin(), v.end(), x);
  if (it != v.end() && *it == x) v.erase(it);
}

int64_t PrefixTree::add(const int32_t* tokens, int64_t n, std::vector<int32_t>* new_chunks,
                        int64_t* matched) {
  std::vector<int32_t> path = match(tokens, n);
  const int64_t m = (int64_t)path.size() * c_;
  const int64_t need = (n - m + c_ - 1) / c_;
  if (need > pool_.available()) throw PoolExhausted{};
  int32_t parent = path.empty() ? -1 : path.back();
  new_chunks->clear();
  for (int64_t k = 0; k < need; ++k) {
    const int64_t start = m + k * c_;
    const int32_t id = acquire_node(parent, (int32_t)start);
    const int32_t len = (int32_t)std::min<int64_t>(c_, n - start);
    std::memcpy(&tok_[(size_t)id * c_], tokens + start, sizeof(int32_t) * len);
    nodes_[id].len = len;
    new_chunks->push_back(id);
    path.push_back(id);
    parent = id;
  }
  const int64_t sid = next_seq_++;
  for (int32_t id : path) nodes_[id].ref += 1;
  insert_sorted(nodes_[path.back()].terms, sid);
  Sequence s;
  s.path = std::move(path);
  s.len = n;
  seqs_.emplace(sid, std::move(s));
  ++epoch_;
  *matched = m;
  return sid;
}

int64_t PrefixTree::append_needs(const int64_t* sids, int64_t n) const {
  int64_t need = 0;
  for (int64_t k = 0; k < n; ++k) {
    const Sequence& s = seqs_.at(sids[k]);
    const Node& last = nodes_[s.path.back()];
    if (!(last.ref == 1 && last.len < c_)) ++need;
  }
  return need;
}

bool PrefixTree::append_grow(const int64_t* sids, int64_t n) {
  bool grew = false;
  for (int64_t k = 0; k < n; ++k) {  // call order (T2)
    Sequence& s = seqs_.at(sids[k]);
    const int32_t last = s.path.back();
    if (nodes_[last].ref == 1 && nodes_[last].len < c_) continue;
    // PAPER.md:507 "grow a new chunk when the leaf chunk is full"; a shared leaf
    // is never mutated (it is full by T1), the sequence branches privately.
    const int32_t id = acquire_node(last, (int32_t)s.len);
    nodes_[id].ref = 1;
    erase_value(nodes_[last].terms, sids[k]);
    insert_sorted(nodes_[id].terms, sids[k]);
    s.path.push_back(id);
    ++epoch_;
    grew = true;
  }
  return grew;
}

void PrefixTree::append_tokens(const int64_t* sids, const int32_t* toks, int64_t n) {
  for (int64_t k = 0; k < n; ++k) {
    Sequence& s = seqs_.at(sids[k]);
    const int32_t id = s.path.back();
    Node& nd = nodes_[id];
    tok_[(size_t)id * c_ + nd.len] = toks[k];
    nd.len += 1;
    s.len += 1;
  }
}

std::vector<int32_t> PrefixTree::remove(int64_t sid) {
  auto it = seqs_.find(sid);
  std::vector<int32_t> released;
  Sequence s = std::move(it->second);
  seqs_.erase(it);
  erase_value(nodes_[s.path.back()].terms, sid);
  for (auto r = s.path.rbegin(); r != s.path.rend(); ++r) {  // leaf -> root (T2)
    Node& nd = nodes_[*r];
    if (--nd.ref == 0) {
      detach_release(*r);
      released.push_back(*r);
    }
  }
  ++epoch_;
  return released;
}

void PrefixTree::dfs(std::vector<int64_t>* order, std::vector<ChunkRec>* recs) const {
  order->clear();
  recs->clear();
  // explicit stack: (node, child cursor, rec index)
  struct Frame {
    int32_t id;
    size_t next;
    size_t rec;
  };
  std::vector<Frame> st;
  for (int32_t root : roots_) {
    st.push_back({root, 0, recs->size()});
    recs->push_back({root, (int32_t)order->size(), -1});
    for (int64_t s : nodes_[root].terms) order->push_back(s);
    while (!st.empty()) {
      Frame& f = st.back();
      const Node& nd = nodes_[f.id];
      if (f.next < nd.children.size()) {
        const int32_t kid = nd.children[f.next++];
        const size_t ri = recs->size();
        recs->push_back({kid, (int32_t)order->size(), -1});
        for (int64_t s : nodes_[kid].terms) order->push_back(s);
        st.push_back({kid, 0, ri});
      } else {
        (*recs)[f.rec].j = (int32_t)order->size() - 1;
        st.pop_back();
      }
    }
  }
}

int64_t PrefixTree::waste_slots() const {
  int64_t w = 0;
  for (size_t id = 0; id < nodes_.size(); ++id)
    if (nodes_[id].live) w += c_ - nodes_[id].len;
  return w;
}

}  // namespace pakv
