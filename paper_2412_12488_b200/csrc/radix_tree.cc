// radix_tree.cc — see radix_tree.h for the semantics and reference lines.
#include "radix_tree.h"

#include <algorithm>
#include <utility>

namespace mkv {

namespace {
constexpr int32_t kRoot = 0;
}

RadixTree::RadixTree() { NewNode(); }

int32_t RadixTree::NewNode() {
  int32_t idx;
  if (!free_.empty()) {
    idx = free_.back();
    free_.pop_back();
    nodes_[idx] = Node{};
  } else {
    idx = static_cast<int32_t>(nodes_.size());
    nodes_.emplace_back();
  }
  ++live_;
  return idx;
}

void RadixTree::FreeSubtree(int32_t idx) {
  std::vector<int32_t> stack{idx};
  while (!stack.empty()) {
    int32_t i = stack.back();
    stack.pop_back();
    for (const auto& kv : nodes_[i].kids) stack.push_back(kv.second);
    nodes_[i] = Node{};
    free_.push_back(i);
    --live_;
  }
}

size_t RadixTree::Common(const Node& n, std::span<const Token> tokens, size_t pos) const {
  size_t limit = std::min(n.edge.size(), tokens.size() - pos);
  size_t c = 0;
  while (c < limit && n.edge[c] == tokens[pos + c]) ++c;
  return c;
}

// radix_tree.cc:28-53
RadixTree::MatchResult RadixTree::MatchPrefix(std::span<const Token> tokens) {
  MatchResult res;
  ++clock_;
  int32_t cur = kRoot;
  size_t pos = 0;
  while (pos < tokens.size()) {
    auto it = nodes_[cur].kids.find(tokens[pos]);
    if (it == nodes_[cur].kids.end()) break;
    Node& child = nodes_[it->second];
    size_t c = Common(child, tokens, pos);
    if (c > 0) {
      child.lru = clock_;
      res.match_len = static_cast<int64_t>(pos + c);
      res.seq = child.ref;
    }
    if (c < child.edge.size()) break;
    pos += c;
    cur = it->second;
  }
  Touch(res.seq);
  return res;
}

// radix_tree.cc:55-94
void RadixTree::Insert(std::span<const Token> tokens, SeqId seq) {
  ++clock_;
  int32_t cur = kRoot;
  size_t pos = 0;
  while (pos < tokens.size()) {
    auto it = nodes_[cur].kids.find(tokens[pos]);
    if (it == nodes_[cur].kids.end()) {
      int32_t fresh = NewNode();
      Node& f = nodes_[fresh];
      f.edge.assign(tokens.begin() + pos, tokens.end());
      f.ref = seq;
      f.lru = clock_;
      nodes_[cur].kids.emplace(tokens[pos], fresh);
      Touch(seq);
      return;
    }
    int32_t ci = it->second;
    size_t c = Common(nodes_[ci], tokens, pos);
    if (c < nodes_[ci].edge.size()) {
      // Split: the tail keeps everything below the divergence point.
      int32_t ti = NewNode();
      Node& child = nodes_[ci];
      Node& tail = nodes_[ti];
      tail.edge.assign(child.edge.begin() + c, child.edge.end());
      tail.ref = child.ref;
      tail.lru = child.lru;
      tail.pinned = child.pinned;
      tail.kids = std::move(child.kids);
      child.kids.clear();
      child.edge.resize(c);
      child.kids.emplace(tail.edge[0], ti);
    }
    Node& child = nodes_[ci];
    child.ref = seq;
    child.lru = clock_;
    pos += c;
    cur = ci;
  }
  Touch(seq);
}

// radix_tree.cc:96-124 (post-order prune, re-point to the first child's ref)
bool RadixTree::RemoveVisit(int32_t idx, SeqId seq) {
  Node& n = nodes_[idx];
  for (auto it = n.kids.begin(); it != n.kids.end();) {
    int32_t k = it->second;
    if (RemoveVisit(k, seq)) {
      ++it;
    } else {
      FreeSubtree(k);
      it = nodes_[idx].kids.erase(it);
    }
  }
  Node& m = nodes_[idx];
  if (m.ref == seq) {
    if (m.kids.empty()) return false;
    m.ref = nodes_[m.kids.begin()->second].ref;
  }
  return true;
}

void RadixTree::Remove(SeqId seq) {
  Node& root = nodes_[kRoot];
  for (auto it = root.kids.begin(); it != root.kids.end();) {
    int32_t k = it->second;
    if (RemoveVisit(k, seq)) {
      ++it;
    } else {
      FreeSubtree(k);
      it = nodes_[kRoot].kids.erase(it);
    }
  }
  touch_.erase(seq);
}

// radix_tree.cc:126-143
void RadixTree::Pin(std::span<const Token> prefix, bool flag) {
  int32_t cur = kRoot;
  size_t pos = 0;
  while (pos < prefix.size()) {
    auto it = nodes_[cur].kids.find(prefix[pos]);
    if (it == nodes_[cur].kids.end()) return;
    Node& child = nodes_[it->second];
    size_t c = Common(child, prefix, pos);
    if (c > 0) child.pinned = flag;
    if (c < child.edge.size()) return;
    pos += c;
    cur = it->second;
  }
}

// radix_tree.cc:145-157 (the root participates, as in the reference)
bool RadixTree::HasPinnedNode(SeqId seq) const {
  std::vector<int32_t> stack{kRoot};
  while (!stack.empty()) {
    int32_t i = stack.back();
    stack.pop_back();
    const Node& n = nodes_[i];
    if (n.ref == seq && n.pinned) return true;
    for (const auto& kv : n.kids) stack.push_back(kv.second);
  }
  return false;
}

uint64_t RadixTree::LastTouch(SeqId seq) const {
  auto it = touch_.find(seq);
  return it == touch_.end() ? 0 : it->second;
}

// radix_tree.cc:166-175: ascending (stamp, seq).
std::vector<SeqId> RadixTree::SequencesByLru() const {
  std::vector<std::pair<uint64_t, SeqId>> order;
  order.reserve(touch_.size());
  for (const auto& [s, t] : touch_) order.emplace_back(t, s);
  std::sort(order.begin(), order.end());
  std::vector<SeqId> out;
  out.reserve(order.size());
  for (const auto& p : order) out.push_back(p.second);
  return out;
}

}  // namespace mkv
