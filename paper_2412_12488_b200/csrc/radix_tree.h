// radix_tree.h — token-level prefix index (the context cache), host C++.
//
// Semantics follow /root/reference/proj/core/src/radix_tree.cc exactly,
// including the behaviours parity tests pin:
//  * MatchPrefix counts partial-edge matches and reports the ref of the
//    deepest touched node (radix_tree.cc:28-53);
//  * Insert re-points every traversed node to the inserting sequence and
//    splits edges at the divergence point (radix_tree.cc:55-94);
//  * Remove prunes childless nodes of the sequence and re-points survivors
//    to their first child's ref, keeping touch stamps of other sequences
//    (radix_tree.cc:96-124);
//  * one logical clock drives node LRU stamps and per-sequence touches.
// Storage is an index arena instead of owning pointers: nodes are recycled
// through a free list, children are kept ordered by first token.
#pragma once

#include <cstdint>
#include <map>
#include <span>
#include <vector>

namespace mkv {

using Token = int32_t;
using SeqId = int64_t;
using Rank = int32_t;

class RadixTree {
 public:
  struct MatchResult {
    int64_t match_len = 0;
    SeqId seq = -1;
  };

  RadixTree();

  MatchResult MatchPrefix(std::span<const Token> tokens);
  void Insert(std::span<const Token> tokens, SeqId seq);
  void Remove(SeqId seq);
  void Pin(std::span<const Token> prefix, bool flag);
  bool HasPinnedNode(SeqId seq) const;
  bool Contains(SeqId seq) const { return touch_.count(seq) > 0; }
  uint64_t LastTouch(SeqId seq) const;
  std::vector<SeqId> SequencesByLru() const;
  size_t NodeCount() const { return live_ - 1; }

 private:
  struct Node {
    std::vector<Token> edge;
    std::map<Token, int32_t> kids;  // first token -> node index
    SeqId ref = -1;
    uint64_t lru = 0;
    bool pinned = false;
  };

  int32_t NewNode();
  void FreeSubtree(int32_t idx);
  // Length of the common prefix of node.edge and tokens[pos:].
  size_t Common(const Node& n, std::span<const Token> tokens, size_t pos) const;
  // Returns false when `idx` must be detached from its parent.
  bool RemoveVisit(int32_t idx, SeqId seq);
  void Touch(SeqId seq) {
    if (seq >= 0) touch_[seq] = ++clock_;
  }

  std::vector<Node> nodes_;
  std::vector<int32_t> free_;
  size_t live_ = 0;
  uint64_t clock_ = 0;
  std::map<SeqId, uint64_t> touch_;
};

}  // namespace mkv
