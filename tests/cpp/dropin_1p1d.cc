// dropin_1p1d.cc — the C++ drop-in, exercised the way engine code uses it.
//
// One template, Run1P1D<Cache>, composes SURVEY.md §3's 1P1D flow from
// splitserve::KVCache calls only (prep_recv on D; CreateSequence +
// EnsureAllocated + MarkSend + BeginForward + Attention per layer with a
// FrameSink on P; DrainReceiveCompletions + BeginForward + Attention +
// SampleToken and a few decode steps on D).  It is instantiated three times
// in this one binary:
//   reference    splitserve::KVCache — the unmodified reference sources,
//                linked as objects (oracle/_ref/obj/*.o)
//   b200-frames  splitserve::b200::KVCache (include/splitserve_b200.h over
//                libmicrokv.so), rows shipped through the sink as host
//                payloads -> D.ApplyRemoteWrite, exactly like the reference
//   b200-direct  the same, with P.AttachPeer(D): rows stored device-direct
//                into D's pages, the sink is never called
// and the three outcomes must agree: PrepRecv's match length and KVAddrInfo,
// generated tokens (also = HashModel::Generate), Committed, fill states and
// the EntryDigest of every (position, layer) entry D holds.
//
// Test infrastructure (built by __graft_entry__.build() where
// /root/reference exists; run by tests/test_dropin_cpp_gpu.py).
#include <cstdio>
#include <cstdlib>
#include <random>
#include <string>
#include <type_traits>
#include <vector>

#include "splitserve/hash_model.h"
#include "splitserve/kv_cache.h"
#include "splitserve_b200.h"

using namespace splitserve;

struct Outcome {
  int64_t match_len = -1;
  KVAddrInfo addr;
  std::vector<Token> tokens;
  int64_t committed = -1;
  int64_t sink_calls = 0;
  std::vector<uint64_t> digests;  // EntryDigest of D's entries, [pos][layer]
  std::vector<int> fills;         // FillOf of D's entries, [pos][layer]
};

template <class Cache>
void Sync(Cache& c) {
  if constexpr (std::is_same_v<Cache, b200::KVCache>) c.Synchronize();
}

template <class Cache, class Setup>
Outcome Run1P1D(const HashModel& m, const CacheConfig& cc, const TokenList& prompt,
                int32_t max_tokens, Setup setup) {
  Outcome out;
  const int32_t L = m.config().layers;
  const int64_t n = static_cast<int64_t>(prompt.size()), e = n - 1;
  Cache P = setup.make(cc, &m, 0);
  Cache D = setup.make(cc, &m, 1);
  setup.attach(P, D);
  // prep_recv on the decode engine.
  auto r = D.PrepRecv(10, prompt, -1);
  out.match_len = r.match_len;
  out.addr = r.addr;
  // remote_send on the prefill engine.
  P.CreateSequence(20, prompt);
  P.EnsureAllocated(20, e);
  P.MarkSend(20, TokenRange{r.match_len, e}, 1, r.addr, 7);
  auto plan = P.BeginForward({BatchEntry{20, TokenRange{0, e}, false}});
  std::vector<uint64_t> x(e);
  for (int64_t i = 0; i < e; ++i) x[i] = m.Embed(prompt[i], i);
  FrameSink sink = [&](int32_t layer, const PlanSend& s, std::vector<uint64_t> payload) {
    ++out.sink_calls;
    if (D.ApplyRemoteWrite(s.dest_addr, layer, payload, s.user_tag) != Cache::ApplyStatus::kOk) {
      std::fprintf(stderr, "ApplyRemoteWrite rejected a frame\n");
      std::exit(3);
    }
  };
  for (int32_t l = 0; l < L; ++l) x = P.Attention(l, &plan, x, sink);
  Sync(P);
  // start_generate on the decode engine.
  const auto done = D.DrainReceiveCompletions();
  if (done.size() != 1 || done[0] != 10) {
    std::fprintf(stderr, "receive window did not complete\n");
    std::exit(3);
  }
  out.committed = D.Committed(10);
  D.EnsureAllocated(10, n);
  auto pd = D.BeginForward({BatchEntry{10, TokenRange{e, n}, false}});
  std::vector<uint64_t> h{m.Embed(prompt[e], e)};
  for (int32_t l = 0; l < L; ++l) h = D.Attention(l, &pd, h, FrameSink{});
  out.tokens.push_back(m.SampleToken(h.back()));
  for (int32_t k = 1; k < max_tokens; ++k) {
    const Token t = out.tokens.back();
    D.AppendToken(10, t);
    D.EnsureAllocated(10, n + k);
    auto pk = D.BeginForward({BatchEntry{10, TokenRange{n + k - 1, n + k}, true}});
    std::vector<uint64_t> y{m.Embed(t, n + k - 1)};
    for (int32_t l = 0; l < L; ++l) y = D.Attention(l, &pk, y, FrameSink{});
    out.tokens.push_back(m.SampleToken(y.back()));
  }
  for (int64_t pos = 0; pos < n; ++pos) {
    for (int32_t l = 0; l < L; ++l) {
      const std::vector<uint64_t> w = D.ReadEntryWords(10, pos, l);
      out.digests.push_back(m.EntryDigest(w));
      out.fills.push_back(static_cast<int>(D.FillOf(10, pos, l)));
    }
  }
  return out;
}

struct RefSetup {
  KVCache make(const CacheConfig& cc, const HashModel* m, Rank) const { return KVCache(cc, m); }
  void attach(KVCache&, KVCache&) const {}
};

struct B200Setup {
  bool direct;
  b200::KVCache make(const CacheConfig& cc, const HashModel* m, Rank r) const {
    return b200::KVCache(cc, m, /*device=*/0, r);
  }
  void attach(b200::KVCache& P, b200::KVCache& D) const {
    if (direct) P.AttachPeer(1, D);
  }
};

// splitserve::KVCache is not movable (it owns a mutex); the factories above
// rely on guaranteed copy elision of a prvalue, which C++17 provides.

static bool Same(const char* what, const Outcome& a, const Outcome& b, const char* an,
                 const char* bn) {
  bool ok = a.match_len == b.match_len && a.addr == b.addr && a.tokens == b.tokens &&
            a.committed == b.committed && a.digests == b.digests && a.fills == b.fills;
  std::printf("%s %s vs %s: match_len %lld/%lld ranges %zu/%zu tokens %s committed %lld/%lld "
              "entries %zu -> %s\n",
              what, an, bn, (long long)a.match_len, (long long)b.match_len, a.addr.ranges.size(),
              b.addr.ranges.size(), a.tokens == b.tokens ? "equal" : "DIFFER",
              (long long)a.committed, (long long)b.committed, a.digests.size(),
              ok ? "IDENTICAL" : "MISMATCH");
  return ok;
}

int main() {
  struct Case {
    const char* name;
    int32_t layers, dim;
    int64_t prompt, pages;
  };
  const Case cases[] = {{"tiny(L4,W128,512)", 4, 128, 512, 64},
                        {"llama(L8,W512,1024)", 8, 512, 1024, 96}};
  bool all = true;
  for (const Case& c : cases) {
    ModelConfig mc;
    mc.layers = c.layers;
    mc.dim = c.dim;
    HashModel m(mc);
    CacheConfig cc;
    cc.num_pages = c.pages;
    cc.page_size = 16;
    std::mt19937_64 rng(1);
    TokenList prompt(c.prompt);
    for (auto& t : prompt) t = static_cast<Token>(rng() % 256);
    const int32_t gen = 4;
    const Outcome ref = Run1P1D<KVCache>(m, cc, prompt, gen, RefSetup{});
    const Outcome fr = Run1P1D<b200::KVCache>(m, cc, prompt, gen, B200Setup{false});
    const Outcome dd = Run1P1D<b200::KVCache>(m, cc, prompt, gen, B200Setup{true});
    const std::vector<Token> want = m.Generate(prompt, gen);
    const bool gen_ok = ref.tokens == want;
    std::printf("%s HashModel::Generate: %s; sink calls ref %lld frames %lld direct %lld\n", c.name,
                gen_ok ? "reference tokens equal" : "MISMATCH", (long long)ref.sink_calls,
                (long long)fr.sink_calls, (long long)dd.sink_calls);
    all &= gen_ok;
    all &= Same(c.name, ref, fr, "reference", "b200-frames");
    all &= Same(c.name, ref, dd, "reference", "b200-direct");
    all &= ref.sink_calls == c.layers && fr.sink_calls == c.layers && dd.sink_calls == 0;
  }
  // Errors keep the reference's exception contract through the facade.
  {
    ModelConfig mc;
    HashModel m(mc);
    CacheConfig cc;
    cc.num_pages = 4;
    b200::KVCache D(cc, &m, 0, 1);
    bool threw = false;
    try {
      D.PrepRecv(1, TokenList(1000, 3), -1);  // needs 63 pages, 4 free
    } catch (const Error& e) {
      threw = e.code() == ErrorCode::kOutOfPages && e.retryable();
    }
    std::printf("OutOfPages through the facade: %s\n", threw ? "splitserve::Error(kOutOfPages)" : "MISSING");
    all &= threw && D.SequenceCount() == 0;
  }
  std::printf("%s\n", all ? "DROPIN OK" : "DROPIN FAILED");
  return all ? 0 : 1;
}
