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
//   b200-ipc     the same flow across two processes: this binary re-executes
//                itself as the decode engine, which exports its receive
//                surface (ExportIpc); the prefill engine imports it
//                (ImportIpc) and stores every layer into the other
//                process's pages; KVAddrInfo travels as the reference's JSON
// and the outcomes must agree: PrepRecv's match length and KVAddrInfo,
// generated tokens (also = HashModel::Generate), Committed, fill states and
// the EntryDigest of every (position, layer) entry D holds.
//
// Test infrastructure (built by __graft_entry__.build() where
// /root/reference exists; run by tests/test_dropin_cpp_gpu.py).
#include <spawn.h>
#include <sys/wait.h>
#include <unistd.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
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

// ---- b200-ipc: the decode engine in a child process ------------------------
// Pipe messages: a 64-bit length, then the bytes.
static void PutBytes(int fd, const void* p, uint64_t n) {
  const auto* b = static_cast<const uint8_t*>(p);
  if (write(fd, &n, sizeof(n)) != static_cast<ssize_t>(sizeof(n))) std::exit(5);
  for (uint64_t done = 0; done < n;) {
    const ssize_t k = write(fd, b + done, n - done);
    if (k <= 0) std::exit(5);
    done += static_cast<uint64_t>(k);
  }
}
static std::vector<uint8_t> GetBytes(int fd) {
  uint64_t n = 0;
  if (read(fd, &n, sizeof(n)) != static_cast<ssize_t>(sizeof(n))) std::exit(5);
  std::vector<uint8_t> v(n);
  for (uint64_t done = 0; done < n;) {
    const ssize_t k = read(fd, v.data() + done, n - done);
    if (k <= 0) std::exit(5);
    done += static_cast<uint64_t>(k);
  }
  return v;
}
template <class T>
static void PutVec(int fd, const std::vector<T>& v) {
  PutBytes(fd, v.data(), v.size() * sizeof(T));
}
template <class T>
static std::vector<T> GetVec(int fd) {
  const std::vector<uint8_t> b = GetBytes(fd);
  std::vector<T> v(b.size() / sizeof(T));
  if (!b.empty()) std::memcpy(v.data(), b.data(), b.size());
  return v;
}

struct IpcCase {
  int32_t layers, dim;
  int64_t prompt, pages;
};

static TokenList CasePrompt(int64_t n) {
  std::mt19937_64 rng(1);
  TokenList prompt(n);
  for (auto& t : prompt) t = static_cast<Token>(rng() % 256);
  return prompt;
}

// Child (decode engine): prep_recv, export, wait for the sender, then
// start_generate + decode steps; reports the outcome.
static int IpcChild(int rfd, int wfd, const IpcCase& c, int32_t max_tokens) {
  ModelConfig mc;
  mc.layers = c.layers;
  mc.dim = c.dim;
  HashModel m(mc);
  CacheConfig cc;
  cc.num_pages = c.pages;
  cc.page_size = 16;
  const TokenList prompt = CasePrompt(c.prompt);
  const int32_t L = c.layers;
  const int64_t n = c.prompt, e = n - 1;
  b200::KVCache D(cc, &m, /*device=*/0, /*rank=*/1);
  auto r = D.PrepRecv(10, prompt, -1);
  const ss_ipc_handle h = D.ExportIpc();
  const int64_t ml = r.match_len;
  PutBytes(wfd, &ml, sizeof(ml));
  const std::string addr = r.addr.ToJson();
  PutBytes(wfd, addr.data(), addr.size());
  PutBytes(wfd, &h, sizeof(h));
  GetBytes(rfd);  // the prefill engine has sent every layer
  std::vector<SeqId> done;
  for (int spin = 0; spin < 100000 && done.empty(); ++spin) done = D.DrainReceiveCompletions();
  if (done.size() != 1 || done[0] != 10) {
    std::fprintf(stderr, "ipc child: receive window did not complete\n");
    return 3;
  }
  const int64_t committed = D.Committed(10);
  std::vector<Token> tokens;
  D.EnsureAllocated(10, n);
  auto pd = D.BeginForward({BatchEntry{10, TokenRange{e, n}, false}});
  std::vector<uint64_t> x{m.Embed(prompt[e], e)};
  for (int32_t l = 0; l < L; ++l) x = D.Attention(l, &pd, x, FrameSink{});
  tokens.push_back(m.SampleToken(x.back()));
  for (int32_t k = 1; k < max_tokens; ++k) {
    const Token t = tokens.back();
    D.AppendToken(10, t);
    D.EnsureAllocated(10, n + k);
    auto pk = D.BeginForward({BatchEntry{10, TokenRange{n + k - 1, n + k}, true}});
    std::vector<uint64_t> y{m.Embed(t, n + k - 1)};
    for (int32_t l = 0; l < L; ++l) y = D.Attention(l, &pk, y, FrameSink{});
    tokens.push_back(m.SampleToken(y.back()));
  }
  std::vector<uint64_t> digests;
  std::vector<int> fills;
  for (int64_t pos = 0; pos < n; ++pos) {
    for (int32_t l = 0; l < L; ++l) {
      digests.push_back(m.EntryDigest(D.ReadEntryWords(10, pos, l)));
      fills.push_back(static_cast<int>(D.FillOf(10, pos, l)));
    }
  }
  PutBytes(wfd, &committed, sizeof(committed));
  PutVec(wfd, tokens);
  PutVec(wfd, digests);
  PutVec(wfd, fills);
  GetBytes(rfd);  // the parent has what it needs: the exported memory may go
  return 0;
}

// Parent (prefill engine): imports the child's receive surface and runs
// remote_send into it.
static Outcome RunIpc(const char* self, const IpcCase& c, int32_t max_tokens) {
  Outcome out;
  int to_child[2], from_child[2];
  if (pipe(to_child) != 0 || pipe(from_child) != 0) std::exit(4);
  char a_rfd[16], a_wfd[16], a_layers[16], a_dim[16], a_prompt[16], a_pages[16], a_gen[16];
  std::snprintf(a_rfd, sizeof(a_rfd), "%d", to_child[0]);
  std::snprintf(a_wfd, sizeof(a_wfd), "%d", from_child[1]);
  std::snprintf(a_layers, sizeof(a_layers), "%d", c.layers);
  std::snprintf(a_dim, sizeof(a_dim), "%d", c.dim);
  std::snprintf(a_prompt, sizeof(a_prompt), "%lld", static_cast<long long>(c.prompt));
  std::snprintf(a_pages, sizeof(a_pages), "%lld", static_cast<long long>(c.pages));
  std::snprintf(a_gen, sizeof(a_gen), "%d", max_tokens);
  char arg0[] = "--ipc-child";
  char* argv[] = {const_cast<char*>(self), arg0, a_rfd, a_wfd, a_layers, a_dim, a_prompt, a_pages,
                  a_gen, nullptr};
  pid_t pid = 0;
  if (posix_spawn(&pid, self, nullptr, nullptr, argv, environ) != 0) std::exit(4);
  close(to_child[0]);
  close(from_child[1]);
  const int rfd = from_child[0], wfd = to_child[1];
  ModelConfig mc;
  mc.layers = c.layers;
  mc.dim = c.dim;
  HashModel m(mc);
  CacheConfig cc;
  cc.num_pages = c.pages;
  cc.page_size = 16;
  const TokenList prompt = CasePrompt(c.prompt);
  const int32_t L = c.layers;
  const int64_t e = c.prompt - 1;
  {
    const std::vector<uint8_t> mlb = GetBytes(rfd);
    std::memcpy(&out.match_len, mlb.data(), sizeof(out.match_len));
    const std::vector<uint8_t> ab = GetBytes(rfd);
    out.addr = KVAddrInfo::FromJson(std::string(ab.begin(), ab.end()));
    const std::vector<uint8_t> hb = GetBytes(rfd);
    ss_ipc_handle h{};
    std::memcpy(&h, hb.data(), sizeof(h));
    b200::KVCache P(cc, &m, /*device=*/0, /*rank=*/0);
    P.ImportIpc(1, h);
    P.CreateSequence(20, prompt);
    P.EnsureAllocated(20, e);
    P.MarkSend(20, TokenRange{out.match_len, e}, 1, out.addr, 7);
    auto plan = P.BeginForward({BatchEntry{20, TokenRange{0, e}, false}});
    std::vector<uint64_t> x(e);
    for (int64_t i = 0; i < e; ++i) x[i] = m.Embed(prompt[i], i);
    FrameSink sink = [&](int32_t, const PlanSend&, std::vector<uint64_t>) { ++out.sink_calls; };
    for (int32_t l = 0; l < L; ++l) x = P.Attention(l, &plan, x, sink);
    P.Synchronize();
    const char go = 1;
    PutBytes(wfd, &go, 1);
    const std::vector<uint8_t> cb = GetBytes(rfd);
    std::memcpy(&out.committed, cb.data(), sizeof(out.committed));
    out.tokens = GetVec<Token>(rfd);
    out.digests = GetVec<uint64_t>(rfd);
    out.fills = GetVec<int>(rfd);
    P.DetachPeer(1);
  }
  const char bye = 1;
  PutBytes(wfd, &bye, 1);
  int status = 0;
  waitpid(pid, &status, 0);
  if (!WIFEXITED(status) || WEXITSTATUS(status) != 0) {
    std::fprintf(stderr, "ipc child failed (status %d)\n", status);
    out.match_len = -2;
  }
  close(rfd);
  close(wfd);
  return out;
}

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

int main(int argc, char** argv) {
  if (argc == 9 && std::strcmp(argv[1], "--ipc-child") == 0) {
    const IpcCase c{std::atoi(argv[4]), std::atoi(argv[5]), std::atoll(argv[6]), std::atoll(argv[7])};
    return IpcChild(std::atoi(argv[2]), std::atoi(argv[3]), c, std::atoi(argv[8]));
  }
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
    // The decode engine in another process, device-direct over CUDA IPC.
    const Outcome ip = RunIpc(argv[0], IpcCase{c.layers, c.dim, c.prompt, c.pages}, gen);
    all &= Same(c.name, ref, ip, "reference", "b200-ipc");
    all &= ip.sink_calls == 0;
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
