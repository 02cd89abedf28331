// Schedule generator + unit expansion.
//
// Builders:
//   STP (R-STP)  PAPER.md §4.2, App. A P:L592 — slot grid, warm-up
//                W-separation except on the last device, degraded-phase
//                separation after the last chunk-0 forward, FIFO deferred-W
//                placement (F -> F&W, one W after each lone full backward,
//                rest at the end).
//   1F1B-I       Megatron interleaved, two virtual stages.
//   ZB           ZB-V-style greedy (V-shape, B/W split, 2p memory cap).
//   1F1B         PipeDream one-forward-one-backward (v = 1).
// Unit expansion (Fig. 3): each action becomes compute units on
// the compute stream (F_ATTN/F_MLP/B_*/W_*/EMB/HEAD), TP comm phases on the
// comm stream (CF/CB) and PP send/recv on the PP stream; a braided action
// interleaves its two lanes unit by unit so each comm phase of one lane runs
// under the next compute unit of the other lane.
//
// This is an independent implementation of the definition the CPU oracle
// (oracle/schedule.py) also implements; tests compare the canonical text
// byte for byte.
#include "schedule.h"

#include <algorithm>
#include <cstdio>
#include <deque>
#include <functional>
#include <map>
#include <stdexcept>
#include <string>

#include "common.h"

namespace stp {

int sched_n_vstages(int kind, int p) { return kind == STP_SCHED_1F1B ? p : 2 * p; }
int sched_n_chunks(int kind) { return kind == STP_SCHED_1F1B ? 1 : 2; }

int sched_vstage(int kind, int p, int d, int c) {
  if (kind == STP_SCHED_1F1B) return d;
  if (kind == STP_SCHED_1F1B_I || kind == STP_SCHED_1F1B_I_NAIVE) return c * p + d;
  return c == 0 ? d : 2 * p - 1 - d;
}

int sched_vstage_device(int kind, int p, int vs) {
  if (kind == STP_SCHED_1F1B) return vs;
  if (kind == STP_SCHED_1F1B_I || kind == STP_SCHED_1F1B_I_NAIVE) return vs % p;
  return vs < p ? vs : 2 * p - 1 - vs;
}

namespace {

stp_action mk(int kind, int chunk, int f = -1, int b = -1, int w = -1, int wc = -1) {
  stp_action a;
  a.kind = kind;
  a.chunk = chunk;
  a.f_mb = f;
  a.b_mb = b;
  a.w_mb = w;
  a.w_chunk = wc;
  return a;
}

std::vector<stp_action> rstp(int p, int m, int d, bool separate) {
  std::vector<stp_action> g;
  auto ok = [&](int x) { return x >= 1 && x <= m; };
  for (int k = 1; k <= m + 2 * p + 1; ++k) {
    const int slots[2][3] = {{1, k - p + d, k - p - 1}, {0, k, k - 2 * p + d}};
    for (auto& s : slots) {
      const int c = s[0], f = s[1], b = s[2];
      if (ok(f) && ok(b)) g.push_back(mk(STP_A_FB, c, f, b));
      else if (ok(f)) g.push_back(mk(STP_A_F, c, f));
      else if (ok(b)) g.push_back(mk(STP_A_BFULL, c, -1, b));
    }
  }
  if (!separate) return g;
  if (d != p - 1) {  // warm-up separation: first p-1 braids, all devices but the last
    int n = 0;
    for (auto& a : g)
      if (a.kind == STP_A_FB && n < p - 1) {
        a.kind = STP_A_FBS;
        ++n;
      }
  }
  int last_f0 = -1;
  for (int i = 0; i < (int)g.size(); ++i)
    if (g[i].chunk == 0 && (g[i].kind == STP_A_F || g[i].kind == STP_A_FB || g[i].kind == STP_A_FBS)) last_f0 = i;
  for (int i = last_f0 + 1; i < (int)g.size(); ++i)
    if (g[i].kind == STP_A_FB) g[i].kind = STP_A_FBS;  // degraded phase
  std::deque<std::pair<int, int>> q;                    // (chunk, mb) of deferred W
  std::vector<stp_action> out;
  for (const auto& a : g) {
    if (a.kind == STP_A_F && !q.empty()) {
      auto w = q.front();
      q.pop_front();
      out.push_back(mk(STP_A_FW, a.chunk, a.f_mb, -1, w.second, w.first));
    } else if (a.kind == STP_A_FBS) {
      out.push_back(a);
      q.push_back({a.chunk, a.b_mb});
    } else if (a.kind == STP_A_BFULL) {
      out.push_back(a);
      if (!q.empty()) {
        auto w = q.front();
        q.pop_front();
        out.push_back(mk(STP_A_W, w.first, -1, -1, w.second, w.first));
      }
    } else {
      out.push_back(a);
    }
  }
  for (auto& w : q) out.push_back(mk(STP_A_W, w.first, -1, -1, w.second, w.first));
  return out;
}

std::vector<stp_action> interleaved(int p, int m, int d) {
  const int v = 2, total = m * v;
  const int nw = std::min(2 * (p - d - 1) + (v - 1) * p, total);
  auto fwd = [&](int k, int& c, int& mb) {
    c = (k % (p * v)) / p;
    mb = (k / (p * v)) * p + (k % p) + 1;
  };
  auto bwd = [&](int k, int& c, int& mb) {
    c = v - 1 - (k % (p * v)) / p;
    mb = (k / (p * v)) * p + (k % p) + 1;
  };
  std::vector<stp_action> out;
  int c, mb;
  for (int k = 0; k < nw; ++k) {
    fwd(k, c, mb);
    out.push_back(mk(STP_A_F, c, mb));
  }
  for (int i = 0; i < total - nw; ++i) {
    fwd(nw + i, c, mb);
    out.push_back(mk(STP_A_F, c, mb));
    bwd(i, c, mb);
    out.push_back(mk(STP_A_BFULL, c, -1, mb));
  }
  for (int i = total - nw; i < total; ++i) {
    bwd(i, c, mb);
    out.push_back(mk(STP_A_BFULL, c, -1, mb));
  }
  return out;
}

std::vector<stp_action> one_f_one_b(int p, int m, int d) {
  const int nw = std::min(p - d - 1, m);
  std::vector<stp_action> out;
  for (int f = 1; f <= nw; ++f) out.push_back(mk(STP_A_F, 0, f));
  for (int i = 0; i < m - nw; ++i) {
    out.push_back(mk(STP_A_F, 0, nw + i + 1));
    out.push_back(mk(STP_A_BFULL, 0, -1, i + 1));
  }
  for (int i = m - nw; i < m; ++i) out.push_back(mk(STP_A_BFULL, 0, -1, i + 1));
  return out;
}

// ZB-V-style greedy list schedule under unit costs: every time step each
// device takes (in priority) a ready B (smallest mb, chunk 1 first), else a
// ready F if fewer than 2p chunk-microbatches are live (chunk 1 first), else
// the oldest deferred W.
// Durations (F, B, W) of the ZB list schedule: B200's per-layer unit times at
// TP4 (F : B : W = 1 : 1.28 : 0.86, plus a lone F / B's exposed TP phase), the
// same constants as oracle/schedule.py ZB_COSTS.
constexpr long kZbF = 12, kZbB = 15, kZbW = 9;

bool zb_greedy(int p, int m, std::vector<std::vector<stp_action>>& progs) {
  const int V = 2 * p, cap = 2 * p;
  std::map<std::pair<int, int>, long> fdone, bdone;
  std::vector<std::array<int, 2>> nextf(p, {1, 1}), nextb(p, {1, 1});
  std::vector<std::deque<std::pair<int, int>>> wq(p);
  std::vector<int> live(p, 0);
  std::vector<long> busy(p, 0);
  progs.assign(p, {});
  const long total = 3L * 2 * m * p;
  long n = 0, t = 0;
  auto done_by = [](const std::map<std::pair<int, int>, long>& mp, std::pair<int, int> k, long t) {
    auto it = mp.find(k);
    return it != mp.end() && it->second <= t;
  };
  while (n < total) {
    if (t > 100 * kZbB * (total + 10)) return false;
    for (int d = 0; d < p; ++d) {
      if (busy[d] > t) continue;
      int bc = -1, bb = 0;
      for (int c : {1, 0}) {
        const int b = nextb[d][c];
        if (b > m) continue;
        const int vs = sched_vstage(STP_SCHED_ZB, p, d, c);
        bool ok = done_by(fdone, {b, vs}, t);
        if (vs < V - 1) ok = ok && done_by(bdone, {b, vs + 1}, t);
        if (ok && (bc < 0 || b < bb)) {
          bc = c;
          bb = b;
        }
      }
      if (bc >= 0) {
        const int vs = sched_vstage(STP_SCHED_ZB, p, d, bc);
        bdone[{bb, vs}] = busy[d] = t + kZbB;
        nextb[d][bc]++;
        wq[d].push_back({bc, bb});
        progs[d].push_back(mk(STP_A_B, bc, -1, bb));
        ++n;
        continue;
      }
      int fc = -1, ff = 0;
      if (live[d] < cap) {
        for (int c : {1, 0}) {
          const int f = nextf[d][c];
          if (f > m) continue;
          const int vs = sched_vstage(STP_SCHED_ZB, p, d, c);
          if (vs == 0 || done_by(fdone, {f, vs - 1}, t)) {
            fc = c;
            ff = f;
            break;
          }
        }
      }
      if (fc >= 0) {
        const int vs = sched_vstage(STP_SCHED_ZB, p, d, fc);
        fdone[{ff, vs}] = busy[d] = t + kZbF;
        nextf[d][fc]++;
        live[d]++;
        progs[d].push_back(mk(STP_A_F, fc, ff));
        ++n;
        continue;
      }
      if (!wq[d].empty()) {
        auto w = wq[d].front();
        wq[d].pop_front();
        live[d]--;
        busy[d] = t + kZbW;
        progs[d].push_back(mk(STP_A_W, w.first, -1, -1, w.second, w.first));
        ++n;
      }
    }
    ++t;
  }
  return true;
}

// Ours^ (STP_SCHED_STP_MEM; memory-efficient warm-up, App. A Fig. 8b and
// App. B schedule (d); reading R4): V-shape list
// schedule under unit costs (F = B = W = 1, FBS / FW = 2) with ZB-V's memory
// budget of 2p chunk-microbatches; each idle device takes the first feasible
// of: braided F(f)&B(b) of one chunk with f > b and W deferred (FBS), lone B,
// forward braided with the oldest deferred W (FW) or lone F, lone W; chunk 1
// before chunk 0.  Same algorithm as oracle/schedule.py build_stp_mem.
bool stp_mem(int p, int m, std::vector<std::vector<stp_action>>& progs) {
  const int V = 2 * p, cap = 2 * p;
  const long total = 3L * 2 * m * p;
  std::map<std::pair<int, int>, long> fend, bend;
  std::vector<std::array<int, 2>> nextf(p, {1, 1}), nextb(p, {1, 1});
  std::vector<std::deque<std::pair<int, int>>> wq(p);
  std::vector<int> live(p, 0);
  std::vector<long> busy(p, 0);
  progs.assign(p, {});
  long n = 0, t = 0;
  auto end_of = [&](const std::map<std::pair<int, int>, long>& mp, int mb, int vs) {
    auto it = mp.find({mb, vs});
    return it == mp.end() ? total + 1 : it->second;
  };
  auto vs_of = [&](int d, int c) { return sched_vstage(STP_SCHED_STP_MEM, p, d, c); };
  auto f_ready = [&](int d, int c) {
    const int f = nextf[d][c], vs = vs_of(d, c);
    return f <= m && (vs == 0 || end_of(fend, f, vs - 1) <= t);
  };
  auto b_ready = [&](int d, int c) {
    const int b = nextb[d][c], vs = vs_of(d, c);
    if (b > m || end_of(fend, b, vs) > t) return false;
    return vs == V - 1 || end_of(bend, b, vs + 1) <= t;
  };
  while (n < total) {
    if (t > 100 * (total + 10)) return false;
    for (int d = 0; d < p; ++d) {
      if (busy[d] > t) continue;
      bool done = false;
      for (int c : {1, 0}) {
        if (live[d] < cap && b_ready(d, c) && f_ready(d, c) && nextf[d][c] > nextb[d][c]) {
          const int f = nextf[d][c], b = nextb[d][c], vs = vs_of(d, c);
          fend[{f, vs}] = bend[{b, vs}] = busy[d] = t + 2;
          nextf[d][c]++;
          nextb[d][c]++;
          live[d]++;
          wq[d].push_back({c, b});
          progs[d].push_back(mk(STP_A_FBS, c, f, b));
          n += 2;
          done = true;
          break;
        }
      }
      if (done) continue;
      for (int c : {1, 0}) {
        if (b_ready(d, c)) {
          const int b = nextb[d][c], vs = vs_of(d, c);
          bend[{b, vs}] = busy[d] = t + 1;
          nextb[d][c]++;
          wq[d].push_back({c, b});
          progs[d].push_back(mk(STP_A_B, c, -1, b));
          n += 1;
          done = true;
          break;
        }
      }
      if (done) continue;
      if (live[d] < cap) {
        for (int c : {1, 0}) {
          if (f_ready(d, c)) {
            const int f = nextf[d][c], vs = vs_of(d, c);
            nextf[d][c]++;
            live[d]++;
            if (!wq[d].empty()) {
              const auto w = wq[d].front();
              wq[d].pop_front();
              live[d]--;
              fend[{f, vs}] = busy[d] = t + 2;
              progs[d].push_back(mk(STP_A_FW, c, f, -1, w.second, w.first));
              n += 2;
            } else {
              fend[{f, vs}] = busy[d] = t + 1;
              progs[d].push_back(mk(STP_A_F, c, f));
              n += 1;
            }
            done = true;
            break;
          }
        }
      }
      if (done) continue;
      if (!wq[d].empty()) {
        const auto w = wq[d].front();
        wq[d].pop_front();
        live[d]--;
        busy[d] = t + 1;
        progs[d].push_back(mk(STP_A_W, w.first, -1, -1, w.second, w.first));
        n += 1;
      }
    }
    ++t;
  }
  return true;
}

const char* kind_name(int kind) {
  switch (kind) {
    case STP_SCHED_STP: return "stp";
    case STP_SCHED_1F1B_I: return "1f1b-i";
    case STP_SCHED_ZB: return "zb";
    case STP_SCHED_STP_NOBRAID: return "stp-nobraid";
    case STP_SCHED_STP_NOSEP: return "stp-nosep";
    case STP_SCHED_1F1B_I_NAIVE: return "1f1b-i-naive";
    case STP_SCHED_1F1B: return "1f1b";
    case STP_SCHED_STP_MEM: return "stp-mem";
  }
  return "?";
}

}  // namespace

stp_status schedule_build(int p, int vpp, int tp, int m, int kind, Schedule& s) {
  STP_CHECK_ARG(p >= 1 && m >= 1 && tp >= 1, "pp >= 1, tp >= 1, n_micro >= 1");
  STP_CHECK_ARG(kind >= 0 && kind <= STP_SCHED_STP_MEM, "schedule kind");
  if (kind == STP_SCHED_1F1B) {
    if (vpp != 1) return fail(STP_EUNSUPPORTED, "1F1B needs vpp == 1");
  } else if (vpp != 2) {
    return fail(STP_EUNSUPPORTED, "STP / 1F1B-I / ZB need vpp == 2 (P:L173)");
  }
  if ((kind == STP_SCHED_1F1B_I || kind == STP_SCHED_1F1B_I_NAIVE) && m % p != 0)
    return fail(STP_EUNSUPPORTED, "1F1B-I needs n_micro % pp == 0 (Megatron rule)");
  s.kind = kind;
  s.pp = p;
  s.vpp = vpp;
  s.tp = tp;
  s.m = m;
  s.ranks.clear();
  if (kind == STP_SCHED_ZB) {
    if (!zb_greedy(p, m, s.ranks)) return fail(STP_ESCHEDULE, "ZB greedy did not terminate");
    return STP_OK;
  }
  if (kind == STP_SCHED_STP_MEM) {
    if (!stp_mem(p, m, s.ranks)) return fail(STP_ESCHEDULE, "STP-MEM list schedule did not terminate");
    return STP_OK;
  }
  for (int d = 0; d < p; ++d) {
    switch (kind) {
      case STP_SCHED_STP:
      case STP_SCHED_STP_NOBRAID: s.ranks.push_back(rstp(p, m, d, true)); break;
      case STP_SCHED_STP_NOSEP: s.ranks.push_back(rstp(p, m, d, false)); break;
      case STP_SCHED_1F1B_I:
      case STP_SCHED_1F1B_I_NAIVE: s.ranks.push_back(interleaved(p, m, d)); break;
      case STP_SCHED_1F1B: s.ranks.push_back(one_f_one_b(p, m, d)); break;
    }
  }
  return STP_OK;
}

// ------------------------------------------------------------- expansion
namespace {

struct Lane {
  std::vector<std::function<void()>> pre, steps, post;
};

}  // namespace

// vit_first (MLLM; reading V5): virtual stage 0 holds the
// ViT layers 0..lay[0]-1 and ends its forward with F_MERGE (2x2 merger + text
// embedding -> LM input); its backward starts with B_MERGE / W_MERGE.
stp_status schedule_expand(const Schedule& s, int d, const std::vector<int>& lay, std::vector<stp_unit>& units,
                           bool vit_first) {
  const int kind = s.kind, p = s.pp;
  const int V = sched_n_vstages(kind, p);
  STP_CHECK_ARG((int)lay.size() == V, "layers_per_vstage must have pp*vpp entries");
  STP_CHECK_ARG(d >= 0 && d < p, "pp_rank");
  units.clear();
  const bool braid = kind != STP_SCHED_STP_NOBRAID;
  const bool naive = kind == STP_SCHED_1F1B_I_NAIVE;
  std::map<std::pair<int, int>, int> fwd_tail, bwd_tail;
  auto emit = [&](int ai, int stream, int op, int layer, int c, int mb, int d0 = -1, int d1 = -1) {
    stp_unit u;
    u.action = ai;
    u.stream = stream;
    u.op = op;
    u.layer = layer;
    u.chunk = c;
    u.mb = mb;
    u.dep0 = d0;
    u.dep1 = d1;
    units.push_back(u);
    return (int)units.size() - 1;
  };
  auto first_layer = [&](int vs) {
    int f = 0;
    for (int i = 0; i < vs; ++i) f += lay[i];
    return f;
  };
  auto dev_of = [&](int vs) { return sched_vstage_device(kind, p, vs); };

  // A lane's callables capture shared state by pointer (kept alive below).
  std::vector<std::shared_ptr<int>> keep;

  auto fwd_lane = [&](int ai, int c, int mb) {
    Lane ln;
    const int vs = sched_vstage(kind, p, d, c);
    const int l0 = first_layer(vs), nl = lay[vs];
    std::vector<std::pair<int, int>> heavy;
    if (vs == 0) heavy.push_back({STP_U_F_EMB, -1});
    for (int l = l0; l < l0 + nl; ++l) {
      heavy.push_back({STP_U_F_ATTN, l});
      heavy.push_back({STP_U_F_MLP, l});
    }
    if (vs == 0 && vit_first) heavy.push_back({STP_U_F_MERGE, -1});
    if (vs == V - 1) heavy.push_back({STP_U_F_HEAD, -1});
    auto last = std::make_shared<int>(-1);
    keep.push_back(last);
    ln.pre.push_back([=, &emit, &dev_of]() {
      int rv = -1;
      if (vs > 0 && dev_of(vs - 1) != d) rv = emit(ai, 2, STP_U_PP_RECV, dev_of(vs - 1), c, mb);
      if (vs > 0) *last = emit(ai, 1, STP_U_CF, 0, c, mb, rv);
    });
    for (size_t k = 0; k < heavy.size(); ++k) {
      const int op = heavy[k].first, l = heavy[k].second, kk = (int)k + 1;
      ln.steps.push_back([=, &emit]() {
        int u = emit(ai, 0, op, l, c, mb, *last);
        *last = emit(ai, 1, STP_U_CF, kk, c, mb, u);
      });
    }
    ln.post.push_back([=, &emit, &dev_of, &fwd_tail]() {
      fwd_tail[{c, mb}] = *last;
      if (vs < V - 1 && dev_of(vs + 1) != d) emit(ai, 2, STP_U_PP_SEND, dev_of(vs + 1), c, mb, *last);
    });
    return ln;
  };

  auto w_list = [&](int vs) {
    std::vector<std::pair<int, int>> wl;
    const int l0 = first_layer(vs), nl = lay[vs];
    if (vs == V - 1) wl.push_back({STP_U_W_HEAD, -1});
    if (vs == 0 && vit_first) wl.push_back({STP_U_W_MERGE, -1});
    for (int l = l0 + nl - 1; l >= l0; --l) {
      wl.push_back({STP_U_W_MLP, l});
      wl.push_back({STP_U_W_ATTN, l});
    }
    return wl;
  };

  auto bwd_lane = [&](int ai, int c, int mb, bool with_w) {
    Lane ln;
    const int vs = sched_vstage(kind, p, d, c);
    const int l0 = first_layer(vs), nl = lay[vs];
    std::vector<std::pair<int, int>> heavy;
    if (vs == V - 1) heavy.push_back({STP_U_B_HEAD, -1});
    if (vs == 0 && vit_first) heavy.push_back({STP_U_B_MERGE, -1});
    for (int l = l0 + nl - 1; l >= l0; --l) {
      heavy.push_back({STP_U_B_MLP, l});
      heavy.push_back({STP_U_B_ATTN, l});
    }
    const auto wl = w_list(vs);
    auto last = std::make_shared<int>(-1);
    keep.push_back(last);
    ln.pre.push_back([=, &emit, &dev_of]() {
      int rv = -1;
      if (vs < V - 1 && dev_of(vs + 1) != d) rv = emit(ai, 2, STP_U_PP_RECV, dev_of(vs + 1), c, mb);
      if (vs < V - 1) *last = emit(ai, 1, STP_U_CB, 0, c, mb, rv);
    });
    for (size_t k = 0; k < heavy.size(); ++k) {
      const int op = heavy[k].first, l = heavy[k].second, kk = (int)k + 1;
      const int wop = wl[k].first, wlay = wl[k].second;
      ln.steps.push_back([=, &emit, &fwd_tail]() {
        const int dep = (op == STP_U_B_HEAD) ? fwd_tail.at({c, mb}) : *last;
        int u = emit(ai, 0, op, l, c, mb, dep);
        *last = emit(ai, 1, STP_U_CB, kk, c, mb, u);
        if (with_w) emit(ai, 0, wop, wlay, c, mb, naive ? *last : -1);
      });
    }
    ln.post.push_back([=, &emit, &dev_of, &bwd_tail]() {
      bwd_tail[{c, mb}] = *last;
      if (with_w && vs == 0) emit(ai, 0, STP_U_W_EMB, -1, c, mb, *last);
      if (vs > 0 && dev_of(vs - 1) != d) emit(ai, 2, STP_U_PP_SEND, dev_of(vs - 1), c, mb, *last);
    });
    return ln;
  };

  auto w_lane = [&](int ai, int c, int mb) {
    Lane ln;
    const int vs = sched_vstage(kind, p, d, c);
    for (auto& w : w_list(vs)) {
      const int op = w.first, l = w.second;
      ln.steps.push_back([=, &emit]() { emit(ai, 0, op, l, c, mb); });
    }
    ln.post.push_back([=, &emit, &bwd_tail]() {
      if (vs == 0) emit(ai, 0, STP_U_W_EMB, -1, c, mb, bwd_tail.at({c, mb}));
    });
    return ln;
  };

  auto run = [&](std::vector<Lane> lanes, bool inter) {
    if (inter) {
      for (auto& ln : lanes)
        for (auto& f : ln.pre) f();
      size_t n = 0;
      for (auto& ln : lanes) n = std::max(n, ln.steps.size());
      for (size_t k = 0; k < n; ++k)
        for (auto& ln : lanes)
          if (k < ln.steps.size()) ln.steps[k]();
      for (auto& ln : lanes)
        for (auto& f : ln.post) f();
    } else {
      for (auto& ln : lanes) {
        for (auto& f : ln.pre) f();
        for (auto& f : ln.steps) f();
        for (auto& f : ln.post) f();
      }
    }
  };

  try {
    const auto& acts = s.ranks[d];
    for (int ai = 0; ai < (int)acts.size(); ++ai) {
      const stp_action& a = acts[ai];
      switch (a.kind) {
        case STP_A_F: run({fwd_lane(ai, a.chunk, a.f_mb)}, true); break;
        case STP_A_BFULL: run({bwd_lane(ai, a.chunk, a.b_mb, true)}, true); break;
        case STP_A_B: run({bwd_lane(ai, a.chunk, a.b_mb, false)}, true); break;
        case STP_A_W: run({w_lane(ai, a.w_chunk, a.w_mb)}, true); break;
        case STP_A_FB: run({fwd_lane(ai, a.chunk, a.f_mb), bwd_lane(ai, a.chunk, a.b_mb, true)}, braid); break;
        case STP_A_FBS: run({fwd_lane(ai, a.chunk, a.f_mb), bwd_lane(ai, a.chunk, a.b_mb, false)}, braid); break;
        case STP_A_FW: run({fwd_lane(ai, a.chunk, a.f_mb), w_lane(ai, a.w_chunk, a.w_mb)}, braid); break;
        default: return fail(STP_ESCHEDULE, "unknown action kind");
      }
    }
  } catch (const std::out_of_range&) {
    return fail(STP_ESCHEDULE, "expansion: backward/W before its forward/backward");
  }
  return STP_OK;
}

int schedule_stash_slots(const Schedule& s, int d) {
  int cur = 0, best = 0;
  for (const auto& a : s.ranks[d]) {
    const bool f = a.kind == STP_A_F || a.kind == STP_A_FB || a.kind == STP_A_FBS || a.kind == STP_A_FW;
    const bool bfull = a.kind == STP_A_BFULL || a.kind == STP_A_FB;
    const bool w = a.kind == STP_A_W || a.kind == STP_A_FW;
    if (f) best = std::max(best, ++cur);
    if (bfull) --cur;
    if (w) --cur;
  }
  return best;
}

std::string schedule_text(const Schedule& s, const int* lay, bool vit_first) {
  std::string out;
  char buf[256];
  snprintf(buf, sizeof(buf), "sched %s p %d v %d t %d m %d%s\n", kind_name(s.kind), s.pp, s.vpp, s.tp, s.m,
           vit_first ? " mllm" : "");
  out += buf;
  const int V = sched_n_vstages(s.kind, s.pp);
  std::vector<int> layv;
  if (lay) layv.assign(lay, lay + V);
  for (int d = 0; d < s.pp; ++d) {
    snprintf(buf, sizeof(buf), "rank %d\n", d);
    out += buf;
    const auto& acts = s.ranks[d];
    for (size_t i = 0; i < acts.size(); ++i) {
      const auto& a = acts[i];
      snprintf(buf, sizeof(buf), "A %zu %d %d %d %d %d %d\n", i, a.kind, a.chunk, a.f_mb, a.b_mb, a.w_mb, a.w_chunk);
      out += buf;
    }
    if (lay) {
      std::vector<stp_unit> units;
      if (schedule_expand(s, d, layv, units, vit_first) != STP_OK) return std::string();
      for (size_t j = 0; j < units.size(); ++j) {
        const auto& u = units[j];
        snprintf(buf, sizeof(buf), "U %zu %d %d %d %d %d %d %d %d\n", j, u.action, u.stream, u.op, u.layer, u.chunk,
                 u.mb, u.dep0, u.dep1);
        out += buf;
      }
    }
  }
  return out;
}

stp_status layer_split(int n_layers, int n_slots, int* out) {
  STP_CHECK_ARG(n_layers >= 1 && n_slots >= 1, "n_layers, n_slots >= 1");
  const int total = n_layers + 2, base = total / n_slots, rem = total % n_slots;
  for (int i = 0; i < n_slots; ++i) out[i] = base + (i < rem ? 1 : 0);
  out[n_slots - 1] -= 2;
  int sum = 0, mn = 1 << 30;
  for (int i = 0; i < n_slots; ++i) {
    sum += out[i];
    mn = std::min(mn, out[i]);
  }
  if (mn < 1 || sum != n_layers)
    return fail(STP_EINVAL, "IndivisibleLayers: " + std::to_string(n_layers) + " layers over " +
                                std::to_string(n_slots) + " slots");
  return STP_OK;
}

}  // namespace stp

// ------------------------------------------------------------------- C ABI
struct stp_schedule {
  stp::Schedule s;
};

extern "C" {

stp_status stp_build_schedule(int32_t pp, int32_t vpp, int32_t tp, int32_t n_micro, int32_t kind,
                              stp_schedule** out) {
  if (!out) return stp::fail(STP_EINVAL, "out is NULL");
  *out = nullptr;
  auto* h = new (std::nothrow) stp_schedule;
  if (!h) return stp::fail(STP_ENOMEM, "schedule handle");
  stp_status st = stp::schedule_build(pp, vpp, tp, n_micro, kind, h->s);
  if (st != STP_OK) {
    delete h;
    return st;
  }
  *out = h;
  return STP_OK;
}

stp_status stp_schedule_actions(const stp_schedule* s, int32_t r, stp_action* buf, int32_t cap, int32_t* n_out) {
  if (!s || !n_out) return stp::fail(STP_EINVAL, "NULL handle / n_out");
  if (r < 0 || r >= s->s.pp) return stp::fail(STP_EINVAL, "pp_rank out of range");
  const auto& a = s->s.ranks[r];
  *n_out = (int32_t)a.size();
  if (cap < (int32_t)a.size()) return stp::fail(STP_ECAPACITY, "buffer too small");
  std::copy(a.begin(), a.end(), buf);
  return STP_OK;
}

static stp_status units_impl(const stp_schedule* s, int32_t r, const int32_t* lay, bool vit_first, stp_unit* buf,
                             int32_t cap, int32_t* n_out) {
  if (!s || !n_out || !lay) return stp::fail(STP_EINVAL, "NULL handle / layers / n_out");
  if (r < 0 || r >= s->s.pp) return stp::fail(STP_EINVAL, "pp_rank out of range");
  std::vector<int> layv(lay, lay + stp::sched_n_vstages(s->s.kind, s->s.pp));
  std::vector<stp_unit> u;
  stp_status st = stp::schedule_expand(s->s, r, layv, u, vit_first);
  if (st != STP_OK) return st;
  *n_out = (int32_t)u.size();
  if (cap < (int32_t)u.size()) return stp::fail(STP_ECAPACITY, "buffer too small");
  std::copy(u.begin(), u.end(), buf);
  return STP_OK;
}

stp_status stp_schedule_units(const stp_schedule* s, int32_t r, const int32_t* lay, stp_unit* buf, int32_t cap,
                              int32_t* n_out) {
  return units_impl(s, r, lay, false, buf, cap, n_out);
}

stp_status stp_schedule_units_mllm(const stp_schedule* s, int32_t r, const int32_t* lay, stp_unit* buf, int32_t cap,
                                   int32_t* n_out) {
  return units_impl(s, r, lay, true, buf, cap, n_out);
}

static stp_status serialize_impl(const stp_schedule* s, const int32_t* lay, bool vit_first, char* buf, int64_t cap,
                                 int64_t* n_out) {
  if (!s || !n_out) return stp::fail(STP_EINVAL, "NULL handle / n_out");
  std::string t = stp::schedule_text(s->s, lay, vit_first);
  if (t.empty()) return STP_ESCHEDULE;
  *n_out = (int64_t)t.size();
  if (cap < (int64_t)t.size() + 1) return stp::fail(STP_ECAPACITY, "buffer too small");
  std::copy(t.begin(), t.end(), buf);
  buf[t.size()] = '\0';
  return STP_OK;
}

stp_status stp_schedule_serialize(const stp_schedule* s, const int32_t* lay, char* buf, int64_t cap, int64_t* n_out) {
  return serialize_impl(s, lay, false, buf, cap, n_out);
}

stp_status stp_schedule_serialize_mllm(const stp_schedule* s, const int32_t* lay, char* buf, int64_t cap,
                                       int64_t* n_out) {
  return serialize_impl(s, lay, true, buf, cap, n_out);
}

stp_status stp_schedule_stash_slots(const stp_schedule* s, int32_t r, int32_t* n_out) {
  if (!s || !n_out) return stp::fail(STP_EINVAL, "NULL handle / n_out");
  if (r < 0 || r >= s->s.pp) return stp::fail(STP_EINVAL, "pp_rank out of range");
  *n_out = stp::schedule_stash_slots(s->s, r);
  return STP_OK;
}

void stp_free_schedule(stp_schedule* s) { delete s; }

stp_status stp_layer_split(int32_t n_layers, int32_t n_slots, int32_t* out) {
  if (!out) return stp::fail(STP_EINVAL, "out is NULL");
  return stp::layer_split(n_layers, n_slots, out);
}

}  // extern "C"
