// oracle/rei_oracle.cpp -- TEST INFRASTRUCTURE, NOT THE PRODUCT.
//
// A plain, slow, sequential CPU implementation of the Paresy search
// (Valizadeh & Berger, arXiv 2305.18575).  Only tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline / --impl reference legs may load this library.
// It shares no code, header, table or constant with the CUDA path under
// paper_2305_18575_b200/.
//
// Citations: P:n = PAPER.md line n (section / algorithm named alongside).
//
//  * Specification and satisfaction  L |= (P,N)   Def. def_specification
//  * Cost homomorphism (c1..c5)
//  * Shortlex order on Sigma^*                    P:324-336
//  * Infix closure IC(P u N)
//  * Infix power series ops 0,1,+,.,*             Def. definition_infix_power_series
//  * Guide table gt(w) = {(s1,s2) | s1 s2 = w}
//  * Main loop (Q, S, C, U per cost level)        Algorithm 1
//  * buildConcat                                  Algorithm 2
//  * Provenance / reconstruction
//  * REI with allowed error
//
// Every operation is the definition written out: concatenation is the fold of
// Alg. 2 lines 7-14 over ALL guide-table splits (including epsilon splits);
// star is the least fixpoint  acc_{k+1} = 1 + acc_k . x  of  r* = (+)_n r^n
// (P:636); dedup is a std::unordered_set over whole CSs.  No
// blocking, no bit tricks beyond "test bit / set bit", no reordering.
//
// Readings of silent / ambiguous points follow SURVEY.md 8(c) A1-A20 and are
// listed in DESIGN.md ("Readings").  Candidate counting follows reading A9.
//
// Pins (tests/test_oracle_pins.py): E1, the introduction
// (P:142-161), the Section 5 allowed-error table -- costs and regex text
// (P:1794-1808), Table 1 row 1's printed regex, brute-force enumeration of
// syntactic regexes matched with Python re, semiring laws, overfit bound
// (P:1540-1545), OnTheFly minimality.
// Parity unpinned: the paper's exact |REs| counts (reading A9 only brackets them
// between the counts before and after the solution's level) and, in OnTheFly mode,
// the level at which the cache fills (it depends on the cache size, reading B3).

#include <algorithm>
#include <array>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <functional>
#include <map>
#include <memory>
#include <string>
#include <unordered_set>
#include <vector>

namespace {

constexpr int kMaxWords = 8;  // |IC| <= 512 bits (the C ABI below always uses 8 words)

// A CS is stored in W 64-bit words, W = the smallest of 1, 2, 4, 8 with 64 W >= |IC|
// (power-of-two width, reading A16: the width is invisible to results;
// it only sets the oracle's memory per cached CS).
template <int W>
using CSW = std::array<uint64_t, W>;

template <int W>
struct CSHash {
  size_t operator()(const CSW<W>& c) const noexcept {
    size_t h = 1469598103934665603ull;
    for (uint64_t w : c) {
      h ^= std::hash<uint64_t>()(w) + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
    }
    return h;
  }
};

template <size_t W>
bool test_bit(const std::array<uint64_t, W>& c, int i) { return (c[i / 64] >> (i % 64)) & 1ull; }
template <size_t W>
void set_bit(std::array<uint64_t, W>& c, int i) { c[i / 64] |= 1ull << (i % 64); }
template <int W>
CSW<W> zero_cs() { CSW<W> c; c.fill(0); return c; }

enum Kind : int { K_SYM = 0, K_QUESTION = 1, K_STAR = 2, K_CONCAT = 3, K_UNION = 4,
                  K_EMPTY = 5, K_EPS = 6 };

struct Prov {
  int32_t kind;  // Kind
  int32_t L;     // cost level of the left / only operand (or symbol index for K_SYM)
  uint32_t i;    // index of the left / only operand in level L
  int32_t R;     // cost level of the right operand
  uint32_t j;    // index of the right operand in level R
};

template <int W>
struct Entry {
  CSW<W> cs;
  Prov prov;
};

struct LevelStat {
  int cost;
  uint64_t cand_q, cand_s, cand_c, cand_u;
  uint64_t unique;
  int complete;
};

// The ABI's view of one oracle instance (CSs cross it as 8 words).
struct Search {
  virtual ~Search() {}
  virtual int n() const = 0;
  virtual const std::string& ic_word(int k) const = 0;
  virtual const std::vector<std::pair<int, int>>& gt_row(int w) const = 0;
  virtual void masks8(uint64_t* pos8, uint64_t* neg8) const = 0;
  virtual void op8(int op, const uint64_t* a, const uint64_t* b, uint64_t* out) const = 0;
  virtual int run(int max_cost, long err_num, long err_den, bool complete_final_level,
                  uint64_t max_entries, bool onthefly) = 0;
  virtual int otf() const = 0;
  virtual void result6(long long* out6, double* seconds) const = 0;
  virtual const std::string& regex_text() const = 0;
  virtual const std::vector<LevelStat>& level_stats() const = 0;
  virtual long level_size(int cost) const = 0;
  virtual long level_cs8(int cost, uint64_t* out, long cap) const = 0;
  virtual std::string entry_regex(int cost, long i) const = 0;
};

template <int W>
struct Oracle : Search {
  using CS = CSW<W>;
  using Entry = ::Entry<W>;
  using CSHash = ::CSHash<W>;
  static CS zero_cs() { return ::zero_cs<W>(); }

  std::string alphabet;
  std::vector<std::string> P, N;
  int c[5];  // (sym, ?, *, concat, union)

  // IC and its shortlex index.
  std::vector<std::string> ic;
  std::map<std::string, int> index_of;
  // gt[w] = [(idx(w[:k]), idx(w[k:])) for k = 0..|w|].
  std::vector<std::vector<std::pair<int, int>>> gt;
  CS pos_mask, neg_mask;

  // Language cache: levels[c] = unique CSs of minimal cost c, in creation order.
  std::map<int, std::deque<Entry>> levels;  // deque: no 2x peak while a level grows
  std::unordered_set<CS, CSHash> seen;
  std::vector<LevelStat> stats;

  // Result.
  int status = -1;  // 0 found, 2 not found, 3 out of memory
  int result_cost = 0;
  std::string regex;
  uint64_t candidates = 0;          // through the found candidate (sequential)
  uint64_t cand_complete = 0;       // through the last complete level
  int last_complete_cost = 0;
  double seconds = 0;

  // allowed error: errors * den <= num * |P u N|; num = 0 = exact.
  long err_num = 0, err_den = 1;
  bool complete_final_level = false;
  uint64_t max_entries = 0;  // 0 = unlimited

  std::string err;

  int sym_rank(char ch) const {
    size_t p = alphabet.find(ch);
    return p == std::string::npos ? -1 : (int)p;
  }

  // Shortlex comparison with Sigma ordered as given.
  bool shortlex_less(const std::string& a, const std::string& b) const {
    if (a.size() != b.size()) return a.size() < b.size();
    for (size_t k = 0; k < a.size(); ++k) {
      int ra = sym_rank(a[k]), rb = sym_rank(b[k]);
      if (ra != rb) return ra < rb;
    }
    return false;
  }

  bool validate() {
    if (alphabet.empty()) { err = "empty alphabet"; return false; }
    for (size_t i = 0; i < alphabet.size(); ++i)
      for (size_t j = i + 1; j < alphabet.size(); ++j)
        if (alphabet[i] == alphabet[j]) { err = "duplicate alphabet symbol"; return false; }
    for (int k = 0; k < 5; ++k)
      if (c[k] < 1) { err = "costs must be >= 1"; return false; }
    for (auto* S : {&P, &N})
      for (auto& w : *S)
        for (char ch : w)
          if (sym_rank(ch) < 0) { err = "symbol not in alphabet"; return false; }
    for (auto& p : P)
      for (auto& q : N)
        if (p == q) { err = "P and N intersect"; return false; }
    return true;
  }

  // IC(P u N): every infix of every example, sorted shortlex, deduplicated.
  void build_ic() {
    std::vector<std::string> all;
    for (auto* S : {&P, &N})
      for (auto& w : *S)
        for (size_t i = 0; i <= w.size(); ++i)
          for (size_t j = i; j <= w.size(); ++j) all.push_back(w.substr(i, j - i));
    std::sort(all.begin(), all.end(),
              [this](const std::string& a, const std::string& b) { return shortlex_less(a, b); });
    all.erase(std::unique(all.begin(), all.end()), all.end());
    ic = all;
    index_of.clear();
    for (size_t i = 0; i < ic.size(); ++i) index_of[ic[i]] = (int)i;
    gt.assign(ic.size(), {});
    for (size_t w = 0; w < ic.size(); ++w)
      for (size_t k = 0; k <= ic[w].size(); ++k)
        gt[w].push_back({index_of.at(ic[w].substr(0, k)), index_of.at(ic[w].substr(k))});
    pos_mask = zero_cs();
    neg_mask = zero_cs();
    for (auto& p : P) set_bit(pos_mask, index_of.at(p));
    for (auto& q : N) set_bit(neg_mask, index_of.at(q));
  }

  int n() const override { return (int)ic.size(); }

  // ---- IPS operations -------------------------------------
  CS one() const {  // 1(sigma) = [sigma = eps]
    CS r = zero_cs();
    set_bit(r, index_of.at(""));
    return r;
  }
  CS op_union(const CS& a, const CS& b) const {  // (r + s)(sigma) = r(sigma) v s(sigma)
    CS r;
    for (int k = 0; k < W; ++k) r[k] = a[k] | b[k];
    return r;
  }
  // Algorithm 2, lines 5-14: fold over every split in gt[w].
  CS op_concat(const CS& a, const CS& b) const {
    CS r = zero_cs();
    for (int w = 0; w < n(); ++w)
      for (auto& lr : gt[w])
        if (test_bit(a, lr.first) && test_bit(b, lr.second)) set_bit(r, w);
    return r;
  }
  // r* = (+)_{n>=0} r^n with r^0 = 1, r^{n+1} = r^n . r:
  // iterate acc <- 1 + acc . x until it stops changing (finite IC).
  CS op_star(const CS& x) const {
    CS acc = one();
    for (;;) {
      CS next = op_union(one(), op_concat(acc, x));
      if (next == acc) return acc;
      acc = next;
    }
  }
  // r? has the language of eps + r.
  CS op_question(const CS& x) const { return op_union(one(), x); }

  // L |= (P, N); with allowed error, the number of misclassified
  // examples is at most the allowed fraction of |P u N|.
  bool satisfies(const CS& cs) const {
    if (err_num == 0) {
      for (int k = 0; k < W; ++k) {
        if ((cs[k] & pos_mask[k]) != pos_mask[k]) return false;
        if ((cs[k] & neg_mask[k]) != 0) return false;
      }
      return true;
    }
    long errors = 0;
    for (auto& p : P) errors += test_bit(cs, index_of.at(p)) ? 0 : 1;
    for (auto& q : N) errors += test_bit(cs, index_of.at(q)) ? 1 : 0;
    long total = (long)(P.size() + N.size());
    return errors * err_den <= err_num * total;
  }

  // ---- reconstruction ---------------------------------------
  // Printer: postfix > concat > union; concat and union are associative so
  // nested same-operator children need no parentheses.
  enum Prec { PREC_UNION = 0, PREC_CONCAT = 1, PREC_POSTFIX = 2 };

  std::string print_prov(const Prov& p, int* prec_out) const {
    switch (p.kind) {
      case K_EMPTY: *prec_out = PREC_POSTFIX; return "empty";
      case K_EPS: *prec_out = PREC_POSTFIX; return "eps";
      case K_SYM: *prec_out = PREC_POSTFIX; return std::string(1, alphabet[p.L]);
      case K_QUESTION:
      case K_STAR: {
        int cp;
        const Prov& child = levels.at(p.L)[p.i].prov;
        std::string s = print_prov(child, &cp);
        // a postfix operator binds to one atom: parenthesise anything but a symbol
        if (child.kind != K_SYM) s = "(" + s + ")";
        *prec_out = PREC_POSTFIX;
        return s + (p.kind == K_QUESTION ? "?" : "*");
      }
      case K_CONCAT: {
        int cl, cr;
        std::string l = print_prov(levels.at(p.L)[p.i].prov, &cl);
        std::string r = print_prov(levels.at(p.R)[p.j].prov, &cr);
        if (cl < PREC_CONCAT) l = "(" + l + ")";
        if (cr < PREC_CONCAT) r = "(" + r + ")";
        *prec_out = PREC_CONCAT;
        return l + r;
      }
      case K_UNION: {
        int cl, cr;
        std::string l = print_prov(levels.at(p.L)[p.i].prov, &cl);
        std::string r = print_prov(levels.at(p.R)[p.j].prov, &cr);
        *prec_out = PREC_UNION;
        return l + "+" + r;
      }
    }
    return "?";
  }
  std::string print(const Prov& p) const { int pr; return print_prov(p, &pr); }

  // ---- Algorithm 1 --------------------------------------------
  uint64_t cand_level = 0;
  std::deque<Entry>* cur = nullptr;
  bool found = false;
  Prov found_prov{};
  bool oom = false;
  uint64_t n_entries = 0;

  // OnTheFly: once the cache is full, a level is only checked --
  // candidates are neither deduplicated nor cached (reading B3: the whole level that
  // overflowed is re-run this way).  checking = true while such a level runs.
  bool onthefly = false;
  bool checking = false;
  int otf_level = 0;  // first level not cached (0 = none)

  // One candidate: Alg. 2 lines 15-20.  Every candidate is
  // counted (reading A9) and tested (reading A11).
  void emit(const CS& cs, const Prov& prov) {
    ++cand_level;
    if (!found) ++candidates;
    bool sat = satisfies(cs);
    if (sat && !found) { found = true; found_prov = prov; }
    if (checking) return;
    if (seen.count(cs)) return;
    if (max_entries && n_entries >= max_entries) { oom = true; return; }
    seen.insert(cs);
    cur->push_back({cs, prov});
    ++n_entries;
  }

  // Level `cost` needs a level that OnTheFly did not cache?
  bool needs_uncached(int cost) {
    if (!otf_level) return false;
    const int c1 = c[0], c2 = c[1], c3 = c[2], c4 = c[3], c5 = c[4];
    auto unk = [&](int L) { return L >= otf_level; };
    auto maybe = [&](int L) { return L >= c1 && (unk(L) || has_level(L)); };
    if (unk(cost - c2) || unk(cost - c3)) return true;
    for (int L = c1; L <= cost - c4 - c1; ++L) {
      int R = cost - c4 - L;
      if ((unk(L) && maybe(R)) || (unk(R) && maybe(L))) return true;
    }
    for (int L = c1; L <= cost - c5 - L; ++L) {
      int R = cost - c5 - L;
      if ((unk(L) && maybe(R)) || (unk(R) && maybe(L))) return true;
    }
    return false;
  }

  bool has_level(int cost) const {
    auto it = levels.find(cost);
    return it != levels.end() && !it->second.empty();
  }

  int solve(int max_cost) {
    auto t0 = std::chrono::steady_clock::now();
    levels.clear(); seen.clear(); stats.clear();
    candidates = 0; cand_complete = 0; found = false; oom = false; n_entries = 0;
    checking = false; otf_level = 0;
    last_complete_cost = 0; regex.clear(); result_cost = 0;
    auto done = [&](int st) {
      status = st;
      seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      return st;
    };
    const int c1 = c[0], c2 = c[1], c3 = c[2], c4 = c[3], c5 = c[4];

    // Alg.1 line 1: the empty regex is the first candidate (reading A9).
    candidates = 1;
    {
      CS z = zero_cs();
      bool sat_empty = P.empty() || (err_num != 0 && satisfies(z));
      if (sat_empty) { regex = "empty"; result_cost = c1; return done(0); }
    }
    // Alg.1 line 2.
    if (P.size() == 1 && P[0].empty()) { regex = "eps"; result_cost = c1; return done(0); }

    // Alg.1 line 3: level c1 = CSs of the alphabet symbols, deduplicated and
    // tested (readings A2, A3).
    cur = &levels[c1];
    cand_level = 0;
    for (size_t a = 0; a < alphabet.size(); ++a) {
      CS cs = zero_cs();
      auto it = index_of.find(std::string(1, alphabet[a]));
      if (it != index_of.end()) set_bit(cs, it->second);
      emit(cs, Prov{K_SYM, (int)a, 0, 0, 0});
      if (found) break;
    }
    if (found) {
      regex = print(found_prov); result_cost = c1;
      stats.push_back({c1, 0, 0, 0, 0, (uint64_t)cur->size(), 0});
      return done(0);
    }
    stats.push_back({c1, 0, 0, 0, 0, (uint64_t)cur->size(), 1});
    cand_complete = candidates;
    last_complete_cost = c1;

    // Alg.1 lines 4-9.
    otf_level = 0;
    checking = false;
    for (int cost = c1 + 1; cost <= max_cost; ++cost) {
     if (needs_uncached(cost)) return done(3);  // OnTheFly ran out of cached operands
     const uint64_t cand_before = candidates, entries_before = n_entries;
     for (int attempt = 0; attempt < 2; ++attempt) {
      std::deque<Entry> fresh;
      cur = &fresh;
      LevelStat st{cost, 0, 0, 0, 0, 0, 0};
      bool stop_emitting = false;
      auto stop = [&]() { return (found && !complete_final_level) || oom; };

      // buildQuestionMark(c - cost(?))
      if (has_level(cost - c2)) {
        cand_level = 0;
        auto& A = levels[cost - c2];
        for (size_t i = 0; i < A.size() && !stop(); ++i)
          emit(op_question(A[i].cs), Prov{K_QUESTION, cost - c2, (uint32_t)i, 0, 0});
        st.cand_q = cand_level;
      }
      // buildStar(c - cost(*))
      if (!stop() && has_level(cost - c3)) {
        cand_level = 0;
        auto& A = levels[cost - c3];
        for (size_t i = 0; i < A.size() && !stop(); ++i)
          emit(op_star(A[i].cs), Prov{K_STAR, cost - c3, (uint32_t)i, 0, 0});
        st.cand_s = cand_level;
      }
      // buildConcat(c - cost(.)) -- Algorithm 2: all (L, R) with L + R = c - c4,
      // all lCS in level L, all rCS in level R (ordered pairs, reading A7).
      cand_level = 0;
      for (int L = c1; L <= cost - c4 - c1 && !stop(); ++L) {
        int R = cost - c4 - L;
        if (!has_level(L) || !has_level(R)) continue;
        auto& A = levels[L];
        auto& B = levels[R];
        for (size_t i = 0; i < A.size() && !stop(); ++i)
          for (size_t j = 0; j < B.size() && !stop(); ++j)
            emit(op_concat(A[i].cs, B[j].cs), Prov{K_CONCAT, L, (uint32_t)i, R, (uint32_t)j});
      }
      st.cand_c = cand_level;
      // buildUnion(c - cost(+)) -- unordered pairs L <= R, i < j when L = R (A8).
      cand_level = 0;
      for (int L = c1; L <= cost - c5 - L && !stop(); ++L) {
        int R = cost - c5 - L;
        if (!has_level(L) || !has_level(R)) continue;
        auto& A = levels[L];
        auto& B = levels[R];
        for (size_t i = 0; i < A.size() && !stop(); ++i)
          for (size_t j = (L == R ? i + 1 : 0); j < B.size() && !stop(); ++j)
            emit(op_union(A[i].cs, B[j].cs), Prov{K_UNION, L, (uint32_t)i, R, (uint32_t)j});
      }
      st.cand_u = cand_level;
      (void)stop_emitting;

      if (oom && onthefly && !checking) {
        // the cache is full: forget this level's entries and check it on the fly
        for (auto& e : fresh) seen.erase(e.cs);
        n_entries = entries_before;
        candidates = cand_before;
        found = false;
        oom = false;
        checking = true;
        otf_level = cost;
        continue;
      }
      st.unique = checking ? 0 : fresh.size();
      bool complete = !oom && (!found || complete_final_level);
      st.complete = complete ? (checking ? 2 : 1) : 0;
      if (st.cand_q + st.cand_s + st.cand_c + st.cand_u > 0 || !fresh.empty() || checking)
        stats.push_back(st);
      if (!checking) levels[cost] = std::move(fresh);  // Alg.1 line 9
      if (found) {
        regex = print(found_prov);
        result_cost = cost;
        if (complete) { last_complete_cost = cost; }
        return done(0);
      }
      if (oom) return done(3);
      cand_complete = candidates;
      last_complete_cost = cost;
      if (std::getenv("ORACLE_PROGRESS") && (st.cand_q + st.cand_s + st.cand_c + st.cand_u))
        std::fprintf(stderr, "[oracle] level %d unique %llu cand %llu entries %llu %.1f s\n", cost,
                     (unsigned long long)st.unique,
                     (unsigned long long)(st.cand_q + st.cand_s + st.cand_c + st.cand_u),
                     (unsigned long long)n_entries,
                     std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
      break;
     }
    }
    return done(2);
  }

  // ---- the ABI's view (8-word CSs in and out) -------------------------------
  static CS from8(const uint64_t* a) {
    CS x = zero_cs();
    for (int k = 0; k < W; ++k) x[k] = a ? a[k] : 0;
    return x;
  }
  static void to8(const CS& x, uint64_t* out) {
    for (int k = 0; k < kMaxWords; ++k) out[k] = k < W ? x[k] : 0;
  }
  const std::string& ic_word(int k) const override { return ic.at(k); }
  const std::vector<std::pair<int, int>>& gt_row(int w) const override { return gt.at(w); }
  void masks8(uint64_t* pos8, uint64_t* neg8) const override {
    to8(pos_mask, pos8);
    to8(neg_mask, neg8);
  }
  // op 0 union, 1 concat, 2 star(a), 3 question(a), 4 satisfies(a) (out[0] = 0/1)
  void op8(int op, const uint64_t* a, const uint64_t* b, uint64_t* out) const override {
    CS x = from8(a), y = from8(b), r = zero_cs();
    switch (op) {
      case 0: r = op_union(x, y); break;
      case 1: r = op_concat(x, y); break;
      case 2: r = op_star(x); break;
      case 3: r = op_question(x); break;
      case 4: r[0] = satisfies(x) ? 1 : 0; break;
    }
    to8(r, out);
  }
  int run(int max_cost, long en, long ed, bool cfl, uint64_t me, bool otf_mode) override {
    err_num = en;
    err_den = ed > 0 ? ed : 1;
    complete_final_level = cfl;
    max_entries = me;
    onthefly = otf_mode;
    return solve(max_cost);
  }
  int otf() const override { return otf_level; }
  void result6(long long* out6, double* secs) const override {
    out6[0] = result_cost;
    out6[1] = status;
    out6[2] = (long long)candidates;
    out6[3] = (long long)cand_complete;
    out6[4] = last_complete_cost;
    out6[5] = (long long)n_entries;
    *secs = seconds;
  }
  const std::string& regex_text() const override { return regex; }
  const std::vector<LevelStat>& level_stats() const override { return stats; }
  long level_size(int cost) const override {
    auto it = levels.find(cost);
    return it == levels.end() ? 0 : (long)it->second.size();
  }
  long level_cs8(int cost, uint64_t* out, long cap) const override {
    auto it = levels.find(cost);
    if (it == levels.end()) return 0;
    long m = (long)it->second.size();
    for (long i = 0; i < m && i < cap; ++i) to8(it->second[i].cs, out + i * kMaxWords);
    return m;
  }
  std::string entry_regex(int cost, long i) const override {
    return print(levels.at(cost).at(i).prov);
  }
};

template <int W>
Search* make_oracle(const char* alphabet, const char* const* P, int nP, const char* const* N,
                    int nN, const int* costs5, std::string* err, int* n_out) {
  auto* o = new Oracle<W>();
  o->alphabet = alphabet;
  for (int i = 0; i < nP; ++i) o->P.push_back(P[i]);
  for (int i = 0; i < nN; ++i) o->N.push_back(N[i]);
  for (int k = 0; k < 5; ++k) o->c[k] = costs5[k];
  if (!o->validate()) {
    *err = o->err;
    delete o;
    return nullptr;
  }
  // build_ic sets bits of the masks: it needs |IC| <= 64 W (checked first).
  {
    std::vector<std::string> all;
    for (auto* S : {&o->P, &o->N})
      for (auto& w : *S)
        for (size_t i = 0; i <= w.size(); ++i)
          for (size_t j = i; j <= w.size(); ++j) all.push_back(w.substr(i, j - i));
    std::sort(all.begin(), all.end());
    all.erase(std::unique(all.begin(), all.end()), all.end());
    *n_out = (int)all.size();
    if (*n_out > 64 * W) {
      delete o;
      return nullptr;
    }
  }
  o->build_ic();
  return o;
}

}  // namespace

// ============================ C ABI for ctypes ================================
extern "C" {

// The CS width W is the smallest of 1, 2, 4, 8 words holding |IC| bits.
void* orc_create(const char* alphabet, const char* const* P, int nP, const char* const* N,
                 int nN, const int* costs5, char* errbuf, int errlen) {
  std::string err;
  int n = 0;
  Search* o = make_oracle<8>(alphabet, P, nP, N, nN, costs5, &err, &n);
  if (o && n <= 64 * 4) {
    delete o;
    if (n <= 64) o = make_oracle<1>(alphabet, P, nP, N, nN, costs5, &err, &n);
    else if (n <= 128) o = make_oracle<2>(alphabet, P, nP, N, nN, costs5, &err, &n);
    else o = make_oracle<4>(alphabet, P, nP, N, nN, costs5, &err, &n);
  }
  if (!o && err.empty()) err = "|IC| > 512";
  if (!o && errbuf && errlen > 0) {
    strncpy(errbuf, err.c_str(), errlen - 1);
    errbuf[errlen - 1] = 0;
  }
  return o;
}

void orc_destroy(void* h) { delete static_cast<Search*>(h); }

int orc_n(void* h) { return static_cast<Search*>(h)->n(); }

// Copies IC word k into buf (NUL-terminated); returns its length.
int orc_ic_word(void* h, int k, char* buf, int buflen) {
  const std::string& w = static_cast<Search*>(h)->ic_word(k);
  int len = (int)w.size();
  if (buf && buflen > len) { memcpy(buf, w.data(), len); buf[len] = 0; }
  return len;
}

// Guide-table row of word w: writes up to cap (l, r) pairs; returns row length.
int orc_gt_row(void* h, int w, int* pairs, int cap) {
  auto& row = static_cast<Search*>(h)->gt_row(w);
  for (int k = 0; k < (int)row.size() && k < cap; ++k) {
    pairs[2 * k] = row[k].first;
    pairs[2 * k + 1] = row[k].second;
  }
  return (int)row.size();
}

void orc_masks(void* h, uint64_t* pos8, uint64_t* neg8) {
  static_cast<Search*>(h)->masks8(pos8, neg8);
}

// CS operations on 8-word CSs: op 0 union, 1 concat, 2 star(a), 3 question(a),
// 4 satisfies(a) (out[0] = 0/1).
void orc_op(void* h, int op, const uint64_t* a, const uint64_t* b, uint64_t* out) {
  static_cast<Search*>(h)->op8(op, a, b, out);
}

int orc_solve(void* h, int max_cost, long err_num, long err_den, int complete_final_level,
              unsigned long long max_entries, int onthefly) {
  return static_cast<Search*>(h)->run(max_cost, err_num, err_den, complete_final_level != 0,
                                      max_entries, onthefly != 0);
}

int orc_otf_level(void* h) { return static_cast<Search*>(h)->otf(); }

// result: cost, status, candidates (through found), cand_complete, last_complete_cost, entries
void orc_result(void* h, long long* out6, double* seconds) {
  static_cast<Search*>(h)->result6(out6, seconds);
}

int orc_regex(void* h, char* buf, int buflen) {
  const std::string& r = static_cast<Search*>(h)->regex_text();
  int len = (int)r.size();
  if (buf && buflen > len) { memcpy(buf, r.data(), len); buf[len] = 0; }
  return len;
}

int orc_num_stats(void* h) { return (int)static_cast<Search*>(h)->level_stats().size(); }

// stat k: cost, cand_q, cand_s, cand_c, cand_u, unique, complete
void orc_stat(void* h, int k, unsigned long long* out7) {
  auto& s = static_cast<Search*>(h)->level_stats().at(k);
  out7[0] = s.cost; out7[1] = s.cand_q; out7[2] = s.cand_s; out7[3] = s.cand_c;
  out7[4] = s.cand_u; out7[5] = s.unique; out7[6] = s.complete;
}

// Number of cached entries at cost level c (0 if none).
long orc_level_size(void* h, int cost) { return static_cast<Search*>(h)->level_size(cost); }

// Copies the CSs of level c (8 words each) into out (cap entries).
long orc_level_cs(void* h, int cost, uint64_t* out, long cap) {
  return static_cast<Search*>(h)->level_cs8(cost, out, cap);
}

// Regex of cached entry i at level c (reconstruction audit).
int orc_entry_regex(void* h, int cost, long i, char* buf, int buflen) {
  std::string s = static_cast<Search*>(h)->entry_regex(cost, i);
  int len = (int)s.size();
  if (buf && buflen > len) { memcpy(buf, s.data(), len); buf[len] = 0; }
  return len;
}

}  // extern "C"
