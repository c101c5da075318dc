// Kernel JIT: fused-task IR -> sm_100a CUDA C++ (hand-written templates) -> NVRTC.
//
// Input is the slot-form program of paper_2406_18109_b200/ir.py (KProg.wire),
// i.e. the reference's optimized Kernel (diffusekit kernels.py:134-151) with
// names resolved.  One generated __global__ per loop nest.  Semantics follow
// interpret() (kernels.py:717-784):
//   * every SetTemp lives in registers; a fused window's temporaries never
//     touch HBM (their stores were demoted to locals and scalarised by the
//     front end, kernels.py:519-615);
//   * operands are numpy-broadcast to the nest domain (the domain buffer's
//     extents, kernels.py:750) -- rank-0 loads become uniform registers;
//   * element pairs along the innermost dimension move as 16-byte
//     LDG.E.128/STG.E.128 when the view is 16-byte aligned, else as two 8-byte
//     accesses (the +-1 views of the stencil);
//   * no FMA contraction: every + - * / is __d{add,sub,mul,div}_rn and NVRTC
//     runs with --fmad=false, so a fused (s*x)+y rounds like numpy's two ufuncs;
//   * min/max propagate NaN and return the second operand on ties like
//     np.minimum/np.maximum; neg flips the sign bit (np.negative);
//     comparisons give 1.0/0.0 and select tests != 0 (kernels.py:645-679);
//   * ReduceStmt: per-thread register accumulator -> warp shuffle tree ->
//     fixed-order block tree -> per-CTA partial -> the last CTA (ticket)
//     folds the partials in a fixed order and performs buf[()] += total in
//     statement order (kernels.py:765).  A scalar-valued expression adds
//     value * volume, like np.sum on a 0-d value does not.
// Grids: a streaming nest launches one CTA per chunk of 256 x unroll element
// pairs (the hardware CTA scheduler then sweeps HBM in order; persistent
// grid-stride CTAs drift apart and lose 15-25 %); a reducing nest keeps a
// bounded grid (one partial per CTA); a TMA-staged nest runs persistent CTAs
// that take tiles from an atomic queue.
// Loads hoisted ahead of the pair's stores are legal because the host rejects
// bindings where a written view overlaps another view of the same store
// (the fusion constraints already exclude that for fused windows,
// fusion.py:72-122).

#include <nvrtc.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <fstream>
#include <functional>
#include <set>
#include <sstream>

#include "dk_internal.h"

namespace dk {

// ---------------------------------------------------------------- IR -----

struct Expr {
  char tag = 0;  // L P C V B N Q
  int i = 0;
  std::string op;
  uint64_t bits = 0;
  std::vector<int64_t> offs;
  std::vector<Expr> k;
};

struct Stmt {
  char tag = 0;  // T S A
  int target = 0;
  std::vector<int64_t> offs;
  Expr e;
};

struct NestIR {
  int dom = 0;
  int decl_rank = 0;
  std::vector<Stmt> stmts;
};

struct Prog {
  int nslots = 0, nscal = 0, ntemps = 0;
  std::vector<char> local;
  std::vector<std::string> priv;
  std::vector<NestIR> nests;
  int nreduce = 0;
};

class Parser {
 public:
  explicit Parser(const std::string& s) {
    std::string cur;
    for (char c : s) {
      if (c == '(' || c == ')') {
        if (!cur.empty()) toks_.push_back(cur), cur.clear();
        toks_.push_back(std::string(1, c));
      } else if (isspace((unsigned char)c)) {
        if (!cur.empty()) toks_.push_back(cur), cur.clear();
      } else {
        cur += c;
      }
    }
    if (!cur.empty()) toks_.push_back(cur);
  }
  std::string next() {
    if (pos_ >= toks_.size()) fail(DK_ERR_ARG, "kernel program: unexpected end");
    return toks_[pos_++];
  }
  void expect(const char* t) {
    std::string x = next();
    if (x != t) fail(DK_ERR_ARG, "kernel program: expected '%s', got '%s'", t, x.c_str());
  }
  int64_t integer() {
    std::string x = next();
    char* end = nullptr;
    long long v = strtoll(x.c_str(), &end, 10);
    if (!end || *end) fail(DK_ERR_ARG, "kernel program: bad integer '%s'", x.c_str());
    return v;
  }
  std::vector<int64_t> offsets() {
    std::string x = next();
    std::vector<int64_t> o;
    if (x == "-") return o;
    std::stringstream ss(x);
    std::string part;
    while (std::getline(ss, part, ',')) o.push_back(strtoll(part.c_str(), nullptr, 10));
    return o;
  }
  Expr expr() {
    expect("(");
    Expr e;
    std::string t = next();
    if (t.size() != 1) fail(DK_ERR_ARG, "kernel program: bad expression tag '%s'", t.c_str());
    e.tag = t[0];
    switch (e.tag) {
      case 'L':
        e.i = (int)integer();
        e.offs = offsets();
        break;
      case 'P':
      case 'V':
        e.i = (int)integer();
        break;
      case 'C':
        e.bits = strtoull(next().c_str(), nullptr, 16);
        break;
      case 'B':
        e.op = next();
        e.k.push_back(expr());
        e.k.push_back(expr());
        break;
      case 'N':
        e.k.push_back(expr());
        break;
      case 'Q':
        e.k.push_back(expr());
        e.k.push_back(expr());
        e.k.push_back(expr());
        break;
      default:
        fail(DK_ERR_ARG, "kernel program: unknown expression tag '%c'", e.tag);
    }
    expect(")");
    return e;
  }

 private:
  std::vector<std::string> toks_;
  size_t pos_ = 0;
};

static Prog parse_prog(const std::string& text) {
  Parser p(text);
  p.expect("DK1");
  Prog g;
  g.nslots = (int)p.integer();
  g.nscal = (int)p.integer();
  g.ntemps = (int)p.integer();
  int nn = (int)p.integer();
  for (int i = 0; i < g.nslots; ++i) {
    p.expect("slot");
    if (p.integer() != i) fail(DK_ERR_ARG, "kernel program: slots out of order");
    p.integer();  // declared rank (actual ranks come from the bound views)
    std::string kind = p.next();
    g.local.push_back(kind == "L");
    g.priv.push_back(p.next());
  }
  for (int n = 0; n < nn; ++n) {
    p.expect("nest");
    NestIR ne;
    ne.dom = (int)p.integer();
    ne.decl_rank = (int)p.integer();
    int ns = (int)p.integer();
    for (int s = 0; s < ns; ++s) {
      Stmt st;
      std::string t = p.next();
      st.tag = t[0];
      if (st.tag == 'T') {
        st.target = (int)p.integer();
        st.e = p.expr();
      } else if (st.tag == 'S') {
        st.target = (int)p.integer();
        st.offs = p.offsets();
        st.e = p.expr();
      } else if (st.tag == 'A') {
        st.target = (int)p.integer();
        st.e = p.expr();
        g.nreduce++;
      } else {
        fail(DK_ERR_ARG, "kernel program: unknown statement '%s'", t.c_str());
      }
      ne.stmts.push_back(std::move(st));
    }
    g.nests.push_back(std::move(ne));
  }
  p.expect("end");
  for (auto& ne : g.nests)
    if (ne.dom < 0 || ne.dom >= g.nslots) fail(DK_ERR_ARG, "kernel program: bad domain slot");
  return g;
}

// ------------------------------------------------------- binding spec -----

// Parameter blocks.  Must match the device-side declarations in kPrelude.
struct DkHdr {
  int64_t ext[4];
  int64_t nrows, ninner, nelem;
  uint64_t red_part, red_ticket, red_totals;
  int64_t red_mode;
};
struct DkSite {
  uint64_t p;
  int64_t st[3];
  int64_t sti;
  int64_t mode;  // 0 pair-aligned contiguous, 1 contiguous, 2 broadcast, 3 strided
};
// peer publish of a point's totals (last reducing nest of a dk_launch_pub launch)
struct DkPub {
  uint64_t src;      // this point's totals block (local board)
  uint64_t dst[8];   // the same block in every rank's board
  uint64_t flag[8];  // the point's flag in every rank's board
  int64_t n, nred;   // ranks to publish to (0: no publish), doubles per block
  int64_t tag;       // flag value: the reduction epoch's tag (never 0)
};
// union region of a register-swept K3 nest
struct DkUni {
  uint64_t base;
  int64_t rs, cols, rows;
};
static_assert(sizeof(DkHdr) == 8 * 11, "DkHdr layout");
static_assert(sizeof(DkPub) == 8 * 20, "DkPub layout");
static_assert(sizeof(DkSite) == 48, "DkSite layout");
static_assert(sizeof(dk_view) == 80, "dk_view layout");

struct Site {
  int slot;
  std::vector<int64_t> offs;  // empty = zero offsets
  char cls;                   // S scalar, A aligned contiguous, C contiguous inner, B broadcast inner, G strided inner
  int par = -1;               // contiguous with even row strides: element parity of the view origin
  bool staged = false;        // read through the CTA's TMA-staged tile (K3)
  int dr = 0, dc = 0;         // element offset of this view within the staged tile
};

// K3: aliased views of one store (the stencil's shifted interior views) are
// staged tile by tile in shared memory by TMA and read from there; each
// persistent CTA takes TR x TC output tiles from an atomic queue (in order
// across the GPU) through an S-stage mbarrier ring, refilled by a producer
// warp (full/empty barriers) while 8 consumer warps compute.
// output rows per tile (DK_K3_TR: 8, 12 or 16; thread t owns rows (t >> 6) + 4u)
static int k_tr() {
  static int v = [] {
    const char* e = getenv("DK_K3_TR");
    int t = e ? atoi(e) : 8;
    return t >= 16 ? 16 : t >= 12 ? 12 : 8;
  }();
  return v;
}
#define kTR (k_tr())
static const int kTC = 128;   // output columns per tile (64 element pairs)
static const int kBW = 136;   // TMA box width (tile + column halo + alignment), 1088 B per row
// TMA ring depth: S-1 boxes in flight per CTA (DK_K3_STAGES, 2..4)
static int kStages() {
  static int s = [] {
    const char* e = getenv("DK_K3_STAGES");
    int v = e ? atoi(e) : 3;
    return std::min(4, std::max(2, v));
  }();
  return s;
}

// K3 register sweep (DK_K3S=1, opt-in): instead of TMA tiles, each thread
// walks a column of element pairs down a block of kSweepRows() rows, keeping
// the stencil's row window in registers and the next kSweepAhead() rows in
// flight.  Measured slower than the TMA ring for the 32768^2 stencil window
// (3.42-3.48 ms vs 3.01 ms on the same box for RB 32..256, PF 2..6, 3..5
// CTAs/SM), so the TMA path stays the default.
static int kSweepRows() {
  static int v = [] {
    const char* e = getenv("DK_K3S_RB");
    return std::min(1024, std::max(8, e ? atoi(e) : 64));
  }();
  return v;
}
static int kSweepAhead() {
  static int v = [] {
    const char* e = getenv("DK_K3S_PF");
    return std::min(8, std::max(1, e ? atoi(e) : 3));
  }();
  return v;
}

// grid of a reducing nest: red_waves() x (SMs x resident CTAs) CTAs, one
// partial per CTA (DK_JIT_RWAVES)
static int red_waves() {
  static int w = [] {
    const char* e = getenv("DK_JIT_RWAVES");
    return std::min(64, std::max(1, e ? atoi(e) : 4));  // CG windows: 4-8 best, 1 = +2 %
  }();
  return w;
}

struct NestPlan {
  int rank = 0;  // actual domain rank
  int shift = 0;  // 1: element pairs start at column -1 (aligns the odd-parity views)
  bool st_queue = false;  // K3 tiles handed out by an atomic queue (else cyclic by CTA)
  bool oneshot = false;  // one CTA per chunk of pairs (no persistent grid-stride loop)
  bool staged = false;
  int st_rows = 0;         // box rows = kTR + max dr
  int st_sh = 0;           // column shift that 16-byte aligns the tensor base
  int st_anchor = -1;      // site whose view origin is the group's minimum address
  int st_min_dc = 0;
  uint64_t st_base = 0;    // tensor base address (aligned)
  int64_t st_cols = 0, st_nrows = 0, st_rowstride = 0;
  std::vector<Site> sites;
  std::vector<char> site_loaded;   // site read before any store to its slot (phase-1 load)
  std::vector<int> red_slots;      // target slot per reduce statement (statement order)
  std::vector<char> red_is_array;  // per reduce statement
  int n_array_red = 0;
  bool st_ws = false;  // K3 with a producer warp (full/empty mbarriers, no CTA barrier per tile)
  bool sweep = false;  // K3 as a register sweep (no TMA): see nest_sweep
  int sw_np = 1;       // union element pairs per row per thread
  int st_maxdr = 0;
};

static bool nonzero(const std::vector<int64_t>& o) {
  for (auto v : o)
    if (v) return true;
  return false;
}

static void walk_loads(const Expr& e, const std::function<void(const Expr&)>& f) {
  if (e.tag == 'L') f(e);
  for (auto& c : e.k) walk_loads(c, f);
}

// per-dim strides of a view broadcast against the domain shape (numpy rules)
static bool bcast_strides(const dk_view& v, const int64_t* D, int r, int64_t* out) {
  if (v.rank > r) {
    for (int d = 0; d < v.rank - r; ++d)
      if (v.ext[d] != 1) return false;
  }
  for (int j = 0; j < r; ++j) {
    int jj = j - (r - v.rank);
    if (jj < 0) {
      out[j] = 0;
    } else if (v.ext[jj] == D[j]) {
      out[j] = v.stride[jj];  // extent-1 dims keep their (irrelevant) stride: innermost stays contiguous
    } else if (v.ext[jj] == 1) {
      out[j] = 0;
    } else {
      return false;
    }
  }
  return true;
}

// Decide whether a rank-2 nest reads >= 3 views of one store at small constant
// offsets (read-only in the whole kernel): those views are served from one TMA
// tile per CTA instead of 3-5 overlapping global streams.
static void plan_staging(NestPlan& np, const dk_view* views, const int64_t* D, int r, const std::set<int>& kstored) {
  if (r != 2 || D[0] < kTR || D[1] < 64 || getenv("DK_JIT_NO_K3")) return;
  std::vector<int> cand;
  for (size_t i = 0; i < np.sites.size(); ++i) {
    const Site& s = np.sites[i];
    if (!np.site_loaded[i] || !s.offs.empty() || (s.cls != 'A' && s.cls != 'C') || kstored.count(s.slot)) continue;
    const dk_view& v = views[s.slot];
    if (v.rank != 2 || v.ext[0] != D[0] || v.ext[1] != D[1] || v.stride[1] != 1) continue;
    cand.push_back((int)i);
  }
  // group by row stride; take the largest group
  std::map<int64_t, std::vector<int>> by;
  for (int i : cand) by[views[np.sites[i].slot].stride[0]].push_back(i);
  std::vector<int> best;
  int64_t rs = 0;
  for (auto& kv : by)
    if (kv.second.size() > best.size()) best = kv.second, rs = kv.first;
  if (best.size() < 3 || (rs * 8) % 16 != 0 || rs <= 16) return;
  uint64_t anchor = ~0ull;
  int anchor_i = -1;
  for (int i : best)
    if (views[np.sites[i].slot].ptr < anchor) anchor = views[np.sites[i].slot].ptr, anchor_i = i;
  std::vector<int> grp;
  int min_dc = 0, max_dc = 0, max_dr = 0;
  for (int i : best) {
    int64_t d = (int64_t)(views[np.sites[i].slot].ptr - anchor);
    if (d % 8) continue;
    d /= 8;
    int64_t dr = (d + 8) / rs, dc = d - dr * rs;
    if (dr > 4 || dc < -8 || dc > 8) continue;
    np.sites[i].dr = (int)dr;
    np.sites[i].dc = (int)dc;
    grp.push_back(i);
  }
  if (grp.size() < 3) return;
  for (int i : grp) {
    min_dc = std::min(min_dc, np.sites[i].dc);
    max_dc = std::max(max_dc, np.sites[i].dc);
    max_dr = std::max(max_dr, np.sites[i].dr);
  }
  uint64_t base = anchor + 8ull * (uint64_t)(int64_t)min_dc;  // min_dc <= 0
  int sh = (int)((base % 16) / 8);
  base -= 8ull * sh;
  if (max_dc - min_dc + sh + kTC > kBW) return;
  if (D[1] + (max_dc - min_dc) + sh > rs) return;  // the union must not wrap across rows
  np.staged = true;
  np.st_rows = kTR + max_dr;
  np.st_maxdr = max_dr;
  np.st_sh = sh;
  np.st_anchor = anchor_i;
  np.st_min_dc = min_dc;
  np.st_base = base;
  np.st_cols = D[1] + (max_dc - min_dc) + sh;
  np.st_nrows = D[0] + max_dr;
  np.st_rowstride = rs;
  for (int i : grp) np.sites[i].staged = true;
}

static std::vector<NestPlan> plan_nests(const Prog& g, const dk_view* views, std::string* key) {
  std::vector<NestPlan> plans;
  std::ostringstream ks;
  std::set<int> kstored;  // slots stored anywhere in the kernel
  for (const NestIR& ne : g.nests)
    for (const Stmt& s : ne.stmts)
      if (s.tag == 'S') kstored.insert(s.target);
  for (size_t n = 0; n < g.nests.size(); ++n) {
    const NestIR& ne = g.nests[n];
    const dk_view& dv = views[ne.dom];
    NestPlan np;
    np.rank = dv.rank;
    const int r = dv.rank;
    int64_t D[4] = {1, 1, 1, 1};
    for (int d = 0; d < r; ++d) D[d] = dv.ext[d];
    std::set<int> stored;
    std::vector<char> temp_array(g.ntemps, 0);
    std::function<bool(const Expr&)> is_array = [&](const Expr& e) -> bool {
      if (e.tag == 'L') return views[e.i].rank > 0;
      if (e.tag == 'V') return e.i < (int)temp_array.size() && temp_array[e.i];
      for (auto& c : e.k)
        if (is_array(c)) return true;
      return false;
    };
    auto site_of = [&](int slot, const std::vector<int64_t>& offs) -> int {
      std::vector<int64_t> o = nonzero(offs) ? offs : std::vector<int64_t>();
      for (size_t i = 0; i < np.sites.size(); ++i)
        if (np.sites[i].slot == slot && np.sites[i].offs == o) return (int)i;
      Site s;
      s.slot = slot;
      s.offs = o;
      const dk_view& v = views[slot];
      if (v.dtype != DK_F64) fail(DK_ERR_UNSUPPORTED, "kernel access to a non-f64 store (slot %d)", slot);
      if (v.rank == 0) {
        s.cls = 'S';
      } else {
        int64_t str[4];
        if (!bcast_strides(v, D, r, str))
          fail(DK_ERR_UNSUPPORTED, "operands could not be broadcast together (slot %d rank %d vs domain rank %d)",
               slot, v.rank, r);
        int64_t inner = r ? str[r - 1] : 0;
        s.cls = inner == 1 ? 'C' : inner == 0 ? 'B' : 'G';
        if (s.cls == 'C') {
          // 'A': every row's element pairs are 16-byte aligned -> LDG.E.128 / STG.E.128
          int64_t shift = 0;
          for (size_t d = 0; d < o.size(); ++d) shift += o[d] * v.stride[d];
          const uint64_t a = v.ptr + 8ull * (uint64_t)shift;
          bool even = a % 8 == 0;
          for (int d = 0; d + 1 < r; ++d)
            if (str[d] % 2) even = false;
          if (even) s.par = (int)((a / 8) % 2);
          if (s.par == 0) s.cls = 'A';
        }
      }
      if (!o.empty()) {
        if ((int)o.size() != r || v.rank != r)
          fail(DK_ERR_UNSUPPORTED, "offset access with mismatched ranks (slot %d)", slot);
        for (int d = 0; d < r; ++d)
          if (D[d] > 0 && (o[d] < 0 || o[d] + D[d] > v.ext[d]))
            fail(DK_ERR_BOUNDS, "access at offset %lld outside buffer slot %d extent %lld", (long long)o[d], slot,
                 (long long)v.ext[d]);
      }
      np.sites.push_back(s);
      return (int)np.sites.size() - 1;
    };
    for (const Stmt& stt : ne.stmts) {
      walk_loads(stt.e, [&](const Expr& ld) {
        if (ld.i < 0 || ld.i >= g.nslots) fail(DK_ERR_ARG, "load of bad slot");
        if (stored.count(ld.i) && nonzero(ld.offs))
          fail(DK_ERR_UNSUPPORTED, "offset load of a buffer written in the same nest");
        for (int rs : np.red_slots)
          if (rs == ld.i) fail(DK_ERR_UNSUPPORTED, "nest reads a buffer it reduces into");
        if (!stored.count(ld.i)) {
          int si = site_of(ld.i, ld.offs);
          if ((int)np.site_loaded.size() <= si) np.site_loaded.resize(si + 1, 0);
          np.site_loaded[si] = 1;
        }
      });
      if (stt.tag == 'T') {
        if (stt.target >= g.ntemps) fail(DK_ERR_ARG, "bad temp index");
        temp_array[stt.target] = is_array(stt.e);
      } else if (stt.tag == 'S') {
        const std::string& pv = g.priv[stt.target];
        if (!g.local[stt.target] && pv != "W" && pv != "RW")
          fail(DK_ERR_PRIVILEGE, "store to read-only param (slot %d)", stt.target);
        if (nonzero(stt.offs)) fail(DK_ERR_UNSUPPORTED, "store with non-zero offsets");
        const dk_view& tv = views[stt.target];
        if (tv.rank != r) fail(DK_ERR_UNSUPPORTED, "store target rank %d differs from nest rank %d", tv.rank, r);
        for (int d = 0; d < r; ++d)
          if (tv.ext[d] != D[d]) fail(DK_ERR_UNSUPPORTED, "store target extents differ from the nest domain");
        if (r > 0 && !is_array(stt.e)) {
          // broadcast scalar value: still a plain pair store
        }
        stored.insert(stt.target);
        int si = site_of(stt.target, {});
        if (np.sites[si].cls == 'B') fail(DK_ERR_UNSUPPORTED, "store into a broadcast view");
      } else {
        const std::string& pv = g.priv[stt.target];
        if (!g.local[stt.target] && pv != "W" && pv != "RW" && pv != "Rd")
          fail(DK_ERR_PRIVILEGE, "reduce into read-only param (slot %d)", stt.target);
        if (views[stt.target].dtype != DK_F64) fail(DK_ERR_UNSUPPORTED, "reduce into non-f64 view");
        bool arr = is_array(stt.e);
        if (arr && r == 0) fail(DK_ERR_UNSUPPORTED, "array-valued reduction in a rank-0 nest");
        np.red_slots.push_back(stt.target);
        np.red_is_array.push_back(arr);
        if (arr) np.n_array_red++;
        for (int sl : stored)
          if (sl == stt.target) fail(DK_ERR_UNSUPPORTED, "reduce into a buffer stored in the same nest");
      }
    }
    np.site_loaded.resize(np.sites.size(), 0);
    for (const Site& s : np.sites) {
      if (r == 0 && s.cls != 'S') fail(DK_ERR_UNSUPPORTED, "rank-0 nest over an array operand");
    }
    plan_staging(np, views, D, r, kstored);
    if (np.staged && getenv("DK_K3S")) {
      int maxcol = 0;
      for (const Site& st : np.sites)
        if (st.staged) maxcol = std::max(maxcol, st.dc - np.st_min_dc + np.st_sh);
      if (maxcol <= 4) {
        np.sweep = true;
        np.sw_np = (maxcol + 1) / 2 + 1;
      }
    }
    if (!np.staged && r > 0 && !getenv("DK_JIT_NO_SHIFT")) {
      // pick the pair grid (start column 0 or -1) that 16-byte aligns the most
      // operands; the others move as shuffled pairs ('H')
      int score[2] = {0, 0};
      for (size_t i = 0; i < np.sites.size(); ++i) {
        const Site& st = np.sites[i];
        if (st.par < 0) continue;
        score[st.par] += (np.site_loaded[i] ? 1 : 0) + (st.offs.empty() && stored.count(st.slot) ? 1 : 0);
      }
      if (score[1] > score[0]) np.shift = 1;
      // 'H' (shuffled odd-parity pairs) is opt-in: measured slower than split
      // 8-byte accesses for the stencil COPY (3.39 vs 3.22 ms)
      const bool useH = getenv("DK_JIT_H") != nullptr;
      for (Site& st : np.sites)
        if (st.cls == 'A' || st.cls == 'C') st.cls = st.par < 0 ? 'C' : st.par == np.shift ? 'A' : useH ? 'H' : 'C';
    }
    np.oneshot = !np.staged && r > 0 && !getenv("DK_JIT_PERSIST");
    ks << "n" << n << ":r" << r << ":h" << np.shift << (np.oneshot ? "o" : "") << ":";
    // queue: stencil window 2.82 ms vs 3.20 ms with a cyclic tile walk (DK_K3_CYCLIC)
    np.st_queue = np.staged && getenv("DK_K3_CYCLIC") == nullptr;
    const bool k3pref = getenv("DK_K3_NOPREF") == nullptr;
    // producer warp: stencil window 2.72 ms vs 2.85-2.88 ms with thread 0
    // refilling between CTA barriers (same box; DK_K3_NOWS=1 restores that)
    np.st_ws = np.st_queue && getenv("DK_K3_NOWS") == nullptr;
    if (np.sweep) np.st_queue = false;
    if (np.staged) ks << "K3:" << np.st_rows << "," << np.st_sh << "," << np.st_min_dc << (np.st_queue ? (k3pref ? "qp" : "q") : "") << (np.st_ws ? "w" : "") << ";";
    if (np.sweep) ks << "K3S:" << np.sw_np << "," << kSweepRows() << "," << kSweepAhead() << ";";
    for (const Site& s : np.sites) {
      if (s.staged) ks << "s" << s.dr << "," << s.dc;
      ks << s.slot << s.cls;
      for (auto o : s.offs) ks << "," << o;
      ks << ";";
    }
    for (size_t k = 0; k < np.red_slots.size(); ++k) ks << "R" << np.red_slots[k] << (np.red_is_array[k] ? "a" : "s");
    ks << "|";
    plans.push_back(std::move(np));
  }
  *key = ks.str();
  return plans;
}

// ------------------------------------------------------------ codegen -----

static const char* kPrelude = R"DK(
typedef long long int64_t;
typedef unsigned long long uint64_t;
typedef int int32_t;
typedef unsigned int uint32_t;
struct dk_view { uint64_t ptr; int32_t rank; int32_t dtype; int64_t ext[4]; int64_t stride[4]; };
struct DkHdr { int64_t ext[4]; int64_t nrows, ninner, nelem; uint64_t red_part, red_ticket, red_totals; int64_t red_mode; };
struct DkSite { uint64_t p; int64_t st[3]; int64_t sti; int64_t mode; };
struct DkPub { uint64_t src; uint64_t dst[8]; uint64_t flag[8]; int64_t n, nred, tag; };
struct DkUni { uint64_t base; int64_t rs, cols, rows; };
// element pair q of row r of a K3 union region (16-byte aligned base, even row stride)
__device__ __forceinline__ double2 dk_ldu(const DkUni& u, int64_t r, int64_t q) {
  double2 v; v.x = 0.0; v.y = 0.0;
  if (r < u.rows) {
    const double* p = (const double*)u.base + r * u.rs + 2 * q;
    if (2 * q + 1 < u.cols) v = __ldg(reinterpret_cast<const double2*>(p));
    else if (2 * q < u.cols) v.x = __ldg(p);
  }
  return v;
}

__device__ __forceinline__ double dk_add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dk_sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dk_mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dk_div(double a, double b) { return __ddiv_rn(a, b); }
// ---- '**' (np.power, kernels.py:650) --------------------------------------
// np.power is libm pow (or SVML on AVX-512 hosts: the two differ by 1 ulp on
// ~5 % of random inputs, so the reference itself is host-dependent).  CUDA's
// pow is within 2 ulp.  dk_pow evaluates y*log(x) and exp() in double-double
// (~2^-100 relative) and rounds once, so its result is the correctly rounded
// x**y except for subnormal results -- exact whenever x**y is representable
// (integer data) and within 1 ulp of either host implementation otherwise.
// Special values follow C99 pow, as numpy does.
struct dk_dd { double h, l; };
__device__ __forceinline__ dk_dd dk_dd_fast(double a, double b) { double s = a + b; return {s, b - (s - a)}; }
__device__ __forceinline__ dk_dd dk_dd_sum(double a, double b) {
  double s = a + b, bb = s - a;
  return {s, (a - (s - bb)) + (b - bb)};
}
__device__ __forceinline__ dk_dd dk_dd_add(dk_dd a, dk_dd b) {
  dk_dd s = dk_dd_sum(a.h, b.h), t = dk_dd_sum(a.l, b.l);
  s.l = s.l + t.h;
  s = dk_dd_fast(s.h, s.l);
  s.l = s.l + t.l;
  return dk_dd_fast(s.h, s.l);
}
__device__ __forceinline__ dk_dd dk_dd_mul(dk_dd a, dk_dd b) {
  double p = a.h * b.h;
  double e = __fma_rn(a.h, b.h, -p);
  e = e + (a.h * b.l + a.l * b.h);
  return dk_dd_fast(p, e);
}
__device__ __forceinline__ dk_dd dk_dd_muld(dk_dd a, double b) {
  double p = a.h * b;
  if (!isfinite(p)) return {p, 0.0};
  double e = __fma_rn(a.h, b, -p) + a.l * b;
  return dk_dd_fast(p, e);
}
__device__ __forceinline__ dk_dd dk_dd_div(dk_dd a, dk_dd b) {
  double q1 = a.h / b.h;
  dk_dd r = dk_dd_add(a, dk_dd_muld(b, -q1));
  double q2 = r.h / b.h;
  r = dk_dd_add(r, dk_dd_muld(b, -q2));
  double q3 = r.h / b.h;
  return dk_dd_add(dk_dd_fast(q1, q2), dk_dd{q3, 0.0});
}
__device__ __forceinline__ dk_dd dk_dd_ln2() { return {__longlong_as_double(0x3FE62E42FEFA39EFll), __longlong_as_double(0x3C7ABC9E3B39803Fll)}; }
// log(x), x > 0 finite: e*ln2 + 2*atanh((m-1)/(m+1)), m in [sqrt(1/2), sqrt(2))
static __device__ __noinline__ dk_dd dk_dd_log(double x) {
  int e;
  double m = frexp(x, &e);
  if (m < 0.70710678118654752) { m = m * 2.0; e -= 1; }
  dk_dd s = dk_dd_div(dk_dd{m - 1.0, 0.0}, dk_dd_sum(m, 1.0));  // m - 1 is exact (Sterbenz)
  dk_dd s2 = dk_dd_mul(s, s);                                      // <= 0.0295
  dk_dd p = {1.0 / 51.0, 0.0};
  for (int k = 24; k >= 0; --k) {
    dk_dd c = k < 12 ? dk_dd_div(dk_dd{1.0, 0.0}, dk_dd{2.0 * k + 1.0, 0.0}) : dk_dd{1.0 / (2.0 * k + 1.0), 0.0};
    p = dk_dd_add(dk_dd_mul(p, s2), c);
  }
  dk_dd lm = dk_dd_mul(s, p);
  lm.h = lm.h * 2.0;
  lm.l = lm.l * 2.0;
  return dk_dd_add(dk_dd_muld(dk_dd_ln2(), (double)e), lm);
}
// exp(z) rounded once to double
static __device__ __noinline__ double dk_dd_exp(dk_dd z) {
  if (z.h != z.h) return z.h;
  if (z.h > 709.9) return __longlong_as_double(0x7FF0000000000000ll);
  if (z.h < -745.3) return 0.0;
  double kf = rint(z.h * 1.4426950408889634);
  dk_dd r = dk_dd_add(z, dk_dd_muld(dk_dd_ln2(), -kf));  // |r| <= 0.35
  r.h = ldexp(r.h, -10);
  r.l = ldexp(r.l, -10);                                  // |r| < 3.5e-4
  // e^r - 1 = r (1 + r/2 (1 + r/3 (1 + ... )))
  dk_dd q = {1.0, 0.0};
  for (int n = 11; n >= 2; --n) q = dk_dd_add(dk_dd{1.0, 0.0}, dk_dd_div(dk_dd_mul(r, q), dk_dd{(double)n, 0.0}));
  dk_dd em1 = dk_dd_mul(r, q);
  for (int i = 0; i < 10; ++i) em1 = dk_dd_mul(em1, dk_dd_add(dk_dd{2.0, 0.0}, em1));  // (1+u)^2 - 1
  dk_dd v = dk_dd_add(dk_dd{1.0, 0.0}, em1);
  int k = (int)kf;
  if (k > 1023) { v.h = v.h * 2.0; v.l = v.l * 2.0; k -= 1; }
  if (k >= -1021) return ldexp(v.h, k);
  // subnormal result: round v * 2^k once on the 2^-1074 grid (scaled so the grid
  // step is 1; both scalings are exact)
  const double hs = ldexp(v.h, k + 1074), ls = ldexp(v.l, k + 1074);
  if (hs >= 4503599627370496.0) return ldexp(v.h, k);  // >= 2^-1022: normal after all
  double g = rint(hs);
  const double d = (hs - g) + ls;
  if (d > 0.5 || (d == 0.5 && fmod(g, 2.0) != 0.0)) g = g + 1.0;
  else if (d < -0.5 || (d == -0.5 && fmod(g, 2.0) != 0.0)) g = g - 1.0;
  return ldexp(g, -1074);
}
static __device__ __noinline__ double dk_pow(double x, double y) {
  const double inf = __longlong_as_double(0x7FF0000000000000ll);
  if (y == 0.0) return 1.0;
  if (x == 1.0) return 1.0;
  if (x != x || y != y) return x + y;
  const double ax = fabs(x);
  if (isinf(y)) {
    if (ax == 1.0) return 1.0;
    return ((ax < 1.0) == (y < 0.0)) ? inf : 0.0;
  }
  const bool yint = floor(y) == y;
  const bool yodd = yint && fabs(y) < 9007199254740992.0 && fmod(y, 2.0) != 0.0;
  if (x == 0.0) {
    if (y < 0.0) return yodd ? copysign(inf, x) : inf;
    return yodd ? x : 0.0;
  }
  if (isinf(x)) {
    if (x > 0.0) return y < 0.0 ? 0.0 : inf;
    if (y < 0.0) return yodd ? -0.0 : 0.0;
    return yodd ? -inf : inf;
  }
  if (x < 0.0 && !yint) return __longlong_as_double(0x7FF8000000000000ll);
  const double r = dk_dd_exp(dk_dd_muld(dk_dd_log(ax), y));
  return (x < 0.0 && yodd) ? -r : r;
}
__device__ __forceinline__ bool dk_isnan(double a) { return a != a; }
__device__ __forceinline__ double dk_min(double a, double b) { return dk_isnan(a) ? a : (a < b ? a : b); }
__device__ __forceinline__ double dk_max(double a, double b) { return dk_isnan(a) ? a : (a > b ? a : b); }
__device__ __forceinline__ double dk_lt(double a, double b) { return a < b ? 1.0 : 0.0; }
__device__ __forceinline__ double dk_le(double a, double b) { return a <= b ? 1.0 : 0.0; }
__device__ __forceinline__ double dk_eq(double a, double b) { return a == b ? 1.0 : 0.0; }
// np.negative flips the sign bit, NaN payload included.  Plain C (-a or an
// integer xor) is turned into DADD -RZ, -a by ptxas, which canonicalises NaN;
// an opaque PTX xor on the high word keeps the bit pattern.
__device__ __forceinline__ double dk_neg(double a) {
  double r;
  asm("{ .reg .b32 lo, hi; mov.b64 {lo, hi}, %1; xor.b32 hi, hi, 0x80000000; mov.b64 %0, {lo, hi}; }"
               : "=d"(r) : "d"(a));
  return r;
}
__device__ __forceinline__ double dk_bits(unsigned long long b) { return __longlong_as_double((long long)b); }

// element-pair access, specialised per site class at code generation time:
//   A aligned contiguous (one 16-byte access), C contiguous (two 8-byte),
//   B broadcast inner dim (one load), G strided inner dim.
// lo / hi: the pair's first / second element lies inside the row (a nest whose
// pair grid is shifted by one element to align its stores has a half first pair)
__device__ __forceinline__ double2 dk_ld_A(const double* p, int64_t e, bool lo, bool hi) {
  if (lo && hi) return *reinterpret_cast<const double2*>(p + e);
  double2 v; v.x = lo ? p[e] : 0.0; v.y = hi ? p[e + 1] : 0.0; return v;
}
__device__ __forceinline__ double2 dk_ld_C(const double* p, int64_t e, bool lo, bool hi) {
  double2 v; v.x = lo ? p[e] : 0.0; v.y = hi ? p[e + 1] : 0.0; return v;
}
__device__ __forceinline__ double2 dk_ld_B(const double* p, int64_t, bool, bool) {
  double2 v; v.x = p[0]; v.y = v.x; return v;
}
__device__ __forceinline__ double2 dk_ld_G(const double* p, int64_t e, bool lo, bool hi, int64_t s) {
  double2 v; v.x = lo ? p[e * s] : 0.0; v.y = hi ? p[(e + 1) * s] : 0.0; return v;
}
__device__ __forceinline__ void dk_st_A(double* p, int64_t e, bool lo, bool hi, double x, double y) {
  if (lo && hi) { double2 v; v.x = x; v.y = y; *reinterpret_cast<double2*>(p + e) = v; return; }
  if (lo) p[e] = x;
  if (hi) p[e + 1] = y;
}
__device__ __forceinline__ double2 dk_ld_Acs(const double* p, int64_t e, bool lo, bool hi) {
  if (lo && hi) return __ldcs(reinterpret_cast<const double2*>(p + e));
  double2 v; v.x = lo ? __ldcs(p + e) : 0.0; v.y = hi ? __ldcs(p + e + 1) : 0.0; return v;
}
__device__ __forceinline__ void dk_st_Acs(double* p, int64_t e, bool lo, bool hi, double x, double y) {
  if (lo && hi) { double2 v; v.x = x; v.y = y; __stcs(reinterpret_cast<double2*>(p + e), v); return; }
  if (lo) __stcs(p + e, x);
  if (hi) __stcs(p + e + 1, y);
}
__device__ __forceinline__ void dk_st_C(double* p, int64_t e, bool lo, bool hi, double x, double y) {
  if (lo) p[e] = x;
  if (hi) p[e + 1] = y;
}
__device__ __forceinline__ void dk_st_G(double* p, int64_t e, bool lo, bool hi, double x, double y, int64_t s) {
  if (lo) p[e * s] = x;
  if (hi) p[(e + 1) * s] = y;
}

// ---- K3: TMA tile staging (cp.async.bulk.tensor + mbarrier) ----
__device__ __forceinline__ uint32_t dk_smem(const void* p) {
  uint64_t a;
  asm("cvta.to.shared.u64 %0, %1;" : "=l"(a) : "l"(p));
  return (uint32_t)a;
}
__device__ __forceinline__ void dk_mbar_init(uint32_t bar, uint32_t cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(bar), "r"(cnt) : "memory");
}
__device__ __forceinline__ void dk_fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void dk_fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void dk_tma_2d(const void* tmap, uint32_t bar, uint32_t dst, int c0, int c1, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(bar), "r"(bytes) : "memory");
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      :: "r"(dst), "l"(tmap), "r"(c0), "r"(c1), "r"(bar) : "memory");
}
__device__ __forceinline__ void dk_mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(bar) : "memory");
}
__device__ __forceinline__ void dk_mbar_wait(uint32_t bar, uint32_t ph) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(ok) : "r"(bar), "r"(ph) : "memory");
}

__device__ __forceinline__ double dk_warp_sum(double v) {
  for (int o = 16; o; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// grid-wide barrier between the nests of a one-launch multi-nest window (cooperative
// launch: every CTA is resident).  bar[0] arrivals, bar[1] generation.
__device__ __forceinline__ void dk_grid_sync(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    unsigned gen;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(gen) : "l"(bar + 1) : "memory");
    __threadfence();
    if (atomicAdd(bar, 1u) == gridDim.x * gridDim.y - 1) {
      bar[0] = 0u;
      __threadfence();
      asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(bar + 1), "r"(gen + 1u) : "memory");
    } else {
      unsigned g = gen;
      while (g == gen) {
        __nanosleep(64);
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(bar + 1) : "memory");
      }
    }
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ double dk_ldcg(const double* p) {
  double v;
  asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

__device__ __forceinline__ void dk_view_add(const dk_view& t, double v) {
  int64_t n = 1;
  for (int d = 0; d < t.rank; ++d) n *= t.ext[d];
  double* p = (double*)t.ptr;
  for (int64_t i = 0; i < n; ++i) {
    int64_t o = 0, rem = i;
    for (int d = t.rank - 1; d >= 0; --d) { o += (rem % t.ext[d]) * t.stride[d]; rem /= t.ext[d]; }
    p[o] = __dadd_rn(p[o], v);
  }
}
)DK";

static const int kTPB = 256;

// Streaming fused nests are latency-bound unless enough bytes are in flight:
// ~1.5 us of HBM latency x 6.5 TB/s needs ~64 KB outstanding per SM.  The
// default asks ptxas for 6 (few operands) or 4 resident 256-thread CTAs per SM
// with 2 element pairs per thread in flight per operand; modules that would
// spill at that budget are regenerated with 4, 3, 2 and then 1 CTA per SM.
struct GenOpts {
  int unroll = 2;
  int min_blocks = 4;
  bool stream_hint = false;  // evict-first (.cs) loads/stores for aligned streaming operands
  bool merged = false;       // all nests in one cooperative launch, grid barriers between them
};

static GenOpts default_opts(const std::vector<NestPlan>& plans) {
  GenOpts o;
  // many-operand nests (the stencil's five views) keep one pair per operand in
  // flight; their bytes in flight per thread are already 5 x 16 B
  size_t most = 0;
  bool staged = false, all_aligned = true;
  for (const NestPlan& np : plans) {
    size_t n = 0;
    for (size_t i = 0; i < np.sites.size(); ++i) {
      n += np.sites[i].cls != 'S' && np.site_loaded[i];
      all_aligned &= np.sites[i].cls == 'S' || np.sites[i].cls == 'A';
    }
    most = std::max(most, n);
    staged |= np.staged;
  }
  const bool persist = getenv("DK_JIT_PERSIST") != nullptr;
  if (persist) {
    // persistent grid-stride CTAs (the round-1 default): same-box sweeps gave
    // 3 CTAs/SM for the TMA-staged stencil window, 4 for nests with an
    // odd-offset operand, 6 for fully aligned few-operand nests
    o.unroll = most <= 3 ? 2 : 1;
    o.min_blocks = staged ? 3 : (most <= 3 && all_aligned ? 6 : 4);
  } else {
    // one CTA per chunk (see NestPlan::oneshot).  Same-box sweeps (U x CTAs/SM):
    // BS window (2 operands) 3.40 ms at U=4 vs 3.45 at U=2 and 4.33 at U=8;
    // stencil COPY 2.47 ms at 6 CTAs/SM vs 2.71 at 4; the staged window keeps 3
    o.unroll = most <= 2 ? 4 : (most <= 3 ? 2 : 1);
    o.min_blocks = staged ? 3 : 6;
  }
  bool sweep = false;
  for (const NestPlan& np : plans) sweep |= np.sweep;
  if (sweep) o.min_blocks = 4;
  if (const char* u = getenv("DK_JIT_UNROLL")) o.unroll = std::max(1, atoi(u));
  if (const char* m = getenv("DK_JIT_MINB")) o.min_blocks = std::max(1, atoi(m));
  if (const char* c = getenv("DK_JIT_CS")) o.stream_hint = atoi(c) != 0;
  return o;
}

class Gen {
 public:
  Gen(const Prog& g, const std::vector<NestPlan>& plans, const std::string& name = "dk", GenOpts opts = GenOpts(),
      std::vector<int> scalar_rep = {})
      : g_(g), plans_(plans), name_(name), kUnroll(opts.unroll), minb_(opts.min_blocks), cs_(opts.stream_hint),
        merged_(opts.merged), opts_rep_(std::move(scalar_rep)) {}

  std::string source() {
    std::ostringstream o;
    o << kPrelude;
    const int NN = (int)g_.nests.size();
    for (int n = 0; n < NN; ++n) {
      if (merged_) o << "#define threadIdx dk_tid\n#define blockDim dk_bdim\n";
      nest(o, n);
      if (merged_) o << "#undef threadIdx\n#undef blockDim\n";
    }
    if (merged_) {
      // one launch for the whole window: each nest's body runs over the same
      // 256-thread CTAs (its own TX x TY view of them), a grid barrier between nests
      o << "\nstruct PM { uint64_t gbar; unsigned tx[" << (NN + 1) / 2 * 2 << "];";
      for (int n = 0; n < NN; ++n) o << " P" << n << " p" << n << ";";
      o << " };\n";
      o << "extern \"C\" __global__ void __launch_bounds__(" << kTPB << ", " << minb_ << ") " << name_
        << "_m(const __grid_constant__ PM P) {\n";
      for (int n = 0; n < NN; ++n) {
        if (n) o << "  dk_grid_sync((unsigned*)P.gbar);\n";
        o << "  " << name_ << "_n" << n << "(P.p" << n << ", make_uint3(threadIdx.x % P.tx[" << n << "], threadIdx.x / P.tx["
          << n << "], 0), dim3(P.tx[" << n << "], " << kTPB << " / P.tx[" << n << "], 1));\n";
      }
      o << "}\n";
    }
    return o.str();
  }

 private:
  const Prog& g_;
  const std::vector<NestPlan>& plans_;
  std::string name_;
  int kUnroll;
  int minb_;
  bool cs_;
  bool merged_;
  std::vector<int> opts_rep_;

  int site_index(const NestPlan& np, int slot, const std::vector<int64_t>& offs) const {
    std::vector<int64_t> o = nonzero(offs) ? offs : std::vector<int64_t>();
    for (size_t i = 0; i < np.sites.size(); ++i)
      if (np.sites[i].slot == slot && np.sites[i].offs == o) return (int)i;
    fail(DK_ERR_STATE, "internal: no site for slot %d", slot);
  }

  static const char* binfn(const std::string& op) {
    if (op == "+") return "dk_add";
    if (op == "-") return "dk_sub";
    if (op == "*") return "dk_mul";
    if (op == "/") return "dk_div";
    if (op == "**") return "dk_pow";
    if (op == "min") return "dk_min";
    if (op == "max") return "dk_max";
    if (op == "lt") return "dk_lt";
    if (op == "le") return "dk_le";
    if (op == "eq") return "dk_eq";
    fail(DK_ERR_ARG, "unknown binary op '%s'", op.c_str());
  }

  // lane: "x" / "y" for element pair lanes, "s" for scalar (epilogue / rank-0)
  std::string expr(const NestPlan& np, const Expr& e, const std::string& lane, const std::set<int>& stored) const {
    char buf[64];
    switch (e.tag) {
      case 'L': {
        if (stored.count(e.i)) return "w" + std::to_string(e.i) + "_" + lane;
        int si = site_index(np, e.i, e.offs);
        const Site& s = np.sites[si];
        if (s.cls == 'S') return "S" + std::to_string(si);
        if (s.cls == 'B' || lane == "s") return "v" + std::to_string(si) + "[u].x";
        return "v" + std::to_string(si) + "[u]." + lane;
      }
      case 'P':
        // scalars equal to an earlier one (bitwise) read that one: ptxas keeps one
        // register per distinct value instead of one per task scalar
        return "P.sc[" + std::to_string(e.i < (int)opts_rep_.size() ? opts_rep_[e.i] : e.i) + "]";
      case 'C':
        snprintf(buf, sizeof buf, "dk_bits(0x%016llxULL)", (unsigned long long)e.bits);
        return buf;
      case 'V':
        return "t" + std::to_string(e.i) + "_" + lane;
      case 'B':
        return std::string(binfn(e.op)) + "(" + expr(np, e.k[0], lane, stored) + ", " + expr(np, e.k[1], lane, stored) + ")";
      case 'N':
        return "dk_neg(" + expr(np, e.k[0], lane, stored) + ")";
      case 'Q':
        return "((" + expr(np, e.k[0], lane, stored) + ") != 0.0 ? (" + expr(np, e.k[1], lane, stored) + ") : (" +
               expr(np, e.k[2], lane, stored) + "))";
    }
    fail(DK_ERR_ARG, "bad expression");
  }

  // K3: persistent CTAs walk kTR x kTC output tiles through an S-stage ring.
  // Default: a producer warp takes tickets from the queue and keeps S-1 TMA
  // boxes in flight; 256 consumer threads compute from shared memory and
  // release each stage per warp.  Without the producer warp (DK_K3_NOWS /
  // DK_K3_CYCLIC) thread 0 refills between CTA barriers.  Consumer t owns the
  // element pair (t & 63) of rows (t >> 6) + 4u of the tile.
  void nest_staged(std::ostringstream& o, int n, const std::vector<int>& wslots) const {
    const NestIR& ne = g_.nests[n];
    const NestPlan& np = plans_[n];
    const int NS = (int)np.sites.size();
    const int NR = (int)np.red_slots.size();
    const int ROWS = np.st_rows;
    const unsigned bytes = (unsigned)(ROWS * kBW * 8);
    for (int a = 0; a < np.n_array_red; ++a) o << "  double racc" << a << " = 0.0;\n";
    // S-stage ring; an even row count per stage keeps every stage on a 128-byte
    // boundary (TMA destination alignment)
    // static shared memory stays within 48 KB: fewer stages for taller boxes
    int S = kStages();
    while (S > 2 && S * ((ROWS + 1) / 2 * 2) * kBW * 8 > 48 * 1024) --S;
    o << "  __shared__ __align__(128) double dk_tile[" << S << "][" << (ROWS + 1) / 2 * 2 << "][" << kBW << "];\n";
    o << "  __shared__ __align__(8) unsigned long long dk_bar[" << S << "];\n";
    o << "  const int tid = threadIdx.x;\n";
    o << "  const int64_t D0 = P.h.ext[0], D1 = P.h.ext[1];\n";
    o << "  const int64_t ntc = (D1 + " << kTC - 1 << ") / " << kTC << ", ntr = (D0 + " << kTR - 1 << ") / " << kTR
      << ", ntiles = ntr * ntc;\n";
    // tile order: row-major (DK_K3_COLMAJOR=1 walks column strips; measured equal time)
    const bool colmaj = getenv("DK_K3_COLMAJOR") != nullptr;
    auto trow = [&](const char* t) { return colmaj ? std::string("(") + t + " % ntr)" : std::string("(") + t + " / ntc)"; };
    auto tcol = [&](const char* t) { return colmaj ? std::string("(") + t + " / ntr)" : std::string("(") + t + " % ntc)"; };
    o << "  if (tid == 0) {\n    for (int s = 0; s < " << S << "; ++s) dk_mbar_init(dk_smem(&dk_bar[s]), 1);\n";
    o << "    dk_fence_mbar_init();\n  }\n  __syncthreads();\n";
    const std::string tma_args_pre = "dk_tma_2d(&P.tm, ";
    auto tma = [&](const std::string& bar, const std::string& dst, const char* t) {
      return tma_args_pre + bar + ", " + dst + ", (int)(" + tcol(t) + " * " + std::to_string(kTC) + "), (int)(" + trow(t) +
             " * " + std::to_string(kTR) + "), " + std::to_string(bytes) + "u);";
    };
    o << "  const int pr = tid & 63, rg = tid >> 6;\n";
    if (np.st_ws) {
      // warp-specialised ring: warp 8 (one lane) takes tickets and issues the
      // TMA refills as soon as the 8 consumer warps have released a stage
      // (empty barrier, one arrive per warp); consumers only wait on the full
      // barrier of their stage -- no CTA-wide barrier per tile
      o << "  __shared__ __align__(8) unsigned long long dk_empty[" << S << "];\n";
      o << "  __shared__ long long dk_tid[" << S << "];\n";
      o << "  unsigned int* const dk_q = (unsigned int*)P.h.red_ticket + 2;\n";
      o << "  if (tid == 0) {\n    for (int s = 0; s < " << S << "; ++s) dk_mbar_init(dk_smem(&dk_empty[s]), 8);\n";
      o << "    dk_fence_mbar_init();\n  }\n  __syncthreads();\n";
      o << "  if (tid >= " << kTPB << ") {\n    if (tid == " << kTPB << ") {\n";
      o << "      long long pend = (long long)atomicAdd(dk_q, 1u);\n";
      o << "      for (int it = 0;; ++it) {\n        const int s = it % " << S << ";\n";
      o << "        if (it >= " << S << ") dk_mbar_wait(dk_smem(&dk_empty[s]), (uint32_t)(((it / " << S << ") - 1) & 1));\n";
      o << "        const long long t = pend; dk_tid[s] = t;\n        dk_fence_proxy_async();\n";
      o << "        if (t >= ntiles) { dk_mbar_arrive(dk_smem(&dk_bar[s])); break; }\n";
      o << "        " << tma("dk_smem(&dk_bar[s])", "dk_smem(&dk_tile[s][0][0])", "t") << "\n";
      o << "        pend = (long long)atomicAdd(dk_q, 1u);\n      }\n    }\n  } else\n";
      o << "  for (int it = 0;; ++it) {\n";
      o << "    const int stg = it % " << S << ";\n    const uint32_t ph = (uint32_t)((it / " << S << ") & 1);\n";
      o << "    dk_mbar_wait(dk_smem(&dk_bar[stg]), ph);\n";
      o << "    const int64_t tile = dk_tid[stg];\n    if (tile >= ntiles) break;\n";
    } else if (np.st_queue) {
      // dynamic tile queue: tiles are handed out in order by an atomic ticket
      // (red_ticket[2]); the CTA's thread 0 publishes each stage's tile index
      // before its TMA (or a plain arrive once the queue is empty)
      o << "  __shared__ long long dk_tid[" << S << "];\n";
      o << "  unsigned int* const dk_q = (unsigned int*)P.h.red_ticket + 2;\n";
      // the ticket for the next refill is requested one iteration early
      // (DK_K3_NOPREF=1 disables): its atomic round trip overlaps the current
      // tile instead of holding every thread at the closing barrier.  Tickets
      // grow per CTA, so the one left unused at exit is past the last tile.
      const bool pref = getenv("DK_K3_NOPREF") == nullptr;
      o << "  long long dk_pend = 0;\n";
      o << "  if (tid == 0) {\n    for (int s = 0; s < " << S - 1 << "; ++s) {\n";
      o << "      const long long t = (long long)atomicAdd(dk_q, 1u); dk_tid[s] = t;\n";
      o << "      if (t < ntiles) " << tma("dk_smem(&dk_bar[s])", "dk_smem(&dk_tile[s][0][0])", "t")
        << " else dk_mbar_arrive(dk_smem(&dk_bar[s]));\n    }\n";
      if (pref) o << "    dk_pend = (long long)atomicAdd(dk_q, 1u);\n";
      o << "  }\n";
      o << "  for (int it = 0;; ++it) {\n";
      o << "    const int stg = it % " << S << ";\n    const uint32_t ph = (uint32_t)((it / " << S << ") & 1);\n";
      o << "    if (tid == 0) {\n      const int ns = (it + " << S - 1 << ") % " << S << ";\n";
      if (pref)
        o << "      const long long nxt = dk_pend; dk_pend = (long long)atomicAdd(dk_q, 1u); dk_tid[ns] = nxt;\n";
      else
        o << "      const long long nxt = (long long)atomicAdd(dk_q, 1u); dk_tid[ns] = nxt;\n";
      o << "      dk_fence_proxy_async();\n";
      o << "      if (nxt < ntiles) " << tma("dk_smem(&dk_bar[ns])", "dk_smem(&dk_tile[ns][0][0])", "nxt")
        << " else dk_mbar_arrive(dk_smem(&dk_bar[ns]));\n    }\n";
      o << "    dk_mbar_wait(dk_smem(&dk_bar[stg]), ph);\n";
      o << "    const int64_t tile = dk_tid[stg];\n    if (tile >= ntiles) break;\n";
    } else {
      o << "  int64_t tile = blockIdx.x;\n";
      // prologue: S-1 tiles in flight
      o << "  if (tid == 0)\n    for (int s = 0; s < " << S - 1 << "; ++s) {\n";
      o << "      const int64_t t = tile + (int64_t)s * gridDim.x;\n      if (t >= ntiles) break;\n";
      o << "      " << tma("dk_smem(&dk_bar[s])", "dk_smem(&dk_tile[s][0][0])", "t") << "\n    }\n";
      o << "  for (int it = 0; tile < ntiles; ++it, tile += gridDim.x) {\n";
      o << "    const int stg = it % " << S << ";\n    const uint32_t ph = (uint32_t)((it / " << S << ") & 1);\n";
      o << "    const int64_t nxt = tile + (int64_t)" << S - 1 << " * gridDim.x;\n";
      // the stage refilled here was read in iteration it-1 and released by its __syncthreads
      o << "    if (tid == 0 && nxt < ntiles) {\n      const int ns = (it + " << S - 1 << ") % " << S << ";\n";
      o << "      dk_fence_proxy_async();\n";
      o << "      " << tma("dk_smem(&dk_bar[ns])", "dk_smem(&dk_tile[ns][0][0])", "nxt") << "\n    }\n";
      o << "    dk_mbar_wait(dk_smem(&dk_bar[stg]), ph);\n";
    }
    o << "    const int64_t r0 = " << trow("tile") << " * " << kTR << ", c0 = " << tcol("tile") << " * " << kTC << ";\n";
    o << "    const double (*T)[" << kBW << "] = dk_tile[stg];\n";
    for (int i = 0; i < NS; ++i)
      if (np.sites[i].cls != 'S' && np.site_loaded[i]) o << "    double2 v" << i << "[" << kTR / 4 << "];\n";
    o << "    #pragma unroll\n    for (int u = 0; u < " << kTR / 4 << "; ++u) {\n";
    o << "      const int a = rg + 4 * u;\n      const int64_t row = r0 + a, e = c0 + 2 * pr;\n";
    o << "      if (row < D0 && e < D1) {\n        const bool full = e + 1 < D1;\n";
    // DK_K3_REUSE=1: an odd-column staged view whose left and right neighbour columns
    // (same row) are staged even-column views is assembled from their registers (W.y,
    // E.x) instead of two more shared-memory loads -- the stencil's centre from its west
    // and east views; source views then always load both elements (in-bounds: the tile
    // has halo columns).  Measured neutral on B200 (2.738 vs 2.745 ms at 32768^2: the
    // window is not bound by its shared-memory loads), so it stays opt-in.
    static const bool no_reuse = getenv("DK_K3_REUSE") == nullptr;
    std::vector<std::pair<int, int>> from(NS, {-1, -1});
    std::vector<bool> is_src(NS, false);
    auto scol = [&](int i) { return np.sites[i].dc - np.st_min_dc + np.st_sh; };
    auto staged_loaded = [&](int i) { return np.sites[i].cls != 'S' && np.site_loaded[i] && np.sites[i].staged; };
    if (!no_reuse)
      for (int i = 0; i < NS; ++i) {
        if (!staged_loaded(i) || scol(i) % 2 == 0) continue;
        int l = -1, r = -1;
        for (int j = 0; j < NS; ++j) {
          if (!staged_loaded(j) || np.sites[j].dr != np.sites[i].dr) continue;
          if (scol(j) == scol(i) - 1) l = j;
          if (scol(j) == scol(i) + 1) r = j;
        }
        if (l >= 0 && r >= 0) {
          from[i] = {l, r};
          is_src[l] = is_src[r] = true;
        }
      }
    for (int i = 0; i < NS; ++i) {
      const Site& s = np.sites[i];
      if (s.cls == 'S' || !np.site_loaded[i] || from[i].first >= 0) continue;
      if (s.staged) {
        const int col = scol(i);  // tile column of element pair 0
        o << "        { const double* t = &T[a + " << s.dr << "][2 * pr + " << col << "]; ";
        if (col % 2 == 0 && is_src[i])
          o << "v" << i << "[u] = *reinterpret_cast<const double2*>(t); }\n";
        else if (col % 2 == 0)
          o << "v" << i << "[u] = full ? *reinterpret_cast<const double2*>(t) : make_double2(t[0], 0.0); }\n";
        else
          o << "v" << i << "[u].x = t[0]; v" << i << "[u].y = full ? t[1] : 0.0; }\n";
      } else {
        const char c = s.cls;
        o << "        v" << i << "[u] = dk_ld_" << c << "((double*)P.s[" << i << "].p + row * P.s[" << i
          << "].st[0], e, true, full";
        if (c == 'G') o << ", P.s[" << i << "].sti";
        o << ");\n";
      }
    }
    for (int i = 0; i < NS; ++i)
      if (from[i].first >= 0)
        o << "        v" << i << "[u].x = v" << from[i].first << "[u].y; v" << i << "[u].y = v" << from[i].second
          << "[u].x;\n";
    o << "      }\n    }\n";
    o << "    #pragma unroll\n    for (int u = 0; u < " << kTR / 4 << "; ++u) {\n";
    o << "      const int a = rg + 4 * u;\n      const int64_t row = r0 + a, e = c0 + 2 * pr;\n";
    o << "      if (row < D0 && e < D1) {\n        const bool full = e + 1 < D1;\n";
    for (int w : wslots) o << "        double w" << w << "_x = 0.0, w" << w << "_y = 0.0;\n";
    o << "        {\n" << lane_code(np, ne, "x") << "        }\n";
    o << "        if (full) {\n" << lane_code(np, ne, "y") << "        }\n";
    for (int w : wslots) {
      int si = site_index(np, w, {});
      const char c = np.sites[si].cls;
      o << "        dk_st_" << c << "((double*)P.s[" << si << "].p + row * P.s[" << si << "].st[0], e, true, full, w" << w
        << "_x, w" << w << "_y";
      if (c == 'G') o << ", P.s[" << si << "].sti";
      o << ");\n";
    }
    o << "      }\n    }\n";
    if (np.st_ws)
      o << "    __syncwarp();\n    if ((tid & 31) == 0) dk_mbar_arrive(dk_smem(&dk_empty[stg]));\n  }\n";
    else
      o << "    __syncthreads();\n  }\n";
    if (np.st_queue) {
      // the last CTA out resets the queue for the next launch (stream order)
      o << "  if (tid == 0) {\n    __threadfence();\n    if (atomicAdd(dk_q + 1, 1u) == gridDim.x - 1) { dk_q[0] = 0u; dk_q[1] = 0u; }\n  }\n";
    }
    if (NR) emit_reduce_epilogue(o, np, ne, wslots);
    o << "}\n";
  }

  // K3 as a register sweep: thread t of a CTA owns domain element pair
  // (task column chunk x 256 + t) and walks kSweepRows() rows of it; the
  // union rows r .. r + max_dr of the aliased views sit in registers (W), the
  // next kSweepAhead() union rows are already loaded (F), every union row is
  // read once per chunk with 16-byte aligned loads (the neighbouring pair comes
  // from L1: the next lane loaded it).  No shared memory, no barriers.
  void nest_sweep(std::ostringstream& o, int n, const std::vector<int>& wslots) const {
    const NestIR& ne = g_.nests[n];
    const NestPlan& np = plans_[n];
    const int NS = (int)np.sites.size();
    const int NR = (int)np.red_slots.size();
    const int NRW = np.st_maxdr + 1, NPR = np.sw_np, PF = kSweepAhead(), RB = kSweepRows();
    for (int a = 0; a < np.n_array_red; ++a) o << "  double racc" << a << " = 0.0;\n";
    o << "  const int64_t D0 = P.h.ext[0], D1 = P.h.ext[1];\n";
    o << "  const int64_t ncc = (((D1 + 1) >> 1) + 255) >> 8, nrb = (D0 + " << RB - 1 << ") / " << RB
      << ", ntask = ncc * nrb;\n";
    o << "  for (int64_t task = blockIdx.x; task < ntask; task += gridDim.x) {\n";
    o << "    const int u = 0; (void)u;\n";
    o << "    const int64_t cc = task % ncc, rb = task / ncc, pp = (cc << 8) + threadIdx.x, e = 2 * pp;\n";
    o << "    if (e >= D1) continue;\n";
    o << "    const bool full = e + 1 < D1;\n";
    o << "    const int64_t r0 = rb * " << RB << ", r1 = r0 + " << RB << " < D0 ? r0 + " << RB << " : D0;\n";
    o << "    double2 W[" << NRW << "][" << NPR << "], F[" << PF << "][" << NPR << "];\n";
    for (int k = 0; k + 1 < NRW; ++k)
      for (int c = 0; c < NPR; ++c) o << "    W[" << k << "][" << c << "] = dk_ldu(P.u, r0 + " << k << ", pp + " << c << ");\n";
    for (int j = 0; j < PF; ++j)
      for (int c = 0; c < NPR; ++c)
        o << "    F[" << j << "][" << c << "] = dk_ldu(P.u, r0 + " << NRW - 1 + j << ", pp + " << c << ");\n";
    o << "    for (int64_t row = r0; row < r1; ++row) {\n";
    for (int c = 0; c < NPR; ++c) o << "      W[" << NRW - 1 << "][" << c << "] = F[0][" << c << "];\n";
    for (int j = 0; j + 1 < PF; ++j)
      for (int c = 0; c < NPR; ++c) o << "      F[" << j << "][" << c << "] = F[" << j + 1 << "][" << c << "];\n";
    for (int c = 0; c < NPR; ++c)
      o << "      F[" << PF - 1 << "][" << c << "] = dk_ldu(P.u, row + " << NRW - 1 + PF << ", pp + " << c << ");\n";
    for (int i = 0; i < NS; ++i) {
      const Site& st = np.sites[i];
      if (st.cls == 'S' || !np.site_loaded[i]) continue;
      o << "      double2 v" << i << "[1];\n";
      if (st.staged) {
        const int col = st.dc - np.st_min_dc + np.st_sh, c2 = col / 2;
        if (col % 2 == 0)
          o << "      v" << i << "[0] = W[" << st.dr << "][" << c2 << "];\n";
        else
          o << "      v" << i << "[0].x = W[" << st.dr << "][" << c2 << "].y; v" << i << "[0].y = W[" << st.dr << "]["
            << c2 + 1 << "].x;\n";
      } else {
        const char c = st.cls;
        o << "      v" << i << "[0] = dk_ld_" << c << "((double*)P.s[" << i << "].p + row * P.s[" << i << "].st[0], e, true, full";
        if (c == 'G') o << ", P.s[" << i << "].sti";
        o << ");\n";
      }
    }
    for (int w : wslots) o << "      double w" << w << "_x = 0.0, w" << w << "_y = 0.0;\n";
    o << "      {\n" << lane_code(np, ne, "x") << "      }\n";
    o << "      if (full) {\n" << lane_code(np, ne, "y") << "      }\n";
    for (int w : wslots) {
      int si = site_index(np, w, {});
      const char c = np.sites[si].cls;
      o << "      dk_st_" << c << "((double*)P.s[" << si << "].p + row * P.s[" << si << "].st[0], e, true, full, w" << w
        << "_x, w" << w << "_y";
      if (c == 'G') o << ", P.s[" << si << "].sti";
      o << ");\n";
    }
    for (int k = 0; k + 1 < NRW; ++k)
      for (int c = 0; c < NPR; ++c) o << "      W[" << k << "][" << c << "] = W[" << k + 1 << "][" << c << "];\n";
    o << "    }\n  }\n";
    if (NR) emit_reduce_epilogue(o, np, ne, wslots);
    o << "}\n";
  }

  void nest(std::ostringstream& o, int n) const {
    const NestIR& ne = g_.nests[n];
    const NestPlan& np = plans_[n];
    const int r = np.rank;
    const int NS = (int)np.sites.size();
    const int NR = (int)np.red_slots.size();
    o << "\nstruct P" << n << " { ";
    if (np.staged && !np.sweep) o << "alignas(64) unsigned char tm[128]; ";
    o << "DkHdr h; " << (NR ? "DkPub pub; " : "") << (np.sweep ? "DkUni u; " : "") << "DkSite s[" << std::max(NS, 1) << "]; dk_view rd[" << std::max(NR, 1)
      << "]; double sc[" << std::max(g_.nscal, 1) << "]; };\n";
    if (merged_)
      o << "static __device__ void " << name_ << "_n" << n << "(const P" << n << "& P, const uint3 dk_tid, const dim3 dk_bdim) {\n";
    else
      o << "extern \"C\" __global__ void __launch_bounds__(" << (np.st_ws ? kTPB + 32 : kTPB) << ", " << minb_ << ") " << name_ << "_n" << n
        << "(const __grid_constant__ P" << n << " P) {\n";
    // hoisted rank-0 operands
    for (int i = 0; i < NS; ++i)
      if (np.sites[i].cls == 'S') o << "  const double S" << i << " = *(const double*)P.s[" << i << "].p;\n";
    // stored slots list
    std::vector<int> wslots;
    for (const Stmt& s : ne.stmts)
      if (s.tag == 'S' && std::find(wslots.begin(), wslots.end(), s.target) == wslots.end()) wslots.push_back(s.target);

    if (r == 0) {
      // a single evaluation, performed by one thread
      o << "  if (blockIdx.x != 0 || threadIdx.x != 0 || threadIdx.y != 0) return;\n";
      o << "  const int u = 0; (void)u;\n";
      for (int w : wslots) o << "  double w" << w << "_s = 0.0;\n";
      emit_scalar_seq(o, np, ne, /*apply_reduce=*/true, wslots);
      o << "}\n";
      return;
    }
    if (np.sweep) {
      nest_sweep(o, n, wslots);
      return;
    }
    if (np.staged) {
      nest_staged(o, n, wslots);
      return;
    }

    for (int a = 0; a < np.n_array_red; ++a) o << "  double racc" << a << " = 0.0;\n";
    // np.shift = 1: element pairs start one element before the row (e = 2q - 1)
    // so that the stored views' pairs are 16-byte aligned
    const int h = np.shift;
    o << "  const int64_t nrows = P.h.nrows, ninner = P.h.ninner, npairs = (ninner + " << 1 + h << ") >> 1;\n";
    o << "  const int TX = blockDim.x;\n";
    if (np.oneshot) {
      // one chunk of TX x unroll pairs (of blockDim.y rows) per CTA, grid = all
      // chunks: measured 2.48 ms vs 3.24 ms for a persistent grid-stride walk
      // over the stencil COPY's 32766 x 32766 interior (tools/gpu/copybench.cu)
      o << "  const int64_t cpr = (npairs + TX * " << kUnroll << " - 1) / (TX * " << kUnroll
        << "), nchunks = (nrows + blockDim.y - 1) / blockDim.y * cpr;\n";
      o << "  for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {\n";
      o << "    const int64_t rg = c / cpr, row = rg * blockDim.y + threadIdx.y;\n";
      o << "    if (row >= nrows) continue;\n";
    } else {
      o << "  for (int64_t row = (int64_t)blockIdx.y * blockDim.y + threadIdx.y; row < nrows; row += (int64_t)gridDim.y * blockDim.y) {\n";
    }
    // outer indices of this row
    if (r == 2) {
      o << "    const int64_t oi[1] = {row};\n";
    } else if (r > 2) {
      o << "    int64_t oi[3] = {0, 0, 0};\n";
      o << "    { int64_t rem = row;\n";
      for (int d = r - 2; d >= 0; --d) o << "      oi[" << d << "] = rem % P.h.ext[" << d << "]; rem /= P.h.ext[" << d << "];\n";
      o << "    }\n";
    }
    for (int i = 0; i < NS; ++i) {
      if (np.sites[i].cls == 'S') continue;
      o << "    double* const b" << i << " = (double*)P.s[" << i << "].p";
      for (int d = 0; d < r - 1; ++d) o << " + oi[" << d << "] * P.s[" << i << "].st[" << d << "]";
      o << ";\n";
    }
    // 'H' sites (odd element parity against the pair grid) move as aligned
    // 16-byte pairs shifted by one element, completed across lanes with a warp
    // shuffle: warps lie along the row (TX is a multiple of 32) and stay
    // converged through the pair loop (the loop bound is per warp)
    bool anyH = false;
    for (const Site& st : np.sites) anyH |= st.cls == 'H';
    o << "    const int lane = threadIdx.x & 31; (void)lane;\n";
    auto qline_of = [&](const std::string& qb) {
      return "        const int64_t q = " + qb + " + (int64_t)u * TX; const bool act = q < npairs;\n"
             "        const int64_t e = 2 * q - " + std::to_string(h) + "; const bool lo = " +
             (h ? "e >= 0" : "true") + ", hi = e + 1 < ninner;\n";
    };
    const std::string qline = qline_of("q0");
    auto emit_loads = [&](const std::string& qb, const std::string& arr, const std::string& ind) {
      o << ind << "#pragma unroll\n" << ind << "for (int u = 0; u < " << kUnroll << "; ++u) {\n" << qline_of(qb);
      o << "        if (act) {\n";
      for (int i = 0; i < NS; ++i) {
        if (np.sites[i].cls == 'S' || np.sites[i].cls == 'H' || !np.site_loaded[i]) continue;
        const char c = np.sites[i].cls;
        o << "          " << arr << i << "[u] = dk_ld_" << c << (c == 'A' && cs_ ? "cs" : "") << "(b" << i << ", e, lo, hi";
        if (c == 'G') o << ", P.s[" << i << "].sti";
        o << ");\n";
      }
      o << "        }\n";
      for (int i = 0; i < NS; ++i) {
        if (np.sites[i].cls != 'H' || !np.site_loaded[i]) continue;
        // lane L loads elements (e+1, e+2); its e comes from lane L-1, lane 0 reads it alone
        o << "        { double2 a = make_double2(0.0, 0.0);\n"
          << "          if (act && hi) { if (e + 2 < ninner) a = *reinterpret_cast<const double2*>(b" << i
          << " + e + 1); else a.x = b" << i << "[e + 1]; }\n"
          << "          double x = __shfl_up_sync(0xffffffffu, a.y, 1);\n"
          << "          if (lane == 0 && act && lo) x = b" << i << "[e];\n"
          << "          " << arr << i << "[u].x = x; " << arr << i << "[u].y = a.x; }\n";
      }
      o << ind << "}\n";
    };
    auto declare = [&](const std::string& arr, const std::string& ind) {
      for (int i = 0; i < NS; ++i)
        if (np.sites[i].cls != 'S' && np.site_loaded[i]) o << ind << "double2 " << arr << i << "[" << kUnroll << "];\n";
    };
    if (np.oneshot) {
      o << "    {\n      const int64_t q0 = (c - rg * cpr) * TX * " << kUnroll << " + threadIdx.x;\n";
    } else {
      o << "    for (int64_t q0 = (int64_t)blockIdx.x * TX * " << kUnroll << " + threadIdx.x; q0" << (anyH ? " - lane" : "")
        << " < npairs; q0 += (int64_t)gridDim.x * TX * " << kUnroll << ") {\n";
    }
    // phase 1: loads
    declare("v", "      ");
    emit_loads("q0", "v", "      ");
    // phase 2: compute + store
    o << "      #pragma unroll\n      for (int u = 0; u < " << kUnroll << "; ++u) {\n" << qline;
    for (int w : wslots) o << "        double w" << w << "_x = 0.0, w" << w << "_y = 0.0;\n";
    o << "        if (act) {\n";
    o << "        if (lo) {\n" << lane_code(np, ne, "x") << "        }\n";
    o << "        if (hi) {\n" << lane_code(np, ne, "y") << "        }\n";
    for (int w : wslots) {
      int si = site_index(np, w, {});
      const char c = np.sites[si].cls;
      if (c == 'H') continue;
      o << "        dk_st_" << c << (c == 'A' && cs_ ? "cs" : "") << "(b" << si << ", e, lo, hi, w" << w << "_x, w" << w
        << "_y";
      if (c == 'G') o << ", P.s[" << si << "].sti";
      o << ");\n";
    }
    o << "        }\n";
    for (int w : wslots) {
      int si = site_index(np, w, {});
      if (np.sites[si].cls != 'H') continue;
      // lane L stores elements (e+1, e+2) = (its y, lane L+1's x); lane 0 stores its x alone
      o << "        { const double nx = __shfl_down_sync(0xffffffffu, w" << w << "_x, 1);\n"
        << "          if (act) {\n"
        << "            if (lane == 0 && lo) b" << si << "[e] = w" << w << "_x;\n"
        << "            if (hi) { if (lane < 31 && q + 1 < npairs) { double2 t; t.x = w" << w << "_y; t.y = nx; "
        << "*reinterpret_cast<double2*>(b" << si << " + e + 1) = t; } else b" << si << "[e + 1] = w" << w << "_y; }\n"
        << "          } }\n";
    }
    o << "      }\n";
    o << "    }\n  }\n";
    if (NR) emit_reduce_epilogue(o, np, ne, wslots);
    o << "}\n";
  }

  // one lane's statement sequence; temps are block-scoped (re-definition safe)
  std::string lane_code(const NestPlan& np, const NestIR& ne, const std::string& lane) const {
    std::ostringstream o;
    std::set<int> stored;
    int k = 0, ka = 0;
    // SetTemp may redefine a temp name; give every definition a fresh C++ name
    std::vector<int> ver(g_.ntemps, 0);
    std::function<std::string(const Expr&)> ex = [&](const Expr& e) -> std::string {
      if (e.tag == 'V') return "t" + std::to_string(e.i) + "v" + std::to_string(ver[e.i]) + "_" + lane;
      if (e.tag == 'B')
        return std::string(binfn(e.op)) + "(" + ex(e.k[0]) + ", " + ex(e.k[1]) + ")";
      if (e.tag == 'N') return "dk_neg(" + ex(e.k[0]) + ")";
      if (e.tag == 'Q') return "((" + ex(e.k[0]) + ") != 0.0 ? (" + ex(e.k[1]) + ") : (" + ex(e.k[2]) + "))";
      return expr(np, e, lane, stored);
    };
    for (const Stmt& s : ne.stmts) {
      if (s.tag == 'T') {
        std::string rhs = ex(s.e);
        ver[s.target]++;
        o << "          const double t" << s.target << "v" << ver[s.target] << "_" << lane << " = " << rhs << ";\n";
      } else if (s.tag == 'S') {
        o << "          w" << s.target << "_" << lane << " = " << ex(s.e) << ";\n";
        stored.insert(s.target);
      } else {
        if (np.red_is_array[k]) {
          o << "          racc" << ka << " = dk_add(racc" << ka << ", " << ex(s.e) << ");\n";
          ka++;
        }
        k++;
      }
    }
    return o.str();
  }

  // scalar-valued statement sequence (rank-0 nest, or the epilogue's scalar reduces)
  void emit_scalar_seq(std::ostringstream& o, const NestPlan& np, const NestIR& ne, bool rank0,
                       const std::vector<int>& wslots) const {
    std::set<int> stored;
    std::vector<int> ver(g_.ntemps, 0);
    std::vector<char> tarr(g_.ntemps, 0);
    std::function<bool(const Expr&)> is_arr = [&](const Expr& e) -> bool {
      if (e.tag == 'L') {
        if (stored.count(e.i)) return false;
        return np.sites[site_index(np, e.i, e.offs)].cls != 'S';
      }
      if (e.tag == 'V') return tarr[e.i];
      for (auto& c : e.k)
        if (is_arr(c)) return true;
      return false;
    };
    std::function<std::string(const Expr&)> ex = [&](const Expr& e) -> std::string {
      if (e.tag == 'V') return "t" + std::to_string(e.i) + "v" + std::to_string(ver[e.i]) + "_s";
      if (e.tag == 'B') return std::string(binfn(e.op)) + "(" + ex(e.k[0]) + ", " + ex(e.k[1]) + ")";
      if (e.tag == 'N') return "dk_neg(" + ex(e.k[0]) + ")";
      if (e.tag == 'Q') return "((" + ex(e.k[0]) + ") != 0.0 ? (" + ex(e.k[1]) + ") : (" + ex(e.k[2]) + "))";
      return expr(np, e, "s", stored);
    };
    int k = 0, ka = 0;
    for (const Stmt& s : ne.stmts) {
      if (s.tag == 'T') {
        bool arr = is_arr(s.e);
        if (!arr) {
          std::string rhs = ex(s.e);
          ver[s.target]++;
          o << "    const double t" << s.target << "v" << ver[s.target] << "_s = " << rhs << ";\n";
        }
        tarr[s.target] = arr;
      } else if (s.tag == 'S') {
        if (rank0) {
          o << "    w" << s.target << "_s = " << ex(s.e) << ";\n";
          stored.insert(s.target);
        }
      } else {
        bool arr = np.red_is_array[k];
        o << "    {\n";
        if (arr) {
          o << "      const double tot = dk_tot[" << ka << "];\n";
          ka++;
        } else {
          o << "      const double tot = dk_mul(" << ex(s.e) << ", (double)P.h.nelem);\n";
        }
        o << "      if (P.h.red_mode == 0) dk_view_add(P.rd[" << k << "], tot); else ((double*)P.h.red_totals)[" << k
          << "] = tot;\n    }\n";
        k++;
      }
    }
    if (rank0) {
      for (int w : wslots) {
        int si = site_index(np, w, {});
        o << "    *(double*)P.s[" << si << "].p = w" << w << "_s;\n";
      }
    }
    if (k) {
      // peer publish (dk_launch_pub): the point's totals block goes straight
      // into every rank's board over NVLink, then each board's flag is raised
      // with release semantics at system scope
      o << "    if (P.pub.n) {\n      const double* src = (const double*)P.pub.src;\n"
        << "      for (int q = 0; q < (int)P.pub.n; ++q) { double* d = (double*)P.pub.dst[q];"
        << " for (int k = 0; k < (int)P.pub.nred; ++k) d[k] = src[k]; }\n"
        << "      __threadfence_system();\n"
        << "      for (int q = 0; q < (int)P.pub.n; ++q)"
        << " asm volatile(\"st.release.sys.global.u32 [%0], %1;\" :: \"l\"(P.pub.flag[q]), \"r\"((unsigned)P.pub.tag) : \"memory\");\n"
        << "    }\n";
    }
  }

  void emit_reduce_epilogue(std::ostringstream& o, const NestPlan& np, const NestIR& ne,
                            const std::vector<int>& wslots) const {
    const int NA = std::max(np.n_array_red, 1);
    o << "  __shared__ double dk_sred[" << NA << "][8];\n  __shared__ int dk_last;\n";
    o << "  const int lin = threadIdx.y * blockDim.x + threadIdx.x, wid = lin >> 5, lane = lin & 31;\n";
    o << "  const int64_t G = (int64_t)gridDim.x * gridDim.y, blin = (int64_t)blockIdx.y * gridDim.x + blockIdx.x;\n";
    o << "  double* red_part = (double*)P.h.red_part;\n";
    for (int a = 0; a < np.n_array_red; ++a)
      o << "  { double v = dk_warp_sum(racc" << a << "); if (lane == 0 && wid < 8) dk_sred[" << a << "][wid] = v; }\n";
    o << "  __syncthreads();\n";
    o << "  if (lin == 0) {\n";
    for (int a = 0; a < np.n_array_red; ++a)
      o << "    { double s = 0.0; for (int w = 0; w < 8; ++w) s = dk_add(s, dk_sred[" << a << "][w]); red_part[" << a
        << " * G + blin] = s; }\n";
    o << "    __threadfence();\n";
    o << "    unsigned int t = atomicAdd((unsigned int*)P.h.red_ticket, 1u);\n";
    o << "    dk_last = (t == (unsigned int)(G - 1));\n  }\n  __syncthreads();\n";
    o << "  if (!dk_last) return;\n  __threadfence();\n";
    o << "  double dk_tot[" << NA << "];\n";
    for (int a = 0; a < np.n_array_red; ++a) {
      // four independent accumulators keep four partial loads in flight per thread
      o << "  { const double* rp = red_part + " << a << " * G; double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0; int64_t i = lin < 256 ? lin : G;\n"
        << "    #pragma unroll 1\n    for (; i + 768 < G; i += 1024) { s0 = dk_add(s0, dk_ldcg(rp + i)); s1 = dk_add(s1, dk_ldcg(rp + i + 256));"
        << " s2 = dk_add(s2, dk_ldcg(rp + i + 512)); s3 = dk_add(s3, dk_ldcg(rp + i + 768)); }\n"
        << "    #pragma unroll 1\n    for (; i < G; i += 256) s0 = dk_add(s0, dk_ldcg(rp + i));\n"
        << "    double s = dk_add(dk_add(s0, s1), dk_add(s2, s3)); s = dk_warp_sum(s); __syncthreads(); if (lane == 0 && wid < 8) dk_sred[" << a << "][wid] = s; }\n";
    }
    o << "  __syncthreads();\n";
    for (int a = 0; a < np.n_array_red; ++a)
      o << "  { double s = 0.0; for (int w = 0; w < 8; ++w) s = dk_add(s, dk_sred[" << a << "][w]); dk_tot[" << a
        << "] = s; }\n";
    o << "  if (lin != 0) return;\n";
    o << "  const int u = 0; (void)u;\n";
    emit_scalar_seq(o, np, ne, false, wslots);
    o << "  *(unsigned int*)P.h.red_ticket = 0u;\n";
  }
};

// -------------------------------------------------------------- NVRTC -----

static uint64_t fnv1a(const std::string& s) {
  uint64_t h = 1469598103934665603ull;
  for (unsigned char c : s) h = (h ^ c) * 1099511628211ull;
  return h;
}

static std::string cache_dir() {
  const char* d = getenv("DK_JIT_CACHE");
  if (d && *d) return d;
  const char* home = getenv("HOME");
  return std::string(home ? home : "/tmp") + "/.cache/dk_b200_jit";
}

// JIT statistics (dk_jit_stats): modules built, NVRTC compiles, disk-cache hits, compile seconds
static int64_t g_jit_modules = 0, g_jit_compiles = 0, g_jit_disk_hits = 0;
static double g_jit_seconds = 0.0;

static std::string compile_cubin(const std::string& src, std::string* log_out) {
  static const char* opts[] = {"--gpu-architecture=sm_100a", "--fmad=false", "-lineinfo", "--std=c++17",
                               "-default-device"};
  const int nopt = sizeof(opts) / sizeof(opts[0]);
  std::string key = src;
  for (int i = 0; i < nopt; ++i) key += opts[i];
  char name[64];
  snprintf(name, sizeof name, "%016llx.cubin", (unsigned long long)fnv1a(key + "dk-jit-v1"));
  std::string dir = cache_dir();
  std::string path = dir + "/" + name;
  {
    std::ifstream f(path, std::ios::binary);
    if (f) {
      std::stringstream ss;
      ss << f.rdbuf();
      std::string bin = ss.str();
      if (!bin.empty()) {
        g_jit_disk_hits++;
        return bin;
      }
    }
  }
  struct Timer {
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    ~Timer() {
      g_jit_seconds += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      g_jit_compiles++;
    }
  } timer;
  nvrtcProgram prog;
  if (nvrtcCreateProgram(&prog, src.c_str(), "dk_fused.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS)
    fail(DK_ERR_NVRTC, "nvrtcCreateProgram failed");
  nvrtcResult rc = nvrtcCompileProgram(prog, nopt, opts);
  size_t logsz = 0;
  nvrtcGetProgramLogSize(prog, &logsz);
  std::string log(logsz, '\0');
  if (logsz) nvrtcGetProgramLog(prog, &log[0]);
  if (log_out) *log_out = log;
  if (rc != NVRTC_SUCCESS) {
    nvrtcDestroyProgram(&prog);
    fail(DK_ERR_NVRTC, "NVRTC: %s\n%s", nvrtcGetErrorString(rc), log.c_str());
  }
  size_t n = 0;
  if (nvrtcGetCUBINSize(prog, &n) != NVRTC_SUCCESS) fail(DK_ERR_NVRTC, "nvrtcGetCUBINSize failed");
  std::string bin(n, '\0');
  nvrtcGetCUBIN(prog, &bin[0]);
  nvrtcDestroyProgram(&prog);
  // best-effort disk cache
  std::string mk = "mkdir -p '" + dir + "' 2>/dev/null";
  if (system(mk.c_str()) == 0) {
    std::string tmp = path + ".tmp" + std::to_string((long long)getpid());
    std::ofstream f(tmp, std::ios::binary);
    if (f) {
      f.write(bin.data(), (std::streamsize)bin.size());
      f.close();
      rename(tmp.c_str(), path.c_str());
    }
  }
  return bin;
}

struct Module {
  CUmodule mod = nullptr;
  std::vector<CUfunction> fn;
  std::vector<int> occ;
  std::vector<NestPlan> plans;
  std::vector<double*> red_part;
  std::vector<unsigned int*> ticket;
  std::string src;
  int unroll = 2;
  bool merged = false;        // fn[0] runs every nest (cooperative launch, grid barriers)
  unsigned int* gbar = nullptr;
  // red_part / ticket (and the K3 tile queue) are per-module scratch: two
  // launches of one module must not overlap.  Launches on one stream are
  // ordered; when a module moves to another stream the new stream first
  // waits for everything already enqueued on the previous one.
  cudaStream_t last_stream = nullptr;
};

static void order_module(Module* m, cudaStream_t s) {
  if (m->last_stream && m->last_stream != s && st().capture_launch0 < 0) {
    static cudaEvent_t ev = [] {
      cudaEvent_t e = nullptr;
      cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
      return e;
    }();
    DK_CUDA(cudaEventRecord(ev, m->last_stream));
    DK_CUDA(cudaStreamWaitEvent(s, ev, 0));
  }
  m->last_stream = s;
}

// A fully prepared launch (parameter blobs, grid shapes) for one exact binding:
// memo-replayed windows re-launch with identical views and scalars every
// iteration, so planning, codegen-key building and blob packing are skipped.
struct Prepared {
  std::string sig;  // raw bytes of views + scalars + totals
  Module* m = nullptr;
  std::vector<std::vector<char>> blobs;
  std::vector<unsigned> grid;  // gx, gy, tx, ty per nest (one entry for a merged module)
};

// a merged module's launch: cooperative (all CTAs resident for the grid barriers)
static void launch_fn(CUfunction f, const unsigned* gd, void* blob, bool coop, CUstream s) {
  void* args[] = {blob};
  if (!coop) {
    DK_CU(cuLaunchKernel(f, gd[0], gd[1], 1, gd[2], gd[3], 1, 0, s, args, nullptr));
    return;
  }
  CUlaunchConfig cfg = {};
  cfg.gridDimX = gd[0];
  cfg.gridDimY = gd[1];
  cfg.gridDimZ = 1;
  cfg.blockDimX = gd[2];
  cfg.blockDimY = gd[3];
  cfg.blockDimZ = 1;
  cfg.hStream = s;
  CUlaunchAttribute at[1];
  at[0].id = CU_LAUNCH_ATTRIBUTE_COOPERATIVE;
  at[0].value.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  DK_CU(cuLaunchKernelEx(&cfg, f, args, nullptr));
}

// one launch per window: every nest a plain streaming nest (or a rank-0 one), the
// parameter block within the 32 KB kernel-parameter limit, and every nest small
// enough (DK_JIT_MERGE_MAX elements, default 2^21) that the launch it saves
// matters more than the one-wave grid-stride walk the grid barrier requires (a
// 32766^2 COPY: 3.24 ms grid-stride vs 2.48 ms one CTA per chunk)
static bool mergeable(const Prog& g, const std::vector<NestPlan>& plans, const dk_view* views) {
  if (plans.size() < 2 || getenv("DK_JIT_SPLIT_NESTS")) return false;
  static const int64_t cap = [] {
    const char* e = getenv("DK_JIT_MERGE_MAX");
    return e ? atoll(e) : (int64_t)1 << 21;
  }();
  size_t bytes = 8 + 4 * (plans.size() + 1);
  for (size_t n = 0; n < plans.size(); ++n) {
    const NestPlan& np = plans[n];
    const dk_view& dv = views[g.nests[n].dom];
    int64_t ne = 1;
    for (int d = 0; d < np.rank; ++d) ne *= dv.ext[d];
    if (ne > cap) return false;
    if (np.rank > 0 && (!np.oneshot || np.staged || np.sweep)) return false;
    bytes += sizeof(DkHdr) + (np.red_slots.empty() ? 0 : sizeof(DkPub)) + 48 * std::max<size_t>(np.sites.size(), 1) +
             sizeof(dk_view) * std::max<size_t>(np.red_slots.size(), 1) + 8 * std::max(g.nscal, 1);
  }
  return bytes <= 30000;
}

struct KernelObj {
  Prog prog;
  std::string text;
  std::unordered_map<std::string, std::unique_ptr<Module>> mods;
  std::string last_src;
  std::vector<Prepared> recent;  // small MRU cache
};

static std::vector<std::unique_ptr<KernelObj>> g_kernels;

static Module* get_module(KernelObj& k, const dk_view* views, const double* scalars, std::vector<NestPlan>* fresh) {
  std::string key;
  std::vector<NestPlan> plans = plan_nests(k.prog, views, &key);
  *fresh = plans;  // pointer-dependent fields (TMA tensor base) come from this binding
  // bitwise-equal scalar classes are part of the binding class
  std::vector<int> rep(k.prog.nscal);
  for (int i = 0; i < k.prog.nscal; ++i) {
    rep[i] = i;
    for (int j = 0; j < i; ++j)
      if (memcmp(&scalars[i], &scalars[j], 8) == 0) {
        rep[i] = rep[j];
        break;
      }
    key += "s" + std::to_string(rep[i]);
  }
  const bool merge = mergeable(k.prog, plans, views);
  key += merge ? "M" : "S";
  auto it = k.mods.find(key);
  if (it != k.mods.end()) return it->second.get();
  auto m = std::make_unique<Module>();
  char name[32];
  snprintf(name, sizeof name, "dkf_%08llx", (unsigned long long)(fnv1a(k.text) & 0xffffffffull));
  GenOpts opts = default_opts(plans);
  opts.merged = m->merged = merge;
  std::vector<CUfunction> fns;
  for (;;) {
    Gen gen(k.prog, plans, name, opts, rep);
    m->src = gen.source();
    k.last_src = m->src;
    std::string log;
    std::string bin = compile_cubin(m->src, &log);
    DK_CU(cuModuleLoadData(&m->mod, bin.data()));
    fns.clear();
    bool spills = false;
    for (size_t n = 0; n < (m->merged ? 1 : k.prog.nests.size()); ++n) {
      CUfunction f;
      std::string nm = std::string(name) + (m->merged ? std::string("_m") : "_n" + std::to_string(n));
      DK_CU(cuModuleGetFunction(&f, m->mod, nm.c_str()));
      int local = 0;
      DK_CU(cuFuncGetAttribute(&local, CU_FUNC_ATTRIBUTE_LOCAL_SIZE_BYTES, f));
      spills |= local > 0;
      fns.push_back(f);
    }
    if (!spills || opts.min_blocks == 1) break;
    DK_CU(cuModuleUnload(m->mod));
    opts.min_blocks = opts.min_blocks > 4 ? 4 : opts.min_blocks - 1;  // 6 -> 4 -> 3 -> 2 -> 1
  }
  m->unroll = opts.unroll;
  g_jit_modules++;
  const int sms = st().sm_count;
  if (m->merged) {
    DK_CUDA(cudaMalloc(&m->gbar, sizeof(unsigned int) * 2));
    DK_CUDA(cudaMemsetAsync(m->gbar, 0, sizeof(unsigned int) * 2, st().stream));
  }
  for (size_t n = 0; n < k.prog.nests.size(); ++n) {
    CUfunction f = fns[m->merged ? 0 : n];
    int occ = 1;
    DK_CU(cuOccupancyMaxActiveBlocksPerMultiprocessor(&occ, f, plans[n].st_ws ? kTPB + 32 : kTPB, 0));
    occ = std::max(occ, 1);
    if (!m->merged || n == 0) m->fn.push_back(f);
    m->occ.push_back(occ);
    double* rp = nullptr;
    unsigned int* tk = nullptr;
    const int na = std::max(plans[n].n_array_red, 1);
    if (!plans[n].red_slots.empty() || plans[n].staged) {
      DK_CUDA(cudaMalloc(&rp, sizeof(double) * (size_t)na * (size_t)sms * occ * red_waves() + 64));
      DK_CUDA(cudaMalloc(&tk, sizeof(unsigned int) * 4));
      DK_CUDA(cudaMemsetAsync(tk, 0, sizeof(unsigned int) * 4, st().stream));
    }
    m->red_part.push_back(rp);
    m->ticket.push_back(tk);
  }
  m->plans = std::move(plans);
  Module* raw = m.get();
  k.mods.emplace(key, std::move(m));
  return raw;
}

// L2 sector promotion of the staged tiles' TMA loads (DK_TMA_L2 = 0 | 64 | 128 | 256)
static CUtensorMapL2promotion tma_l2_promotion() {
  static int v = [] {
    const char* e = getenv("DK_TMA_L2");
    return e ? atoi(e) : 128;
  }();
  switch (v) {
    case 0: return CU_TENSOR_MAP_L2_PROMOTION_NONE;
    case 64: return CU_TENSOR_MAP_L2_PROMOTION_L2_64B;
    case 256: return CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
    default: return CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
  }
}

static int64_t pow2ceil(int64_t v) {
  int64_t p = 1;
  while (p < v) p <<= 1;
  return p;
}

static void launch(KernelObj& k, const dk_view* views, int nviews, const double* scalars, int nscal, uint64_t totals,
                   const DkPub* pub = nullptr) {
  const Prog& g = k.prog;
  if (nviews != g.nslots) fail(DK_ERR_ARG, "launch binds %d views, kernel has %d slots", nviews, g.nslots);
  if (nscal != g.nscal) fail(DK_ERR_ARG, "launch passes %d scalars, kernel expects %d", nscal, g.nscal);
  State& S = st();
  std::string sig((const char*)views, sizeof(dk_view) * (size_t)nviews);
  sig.append((const char*)scalars, 8 * (size_t)nscal);
  sig.append((const char*)&totals, sizeof totals);
  if (pub) sig.append((const char*)pub, sizeof *pub);
  for (size_t i = 0; i < k.recent.size(); ++i) {
    Prepared& pr = k.recent[i];
    if (pr.sig != sig) continue;
    order_module(pr.m, S.stream);
    for (size_t n = 0; n < pr.blobs.size(); ++n) {
      launch_fn(pr.m->fn[n], &pr.grid[4 * n], pr.blobs[n].data(), pr.m->merged, (CUstream)S.stream);
      S.launches++;
    }
    if (i) std::swap(k.recent[i], k.recent[0]);
    return;
  }
  std::vector<NestPlan> fresh;
  Module* m = get_module(k, views, scalars, &fresh);
  Prepared prep;
  prep.sig = sig;
  prep.m = m;
  order_module(m, S.stream);
  int kbase = 0;
  std::vector<char> blob;
  std::vector<char> mblob;      // merged module: the nests' P_n blocks, in order
  std::vector<unsigned> mtx;    // merged module: each nest's TX
  int64_t mgx = 1;              // merged module: the largest per-nest grid
  for (size_t n = 0; n < g.nests.size(); ++n) {
    const NestPlan& np = fresh[n];
    const dk_view& dv = views[g.nests[n].dom];
    const int r = np.rank;
    DkHdr h = {};
    for (int d = 0; d < 4; ++d) h.ext[d] = 1;
    int64_t D[4] = {1, 1, 1, 1};
    h.nelem = 1;
    for (int d = 0; d < r; ++d) {
      h.ext[d] = D[d] = dv.ext[d];
      h.nelem *= dv.ext[d];
    }
    h.ninner = r ? D[r - 1] : 1;
    h.nrows = 1;
    for (int d = 0; d + 1 < r; ++d) h.nrows *= D[d];
    h.red_part = (uint64_t)m->red_part[n];
    h.red_ticket = (uint64_t)m->ticket[n];
    h.red_totals = totals ? totals + 8ull * kbase : 0;
    h.red_mode = totals ? 1 : 0;
    const int NS = (int)np.sites.size(), NR = (int)np.red_slots.size();
    DkPub pb = {};
    if (pub && NR) {
      // only the kernel's last reducing nest publishes (the whole block)
      bool last = true;
      for (size_t n2 = n + 1; n2 < g.nests.size(); ++n2)
        if (!fresh[n2].red_slots.empty()) last = false;
      if (last) pb = *pub;
    }
    std::vector<DkSite> sites(std::max(NS, 1));
    memset(sites.data(), 0, sizeof(DkSite) * sites.size());
    for (int i = 0; i < NS; ++i) {
      const Site& s = np.sites[i];
      const dk_view& v = views[s.slot];
      DkSite& o = sites[i];
      int64_t str[4] = {0, 0, 0, 0};
      if (v.rank > 0) bcast_strides(v, D, r, str);
      int64_t shift = 0;
      for (size_t d = 0; d < s.offs.size(); ++d) shift += s.offs[d] * v.stride[d];
      o.p = v.ptr + 8ull * (uint64_t)shift;
      for (int d = 0; d < 3 && d + 1 < r; ++d) o.st[d] = str[d];
      o.sti = r ? str[r - 1] : 0;
      o.mode = s.cls == 'A' ? 0 : s.cls == 'C' || s.cls == 'H' ? 1 : s.cls == 'G' ? 3 : 2;  // informational: code is specialised
    }
    std::vector<dk_view> rd(std::max(NR, 1));
    memset(rd.data(), 0, sizeof(dk_view) * rd.size());
    for (int q = 0; q < NR; ++q) rd[q] = views[np.red_slots[q]];
    const size_t nsc = std::max(g.nscal, 1);
    const bool tma = np.staged && !np.sweep;
    const size_t tmb = tma ? 128 : 0;  // CUtensorMap (64-byte aligned) leads a TMA-staged nest's params
    size_t total = tmb + sizeof(DkHdr) + (NR ? sizeof(DkPub) : 0) + (np.sweep ? sizeof(DkUni) : 0) +
                   sizeof(DkSite) * sites.size() + sizeof(dk_view) * rd.size() + 8 * nsc;
    if (tma) total = (total + 63) / 64 * 64;
    blob.assign(total + 64, 0);
    char* p = blob.data();
    if (tma) {
      static_assert(sizeof(CUtensorMap) == 128, "CUtensorMap size");
      CUtensorMap tm;
      cuuint64_t gdim[2] = {(cuuint64_t)np.st_cols, (cuuint64_t)np.st_nrows};
      cuuint64_t gstr[1] = {(cuuint64_t)np.st_rowstride * 8};
      cuuint32_t box[2] = {(cuuint32_t)kBW, (cuuint32_t)np.st_rows};
      cuuint32_t estr[2] = {1, 1};
      DK_CU(cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)np.st_base, gdim, gstr, box, estr,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                   tma_l2_promotion(), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
      memcpy(p, &tm, 128);
      p += 128;
    }
    memcpy(p, &h, sizeof h);
    p += sizeof h;
    if (NR) {
      memcpy(p, &pb, sizeof pb);
      p += sizeof pb;
    }
    if (np.sweep) {
      DkUni un = {np.st_base, np.st_rowstride, np.st_cols, np.st_nrows};
      memcpy(p, &un, sizeof un);
      p += sizeof un;
    }
    memcpy(p, sites.data(), sizeof(DkSite) * sites.size());
    p += sizeof(DkSite) * sites.size();
    memcpy(p, rd.data(), sizeof(dk_view) * rd.size());
    p += sizeof(dk_view) * rd.size();
    if (g.nscal) memcpy(p, scalars, 8 * (size_t)g.nscal);
    // launch shape
    unsigned gx = 1, gy = 1, tx = kTPB, ty = 1;
    if (r > 0 && h.nelem > 0) {
      const int64_t npairs = (h.ninner + 1 + np.shift) / 2;
      tx = (unsigned)(npairs >= kTPB ? kTPB : std::max<int64_t>(32, pow2ceil(npairs)));
      ty = kTPB / tx;
      const int64_t maxg = (int64_t)S.sm_count * m->occ[n];
      const int64_t U = m->unroll;
      if (np.oneshot) {
        // reductions keep a bounded grid (one partial per CTA, folded by the last CTA)
        const int64_t cpr = (npairs + (int64_t)tx * U - 1) / ((int64_t)tx * U);
        const int64_t cap = np.red_slots.empty() ? 0x7fffffff : red_waves() * maxg;
        gx = (unsigned)std::max<int64_t>(1, std::min<int64_t>((h.nrows + ty - 1) / ty * cpr, cap));
        gy = 1;
      } else {
        int64_t GX = std::min<int64_t>((npairs + (int64_t)tx * U - 1) / ((int64_t)tx * U), maxg);
        GX = std::max<int64_t>(GX, 1);
        int64_t GY = std::min<int64_t>((h.nrows + ty - 1) / ty, std::max<int64_t>(1, maxg / GX));
        GY = std::min<int64_t>(std::max<int64_t>(GY, 1), 65535);
        gx = (unsigned)GX;
        gy = (unsigned)GY;
      }
    } else if (r == 0) {
      tx = 32;
      ty = 1;
    }
    if (np.sweep) {
      const int64_t ntask = ((((D[1] + 1) / 2) + 255) / 256) * ((D[0] + kSweepRows() - 1) / kSweepRows());
      const int64_t cap = NR ? red_waves() * (int64_t)S.sm_count * m->occ[n] : 0x7fffffff;
      gx = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ntask, cap));
      gy = 1;
      tx = kTPB;
      ty = 1;
    } else if (np.staged) {
      const int64_t ntiles = ((D[0] + kTR - 1) / kTR) * ((D[1] + kTC - 1) / kTC);
      gx = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ntiles, (int64_t)S.sm_count * m->occ[n]));
      gy = 1;
      tx = np.st_ws ? kTPB + 32 : kTPB;
      ty = 1;
    }
    kbase += NR;
    if (m->merged) {
      // the nest's P_n goes into the one PM block; its TX and grid are folded in below
      blob.resize(total);
      mblob.insert(mblob.end(), blob.begin(), blob.end());
      mtx.push_back(r == 0 ? 32u : tx);
      mgx = std::max<int64_t>(mgx, (int64_t)gx * gy);
      continue;
    }
    // one by-value struct parameter; the driver copies sizeof(P_n) bytes from the blob
    launch_fn(m->fn[n], std::vector<unsigned>{gx, gy, tx, ty}.data(), blob.data(), false, (CUstream)S.stream);
    S.launches++;
    prep.blobs.push_back(blob);
    prep.grid.insert(prep.grid.end(), {gx, gy, tx, ty});
  }
  if (m->merged) {
    // PM = { gbar, tx[NN rounded to even], P_0, P_1, ... }; every CTA resident (one wave)
    const size_t NN = g.nests.size(), ntx = (NN + 1) / 2 * 2;
    std::vector<char> pm(8 + 4 * ntx, 0);
    const uint64_t gb = (uint64_t)m->gbar;
    memcpy(pm.data(), &gb, 8);
    memcpy(pm.data() + 8, mtx.data(), 4 * NN);
    pm.insert(pm.end(), mblob.begin(), mblob.end());
    pm.resize(pm.size() + 64, 0);
    const int64_t wave = (int64_t)S.sm_count * m->occ[0];
    const unsigned G = (unsigned)std::max<int64_t>(1, std::min<int64_t>(mgx, wave));
    const unsigned gd[4] = {G, 1, (unsigned)kTPB, 1};
    launch_fn(m->fn[0], gd, pm.data(), true, (CUstream)S.stream);
    S.launches++;
    prep.blobs.push_back(pm);
    prep.grid.insert(prep.grid.end(), {gd[0], gd[1], gd[2], gd[3]});
  }
  if (k.recent.size() >= 8) k.recent.pop_back();
  k.recent.insert(k.recent.begin(), std::move(prep));
}

}  // namespace dk

using namespace dk;

extern "C" {

int dk_kernel_compile(const char* program, int64_t len, int64_t* handle) {
  return guard([&] {
    require_init();
    auto k = std::make_unique<KernelObj>();
    k->text.assign(program, (size_t)len);
    k->prog = parse_prog(k->text);
    g_kernels.push_back(std::move(k));
    *handle = (int64_t)g_kernels.size() - 1;
  });
}

static KernelObj& kernel_of(int64_t h) {
  if (h < 0 || h >= (int64_t)g_kernels.size()) fail(DK_ERR_STATE, "unknown kernel handle %lld", (long long)h);
  return *g_kernels[h];
}

int dk_kernel_source(int64_t handle, char* buf, int64_t cap, int64_t* len) {
  return guard([&] {
    KernelObj& k = kernel_of(handle);
    *len = (int64_t)k.last_src.size();
    if (buf && cap > 0) {
      int64_t n = std::min<int64_t>(cap - 1, *len);
      memcpy(buf, k.last_src.data(), (size_t)n);
      buf[n] = 0;
    }
  });
}

int dk_kernel_codegen(const char* program, int64_t len, const dk_view* views, int nviews, const double* scalars,
                      int compile, char* buf, int64_t cap, int64_t* out_len) {
  return guard([&] {
    Prog g = parse_prog(std::string(program, (size_t)len));
    if (nviews != g.nslots) fail(DK_ERR_ARG, "codegen binds %d views, kernel has %d slots", nviews, g.nslots);
    std::string key;
    std::vector<NestPlan> plans = plan_nests(g, views, &key);
    std::vector<int> rep(g.nscal);
    for (int i = 0; i < g.nscal; ++i) {
      rep[i] = i;
      for (int j = 0; scalars && j < i; ++j)
        if (memcmp(&scalars[i], &scalars[j], 8) == 0) {
          rep[i] = rep[j];
          break;
        }
    }
    GenOpts opts = default_opts(plans);
    opts.merged = mergeable(g, plans, views);
    Gen gen(g, plans, "dk", opts, rep);
    std::string src = gen.source();
    if (compile) {
      std::string log;
      std::string bin = compile_cubin(src, &log);
      if (bin.empty()) fail(DK_ERR_NVRTC, "empty cubin");
    }
    *out_len = (int64_t)src.size();
    if (buf && cap > 0) {
      int64_t n = std::min<int64_t>(cap - 1, *out_len);
      memcpy(buf, src.data(), (size_t)n);
      buf[n] = 0;
    }
  });
}

int dk_jit_stats(int64_t* modules, int64_t* compiles, int64_t* disk_hits, double* seconds) {
  return guard([&] {
    *modules = g_jit_modules;
    *compiles = g_jit_compiles;
    *disk_hits = g_jit_disk_hits;
    *seconds = g_jit_seconds;
  });
}

int dk_kernel_num_reductions(int64_t handle, int* n) {
  return guard([&] { *n = kernel_of(handle).prog.nreduce; });
}

int dk_launch(int64_t handle, const dk_view* views, int nviews, const double* scalars, int nscalars,
              uint64_t totals) {
  return guard([&] {
    require_init();
    NvtxRange nv("dk_launch", handle);
    launch(kernel_of(handle), views, nviews, scalars, nscalars, totals);
  });
}

static void launch_pub(int64_t handle, const dk_view* views, int nviews, const double* scalars, int nscalars,
                       int64_t epoch, int point, int red_offset, int nred_total) {
  require_init();
  require_not_capturing("dk_launch_pub (board slots are epoch-numbered)");
  NvtxRange nv("dk_launch_pub", handle);
  State& S = st();
  if (!S.p2p) fail(DK_ERR_STATE, "dk_p2p_init has not enabled peer-memory reductions");
  if (epoch < 0) fail(DK_ERR_ARG, "negative reduction epoch");
  const int slot = (int)(epoch % DK_P2P_SLOTS);
  if (point < 0 || point >= DK_P2P_POINTS) fail(DK_ERR_ARG, "point %d exceeds the board's %d points per rank", point, DK_P2P_POINTS);
  KernelObj& k = kernel_of(handle);
  const int nred = k.prog.nreduce;
  if (nred_total <= 0) nred_total = nred;
  if (nred == 0 || red_offset < 0 || red_offset + nred > nred_total || nred_total > DK_P2P_RED)
    fail(DK_ERR_UNSUPPORTED, "kernel has %d reductions at %d of %d (board holds 1..%d)", nred, red_offset, nred_total,
         DK_P2P_RED);
  const size_t off = 8ull * (size_t)nred_total * (size_t)(S.rank * DK_P2P_POINTS + point);
  DkPub pub = {};
  pub.n = S.world;
  pub.nred = nred_total;
  pub.tag = p2p_tag(epoch);
  pub.src = (uint64_t)S.board + p2p_data_off(slot) + off;
  for (int q = 0; q < S.world; ++q) {
    pub.dst[q] = S.peer_board[q] + p2p_data_off(slot) + off;
    pub.flag[q] = S.peer_board[q] + p2p_flag_off(slot) + 4ull * (size_t)(S.rank * DK_P2P_POINTS + point);
  }
  launch(k, views, nviews, scalars, nscalars, pub.src + 8ull * (uint64_t)red_offset, &pub);
}

int dk_launch_pub(int64_t handle, const dk_view* views, int nviews, const double* scalars, int nscalars,
                  int64_t epoch, int point) {
  return guard([&] { launch_pub(handle, views, nviews, scalars, nscalars, epoch, point, 0, 0); });
}

int dk_launch_pub_ex(int64_t handle, const dk_view* views, int nviews, const double* scalars, int nscalars,
                     int64_t epoch, int point, int red_offset, int nred_total) {
  return guard([&] { launch_pub(handle, views, nviews, scalars, nscalars, epoch, point, red_offset, nred_total); });
}

int dk_p2p_block(int64_t epoch, int point, int nred_total, uint64_t* ptr) {
  return guard([&] {
    require_init();
    State& S = st();
    if (!S.p2p) fail(DK_ERR_STATE, "dk_p2p_init has not enabled peer-memory reductions");
    if (epoch < 0 || point < 0 || point >= DK_P2P_POINTS || nred_total <= 0 || nred_total > DK_P2P_RED)
      fail(DK_ERR_ARG, "bad board block (epoch %lld, point %d, %d totals)", (long long)epoch, point, nred_total);
    const int slot = (int)(epoch % DK_P2P_SLOTS);
    *ptr = (uint64_t)S.board + p2p_data_off(slot) + 8ull * (size_t)nred_total * (size_t)(S.rank * DK_P2P_POINTS + point);
  });
}

}  // extern "C"
