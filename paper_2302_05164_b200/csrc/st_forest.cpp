// Leaf tables of the growing adaptive voxel mesh, host C++.
//
// The reference keeps its octree forest and DoF map in numpy
// (pkg/src/scantherm/mesh.py).  This file builds the same tables from the
// leaf set with hash-indexed integer lattice work, written for this
// library (no numpy semantics copied, only the published rules):
//
//   st_coarse_grid      level-0 tiling of the build volume   (mesh.py:289-333)
//   st_plan_layer       layer advance: refine / activate / coarsen-gate /
//                       void collapse / 2:1 ripple + lineage  (mesh.py:439-602)
//   st_build_dofmap     vertex numbering, hanging constraints with chains,
//                       Dirichlet plane                       (mesh.py:706-779)
//   st_interface_faces  radiating +z facets (full or quarter) (mesh.py:998-1072)
//   st_transfer_nodal   nodal copy / trilinear interpolation / fresh fill
//   st_transfer_history r_c octant copy down, octant mean up  (mesh.py:803-899)
//
// Outputs must be bit-identical to the reference: integer work is exact by
// construction; the few floating-point results (constraint weights, the
// trilinear transfer, the octant mean) are evaluated in the reference's
// operation order (weights are dyadic, so their sums are exact in any
// order; the transfer and the mean round like numpy's sequential
// accumulation / 8-lane pairwise sum).  Compiled with -ffp-contract=off.
//
// Results of variable size come back in an st_tables bag of named arrays
// (st_tables_get / st_tables_free).

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <limits>
#include <map>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/scantherm_b200.h"

namespace st {
void set_error(const std::string& msg);
}

struct st_tables {
  struct Arr {
    std::string name;
    int dtype;  // ST_DT_*
    std::vector<int64_t> dims;
    std::vector<unsigned char> bytes;
  };
  std::vector<Arr> arrs;

  template <class T>
  void put(const char* name, int dtype, const std::vector<T>& v, std::vector<int64_t> dims = {}) {
    Arr a;
    a.name = name;
    a.dtype = dtype;
    a.dims = dims.empty() ? std::vector<int64_t>{(int64_t)v.size()} : dims;
    a.bytes.resize(v.size() * sizeof(T));
    if (!v.empty()) std::memcpy(a.bytes.data(), v.data(), a.bytes.size());
    arrs.push_back(std::move(a));
  }
};

namespace {

// ---- lattice keys ---------------------------------------------------------
// (x, y, z) -> one int64, 21 bits per axis with an offset of 2^20: the
// reference's key (mesh.py:41-46), so key order is x-major, z-fastest.
constexpr int kBits = 21;
constexpr int64_t kOff = int64_t(1) << (kBits - 1);
constexpr int64_t kMask = (int64_t(1) << kBits) - 1;

struct V3 {
  int64_t x, y, z;
};

inline bool packable(const V3& v) {
  return v.x + kOff >= 0 && v.x + kOff <= kMask && v.y + kOff >= 0 && v.y + kOff <= kMask &&
         v.z + kOff >= 0 && v.z + kOff <= kMask;
}
inline int64_t key_of(const V3& v) {
  return ((v.x + kOff) << (2 * kBits)) | ((v.y + kOff) << kBits) | (v.z + kOff);
}
inline V3 v3_of(int64_t k) {
  return V3{((k >> (2 * kBits)) & kMask) - kOff, ((k >> kBits) & kMask) - kOff, (k & kMask) - kOff};
}
// floor division / floor to a multiple (lattice coordinates can be negative)
inline int64_t fdiv(int64_t a, int64_t b) {
  int64_t q = a / b;
  return (a % b != 0 && ((a < 0) != (b < 0))) ? q - 1 : q;
}
inline int64_t fdown(int64_t a, int64_t s) { return fdiv(a, s) * s; }
inline bool divisible(int64_t a, int64_t s) { return a % s == 0; }

// corner c = ix*4 + iy*2 + iz
inline int cbit(int c, int axis) { return (c >> (2 - axis)) & 1; }

// ---- open-addressing map int64 key -> int64 value -------------------------
class KeyMap {
 public:
  explicit KeyMap(size_t expect = 16) { reset(expect); }
  void reset(size_t expect) {
    size_t cap = 16;
    while (cap < expect * 2 + 1) cap <<= 1;
    keys_.assign(cap, kEmpty);
    vals_.assign(cap, -1);
    mask_ = cap - 1;
    n_ = 0;
  }
  void put(int64_t k, int64_t v) {
    if ((n_ + 1) * 2 > keys_.size()) grow();
    size_t i = slot(k);
    if (keys_[i] == kEmpty) {
      keys_[i] = k;
      n_++;
    }
    vals_[i] = v;
  }
  int64_t get(int64_t k) const {
    size_t i = hash(k) & mask_;
    while (true) {
      if (keys_[i] == k) return vals_[i];
      if (keys_[i] == kEmpty) return -1;
      i = (i + 1) & mask_;
    }
  }
  size_t size() const { return n_; }

 private:
  static constexpr int64_t kEmpty = std::numeric_limits<int64_t>::min();
  static size_t hash(int64_t k) {
    uint64_t z = (uint64_t)k + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return (size_t)(z ^ (z >> 31));
  }
  size_t slot(int64_t k) const {
    size_t i = hash(k) & mask_;
    while (keys_[i] != kEmpty && keys_[i] != k) i = (i + 1) & mask_;
    return i;
  }
  void grow() {
    std::vector<int64_t> k = std::move(keys_), v = std::move(vals_);
    reset(k.size());
    for (size_t i = 0; i < k.size(); i++)
      if (k[i] != kEmpty) put(k[i], v[i]);
  }
  std::vector<int64_t> keys_, vals_;
  size_t mask_ = 0, n_ = 0;
};

// ---- a leaf table ----------------------------------------------------------
struct Leaves {
  int depth = 0, cpl = 1;
  std::vector<int> level;
  std::vector<V3> anchor;
  std::vector<uint8_t> active, consol;

  size_t n() const { return level.size(); }
  int64_t size(size_t i) const { return int64_t(1) << (depth - level[i]); }
  int64_t size_at(int ell) const { return int64_t(1) << (depth - ell); }
};

Leaves from_c(const st_leaves* L) {
  Leaves f;
  f.depth = L->depth;
  f.cpl = L->cpl;
  const size_t n = (size_t)L->n;
  f.level.resize(n);
  f.anchor.resize(n);
  f.active.resize(n);
  f.consol.resize(n);
  for (size_t i = 0; i < n; i++) {
    f.level[i] = L->level[i];
    f.anchor[i] = V3{L->anchor[3 * i], L->anchor[3 * i + 1], L->anchor[3 * i + 2]};
    f.active[i] = L->active[i] ? 1 : 0;
    f.consol[i] = L->init_consol ? (L->init_consol[i] ? 1 : 0) : 0;
  }
  return f;
}

// per-level hash index of a leaf table: (level, anchor key) -> row
class LevelIndex {
 public:
  explicit LevelIndex(const Leaves& f) {
    for (size_t i = 0; i < f.n(); i++) by_level_[f.level[i]].put(key_of(f.anchor[i]), (int64_t)i);
  }
  int64_t find(int ell, const V3& a) const {
    auto it = by_level_.find(ell);
    if (it == by_level_.end() || !packable(a)) return -1;
    return it->second.get(key_of(a));
  }
  // levels present, ascending
  std::vector<int> levels() const {
    std::vector<int> v;
    for (auto& kv : by_level_) v.push_back(kv.first);
    return v;
  }
  // the leaf containing the finest lattice cell p (any level), -1 outside
  int64_t containing(const Leaves& f, const V3& p) const {
    for (auto& kv : by_level_) {
      const int64_t s = f.size_at(kv.first);
      const V3 a{fdown(p.x, s), fdown(p.y, s), fdown(p.z, s)};
      if (!packable(a)) continue;
      const int64_t r = kv.second.get(key_of(a));
      if (r >= 0) return r;
    }
    return -1;
  }

 private:
  std::map<int, KeyMap> by_level_;
};

// canonical leaf order: by anchor key, then level (mesh.py:269-271)
std::vector<size_t> canonical_order(const std::vector<int>& level, const std::vector<V3>& anchor) {
  std::vector<size_t> o(level.size());
  std::iota(o.begin(), o.end(), 0);
  std::vector<int64_t> k(level.size());
  for (size_t i = 0; i < level.size(); i++) k[i] = key_of(anchor[i]);
  std::stable_sort(o.begin(), o.end(), [&](size_t a, size_t b) {
    return k[a] != k[b] ? k[a] < k[b] : level[a] < level[b];
  });
  return o;
}

// An active leaf whose closed box holds lattice vertex v without v being one
// of its corners (the hanging-node host of v).  Levels coarse to fine, the
// eight candidate boxes around v in corner order; first hit wins.
bool hanging_host(const Leaves& f, const LevelIndex& idx, const std::vector<int>& levels,
                  const V3& v, int64_t* row, V3* rel) {
  for (int ell : levels) {
    const int64_t s = f.size_at(ell);
    const int64_t hx = fdown(v.x, s), hy = fdown(v.y, s), hz = fdown(v.z, s);
    const int64_t lx = divisible(v.x, s) ? hx - s : hx, ly = divisible(v.y, s) ? hy - s : hy,
                  lz = divisible(v.z, s) ? hz - s : hz;
    for (int c = 0; c < 8; c++) {
      const V3 a{cbit(c, 0) ? hx : lx, cbit(c, 1) ? hy : ly, cbit(c, 2) ? hz : lz};
      const int64_t r = idx.find(ell, a);
      if (r < 0 || !f.active[r]) continue;
      const V3 d{v.x - a.x, v.y - a.y, v.z - a.z};
      const bool corner = (d.x == 0 || d.x == s) && (d.y == 0 || d.y == s) && (d.z == 0 || d.z == s);
      if (corner) continue;
      *row = r;
      *rel = d;
      return true;
    }
  }
  return false;
}

// trilinear weight of corner c at relative position r (components in [0, 1]),
// multiplied up from 1.0 in axis order
inline double corner_weight(int c, const double r[3]) {
  double w = 1.0;
  for (int d = 0; d < 3; d++) w *= cbit(c, d) ? r[d] : (1.0 - r[d]);
  return w;
}

// numpy's add.reduce summation for n doubles (8-lane pairwise blocks)
double np_pairwise(const double* a, int64_t n) {
  if (n < 8) {
    double r = 0.0;
    for (int64_t i = 0; i < n; i++) r += a[i];
    return r;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; j++) r[j] = a[j];
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; j++) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; i++) res += a[i];
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return np_pairwise(a, n2) + np_pairwise(a + n2, n - n2);
}

// ---- DoF map ---------------------------------------------------------------
struct DofTables {
  std::vector<int64_t> vkeys;   // sorted vertex keys
  std::vector<int32_t> cell_verts;
  std::vector<int64_t> active_rows;
  std::vector<uint8_t> is_slave, is_dir;
  std::vector<int64_t> slaves, ptr, masters;
  std::vector<double> weights;
};

void build_dofs(const Leaves& f, int64_t z_min, bool dirichlet, DofTables& D) {
  for (size_t i = 0; i < f.n(); i++)
    if (f.active[i]) D.active_rows.push_back((int64_t)i);
  const size_t na = D.active_rows.size();
  std::vector<int64_t> ck(na * 8);
  for (size_t e = 0; e < na; e++) {
    const size_t r = (size_t)D.active_rows[e];
    const int64_t s = f.size(r);
    for (int c = 0; c < 8; c++)
      ck[e * 8 + c] = key_of(V3{f.anchor[r].x + cbit(c, 0) * s, f.anchor[r].y + cbit(c, 1) * s,
                                f.anchor[r].z + cbit(c, 2) * s});
  }
  D.vkeys = ck;
  std::sort(D.vkeys.begin(), D.vkeys.end());
  D.vkeys.erase(std::unique(D.vkeys.begin(), D.vkeys.end()), D.vkeys.end());
  const size_t nv = D.vkeys.size();
  D.cell_verts.resize(na * 8);
  std::vector<int32_t> incid(nv, 0);
  for (size_t e = 0; e < na * 8; e++) {
    const int64_t id = std::lower_bound(D.vkeys.begin(), D.vkeys.end(), ck[e]) - D.vkeys.begin();
    D.cell_verts[e] = (int32_t)id;
    incid[id]++;
  }
  // hanging vertices: fewer than 8 incident active cells and an active host
  // leaf that holds them off its corners.  One constraint level per vertex
  // under 2:1 balance; chains (a master hanging on a coarser cell) are
  // expanded below.
  LevelIndex idx(f);
  const std::vector<int> levels = idx.levels();
  std::vector<int64_t> pos_of_row(f.n(), -1);
  for (size_t e = 0; e < na; e++) pos_of_row[D.active_rows[e]] = (int64_t)e;
  std::map<int64_t, std::vector<std::pair<int64_t, double>>> direct;  // slave -> masters
  for (size_t v = 0; v < nv; v++) {
    if (incid[v] >= 8) continue;
    int64_t row;
    V3 rel;
    if (!hanging_host(f, idx, levels, v3_of(D.vkeys[v]), &row, &rel)) continue;
    const double s = (double)f.size((size_t)row);
    const double r[3] = {(double)rel.x / s, (double)rel.y / s, (double)rel.z / s};
    auto& m = direct[(int64_t)v];
    for (int c = 0; c < 8; c++) {
      const double w = corner_weight(c, r);
      if (w > 0.0) m.emplace_back((int64_t)D.cell_verts[pos_of_row[row] * 8 + c], w);
    }
  }
  // full expansion over non-hanging masters; weights are dyadic, so the
  // accumulated sums are exact whatever the order
  std::map<int64_t, std::map<int64_t, double>> full;
  std::vector<int64_t> stack;
  auto expand = [&](int64_t v, auto&& self) -> const std::map<int64_t, double>& {
    auto it = full.find(v);
    if (it != full.end()) return it->second;
    std::map<int64_t, double> acc;
    for (auto& mw : direct[v]) {
      if (direct.count(mw.first)) {
        for (auto& kv : self(mw.first, self)) acc[kv.first] += mw.second * kv.second;
      } else {
        acc[mw.first] += mw.second;
      }
    }
    return full[v] = std::move(acc);
  };
  D.is_slave.assign(nv, 0);
  D.ptr.push_back(0);
  for (auto& kv : direct) {
    const auto& m = expand(kv.first, expand);
    D.slaves.push_back(kv.first);
    D.is_slave[kv.first] = 1;
    for (auto& mw : m) {
      D.masters.push_back(mw.first);
      D.weights.push_back(mw.second);
    }
    D.ptr.push_back((int64_t)D.masters.size());
  }
  D.is_dir.assign(nv, 0);
  if (dirichlet)
    for (size_t v = 0; v < nv; v++) D.is_dir[v] = (v3_of(D.vkeys[v]).z == z_min && !D.is_slave[v]) ? 1 : 0;
}

// ---- layer planner -----------------------------------------------------------
// Mutable leaf list with the reference's row semantics: a split removes the
// rows and appends their eight children (corner order), a merge removes the
// children and appends the parents.
struct Work : Leaves {
  void split(const std::vector<size_t>& rows) {
    if (rows.empty()) return;
    std::vector<uint8_t> drop(n(), 0);
    for (size_t r : rows) drop[r] = 1;
    Leaves nw;
    nw.depth = depth;
    nw.cpl = cpl;
    for (size_t i = 0; i < n(); i++)
      if (!drop[i]) push(nw, level[i], anchor[i], active[i], consol[i]);
    for (size_t r : rows) {
      const int64_t h = size(r) >> 1;
      for (int c = 0; c < 8; c++)
        push(nw, level[r] + 1,
             V3{anchor[r].x + cbit(c, 0) * h, anchor[r].y + cbit(c, 1) * h, anchor[r].z + cbit(c, 2) * h},
             active[r], consol[r]);
    }
    assign(nw);
  }
  void merge(const std::vector<int>& plevel, const std::vector<V3>& pa,
             const std::vector<std::vector<size_t>>& groups, uint8_t act,
             const std::vector<uint8_t>& cons) {
    std::vector<uint8_t> drop(n(), 0);
    for (auto& g : groups)
      for (size_t r : g) drop[r] = 1;
    Leaves nw;
    nw.depth = depth;
    nw.cpl = cpl;
    for (size_t i = 0; i < n(); i++)
      if (!drop[i]) push(nw, level[i], anchor[i], active[i], consol[i]);
    for (size_t g = 0; g < groups.size(); g++) push(nw, plevel[g], pa[g], act, cons[g]);
    assign(nw);
  }
  // complete sibling octets among the given rows: per level ascending, the
  // groups of eight rows sharing a parent, in parent-key order (rows of a
  // group ascending)
  void octets(const std::vector<size_t>& rows, std::vector<int>& plevel, std::vector<V3>& pa,
              std::vector<std::vector<size_t>>& groups) const {
    std::map<int, std::vector<size_t>> by_level;
    for (size_t r : rows) by_level[level[r]].push_back(r);
    for (auto& kv : by_level) {
      const int64_t ps = int64_t(2) << (depth - kv.first);
      std::vector<std::pair<int64_t, size_t>> kr;
      for (size_t r : kv.second)
        kr.emplace_back(key_of(V3{fdown(anchor[r].x, ps), fdown(anchor[r].y, ps), fdown(anchor[r].z, ps)}), r);
      std::stable_sort(kr.begin(), kr.end(),
                       [](const std::pair<int64_t, size_t>& a, const std::pair<int64_t, size_t>& b) {
                         return a.first < b.first;
                       });
      for (size_t s = 0; s < kr.size();) {
        size_t e = s;
        while (e < kr.size() && kr[e].first == kr[s].first) e++;
        if (e - s == 8) {
          std::vector<size_t> g;
          for (size_t t = s; t < e; t++) g.push_back(kr[t].second);
          groups.push_back(g);
          pa.push_back(v3_of(kr[s].first));
          plevel.push_back(kv.first - 1);
        }
        s = e;
      }
    }
  }

 private:
  static void push(Leaves& l, int lev, const V3& a, uint8_t act, uint8_t con) {
    l.level.push_back(lev);
    l.anchor.push_back(a);
    l.active.push_back(act);
    l.consol.push_back(con);
  }
  void assign(Leaves& nw) {
    level.swap(nw.level);
    anchor.swap(nw.anchor);
    active.swap(nw.active);
    consol.swap(nw.consol);
  }
};

// level of the leaf containing each probe (finest cell), -1 outside
struct LevelProbe {
  LevelProbe(const Leaves& f) : f_(f), idx_(f) {}
  int level_at(const V3& p) const {
    const int64_t r = idx_.containing(f_, p);
    return r < 0 ? -1 : f_.level[r];
  }
  const Leaves& f_;
  LevelIndex idx_;
};

// the 26 neighbour directions (dx, dy, dz) != 0, x slowest
const std::vector<V3>& dirs26() {
  static std::vector<V3> d = [] {
    std::vector<V3> v;
    for (int x = -1; x <= 1; x++)
      for (int y = -1; y <= 1; y++)
        for (int z = -1; z <= 1; z++)
          if (x || y || z) v.push_back(V3{x, y, z});
    return v;
  }();
  return d;
}

inline int64_t probe_coord(int64_t a, int64_t s, int64_t d) { return d < 0 ? a - 1 : (d > 0 ? a + s : a + (s >> 1)); }

struct Plan {
  Leaves leaves;
  std::vector<int64_t> same_src, ancestor_src;
  std::vector<int64_t> group_rows, group_ptr{0}, group_kids;
  std::vector<double> coarsened_min_rc;
};

void lineage(const Leaves& old, Plan& P) {
  const Leaves& nw = P.leaves;
  const size_t n = nw.n();
  LevelIndex oidx(old);
  const std::vector<int> olev = oidx.levels();
  P.same_src.assign(n, -1);
  P.ancestor_src.assign(n, -1);
  std::vector<size_t> orphans;
  for (size_t r = 0; r < n; r++) {
    P.same_src[r] = oidx.find(nw.level[r], nw.anchor[r]);
    if (P.same_src[r] >= 0) continue;
    for (int lo : olev) {  // an old leaf strictly coarser that contains it
      if (lo >= nw.level[r]) break;
      const int64_t s = old.size_at(lo);
      const int64_t hit =
          oidx.find(lo, V3{fdown(nw.anchor[r].x, s), fdown(nw.anchor[r].y, s), fdown(nw.anchor[r].z, s)});
      if (hit >= 0) {
        P.ancestor_src[r] = hit;
        break;
      }
    }
    if (P.ancestor_src[r] < 0) orphans.push_back(r);
  }
  // new leaves coarser than old ones: the old leaves inside each
  if (orphans.empty()) return;
  std::map<int, KeyMap> at;  // new level -> anchor key -> new row
  for (size_t r : orphans) at[nw.level[r]].put(key_of(nw.anchor[r]), (int64_t)r);
  std::map<int64_t, std::vector<int64_t>> kids;
  for (size_t r : orphans) kids[(int64_t)r];
  for (auto& kv : at) {
    const int64_t s = nw.size_at(kv.first);
    for (size_t o = 0; o < old.n(); o++) {
      if (old.level[o] <= kv.first) continue;
      const V3 a{fdown(old.anchor[o].x, s), fdown(old.anchor[o].y, s), fdown(old.anchor[o].z, s)};
      const int64_t r = kv.second.get(key_of(a));
      if (r >= 0) kids[r].push_back((int64_t)o);
    }
  }
  for (auto& kv : kids) {
    std::vector<int64_t> k = kv.second;
    std::sort(k.begin(), k.end());
    P.group_rows.push_back(kv.first);
    P.group_kids.insert(P.group_kids.end(), k.begin(), k.end());
    P.group_ptr.push_back((int64_t)P.group_kids.size());
  }
}

bool plan_layer(const Leaves& old, int new_layer, const double* rc, int nq, Plan& P, std::string& err) {
  const int64_t cpl = old.cpl;
  const int64_t z0 = new_layer * cpl, z1 = (new_layer + 1) * cpl, d_haz = 4 * cpl;
  Work w;
  static_cast<Leaves&>(w) = old;
  // 1. the new layer refined to the finest level
  while (true) {
    std::vector<size_t> rows;
    for (size_t i = 0; i < w.n(); i++)
      if (w.level[i] < w.depth && w.anchor[i].z < z1 && w.anchor[i].z + w.size(i) > z0) rows.push_back(i);
    if (rows.empty()) break;
    w.split(rows);
  }
  // 2. activated as powder
  for (size_t i = 0; i < w.n(); i++) {
    if (w.anchor[i].z >= z0 && w.anchor[i].z + w.size(i) <= z1) {
      if (w.level[i] != w.depth || w.active[i]) {
        err = "layer to activate is not a fresh finest-level layer";
        return false;
      }
      w.active[i] = 1;
    }
  }
  // 3. one level of coarsening for settled active octets below the HAZ,
  // gated on min r_c >= 0.9 over their quadrature points when a history is
  // given; active leaves are unchanged old rows here
  std::vector<double> rc_min;  // per old row, +inf off the active set
  if (rc) {
    rc_min.assign(old.n(), std::numeric_limits<double>::infinity());
    size_t e = 0;
    for (size_t r = 0; r < old.n(); r++) {
      if (!old.active[r]) continue;
      double m = rc[e * nq];
      for (int q = 1; q < nq; q++) m = std::min(m, rc[e * nq + q]);
      rc_min[r] = m;
      e++;
    }
  }
  {
    LevelIndex oidx(old);
    std::vector<size_t> elig;
    for (size_t i = 0; i < w.n(); i++) {
      if (!(w.active[i] && w.level[i] >= 1 && w.anchor[i].z + w.size(i) < z0 - d_haz)) continue;
      if (rc) {
        const int64_t o = oidx.find(w.level[i], w.anchor[i]);
        if (o < 0) {
          err = "coarsening candidate is not an old leaf";
          return false;
        }
        if (!(rc_min[o] >= 0.9)) continue;
      }
      elig.push_back(i);
    }
    std::vector<int> pl;
    std::vector<V3> pa;
    std::vector<std::vector<size_t>> g;
    w.octets(elig, pl, pa, g);
    if (!g.empty()) {
      std::vector<uint8_t> cons(g.size());
      for (size_t t = 0; t < g.size(); t++) cons[t] = w.consol[g[t][0]];
      w.merge(pl, pa, g, 1, cons);
    }
  }
  // 4. void octets collapsed as far as they go
  while (true) {
    std::vector<size_t> rows;
    for (size_t i = 0; i < w.n(); i++)
      if (!w.active[i]) rows.push_back(i);
    std::vector<int> pl;
    std::vector<V3> pa;
    std::vector<std::vector<size_t>> g;
    w.octets(rows, pl, pa, g);
    if (g.empty()) break;
    w.merge(pl, pa, g, 0, std::vector<uint8_t>(g.size(), 0));
  }
  // 5. 2:1 balance over faces, edges and vertices by a refinement ripple
  while (true) {
    LevelProbe lp(w);
    std::vector<size_t> rows;
    for (size_t i = 0; i < w.n(); i++) {
      const int64_t s = w.size(i);
      int worst = -1;
      for (const V3& d : dirs26()) {
        const V3 p{probe_coord(w.anchor[i].x, s, d.x), probe_coord(w.anchor[i].y, s, d.y),
                   probe_coord(w.anchor[i].z, s, d.z)};
        worst = std::max(worst, lp.level_at(p));
      }
      if (worst - w.level[i] >= 2) rows.push_back(i);
    }
    if (rows.empty()) break;
    w.split(rows);
  }
  const std::vector<size_t> o = canonical_order(w.level, w.anchor);
  Leaves& L = P.leaves;
  L.depth = w.depth;
  L.cpl = w.cpl;
  for (size_t r : o) {
    L.level.push_back(w.level[r]);
    L.anchor.push_back(w.anchor[r]);
    L.active.push_back(w.active[r]);
    L.consol.push_back(w.consol[r]);
  }
  lineage(old, P);
  if (rc) {
    for (size_t g = 0; g < P.group_rows.size(); g++) {
      if (!L.active[P.group_rows[g]]) continue;
      double m = std::numeric_limits<double>::infinity();
      for (int64_t t = P.group_ptr[g]; t < P.group_ptr[g + 1]; t++) m = std::min(m, rc_min[P.group_kids[t]]);
      P.coarsened_min_rc.push_back(m);
    }
  }
  return true;
}

// ---- radiating facets ---------------------------------------------------------
struct Facet {
  int64_t row, ox, oy, size;
};

void top_facets(const Leaves& f, std::vector<Facet>& out) {
  LevelIndex idx(f);
  // 0 open (no leaf there), 1 active, 2 void
  auto status = [&](int ell, const V3& a) -> int {
    const int64_t r = idx.find(ell, a);
    return r < 0 ? 0 : (f.active[r] ? 1 : 2);
  };
  for (size_t r = 0; r < f.n(); r++) {
    if (!f.active[r]) continue;
    const int ell = f.level[r];
    const int64_t s = f.size(r);
    const V3& a = f.anchor[r];
    const int64_t top = a.z + s;
    int cov = status(ell, V3{a.x, a.y, top});  // same-level neighbour above
    if (cov == 0 && ell > 0) {                  // one coarser, if aligned
      const int64_t ps = 2 * s;
      if (divisible(top, ps)) cov = status(ell - 1, V3{fdown(a.x, ps), fdown(a.y, ps), top});
    }
    if (cov == 1) continue;
    if (cov == 2 || ell >= f.depth) {
      out.push_back(Facet{(int64_t)r, 0, 0, s});
      continue;
    }
    // open: quarters against the finer level; no finer leaf at all means
    // the whole face is exterior
    const int64_t hs = s >> 1;
    int q[2][2];
    bool any = false;
    for (int i = 0; i < 2; i++)
      for (int j = 0; j < 2; j++) {
        q[i][j] = status(ell + 1, V3{a.x + i * hs, a.y + j * hs, top});
        any |= q[i][j] != 0;
      }
    if (!any) {
      out.push_back(Facet{(int64_t)r, 0, 0, s});
      continue;
    }
    for (int i = 0; i < 2; i++)
      for (int j = 0; j < 2; j++)
        if (q[i][j] != 1) out.push_back(Facet{(int64_t)r, i * hs, j * hs, hs});
  }
  std::stable_sort(out.begin(), out.end(), [](const Facet& x, const Facet& y) {
    if (x.row != y.row) return x.row < y.row;
    if (x.ox != y.ox) return x.ox < y.ox;
    return x.oy < y.oy;
  });
}

bool check_leaves(const st_leaves* L, std::string& err) {
  if (!L || L->n < 0 || (L->n > 0 && (!L->level || !L->anchor || !L->active))) {
    err = "invalid leaf table";
    return false;
  }
  for (int64_t i = 0; i < L->n; i++) {
    const V3 a{L->anchor[3 * i], L->anchor[3 * i + 1], L->anchor[3 * i + 2]};
    if (!packable(a) || L->level[i] > L->depth) {
      err = "leaf anchor out of the packable lattice range or level above depth";
      return false;
    }
  }
  return true;
}

st_tables* leaves_tables(st_tables* t, const Leaves& L) {
  std::vector<int8_t> lev(L.n());
  std::vector<int64_t> anc(3 * L.n());
  for (size_t i = 0; i < L.n(); i++) {
    lev[i] = (int8_t)L.level[i];
    anc[3 * i] = L.anchor[i].x;
    anc[3 * i + 1] = L.anchor[i].y;
    anc[3 * i + 2] = L.anchor[i].z;
  }
  t->put("level", ST_DT_I8, lev);
  t->put("anchor", ST_DT_I64, anc, {(int64_t)L.n(), 3});
  t->put("active", ST_DT_U8, L.active);
  t->put("init_consol", ST_DT_U8, L.consol);
  return t;
}

}  // namespace

extern "C" {

int st_tables_get(const st_tables* t, const char* name, int* dtype, int* ndim, int64_t* dims,
                  const void** data) {
  if (!t || !name) {
    st::set_error("st_tables_get: null argument");
    return ST_EINVAL;
  }
  for (auto& a : t->arrs) {
    if (a.name != name) continue;
    if (dtype) *dtype = a.dtype;
    if (ndim) *ndim = (int)a.dims.size();
    if (dims)
      for (size_t d = 0; d < a.dims.size() && d < 4; d++) dims[d] = a.dims[d];
    if (data) *data = a.bytes.empty() ? nullptr : a.bytes.data();
    return ST_OK;
  }
  st::set_error(std::string("st_tables_get: no array named ") + name);
  return ST_EINVAL;
}

void st_tables_free(st_tables* t) { delete t; }

int st_coarse_grid(int32_t depth, int32_t cpl, int64_t n_boxes, const int64_t* boxes,
                   const uint8_t* box_active, st_tables** out) {
  if (!out || (n_boxes > 0 && (!boxes || !box_active)) || depth < 0) {
    st::set_error("st_coarse_grid: invalid arguments");
    return ST_EINVAL;
  }
  const int64_t s0 = int64_t(1) << depth;
  std::vector<std::pair<int64_t, uint8_t>> cells;
  for (int64_t b = 0; b < n_boxes; b++) {
    const int64_t* B = boxes + 6 * b;
    for (int64_t x = B[0]; x < B[3]; x += s0)
      for (int64_t y = B[1]; y < B[4]; y += s0)
        for (int64_t z = B[2]; z < B[5]; z += s0) {
          const V3 a{x, y, z};
          if (!packable(a)) {
            st::set_error("st_coarse_grid: box outside the packable lattice range");
            return ST_EINVAL;
          }
          cells.emplace_back(key_of(a), box_active[b] ? 1 : 0);
        }
  }
  std::stable_sort(cells.begin(), cells.end(),
                   [](const std::pair<int64_t, uint8_t>& a, const std::pair<int64_t, uint8_t>& b) {
                     return a.first < b.first;
                   });
  Leaves L;
  L.depth = depth;
  L.cpl = cpl;
  for (size_t i = 0; i < cells.size(); i++) {
    if (i && cells[i].first == cells[i - 1].first) {
      if (cells[i].second != cells[i - 1].second) {
        st::set_error("st_coarse_grid: an active and a void box overlap");
        return ST_EINVAL;
      }
      continue;
    }
    L.level.push_back(0);
    L.anchor.push_back(v3_of(cells[i].first));
    L.active.push_back(cells[i].second);
    L.consol.push_back(cells[i].second);
  }
  *out = leaves_tables(new st_tables, L);
  return ST_OK;
}

int st_build_dofmap(const st_leaves* leaves, int64_t z_min, int dirichlet_bottom, st_tables** out) {
  std::string err;
  if (!out || !check_leaves(leaves, err)) {
    st::set_error("st_build_dofmap: " + (err.empty() ? std::string("null argument") : err));
    return ST_EINVAL;
  }
  const Leaves f = from_c(leaves);
  DofTables D;
  build_dofs(f, z_min, dirichlet_bottom != 0, D);
  std::vector<int64_t> verts(3 * D.vkeys.size());
  for (size_t v = 0; v < D.vkeys.size(); v++) {
    const V3 c = v3_of(D.vkeys[v]);
    verts[3 * v] = c.x;
    verts[3 * v + 1] = c.y;
    verts[3 * v + 2] = c.z;
  }
  st_tables* t = new st_tables;
  t->put("vertices", ST_DT_I64, verts, {(int64_t)D.vkeys.size(), 3});
  t->put("cell_verts", ST_DT_I32, D.cell_verts, {(int64_t)D.active_rows.size(), 8});
  t->put("active_rows", ST_DT_I64, D.active_rows);
  t->put("is_slave", ST_DT_U8, D.is_slave);
  t->put("is_dirichlet", ST_DT_U8, D.is_dir);
  t->put("slaves", ST_DT_I64, D.slaves);
  t->put("slave_ptr", ST_DT_I64, D.ptr);
  t->put("slave_masters", ST_DT_I64, D.masters);
  t->put("slave_weights", ST_DT_F64, D.weights);
  *out = t;
  return ST_OK;
}

int st_interface_faces(const st_leaves* leaves, st_tables** out) {
  std::string err;
  if (!out || !check_leaves(leaves, err)) {
    st::set_error("st_interface_faces: " + (err.empty() ? std::string("null argument") : err));
    return ST_EINVAL;
  }
  const Leaves f = from_c(leaves);
  std::vector<Facet> fs;
  top_facets(f, fs);
  std::vector<int64_t> rows(fs.size()), off(2 * fs.size()), size(fs.size());
  for (size_t i = 0; i < fs.size(); i++) {
    rows[i] = fs[i].row;
    off[2 * i] = fs[i].ox;
    off[2 * i + 1] = fs[i].oy;
    size[i] = fs[i].size;
  }
  st_tables* t = new st_tables;
  t->put("cell_rows", ST_DT_I64, rows);
  t->put("offset", ST_DT_I64, off, {(int64_t)fs.size(), 2});
  t->put("fsize", ST_DT_I64, size);
  *out = t;
  return ST_OK;
}

int st_plan_layer(const st_leaves* leaves, int32_t new_layer, const double* rc, int32_t nq,
                  st_tables** out) {
  std::string err;
  if (!out || !check_leaves(leaves, err) || (rc && nq <= 0)) {
    st::set_error("st_plan_layer: " + (err.empty() ? std::string("invalid arguments") : err));
    return ST_EINVAL;
  }
  const Leaves old = from_c(leaves);
  Plan P;
  if (!plan_layer(old, new_layer, rc, nq, P, err)) {
    st::set_error("st_plan_layer: " + err);
    return ST_EINVAL;
  }
  st_tables* t = leaves_tables(new st_tables, P.leaves);
  t->put("same_src", ST_DT_I64, P.same_src);
  t->put("ancestor_src", ST_DT_I64, P.ancestor_src);
  t->put("group_rows", ST_DT_I64, P.group_rows);
  t->put("group_ptr", ST_DT_I64, P.group_ptr);
  t->put("group_kids", ST_DT_I64, P.group_kids);
  t->put("coarsened_min_rc", ST_DT_F64, P.coarsened_min_rc);
  *out = t;
  return ST_OK;
}

int st_transfer_nodal(const st_leaves* old_leaves, const int64_t* old_verts, int64_t nv_old,
                      const int32_t* old_cell_verts, const int64_t* new_verts, int64_t nv_new,
                      const int64_t* slave_ptr, const int64_t* slaves, int64_t n_slaves,
                      const int64_t* slave_masters, const double* slave_weights, int32_t n_fields,
                      const double* fields_old, double T_0, double* fields_new, int8_t* source) {
  std::string err;
  if (!check_leaves(old_leaves, err) || (nv_old > 0 && !old_verts) || (nv_new > 0 && !new_verts) ||
      (n_fields > 0 && (!fields_old || !fields_new)) || n_fields < 0 ||
      (n_slaves > 0 && (!slave_ptr || !slaves || !slave_masters || !slave_weights))) {
    st::set_error("st_transfer_nodal: " + (err.empty() ? std::string("invalid arguments") : err));
    return ST_EINVAL;
  }
  const Leaves f = from_c(old_leaves);
  LevelIndex idx(f);
  const std::vector<int> levels = idx.levels();
  std::vector<int64_t> pos_of_row(f.n(), -1);
  int64_t na = 0;
  for (size_t r = 0; r < f.n(); r++)
    if (f.active[r]) pos_of_row[r] = na++;
  KeyMap old_at((size_t)nv_old);
  for (int64_t v = 0; v < nv_old; v++)
    old_at.put(key_of(V3{old_verts[3 * v], old_verts[3 * v + 1], old_verts[3 * v + 2]}), v);
  for (int64_t v = 0; v < nv_new; v++) {
    const V3 c{new_verts[3 * v], new_verts[3 * v + 1], new_verts[3 * v + 2]};
    const int64_t o = packable(c) ? old_at.get(key_of(c)) : -1;
    if (o >= 0) {  // surviving vertex: exact copy
      if (source) source[v] = 0;
      for (int k = 0; k < n_fields; k++) fields_new[k * nv_new + v] = fields_old[k * nv_old + o];
      continue;
    }
    int64_t row;
    V3 rel;
    if (hanging_host(f, idx, levels, c, &row, &rel)) {  // inside an old cell: trilinear
      if (source) source[v] = 1;
      const double s = (double)f.size((size_t)row);
      const double r[3] = {(double)rel.x / s, (double)rel.y / s, (double)rel.z / s};
      const int32_t* cv = old_cell_verts + pos_of_row[row] * 8;
      for (int k = 0; k < n_fields; k++) {
        double acc = 0.0;
        for (int cc = 0; cc < 8; cc++) acc += corner_weight(cc, r) * fields_old[k * nv_old + cv[cc]];
        fields_new[k * nv_new + v] = acc;
      }
      continue;
    }
    if (source) source[v] = 2;  // newly activated
    for (int k = 0; k < n_fields; k++) fields_new[k * nv_new + v] = T_0;
  }
  // slaves re-interpolated from their masters: numpy add.reduceat order
  // (first product, then the 8-lane pairwise sum of the rest)
  std::vector<double> prod;
  for (int k = 0; k < n_fields; k++) {
    double* x = fields_new + k * nv_new;
    for (int64_t s = 0; s < n_slaves; s++) {
      const int64_t b = slave_ptr[s], e = slave_ptr[s + 1];
      prod.resize((size_t)(e - b));
      for (int64_t t = b; t < e; t++) prod[t - b] = slave_weights[t] * x[slave_masters[t]];
      x[slaves[s]] = e - b == 0 ? 0.0 : prod[0] + np_pairwise(prod.data() + 1, e - b - 1);
    }
  }
  return ST_OK;
}

int st_transfer_history(const st_leaves* old_leaves, const st_leaves* new_leaves,
                        const int64_t* same_src, const int64_t* ancestor_src, int64_t n_groups,
                        const int64_t* group_rows, const int64_t* group_ptr,
                        const int64_t* group_kids, const double* rc_old, double* rc_new) {
  std::string err;
  if (!check_leaves(old_leaves, err) || !check_leaves(new_leaves, err) || !same_src ||
      !ancestor_src || (n_groups > 0 && (!group_rows || !group_ptr || !group_kids)) || !rc_new) {
    st::set_error("st_transfer_history: " + (err.empty() ? std::string("invalid arguments") : err));
    return ST_EINVAL;
  }
  const Leaves fo = from_c(old_leaves), fn = from_c(new_leaves);
  std::vector<int64_t> opos(fo.n(), -1);
  int64_t na = 0;
  for (size_t r = 0; r < fo.n(); r++)
    if (fo.active[r]) opos[r] = na++;
  std::map<int64_t, int64_t> group_of;
  for (int64_t g = 0; g < n_groups; g++) group_of[group_rows[g]] = g;
  int64_t e = 0;
  for (size_t r = 0; r < fn.n(); r++) {
    if (!fn.active[r]) continue;
    double* dst = rc_new + e * 8;
    e++;
    std::fill(dst, dst + 8, 0.0);
    const int64_t src = same_src[r];
    if (src >= 0) {  // same leaf: copy (fresh powder stays 0)
      if (fo.active[src]) std::copy(rc_old + opos[src] * 8, rc_old + opos[src] * 8 + 8, dst);
      continue;
    }
    const int64_t anc = ancestor_src[r];
    if (anc >= 0) {  // refined: the old octant holding this leaf's centre
      if (fo.active[anc]) {
        const int64_t sa = fo.size((size_t)anc), sn = fn.size(r);
        const V3& a = fo.anchor[anc];
        const V3& b = fn.anchor[r];
        const int ox = (int)fdiv((b.x + sn / 2 - a.x) * 2, sa), oy = (int)fdiv((b.y + sn / 2 - a.y) * 2, sa),
                  oz = (int)fdiv((b.z + sn / 2 - a.z) * 2, sa);
        const double v = rc_old[opos[anc] * 8 + ox * 4 + oy * 2 + oz];
        std::fill(dst, dst + 8, v);
      }
      continue;
    }
    auto it = group_of.find((int64_t)r);
    if (it == group_of.end()) {
      st::set_error("st_transfer_history: new leaf without lineage");
      return ST_EINVAL;
    }
    const int64_t g = it->second;
    if (group_ptr[g + 1] - group_ptr[g] != 8) {
      st::set_error("st_transfer_history: active coarsening must merge exactly one level");
      return ST_EINVAL;
    }
    const int64_t sp = fn.size(r);
    for (int64_t t = group_ptr[g]; t < group_ptr[g + 1]; t++) {
      const int64_t kid = group_kids[t];
      if (!fo.active[kid]) {
        st::set_error("st_transfer_history: active coarsening of a void child");
        return ST_EINVAL;
      }
      const V3& a = fo.anchor[kid];
      const V3& b = fn.anchor[r];
      const int ox = (int)fdiv((a.x - b.x) * 2, sp), oy = (int)fdiv((a.y - b.y) * 2, sp),
                oz = (int)fdiv((a.z - b.z) * 2, sp);
      dst[ox * 4 + oy * 2 + oz] = np_pairwise(rc_old + opos[kid] * 8, 8) / 8.0;
    }
  }
  return ST_OK;
}

int st_host_distribute(int64_t n_slaves, const int64_t* slaves, const int64_t* slave_ptr,
                       const int64_t* slave_masters, const double* slave_weights, double* values) {
  if (n_slaves < 0 || (n_slaves > 0 && (!slaves || !slave_ptr || !slave_masters || !slave_weights || !values))) {
    st::set_error("st_host_distribute: invalid arguments");
    return ST_EINVAL;
  }
  // every product first (masters are never slaves), then each segment as
  // numpy's add.reduceat sums it
  std::vector<double> prod;
  for (int64_t s = 0; s < n_slaves; s++) {
    const int64_t b = slave_ptr[s], e = slave_ptr[s + 1];
    if (e <= b) continue;
    prod.resize((size_t)(e - b));
    for (int64_t t = b; t < e; t++) prod[t - b] = slave_weights[t] * values[slave_masters[t]];
    values[slaves[s]] = prod[0] + np_pairwise(prod.data() + 1, e - b - 1);
  }
  return ST_OK;
}

int st_host_condense(int64_t n_slaves, const int64_t* slaves, const int64_t* slave_ptr,
                     const int64_t* slave_masters, const double* slave_weights, double* values) {
  if (n_slaves < 0 || (n_slaves > 0 && (!slaves || !slave_ptr || !slave_masters || !slave_weights || !values))) {
    st::set_error("st_host_condense: invalid arguments");
    return ST_EINVAL;
  }
  // transpose of distribute, accumulated in CSR order (numpy add.at order)
  for (int64_t s = 0; s < n_slaves; s++) {
    const double v = values[slaves[s]];
    for (int64_t t = slave_ptr[s]; t < slave_ptr[s + 1]; t++) values[slave_masters[t]] += slave_weights[t] * v;
  }
  for (int64_t s = 0; s < n_slaves; s++) values[slaves[s]] = 0.0;
  return ST_OK;
}

}  // extern "C"
