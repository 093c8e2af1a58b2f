// Host gate DAG of TfheContext, native: node store,
// constant/duplicate elision, hash-consing, MUX lowering, full-adder fusion
// into 3-input bootstraps (majority, XOR3), live-handle counts, the
// live-gate filter of a flush and the carry-save popcount networks of the
// opt-in popcount replacement (csa; paper_1806_03461_b200/popcount.py).  The Python context (backend.py) keeps the
// reference contract (handles, GateStats, scopes, errors) and the engine
// calls; every gate of the reference API lands here once.
//
// Binding: the raw CPython API (vectorcall-style METH_FASTCALL methods, numpy
// C API for the bulk arrays), so one gate costs one cheap native call rather
// than a pybind11 dispatch (~0.3 us) — the host DAG build is on the critical
// path of a BNN's first evaluation.
//
// Refs are (node << 1) | not_flag; node 0 is the constant 0 (ref 0 = false,
// ref 1 = true).  Node operands: AND / MUX / MAJ store refs; XOR / XOR3 store
// node << 1 and push NOT flags to the output ref.  Node n owns logical pool
// slot n - 1.
#define PY_SSIZE_T_CLEAN
#include <Python.h>
#define NPY_NO_DEPRECATED_API NPY_1_7_API_VERSION
#include <numpy/arrayobject.h>

#include <algorithm>
#include <array>
#include <cstdint>
#include <deque>
#include <tuple>
#include <vector>

namespace {

struct IndexErr {};  // node id out of range -> IndexError

enum Op : int8_t { CONST = 0, INPUT = 1, AND = 2, XOR = 3, MUX = 4, MAJ = 5, XOR3 = 6 };
enum State : uint8_t { PENDING = 0, DONE = 1, DORMANT = 2 };
// gate kinds of the reference API (hebnn.backend AND/OR/XOR/XNOR)
enum Kind : int { K_AND = 0, K_OR = 1, K_XOR = 2, K_XNOR = 3 };

// Hash-consing table: open addressing with linear probing over a flat,
// power-of-two array (load <= 1/2), keyed by (op, a, b, c) refs.  A flat
// table keeps a lookup at ~one cache line; a node-based std::unordered_map
// cost ~0.6 us per gate on the cfg2l DAG (565k nodes).
class CseTable {
  public:
    CseTable() : slots_(1u << 12) {}

    // node id of the key, or -1
    int64_t find(int8_t op, int64_t a, int64_t b, int64_t c) const {
        const size_t mask = slots_.size() - 1;
        for (size_t i = hash(op, a, b, c) & mask;; i = (i + 1) & mask) {
            const Slot &e = slots_[i];
            if (e.node < 0) return -1;
            if (e.op == op && e.a == a && e.b == b && e.c == c) return e.node;
        }
    }

    void insert(int8_t op, int64_t a, int64_t b, int64_t c, int64_t node) {
        if (2 * (used_ + 1) > slots_.size()) grow();
        place(Slot{a, b, c, node, op});
        used_++;
    }

  private:
    struct Slot {
        int64_t a = 0, b = 0, c = 0;
        int64_t node = -1;
        int8_t op = 0;
    };
    std::vector<Slot> slots_;
    size_t used_ = 0;

    static size_t hash(int8_t op, int64_t a, int64_t b, int64_t c) {
        uint64_t h = (uint64_t)a * 0x9E3779B97F4A7C15ull;
        h ^= (uint64_t)b * 0xC2B2AE3D27D4EB4Full + (h >> 29);
        h ^= (uint64_t)c * 0x165667B19E3779F9ull + (uint64_t)op + (h >> 32);
        h *= 0xD6E8FEB86659FD93ull;
        return (size_t)(h ^ (h >> 32));
    }
    void place(const Slot &s) {
        const size_t mask = slots_.size() - 1;
        size_t i = hash(s.op, s.a, s.b, s.c) & mask;
        while (slots_[i].node >= 0) i = (i + 1) & mask;
        slots_[i] = s;
    }
    void grow() {
        std::vector<Slot> old(slots_.size() * 2);
        old.swap(slots_);
        for (const Slot &s : old)
            if (s.node >= 0) place(s);
    }
};

class Dag {
  public:
    Dag() { push(CONST, 0, 0, 0, 0, DONE); }

    int64_t size() const { return (int64_t)op_.size(); }
    int64_t pending_count() const { return (int64_t)pending_.size(); }

    int64_t add_input() { return push(INPUT, 0, 0, 0, 0, DONE); }

    // ref of a 2-input gate of the reference API; one live handle is counted on it
    int64_t gate(int kind, int64_t ra, int64_t rb) {
        check_ref(ra);
        check_ref(rb);
        int64_t r;
        switch (kind) {
            case K_AND: r = mk_and(ra, rb); break;
            case K_OR: r = mk_and(ra ^ 1, rb ^ 1) ^ 1; break;
            case K_XOR: r = mk_xor(ra, rb); break;
            default: r = mk_xor(ra, rb) ^ 1; break;
        }
        hcnt_[r >> 1]++;
        return r;
    }
    int64_t mux(int64_t rs, int64_t ra, int64_t rb) {
        check_ref(rs);
        check_ref(ra);
        check_ref(rb);
        const int64_t r = mk_mux(rs, ra, rb);
        hcnt_[r >> 1]++;
        return r;
    }

    // Carry-save popcount of the literals refs[0..n): output refs, LSB first, whose
    // values are the binary digits of the number of true literals; one live handle is
    // counted on each.  Column by column, three bits of a weight go through a full adder
    // (XOR3 + MAJ: two bootstraps), a last pair through a half adder; sums rejoin the
    // back of their column and carries the back of the next one (breadth-first, so the
    // depth stays ~log_1.5 n).  About 2n bootstraps instead of the ~3n of a tree of
    // ripple-carry adders (reference circuits.py:189-216); the digits of a sum are
    // unique, so any consumer sees the same plaintexts.
    //
    // block >= 3: shared first stage.  Every leaf node gets an ordinal the first time a
    // popcount sees it; the literals are sorted by ordinal and cut into blocks of `block`
    // consecutive ordinals, and inside a block full adders (only: they are what removes
    // bits) take the first three bits of a weight until fewer than three are left.  The
    // blocks are the same for every popcount over the same leaves (the neurons of a
    // layer sum subsets of one input vector), so hash-consing computes a block's adders
    // once for all of them; MAJ is stored with its first operand positive (it is
    // self-dual), so the popcounts of negated literals share them too.
    std::vector<int64_t> csa(const int64_t *refs, int64_t n, int64_t block) {
        for (int64_t i = 0; i < n; i++) check_ref(refs[i]);
        std::vector<std::deque<int64_t>> cols(1);
        auto fa_front = [this](std::vector<std::deque<int64_t>> &c, size_t w) {
            const int64_t x = c[w][0], y = c[w][1], z = c[w][2];
            c[w].erase(c[w].begin(), c[w].begin() + 3);
            c[w].push_back(sum3(x, y, z));
            if (c.size() <= w + 1) c.emplace_back();
            c[w + 1].push_back(mk_maj(x, y, z));
        };
        if (block >= 3) {
            if (ord_.size() < op_.size()) ord_.resize(op_.size(), 0);
            std::vector<std::pair<int64_t, int64_t>> lit;  // (ordinal, literal)
            lit.reserve((size_t)n);
            for (int64_t i = 0; i < n; i++) {
                int64_t &o = ord_[refs[i] >> 1];
                if (o == 0) o = ++next_ord_;
                lit.emplace_back(o - 1, refs[i]);
            }
            std::sort(lit.begin(), lit.end());
            std::vector<std::deque<int64_t>> loc;
            for (size_t i = 0; i < lit.size();) {
                const int64_t blk = lit[i].first / block;
                loc.assign(1, {});
                for (; i < lit.size() && lit[i].first / block == blk; i++) loc[0].push_back(lit[i].second);
                for (size_t w = 0; w < loc.size(); w++)
                    while (loc[w].size() >= 3) fa_front(loc, w);
                if (cols.size() < loc.size()) cols.resize(loc.size());
                for (size_t w = 0; w < loc.size(); w++) cols[w].insert(cols[w].end(), loc[w].begin(), loc[w].end());
            }
        } else {
            cols[0].assign(refs, refs + n);
        }
        // global compression: in every column the three shallowest bits (DAG level) go
        // through the next full adder, so late carries are not waited for by early bits
        // (depth ~ the Wallace stages plus one carry chain over the word)
        using Item = std::tuple<int32_t, int64_t, int64_t>;  // (level, arrival, literal)
        auto later = [](const Item &p, const Item &q) { return p > q; };
        std::vector<std::vector<Item>> heap(cols.size());
        int64_t seq = 0;
        auto push = [&](size_t w, int64_t r) {
            if (heap.size() <= w) heap.resize(w + 1);
            heap[w].emplace_back(lv(r), seq++, r);
            std::push_heap(heap[w].begin(), heap[w].end(), later);
        };
        auto pop = [&](size_t w) {
            std::pop_heap(heap[w].begin(), heap[w].end(), later);
            const int64_t r = std::get<2>(heap[w].back());
            heap[w].pop_back();
            return r;
        };
        for (size_t w = 0; w < cols.size(); w++)
            for (int64_t r : cols[w]) push(w, r);
        std::vector<int64_t> out;
        for (size_t w = 0; w < heap.size(); w++) {
            while (heap[w].size() >= 3) {
                const int64_t x = pop(w), y = pop(w), z = pop(w);
                push(w, sum3(x, y, z));
                push(w + 1, mk_maj(x, y, z));
            }
            if (heap[w].size() == 2) {
                const int64_t x = pop(w), y = pop(w);
                push(w, mk_xor(x, y));
                push(w + 1, mk_and(x, y));
            }
            if (heap[w].empty()) break;  // a vanished digit (degenerate operands): the caller falls back
            out.push_back(pop(w));
        }
        for (int64_t r : out) hcnt_[r >> 1]++;
        return out;
    }

    void hinc(int64_t n) { hcnt_[check(n)]++; }
    void hdec(int64_t n) { hcnt_[check(n)]--; }
    int32_t hcount(int64_t n) const { return hcnt_[check(n)]; }
    int op(int64_t n) const { return op_[check(n)]; }
    bool is_done(int64_t n) const { return state_[check(n)] == DONE; }
    bool is_dormant(int64_t n) const { return state_[check(n)] == DORMANT; }

    // dormant node (and its dormant operands) back to pending
    void revive(int64_t n) {
        std::vector<int64_t> stack{check(n)};
        while (!stack.empty()) {
            const int64_t m = stack.back();
            stack.pop_back();
            if (state_[m] != DORMANT) continue;
            state_[m] = PENDING;
            pending_.push_back(m);
            if (op_[m] != INPUT)
                for (int64_t r : {a_[m], b_[m], c_[m]}) stack.push_back(r >> 1);
        }
    }

    // pending nodes reachable from live handles through pending operands, in
    // pending order; with take: the rest become dormant and pending empties
    std::vector<int64_t> live(bool take) {
        const uint32_t ep = ++epoch_;
        if (mark_.size() < op_.size()) mark_.resize(op_.size(), 0);
        std::vector<int64_t> stack;
        for (int64_t n : pending_)
            if (hcnt_[n] > 0) stack.push_back(n);
        while (!stack.empty()) {
            const int64_t n = stack.back();
            stack.pop_back();
            if (mark_[n] == ep) continue;
            mark_[n] = ep;
            if (op_[n] == INPUT) continue;
            for (int64_t r : {a_[n], b_[n], c_[n]}) {
                const int64_t m = r >> 1;
                if (state_[m] == PENDING && mark_[m] != ep) stack.push_back(m);
            }
        }
        std::vector<int64_t> out;
        out.reserve(pending_.size());
        for (int64_t n : pending_) {
            if (mark_[n] == ep) {
                out.push_back(n);
            } else if (take) {
                state_[n] = DORMANT;
            }
        }
        if (take) pending_.clear();
        return out;
    }

    const std::vector<int64_t> &pending() const { return pending_; }

    // pending nodes taken by live(true) but not run: back into the pending list
    void requeue(const int64_t *ids, int64_t n) {
        for (int64_t i = 0; i < n; i++)
            if (state_[check(ids[i])] != PENDING) throw IndexErr{};
        pending_.insert(pending_.end(), ids, ids + n);
    }

    void mark_done(const int64_t *ids, int64_t n) {
        for (int64_t i = 0; i < n; i++) check(ids[i]);
        for (int64_t i = 0; i < n; i++) state_[ids[i]] = DONE;
    }

    // node fields of ids: op int8, a, b, c int64 refs, lvl int64
    void gather(const int64_t *ids, int64_t n, int8_t *o, int64_t *a, int64_t *b, int64_t *c, int64_t *l) const {
        for (int64_t i = 0; i < n; i++) {
            const int64_t k = check(ids[i]);
            o[i] = op_[k];
            a[i] = a_[k];
            b[i] = b_[k];
            c[i] = c_[k];
            l[i] = lvl_[k];
        }
    }

  private:
    std::vector<int8_t> op_;
    std::vector<int64_t> a_, b_, c_;
    std::vector<int32_t> lvl_;
    std::vector<uint8_t> state_;
    std::vector<int32_t> hcnt_;
    std::vector<int64_t> pending_;
    std::vector<uint32_t> mark_;
    uint32_t epoch_ = 0;
    CseTable cse_;
    std::vector<int64_t> ord_;  // csa: leaf ordinal + 1 of a node (0: none yet)
    int64_t next_ord_ = 0;

    int64_t check(int64_t n) const {
        if (n < 0 || n >= (int64_t)op_.size()) throw IndexErr{};
        return n;
    }
    void check_ref(int64_t r) const { check(r >> 1); }

    int64_t push(int8_t op, int64_t a, int64_t b, int64_t c, int32_t lvl, uint8_t state) {
        const int64_t n = (int64_t)op_.size();
        op_.push_back(op);
        a_.push_back(a);
        b_.push_back(b);
        c_.push_back(c);
        lvl_.push_back(lvl);
        state_.push_back(state);
        hcnt_.push_back(0);
        return n;
    }

    // CSE lookup or a new pending node; dormant hits and dormant operands revive
    int64_t node(int8_t op, int64_t a, int64_t b, int64_t c, int32_t lvl) {
        const int64_t hit = cse_.find(op, a, b, c);
        if (hit >= 0) {
            if (state_[hit] == DORMANT) revive(hit);
            return hit;
        }
        for (int64_t r : {a, b, c})
            if (state_[r >> 1] == DORMANT) revive(r >> 1);
        const int64_t n = push(op, a, b, c, lvl, PENDING);
        pending_.push_back(n);
        cse_.insert(op, a, b, c, n);
        return n;
    }

    int32_t lv(int64_t r) const { return lvl_[r >> 1]; }

    int64_t mk_and(int64_t ra, int64_t rb) {
        if ((ra >> 1) == 0) return (ra & 1) ? rb : 0;
        if ((rb >> 1) == 0) return (rb & 1) ? ra : 0;
        if (ra == rb) return ra;
        if (ra == (rb ^ 1)) return 0;
        if (ra & rb & 1) {  // OR(u, v): a full adder's carry folds into one majority
            const int64_t m = try_maj(ra ^ 1, rb ^ 1);
            if (m >= 0) return m ^ 1;
        }
        if (ra > rb) std::swap(ra, rb);
        return node(AND, ra, rb, 0, 1 + std::max(lv(ra), lv(rb))) << 1;
    }

    int64_t mk_xor(int64_t ra, int64_t rb) {
        const int64_t neg = (ra ^ rb) & 1;
        int64_t na = ra >> 1, nb = rb >> 1;
        if (na == 0) return rb ^ (ra & 1);
        if (nb == 0) return ra ^ (rb & 1);
        if (na == nb) return neg;
        // XOR(XOR(p, q), r) = XOR3(p, q, r): one bootstrap at a lower level
        // (the deeper XOR operand is absorbed)
        bool xa = op_[na] == XOR, xb = op_[nb] == XOR;
        if (xa || xb) {
            if (xa && xb && lvl_[nb] > lvl_[na]) xa = false;
            const int64_t x = xa ? na : nb, y = xa ? nb : na;
            const int64_t p = a_[x] >> 1, q = b_[x] >> 1;
            if (y == p) return (q << 1) | neg;
            if (y == q) return (p << 1) | neg;
            return mk_xor3(p, q, y) | neg;
        }
        if (na > nb) std::swap(na, nb);
        return (node(XOR, na << 1, nb << 1, 0, 1 + std::max(lvl_[na], lvl_[nb])) << 1) | neg;
    }

    // ref of OR(u, v) as MAJ(x, y, z) when {u, v} = {AND(x, y), AND(XOR(x, y), z)}
    // (reference circuits.py:101-108 builds a full adder's carry this way); -1 if not
    int64_t try_maj(int64_t u, int64_t v) {
        for (int t = 0; t < 2; t++) {
            const int64_t g = t ? v : u, h = t ? u : v;
            if ((g | h) & 1) continue;
            const int64_t G = g >> 1, H = h >> 1;
            if (op_[G] != AND || op_[H] != AND) continue;
            const int64_t x = a_[G], y = b_[G];
            for (int s = 0; s < 2; s++) {
                const int64_t w = s ? b_[H] : a_[H], z = s ? a_[H] : b_[H];
                const int64_t W = w >> 1;
                if (op_[W] != XOR || (w & 1) != ((x ^ y) & 1)) continue;
                const int64_t p = a_[W] >> 1, q = b_[W] >> 1;
                if ((p == (x >> 1) && q == (y >> 1)) || (p == (y >> 1) && q == (x >> 1))) return mk_maj(x, y, z);
            }
        }
        return -1;
    }

    int64_t mk_maj(int64_t x, int64_t y, int64_t z) {
        const std::array<std::array<int64_t, 3>, 3> pairs{{{x, y, z}, {x, z, y}, {y, z, x}}};
        for (const auto &t : pairs) {
            if (t[0] == t[1]) return t[0];
            if (t[0] == (t[1] ^ 1)) return t[2];
        }
        const std::array<std::array<int64_t, 3>, 3> consts{{{x, y, z}, {y, x, z}, {z, x, y}}};
        for (const auto &t : consts) {
            if ((t[0] >> 1) == 0)  // MAJ(0, q, r) = AND(q, r); MAJ(1, q, r) = OR(q, r)
                return (t[0] & 1) ? (mk_and(t[1] ^ 1, t[2] ^ 1) ^ 1) : mk_and(t[1], t[2]);
        }
        std::array<int64_t, 3> s{x, y, z};
        std::sort(s.begin(), s.end());
        // self-dual: MAJ(~a, ~b, ~c) = ~MAJ(a, b, c); stored with the first operand positive
        const int64_t neg = s[0] & 1;
        if (neg) s = {s[0] ^ 1, s[1] ^ 1, s[2] ^ 1};
        return (node(MAJ, s[0], s[1], s[2], 1 + std::max({lv(s[0]), lv(s[1]), lv(s[2])})) << 1) | neg;
    }

    int64_t mk_xor3(int64_t p, int64_t q, int64_t r) {
        std::array<int64_t, 3> s{p, q, r};
        std::sort(s.begin(), s.end());
        return node(XOR3, s[0] << 1, s[1] << 1, s[2] << 1,
                    1 + std::max({lvl_[s[0]], lvl_[s[1]], lvl_[s[2]]})) << 1;
    }

    // literal a ^ b ^ c: one XOR3 node when the three nodes are distinct non-constants
    int64_t sum3(int64_t a, int64_t b, int64_t c) {
        const int64_t na = a >> 1, nb = b >> 1, nc = c >> 1;
        if (na == 0 || nb == 0 || nc == 0 || na == nb || na == nc || nb == nc) return mk_xor(mk_xor(a, b), c);
        return mk_xor3(na, nb, nc) | ((a ^ b ^ c) & 1);
    }

    int64_t mk_mux(int64_t rs, int64_t ra, int64_t rb) {
        if (rs & 1) {  // MUX(~s, a, b) = MUX(s, b, a)
            rs ^= 1;
            std::swap(ra, rb);
        }
        if ((rs >> 1) == 0) return (rs & 1) ? ra : rb;  // constant selector (only after elision)
        if (ra == rb) return ra;
        if ((ra >> 1) == 0 && (rb >> 1) == 0) return (ra & 1) ? rs : (rs ^ 1);  // both constant, a != b
        if ((ra >> 1) == 0)  // s ? 1 : b = s OR b;  s ? 0 : b = ~s AND b
            return (ra & 1) ? (mk_and(rs ^ 1, rb ^ 1) ^ 1) : mk_and(rs ^ 1, rb);
        if ((rb >> 1) == 0)  // s ? a : 1 = ~s OR a;  s ? a : 0 = s AND a
            return (rb & 1) ? (mk_and(rs, ra ^ 1) ^ 1) : mk_and(rs, ra);
        if (ra == (rb ^ 1)) return mk_xor(rs, ra) ^ 1;          // s ? a : ~a = XNOR(s, a)
        if (ra == rs) return mk_and(rs ^ 1, rb ^ 1) ^ 1;         // s ? s : b = s OR b
        if (ra == (rs ^ 1)) return mk_and(rs ^ 1, rb);           // s ? ~s : b = ~s AND b
        if (rb == rs) return mk_and(rs, ra);                     // s ? a : s = s AND a
        if (rb == (rs ^ 1)) return mk_and(rs, ra ^ 1) ^ 1;       // s ? a : ~s = ~s OR a
        return node(MUX, rs, ra, rb, 1 + std::max({lv(rs), lv(ra), lv(rb)})) << 1;
    }
};

}  // namespace

// ---------------------------------------------------------------------------
// CPython binding
// ---------------------------------------------------------------------------
namespace {

struct PyDag {
    PyObject_HEAD
    Dag *dag;
};

PyObject *index_error() {
    PyErr_SetString(PyExc_IndexError, "gate DAG: node id out of range");
    return nullptr;
}

bool args_i64(PyObject *const *args, Py_ssize_t nargs, Py_ssize_t want, int64_t *out, const char *name) {
    if (nargs != want) {
        PyErr_Format(PyExc_TypeError, "Dag.%s() takes %zd arguments (%zd given)", name, want, nargs);
        return false;
    }
    for (Py_ssize_t i = 0; i < want; i++) {
        const long long v = PyLong_AsLongLong(args[i]);
        if (v == -1 && PyErr_Occurred()) return false;
        out[i] = (int64_t)v;
    }
    return true;
}

PyObject *to_array(const std::vector<int64_t> &v) {
    npy_intp dims[1] = {(npy_intp)v.size()};
    PyObject *arr = PyArray_SimpleNew(1, dims, NPY_INT64);
    if (arr && !v.empty()) std::copy(v.begin(), v.end(), (int64_t *)PyArray_DATA((PyArrayObject *)arr));
    return arr;
}

// int64 C-contiguous view of a 1-d array-like (new reference)
PyArrayObject *as_ids(PyObject *obj) {
    return (PyArrayObject *)PyArray_FROMANY(obj, NPY_INT64, 1, 1, NPY_ARRAY_IN_ARRAY | NPY_ARRAY_FORCECAST);
}

PyObject *Dag_new(PyTypeObject *type, PyObject *, PyObject *) {
    PyDag *self = (PyDag *)type->tp_alloc(type, 0);
    if (!self) return nullptr;
    try {
        self->dag = new Dag();
    } catch (const std::bad_alloc &) {
        Py_DECREF(self);
        return PyErr_NoMemory();
    }
    return (PyObject *)self;
}

void Dag_dealloc(PyDag *self) {
    delete self->dag;
    Py_TYPE(self)->tp_free((PyObject *)self);
}

#define HB_DAG_TRY(expr)                     \
    try {                                    \
        expr;                                \
    } catch (const IndexErr &) {             \
        return index_error();                \
    } catch (const std::bad_alloc &) {       \
        return PyErr_NoMemory();             \
    }

PyObject *Dag_size(PyDag *self, PyObject *) { return PyLong_FromLongLong(self->dag->size()); }
PyObject *Dag_pending_count(PyDag *self, PyObject *) { return PyLong_FromLongLong(self->dag->pending_count()); }
PyObject *Dag_add_input(PyDag *self, PyObject *) {
    int64_t r;
    HB_DAG_TRY(r = self->dag->add_input());
    return PyLong_FromLongLong(r);
}

PyObject *Dag_gate(PyDag *self, PyObject *const *args, Py_ssize_t nargs) {
    int64_t v[3];
    if (!args_i64(args, nargs, 3, v, "gate")) return nullptr;
    int64_t r;
    HB_DAG_TRY(r = self->dag->gate((int)v[0], v[1], v[2]));
    return PyLong_FromLongLong(r);
}

PyObject *Dag_mux(PyDag *self, PyObject *const *args, Py_ssize_t nargs) {
    int64_t v[3];
    if (!args_i64(args, nargs, 3, v, "mux")) return nullptr;
    int64_t r;
    HB_DAG_TRY(r = self->dag->mux(v[0], v[1], v[2]));
    return PyLong_FromLongLong(r);
}

// one-argument node methods
template <typename F>
PyObject *node_call(PyDag *self, PyObject *arg, F f) {
    const long long n = PyLong_AsLongLong(arg);
    if (n == -1 && PyErr_Occurred()) return nullptr;
    HB_DAG_TRY(return f(self->dag, (int64_t)n));
}

PyObject *Dag_hinc(PyDag *self, PyObject *arg) {
    return node_call(self, arg, [](Dag *d, int64_t n) { d->hinc(n); Py_RETURN_NONE; });
}
PyObject *Dag_hdec(PyDag *self, PyObject *arg) {
    return node_call(self, arg, [](Dag *d, int64_t n) { d->hdec(n); Py_RETURN_NONE; });
}
PyObject *Dag_hcount(PyDag *self, PyObject *arg) {
    return node_call(self, arg, [](Dag *d, int64_t n) { return PyLong_FromLong(d->hcount(n)); });
}
PyObject *Dag_op(PyDag *self, PyObject *arg) {
    return node_call(self, arg, [](Dag *d, int64_t n) { return PyLong_FromLong(d->op(n)); });
}
PyObject *Dag_is_done(PyDag *self, PyObject *arg) {
    return node_call(self, arg, [](Dag *d, int64_t n) { return PyBool_FromLong(d->is_done(n)); });
}
PyObject *Dag_is_dormant(PyDag *self, PyObject *arg) {
    return node_call(self, arg, [](Dag *d, int64_t n) { return PyBool_FromLong(d->is_dormant(n)); });
}
PyObject *Dag_revive(PyDag *self, PyObject *arg) {
    return node_call(self, arg, [](Dag *d, int64_t n) { d->revive(n); Py_RETURN_NONE; });
}

PyObject *Dag_live(PyDag *self, PyObject *args, PyObject *kwds) {
    static const char *kwlist[] = {"take", nullptr};
    int take = 0;
    if (!PyArg_ParseTupleAndKeywords(args, kwds, "p", (char **)kwlist, &take)) return nullptr;
    HB_DAG_TRY(return to_array(self->dag->live(take != 0)));
}

PyObject *Dag_pending(PyDag *self, PyObject *) { HB_DAG_TRY(return to_array(self->dag->pending())); }

PyObject *Dag_mark_done(PyDag *self, PyObject *arg) {
    PyArrayObject *ids = as_ids(arg);
    if (!ids) return nullptr;
    try {
        self->dag->mark_done((const int64_t *)PyArray_DATA(ids), (int64_t)PyArray_SIZE(ids));
    } catch (const IndexErr &) {
        Py_DECREF(ids);
        return index_error();
    }
    Py_DECREF(ids);
    Py_RETURN_NONE;
}

PyObject *Dag_requeue(PyDag *self, PyObject *arg) {
    PyArrayObject *ids = as_ids(arg);
    if (!ids) return nullptr;
    try {
        self->dag->requeue((const int64_t *)PyArray_DATA(ids), (int64_t)PyArray_SIZE(ids));
    } catch (const IndexErr &) {
        Py_DECREF(ids);
        PyErr_SetString(PyExc_IndexError, "gate DAG: requeue of a node that is not pending");
        return nullptr;
    }
    Py_DECREF(ids);
    Py_RETURN_NONE;
}

PyObject *Dag_csa(PyDag *self, PyObject *args) {
    PyObject *arg = nullptr;
    long long block = 0;
    if (!PyArg_ParseTuple(args, "O|L", &arg, &block)) return nullptr;
    PyArrayObject *ids = as_ids(arg);
    if (!ids) return nullptr;
    PyObject *res = nullptr;
    try {
        res = to_array(self->dag->csa((const int64_t *)PyArray_DATA(ids), (int64_t)PyArray_SIZE(ids), (int64_t)block));
    } catch (const IndexErr &) {
        Py_DECREF(ids);
        return index_error();
    } catch (const std::bad_alloc &) {
        Py_DECREF(ids);
        return PyErr_NoMemory();
    }
    Py_DECREF(ids);
    return res;
}

PyObject *Dag_gather(PyDag *self, PyObject *arg) {
    PyArrayObject *ids = as_ids(arg);
    if (!ids) return nullptr;
    npy_intp dims[1] = {PyArray_SIZE(ids)};
    PyObject *o = PyArray_SimpleNew(1, dims, NPY_INT8);
    PyObject *a = PyArray_SimpleNew(1, dims, NPY_INT64), *b = PyArray_SimpleNew(1, dims, NPY_INT64);
    PyObject *c = PyArray_SimpleNew(1, dims, NPY_INT64), *l = PyArray_SimpleNew(1, dims, NPY_INT64);
    PyObject *res = nullptr;
    if (o && a && b && c && l) {
        try {
            self->dag->gather((const int64_t *)PyArray_DATA(ids), (int64_t)dims[0],
                              (int8_t *)PyArray_DATA((PyArrayObject *)o), (int64_t *)PyArray_DATA((PyArrayObject *)a),
                              (int64_t *)PyArray_DATA((PyArrayObject *)b), (int64_t *)PyArray_DATA((PyArrayObject *)c),
                              (int64_t *)PyArray_DATA((PyArrayObject *)l));
            res = PyTuple_Pack(5, o, a, b, c, l);
        } catch (const IndexErr &) {
            index_error();
        }
    }
    Py_DECREF(ids);
    Py_XDECREF(o);
    Py_XDECREF(a);
    Py_XDECREF(b);
    Py_XDECREF(c);
    Py_XDECREF(l);
    return res;
}

PyMethodDef Dag_methods[] = {
    {"size", (PyCFunction)Dag_size, METH_NOARGS, "number of nodes (node 0 is the constant)"},
    {"pending_count", (PyCFunction)Dag_pending_count, METH_NOARGS, "pending (not yet executed) nodes"},
    {"add_input", (PyCFunction)Dag_add_input, METH_NOARGS, "new input node id"},
    {"gate", (PyCFunction)(void (*)(void))Dag_gate, METH_FASTCALL,
     "gate(kind, ref_a, ref_b) -> ref of a 2-input gate of the reference API (counts one live handle)"},
    {"mux", (PyCFunction)(void (*)(void))Dag_mux, METH_FASTCALL,
     "mux(ref_s, ref_a, ref_b) -> ref of s ? a : b (counts one live handle)"},
    {"hinc", (PyCFunction)Dag_hinc, METH_O, "one more live handle on node n"},
    {"hdec", (PyCFunction)Dag_hdec, METH_O, "one live handle fewer on node n"},
    {"hcount", (PyCFunction)Dag_hcount, METH_O, "live handles on node n"},
    {"op", (PyCFunction)Dag_op, METH_O, "op code of node n"},
    {"is_done", (PyCFunction)Dag_is_done, METH_O, "node n executed"},
    {"is_dormant", (PyCFunction)Dag_is_dormant, METH_O, "node n skipped by a flush (unreachable then)"},
    {"revive", (PyCFunction)Dag_revive, METH_O, "dormant node n (and dormant operands) back to pending"},
    {"live", (PyCFunction)(void (*)(void))Dag_live, METH_VARARGS | METH_KEYWORDS,
     "live(take) -> int64 ids of pending nodes reachable from live handles"},
    {"pending", (PyCFunction)Dag_pending, METH_NOARGS, "int64 ids of pending nodes"},
    {"mark_done", (PyCFunction)Dag_mark_done, METH_O, "mark node ids executed"},
    {"requeue", (PyCFunction)Dag_requeue, METH_O, "pending node ids taken by live(True) but not run"},
    {"csa", (PyCFunction)Dag_csa, METH_VARARGS,
     "csa(refs, block=0) -> refs of the binary digits (LSB first) of the number of true literals; counts a handle "
     "on each; block >= 3: shared first stage over blocks of leaf ordinals"},
    {"gather", (PyCFunction)Dag_gather, METH_O, "gather(ids) -> (op int8, a, b, c, lvl int64 arrays)"},
    {nullptr, nullptr, 0, nullptr}};

PyTypeObject DagType = {PyVarObject_HEAD_INIT(nullptr, 0)};

PyModuleDef dag_module = {PyModuleDef_HEAD_INIT, "hb_dag",
                          "native gate DAG of paper_1806_03461_b200.backend.TfheContext", -1, nullptr};

}  // namespace

PyMODINIT_FUNC PyInit_hb_dag(void) {
    import_array();
    DagType.tp_name = "hb_dag.Dag";
    DagType.tp_basicsize = sizeof(PyDag);
    DagType.tp_flags = Py_TPFLAGS_DEFAULT;
    DagType.tp_doc = "gate DAG: node store, elision, CSE, full-adder fusion, live-handle filter";
    DagType.tp_new = Dag_new;
    DagType.tp_dealloc = (destructor)Dag_dealloc;
    DagType.tp_methods = Dag_methods;
    if (PyType_Ready(&DagType) < 0) return nullptr;
    PyObject *m = PyModule_Create(&dag_module);
    if (!m) return nullptr;
    Py_INCREF(&DagType);
    if (PyModule_AddObject(m, "Dag", (PyObject *)&DagType) < 0) {
        Py_DECREF(&DagType);
        Py_DECREF(m);
        return nullptr;
    }
    const std::pair<const char *, int> ops[] = {{"OP_CONST", CONST}, {"OP_INPUT", INPUT}, {"OP_AND", AND},
                                                {"OP_XOR", XOR},     {"OP_MUX", MUX},     {"OP_MAJ", MAJ},
                                                {"OP_XOR3", XOR3}};
    for (const auto &kv : ops)
        if (PyModule_AddIntConstant(m, kv.first, kv.second) < 0) {
            Py_DECREF(m);
            return nullptr;
        }
    return m;
}
