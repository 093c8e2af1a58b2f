// Host gate DAG of TfheContext, native: node store,
// constant/duplicate elision, hash-consing, MUX lowering, full-adder fusion
// into 3-input bootstraps (majority, XOR3), live-handle counts and the
// live-gate filter of a flush.  The Python context (backend.py) keeps the
// reference contract (handles, GateStats, scopes, errors) and the engine
// calls; every gate of the reference API lands here once.
//
// Refs are (node << 1) | not_flag; node 0 is the constant 0 (ref 0 = false,
// ref 1 = true).  Node operands: AND / MUX / MAJ store refs; XOR / XOR3 store
// node << 1 and push NOT flags to the output ref.  Node n owns logical pool
// slot n - 1.
#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>

#include <algorithm>
#include <array>
#include <cstdint>
#include <unordered_map>
#include <vector>

namespace py = pybind11;

namespace {

enum Op : int8_t { CONST = 0, INPUT = 1, AND = 2, XOR = 3, MUX = 4, MAJ = 5, XOR3 = 6 };
enum State : uint8_t { PENDING = 0, DONE = 1, DORMANT = 2 };
// gate kinds of the reference API (hebnn.backend AND/OR/XOR/XNOR)
enum Kind : int { K_AND = 0, K_OR = 1, K_XOR = 2, K_XNOR = 3 };

struct Key {
    int64_t op, a, b, c;
    bool operator==(const Key &o) const { return op == o.op && a == o.a && b == o.b && c == o.c; }
};
struct KeyHash {
    size_t operator()(const Key &k) const {
        uint64_t h = (uint64_t)k.op * 0x9E3779B97F4A7C15ull;
        for (int64_t v : {k.a, k.b, k.c}) {
            h ^= (uint64_t)v + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2);
        }
        return (size_t)h;
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
    py::array_t<int64_t> live(bool take) {
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
        return to_array(out);
    }

    py::array_t<int64_t> pending() const { return to_array(pending_); }

    void mark_done(py::array_t<int64_t, py::array::c_style | py::array::forcecast> ids) {
        auto v = ids.unchecked<1>();
        for (py::ssize_t i = 0; i < v.shape(0); i++) state_[check(v(i))] = DONE;
    }

    // node fields of ids: (op int8, a, b, c int64 refs, lvl int64)
    py::tuple gather(py::array_t<int64_t, py::array::c_style | py::array::forcecast> ids) const {
        auto v = ids.unchecked<1>();
        const py::ssize_t n = v.shape(0);
        py::array_t<int8_t> o(n);
        py::array_t<int64_t> a(n), b(n), c(n), l(n);
        auto O = o.mutable_unchecked<1>();
        auto A = a.mutable_unchecked<1>(), B = b.mutable_unchecked<1>(), C = c.mutable_unchecked<1>();
        auto L = l.mutable_unchecked<1>();
        for (py::ssize_t i = 0; i < n; i++) {
            const int64_t k = check(v(i));
            O(i) = op_[k];
            A(i) = a_[k];
            B(i) = b_[k];
            C(i) = c_[k];
            L(i) = lvl_[k];
        }
        return py::make_tuple(o, a, b, c, l);
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
    std::unordered_map<Key, int64_t, KeyHash> cse_;

    int64_t check(int64_t n) const {
        if (n < 0 || n >= (int64_t)op_.size()) throw py::index_error("gate DAG: node id out of range");
        return n;
    }
    void check_ref(int64_t r) const { check(r >> 1); }

    static py::array_t<int64_t> to_array(const std::vector<int64_t> &v) {
        py::array_t<int64_t> out((py::ssize_t)v.size());
        std::copy(v.begin(), v.end(), out.mutable_data());
        return out;
    }

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
        const Key key{op, a, b, c};
        auto it = cse_.find(key);
        if (it != cse_.end()) {
            if (state_[it->second] == DORMANT) revive(it->second);
            return it->second;
        }
        for (int64_t r : {a, b, c})
            if (state_[r >> 1] == DORMANT) revive(r >> 1);
        const int64_t n = push(op, a, b, c, lvl, PENDING);
        pending_.push_back(n);
        cse_.emplace(key, n);
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
        return node(MAJ, s[0], s[1], s[2], 1 + std::max({lv(s[0]), lv(s[1]), lv(s[2])})) << 1;
    }

    int64_t mk_xor3(int64_t p, int64_t q, int64_t r) {
        std::array<int64_t, 3> s{p, q, r};
        std::sort(s.begin(), s.end());
        return node(XOR3, s[0] << 1, s[1] << 1, s[2] << 1,
                    1 + std::max({lvl_[s[0]], lvl_[s[1]], lvl_[s[2]]})) << 1;
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

PYBIND11_MODULE(hb_dag, m) {
    m.doc() = "native gate DAG of paper_1806_03461_b200.backend.TfheContext";
    m.attr("OP_CONST") = (int)CONST;
    m.attr("OP_INPUT") = (int)INPUT;
    m.attr("OP_AND") = (int)AND;
    m.attr("OP_XOR") = (int)XOR;
    m.attr("OP_MUX") = (int)MUX;
    m.attr("OP_MAJ") = (int)MAJ;
    m.attr("OP_XOR3") = (int)XOR3;
    py::class_<Dag>(m, "Dag")
        .def(py::init<>())
        .def("size", &Dag::size)
        .def("pending_count", &Dag::pending_count)
        .def("add_input", &Dag::add_input)
        .def("gate", &Dag::gate)
        .def("mux", &Dag::mux)
        .def("hinc", &Dag::hinc)
        .def("hdec", &Dag::hdec)
        .def("hcount", &Dag::hcount)
        .def("op", &Dag::op)
        .def("is_done", &Dag::is_done)
        .def("is_dormant", &Dag::is_dormant)
        .def("revive", &Dag::revive)
        .def("live", &Dag::live, py::arg("take"))
        .def("pending", &Dag::pending)
        .def("mark_done", &Dag::mark_done)
        .def("gather", &Dag::gather);
}
