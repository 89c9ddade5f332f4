// fusion.cpp -- the paper's gate fusion (Table 2 Depth* /
// Gates* columns): "iterating over the circuit gates and greedily combining
// one-qubit and two-qubit gates that act on the same target qubits" into gates
// of at most `max_qubits` (= 2) qubits, each applied as one dense gate.
//
// Greedy rule (reading R23; reproduces Table 2's fused columns for
// qft / variational / bv exactly, tests/test_fusion.py):
//  * every qubit has an "open" group: the latest group touching it;
//  * a gate whose qubits (targets + controls) are all covered by the single
//    open group of its qubits joins that group;
//  * otherwise, if the union of the open groups on its qubits has <= max
//    qubits and each of those groups is open on all of its own qubits, they are
//    merged with the gate into one group placed at this gate;
//  * otherwise the gate starts a new group, which absorbs the one-qubit groups
//    still open on its qubits;
//  * gates on more than max qubits pass through unchanged.
// Moving a group later (merge / absorb) or a gate earlier (join) is valid
// because the moved gates share no qubit with the gates they pass.
// The group's matrix is the ordered product of its members embedded in the
// group's qubit space (controls become part of the matrix).
#include <algorithm>
#include <vector>

#include "planner.h"

namespace qj {

namespace {

struct Group {
    std::vector<int> qubits;   // first-seen order (matrix bit order, MSB first)
    std::vector<int> members;  // gate indices, program order
    int pos = 0;               // placement: the gate at which it last grew
    bool alive = true;
    bool passthrough = false;
};

bool contains(const std::vector<int>& v, int q) { return std::find(v.begin(), v.end(), q) != v.end(); }

// Dense matrix of gate g embedded in the space of `qubits` (first = MSB).
std::vector<cd> embed(const LGate& g, const std::vector<int>& qubits) {
    const int m = (int)qubits.size(), D = 1 << m;
    auto bitpos = [&](int q) {
        for (int i = 0; i < m; ++i)
            if (qubits[i] == q) return m - 1 - i;
        return -1;
    };
    // the gate's own target matrix (listed order)
    const int k = g.nt, K = 1 << k;
    std::vector<cd> G((size_t)K * K, cd(0, 0));
    switch (g.kind) {
        case QJ_GATE_DENSE: G = g.data; break;
        case QJ_GATE_X: G = {0, 1, 1, 0}; break;
        case QJ_GATE_Z: G = {1, 0, 0, -1}; break;
        case QJ_GATE_SWAP: G[0] = G[6] = G[9] = G[15] = 1; break;
        case QJ_GATE_FSIM:
            G[0] = 1;
            G[5] = g.data[0];
            G[6] = g.data[1];
            G[9] = g.data[2];
            G[10] = g.data[3];
            G[15] = g.data[4];
            break;
        case QJ_GATE_DIAG:
            for (int i = 0; i < K; ++i) G[(size_t)i * K + i] = g.data[i];
            break;
    }
    std::vector<cd> M((size_t)D * D, cd(0, 0));
    for (int col = 0; col < D; ++col) {
        bool active = true;
        for (int i = 0; i < g.nc; ++i) active &= ((col >> bitpos(g.c[i])) & 1) != 0;
        if (!active) {
            M[(size_t)col * D + col] = 1;
            continue;
        }
        int gc = 0;
        for (int i = 0; i < k; ++i) gc = (gc << 1) | ((col >> bitpos(g.t[i])) & 1);
        for (int gr = 0; gr < K; ++gr) {
            const cd v = G[(size_t)gr * K + gc];
            if (v == cd(0, 0)) continue;
            int row = col;
            for (int i = 0; i < k; ++i) {
                const int b = bitpos(g.t[i]);
                row = (row & ~(1 << b)) | (((gr >> (k - 1 - i)) & 1) << b);
            }
            M[(size_t)row * D + col] += v;
        }
    }
    return M;
}

std::vector<cd> matmul(const std::vector<cd>& A, const std::vector<cd>& B, int D) {
    std::vector<cd> C((size_t)D * D, cd(0, 0));
    for (int i = 0; i < D; ++i)
        for (int k = 0; k < D; ++k) {
            const cd a = A[(size_t)i * D + k];
            if (a == cd(0, 0)) continue;
            for (int j = 0; j < D; ++j) C[(size_t)i * D + j] += a * B[(size_t)k * D + j];
        }
    return C;
}

}  // namespace

std::vector<LGate> fuse_gates(const std::vector<LGate>& gates, int n, int max_qubits) {
    std::vector<Group> groups;
    groups.reserve(gates.size());
    std::vector<int> open(n, -1);
    for (int idx = 0; idx < (int)gates.size(); ++idx) {
        const LGate& g = gates[idx];
        std::vector<int> Q;
        for (int i = 0; i < g.nt; ++i) Q.push_back(g.t[i]);
        for (int i = 0; i < g.nc; ++i) Q.push_back(g.c[i]);
        std::vector<int> cands;
        for (int q : Q)
            if (open[q] >= 0 && std::find(cands.begin(), cands.end(), open[q]) == cands.end()) cands.push_back(open[q]);
        auto open_on_all = [&](int gi) {
            for (int q : groups[gi].qubits)
                if (open[q] != gi) return false;
            return true;
        };
        if ((int)Q.size() > max_qubits) {
            Group G;
            G.qubits = Q;
            G.members = {idx};
            G.pos = idx;
            G.passthrough = true;
            groups.push_back(G);
            for (int q : Q) open[q] = (int)groups.size() - 1;
            continue;
        }
        // join the single covering group
        if (cands.size() == 1) {
            bool covered = true;
            for (int q : Q) covered &= contains(groups[cands[0]].qubits, q);
            if (covered && !groups[cands[0]].passthrough) {
                groups[cands[0]].members.push_back(idx);
                continue;
            }
        }
        // merge with the open groups if the union fits
        std::vector<int> uni;
        for (int gi : cands)
            for (int q : groups[gi].qubits)
                if (!contains(uni, q)) uni.push_back(q);
        for (int q : Q)
            if (!contains(uni, q)) uni.push_back(q);
        bool ok = !cands.empty() && (int)uni.size() <= max_qubits;
        for (int gi : cands) ok = ok && !groups[gi].passthrough && open_on_all(gi);
        if (ok) {
            if (cands.size() == 1) {
                Group& G = groups[cands[0]];
                for (int q : Q)
                    if (!contains(G.qubits, q)) G.qubits.push_back(q);
                G.members.push_back(idx);
                G.pos = idx;
                for (int q : G.qubits) open[q] = cands[0];
            } else {
                std::sort(cands.begin(), cands.end(), [&](int x, int y) { return groups[x].pos < groups[y].pos; });
                Group G;
                for (int gi : cands) {
                    for (int q : groups[gi].qubits)
                        if (!contains(G.qubits, q)) G.qubits.push_back(q);
                    G.members.insert(G.members.end(), groups[gi].members.begin(), groups[gi].members.end());
                    groups[gi].alive = false;
                }
                for (int q : Q)
                    if (!contains(G.qubits, q)) G.qubits.push_back(q);
                std::sort(G.members.begin(), G.members.end());
                G.members.push_back(idx);
                G.pos = idx;
                groups.push_back(G);
                for (int q : G.qubits) open[q] = (int)groups.size() - 1;
            }
            continue;
        }
        // new group, absorbing the one-qubit groups still open on its qubits
        Group G;
        G.qubits = Q;
        std::vector<int> absorb;
        for (int gi : cands)
            if (!groups[gi].passthrough && groups[gi].qubits.size() == 1 && contains(Q, groups[gi].qubits[0]) &&
                open[groups[gi].qubits[0]] == gi)
                absorb.push_back(gi);
        for (int gi : absorb) {
            G.members.insert(G.members.end(), groups[gi].members.begin(), groups[gi].members.end());
            groups[gi].alive = false;
        }
        std::sort(G.members.begin(), G.members.end());
        G.members.push_back(idx);
        G.pos = idx;
        groups.push_back(G);
        for (int q : Q) open[q] = (int)groups.size() - 1;
    }
    std::vector<int> order;
    for (int gi = 0; gi < (int)groups.size(); ++gi)
        if (groups[gi].alive) order.push_back(gi);
    std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return groups[x].pos < groups[y].pos; });
    std::vector<LGate> out;
    out.reserve(order.size());
    for (int gi : order) {
        const Group& G = groups[gi];
        if (G.passthrough || G.members.size() == 1) {
            out.push_back(gates[G.members[0]]);
            out.back().src = G.members[0];
            continue;
        }
        const int D = 1 << G.qubits.size();
        std::vector<cd> M((size_t)D * D, cd(0, 0));
        for (int i = 0; i < D; ++i) M[(size_t)i * D + i] = 1;
        for (int mi : G.members) M = matmul(embed(gates[mi], G.qubits), M, D);
        LGate f;
        f.kind = QJ_GATE_DENSE;
        f.nt = (int)G.qubits.size();
        f.nc = 0;
        for (int i = 0; i < f.nt; ++i) f.t[i] = G.qubits[i];
        f.data = std::move(M);
        out.push_back(std::move(f));
    }
    return out;
}

}  // namespace qj
