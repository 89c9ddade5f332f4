// planner.h -- host-side planning of gate lists into device steps.
//
// A logical gate (qubit labels) becomes, per shard, one Pass on physical bit
// positions, after
//   * specialisation: diagonal matrices -> DIAG,
//     single non-unit diagonal entry -> PHASE on a fixed-bit subspace (CU1,
//     CZ touch 1/4 of the state), -1 -> exact sign flip, X / SWAP -> pure
//     data movement, fSim -> dense on the 3 touched members;
//   * global-qubit handling: controls / phase patterns on
//     global bits select shards, diagonal tables are sliced per shard, and a
//     non-diagonal target on a global bit is first swapped with a local bit
//     (EXCHANGE step, a local<->global qubit swap).
// With fusion on, runs of consecutive gates become TILE steps (tile.h).
#pragma once

#include <vector>

#include "qj_internal.h"
#include "tile.h"

namespace qj {

struct LGate {
    int kind = QJ_GATE_DENSE;
    int nt = 0, nc = 0;
    int t[QJ_MAX_TARGETS] = {};
    int c[QJ_MAX_CONTROLS] = {};
    std::vector<cd> data;  // dense 4^nt / diag 2^nt / fsim 5
    int src = -1;          // fusion: index of the input gate this one is (-1: fused group)
};

struct Step {
    enum Type { PASS = 0, EXCHANGE = 1, TILE = 2, SMALL = 3 } type = PASS;
    int shard = 0;
    Pass pass;
    TileSpec tile;
    std::vector<Pass> prog;  // SMALL: the passes the whole-state SMEM kernel runs (small.h)
    int gbit = 0, lbit = 0;  // EXCHANGE: global bit index j (physical nl + j), local bit L
    double alg_bytes = 0;
};

struct PlanContext {
    int n, nl, g, amp_bytes, nshards;
    std::vector<int>* phys;  // logical qubit -> physical bit, updated by remaps
};

class Planner {
  public:
    void plan(const PlanContext& ctx, const std::vector<LGate>& gates, bool fuse, std::vector<Step>& out);
    // with fuse: also plan the gates after the paper's <= 2-qubit fusion and
    // keep the cheaper plan (callers set it when the user asked for no
    // explicit fusion width; QJ_AUTO_FUSE=0 turns it off)
    bool auto_fuse_ = false;

  private:
    void plan_gate(const PlanContext& ctx, const LGate& g, std::vector<Step>& out);
    void plan_fused(const PlanContext& ctx, const std::vector<LGate>& gates, std::vector<Step>& out);
};

// Sharded states: a non-diagonal gate with a target on a global bit first
// swaps it into the local bits (EXCHANGE steps, map updated).
bool needs_exchange(const PlanContext& ctx, const LGate& g);
void exchange_for(const PlanContext& ctx, const LGate& g, std::vector<Step>& out);

// The paper's greedy gate fusion into gates of <= max_qubits qubits
// (fusion.cpp).
std::vector<LGate> fuse_gates(const std::vector<LGate>& gates, int n, int max_qubits);

// Pass specialisation of one logical gate on local physical positions, as
// seen from shard `r` (global bits fixed to r's bits).  Returns false when
// the gate is the identity on that shard.
bool specialise(const PlanContext& ctx, const LGate& g, uint64_t r, Pass& p);

}  // namespace qj
