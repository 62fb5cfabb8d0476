// clv_ctx.h -- the native context behind the opaque clv_ctx handle of include/clover.h
// (shared by the C-ABI translation units).
#pragma once
#include <string>
#include "clv_internal.h"

namespace clv {
struct SimState;                            // clv_sim.cu
void sim_destroy(SimState *s);
}

using clv::Topology; using clv::FamilyTables; using clv::RecP; using clv::EvalConst;

struct clv_ctx {
    int device = 0;
    int sm_count = 148;
    std::string err;
    bool topo_set = false;
    Topology topo{};
    double mem_gb[CLV_K] = {0, 0, 0, 0, 0};
    Topology *topo_dev = nullptr;
    bool fam_set[CLV_MAX_FAMILIES] = {};
    FamilyTables fam[CLV_MAX_FAMILIES];
    uint32_t *pair_list_dev[CLV_MAX_FAMILIES] = {};
    FamilyTables *fam_dev = nullptr;
    // feasibility tables
    int feas_nmax = -1;
    int bdim = 0, cdim = 0;
    uint32_t *feas_bits = nullptr;
    uint32_t *feas_off = nullptr;
    size_t feas_words = 0;
    // selection scratch
    int max_blocks = 0;
    RecP *partials = nullptr;
    unsigned long long *pcnt = nullptr;
    unsigned int *done_counter = nullptr;
    RecP *final_rec = nullptr;
    unsigned long long *final_cnt = nullptr;
    RecP *host_rec = nullptr;                 // pinned
    unsigned long long *host_cnt = nullptr;   // pinned
    int *err_flag = nullptr;
    long long *err_index = nullptr;
    int *host_err = nullptr;                  // pinned [2 ints + 1 ll]
    EvalConst *ec_dev = nullptr;
    int ec_cap = 0;
    int32_t *small_dev = nullptr;             // realize scratch
    clv::SimState *sim = nullptr;             // serving simulator (clv_sim.cu)
    int *mvlog = nullptr;                     // chain move logs (best-graph reconstruction)
    int *chain_counter = nullptr;             // persistent chain launches: next chain (one int)
    size_t mvlog_cap = 0;
    unsigned char *replan_buf = nullptr;      // clv_replan device staging: starts | results | best | final | record
    size_t replan_cap = 0;
};
