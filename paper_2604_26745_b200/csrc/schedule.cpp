// schedule.cpp -- static task schedules of the persistent projector (host, native C++).
//
// A projector task is (batch member, traced angle-bank, detector range).  For each projector kind
// (forward, JVP, adjoint = VJP and GN) the host builds, once per geometry handle, the list of tasks
// every CTA processes, from the exact per-task work (nominal samples of the task's rays, known from
// the clip table):
//   * many tasks per CTA (>= 8): contiguous member-major ranges, whole angle-banks;
//   * otherwise the angle-banks are cut into p equal detector ranges (p = 1..2, the p with the
//     smallest estimated makespan, a part costing work/p + a fixed per-part overhead) and the parts
//     are assigned longest-first to the least-loaded CTA (LPT).
// For the adjoint kind every task also gets a partial-gradient slot: consecutive tasks of one CTA
// with the same (member, orientation class) share a slot (at most kSlotTasks of them, so an fp32
// slot sums a bounded number of angle-banks); the slot lists per (member, class) drive the fixed-order
// fp64 reduction (reduce_slots_kernel).  Comb groups (sweep B lane sets) are built per detector range.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <numeric>
#include <queue>

#include "internal.h"

namespace pget {

constexpr int kSlotTasks = 16;   // 32 and 64 measured without effect on the LM iteration (configs 4, 5)

// comb groups of rays [r_lo, r_hi): <= 32 rays pairwise >= S apart (greedy, comb order)
static void comb_groups(int r_lo, int r_hi, int S, std::vector<int32_t>* out)
{
    std::vector<int32_t> cur;
    auto flush = [&]() {
        if (cur.empty()) return;
        for (int k = 0; k < 32; ++k) out->push_back(k < static_cast<int>(cur.size()) ? cur[k] : -1);
        cur.clear();
    };
    for (int c0 = 0; c0 < S; ++c0)
        for (int r = r_lo + c0; r < r_hi; r += S) {
            bool ok = cur.size() < 32;
            for (int32_t x : cur)
                if (std::abs(x - r) < S) { ok = false; break; }
            if (!ok) flush();
            cur.push_back(r);
        }
    flush();
}

void build_schedule(const Geometry& g, int kind, int C, Schedule* S)
{
    const bool adjoint = kind == kSchedAdj;
    const bool paired = g.pair && kind != kSchedJvp;
    const std::vector<int32_t>& list = paired ? g.task_ab_p : g.task_ab;
    const int B = g.desc.batch, nd = g.desc.n_det, J = g.desc.n_subrays;
    const int ntab = static_cast<int>(list.size());
    S->C = C;
    S->tasks.clear();
    S->groups.clear();
    S->cta_begin.assign(C + 1, 0);

    // work of each traced angle-bank (samples of its rays)
    std::vector<double> cost(ntab, 0.0);
    for (int k = 0; k < ntab; ++k)
        for (int r = 0; r < g.R; ++r) {
            const size_t e = static_cast<size_t>(list[k]) * g.R + r;
            const int32_t lo = g.clip[2 * e], hi = g.clip[2 * e + 1];
            if (hi >= lo) cost[k] += hi - lo + 1;
        }
    const int64_t T0 = static_cast<int64_t>(B) * ntab;

    std::map<std::pair<int, int>, std::pair<int, int>> gcache;   // (p, q) -> comb group range
    auto groups_of = [&](int p, int q) {
        auto key = std::make_pair(p, q);
        auto it = gcache.find(key);
        if (it != gcache.end()) return it->second;
        const int b = static_cast<int>(S->groups.size() / 32);
        comb_groups((nd * q / p) * J, (nd * (q + 1) / p) * J, g.comb_S, &S->groups);
        const auto rg = std::make_pair(b, static_cast<int>(S->groups.size() / 32));
        gcache[key] = rg;
        return rg;
    };
    auto make = [&](int m, int k, int p, int q) {
        TaskD t;
        t.m = m;
        t.ab = list[k];
        t.dlo = nd * q / p;
        t.dhi = nd * (q + 1) / p;
        const auto rg = groups_of(p, q);
        t.gbeg = rg.first;
        t.gend = rg.second;
        t.slot = -1;
        t.flags = g.orient[list[k]] ? kTaskClass1 : 0;
        return t;
    };

    std::vector<std::vector<TaskD>> per(C);
    if (T0 >= 8LL * C || ntab == 0) {
        for (int c = 0; c < C; ++c) {
            const int64_t tb = static_cast<int64_t>(c) * T0 / C, te = static_cast<int64_t>(c + 1) * T0 / C;
            for (int64_t t = tb; t < te; ++t) per[c].push_back(make(static_cast<int>(t / ntab), static_cast<int>(t % ntab), 1, 0));
        }
    } else {
        // per-part overhead (band streaming, barriers, flush) as a fraction of a whole angle-bank; it
        // scales with the band count over the work, ~1/N (measured: 0.06 right at N = 256, too low at 128)
        const double ovh = (adjoint ? 0.06 : 0.04) * 256.0 / g.desc.n_px;
        double best = 1e300;
        int best_p = 1;
        std::vector<int> best_owner;
        struct Item { double w; int m, k, q; };
        // p <= 2: measured on configs 2-4 (scripts/pmax_exp.sh), p = 3 or 4 is never faster than p = 2
        // (narrower parts mean fewer ray groups, so fewer warps per CTA and emptier comb lanes), and
        // p = 2 beats whole angle-banks on configs 2-4 (JVP config 2: p=3 0.198 ms, p=2 0.170 ms)
        int pmax = std::min(2, nd);
        if (const char* e = std::getenv("PGET_SCHED_PMAX")) pmax = std::max(1, std::min(pmax, std::atoi(e)));   // experiments
        for (int p = 1; p <= pmax; ++p) {
            std::vector<Item> items;
            for (int m = 0; m < B; ++m)
                for (int k = 0; k < ntab; ++k)
                    for (int q = 0; q < p; ++q) {
                        const double frac = static_cast<double>(nd * (q + 1) / p - nd * q / p) / nd;
                        items.push_back({cost[k] * (frac + (p > 1 ? ovh : 0.0)), m, k, q});
                    }
            std::vector<int> order(items.size());
            std::iota(order.begin(), order.end(), 0);
            std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return items[a].w > items[b].w; });
            using L = std::pair<double, int>;
            std::priority_queue<L, std::vector<L>, std::greater<L>> heap;
            for (int c = 0; c < C; ++c) heap.push({0.0, c});
            std::vector<int> owner(items.size());
            double mk = 0.0;
            for (int idx : order) {
                L top = heap.top();
                heap.pop();
                owner[idx] = top.second;
                top.first += items[idx].w;
                mk = std::max(mk, top.first);
                heap.push(top);
            }
            if (mk < best * 0.98) { best = mk; best_p = p; best_owner = owner; }
        }
        // rebuild the chosen items in (m, class, k, q) order per CTA
        std::vector<std::vector<std::array<int, 3>>> own(C);
        int idx = 0;
        for (int m = 0; m < B; ++m)
            for (int k = 0; k < ntab; ++k)
                for (int q = 0; q < best_p; ++q) own[best_owner[idx++]].push_back({m, k, q});
        for (int c = 0; c < C; ++c)
            for (const auto& it : own[c]) per[c].push_back(make(it[0], it[1], best_p, it[2]));
    }
    // flatten; slots for the adjoint kind
    S->n_slots = 0;
    std::vector<std::vector<int32_t>> lists(static_cast<size_t>(B) * 2);
    for (int c = 0; c < C; ++c) {
        S->cta_begin[c] = static_cast<int32_t>(S->tasks.size());
        int run = 0, pm = -1, pc = -1;
        for (TaskD t : per[c]) {
            if (adjoint) {
                const int cls = (t.flags & kTaskClass1) ? 1 : 0;
                if (t.m != pm || cls != pc || run == kSlotTasks) {
                    lists[static_cast<size_t>(t.m) * 2 + cls].push_back(S->n_slots);
                    ++S->n_slots;
                    run = 0;
                    t.flags |= kTaskFirst;
                }
                t.slot = S->n_slots - 1;
                ++run;
                pm = t.m;
                pc = cls;
            }
            S->tasks.push_back(t);
        }
    }
    S->cta_begin[C] = static_cast<int32_t>(S->tasks.size());
    S->slot_lo.assign(S->n_slots, 0);
    S->slot_hi.assign(S->n_slots, g.desc.n_px);
    S->red_off.assign(static_cast<size_t>(B) * 2 + 1, 0);
    S->red_slot.clear();
    for (size_t e = 0; e < lists.size(); ++e) {
        S->red_off[e] = static_cast<int32_t>(S->red_slot.size());
        S->red_slot.insert(S->red_slot.end(), lists[e].begin(), lists[e].end());
    }
    S->red_off[lists.size()] = static_cast<int32_t>(S->red_slot.size());
    S->max_slots_member = 0;
    for (int m = 0; m < B; ++m)
        S->max_slots_member = std::max(S->max_slots_member, S->red_off[2 * m + 2] - S->red_off[2 * m]);
    S->max_gA = 1;
    S->max_gB = 1;
    for (const TaskD& t : S->tasks) {
        S->max_gA = std::max(S->max_gA, ((t.dhi - t.dlo) * J + 31) / 32);
        S->max_gB = std::max(S->max_gB, t.gend - t.gbeg);
    }
}

// ------------------------------------------------------------------ segmented adjoint (VJP / GN)
// Units (member, traced angle-bank, row segment) over all detectors: full 32-lane comb groups and the
// most warps per CTA, while K segments per angle-bank give enough units to balance the CTAs.  The
// unit cost is the exact number of its samples (seg_entry of the segment bounds, per ray) plus a
// fixed per-unit overhead; units are assigned longest-first to the least-loaded CTA, separately for
// phase A (CA CTAs) and phase B (C CTAs), and listed per CTA in (member, class, angle-bank, segment)
// order so that consecutive units of one (member, class) share a partial slot (<= kSlotTasks).
void build_adj_schedule(const Geometry& g, const std::vector<RayP>& rays, int CA, int C, Schedule* S, bool unpaired)
{
    const bool paired = g.pair && !unpaired;   // unpaired: the standalone JVP (every traced angle-bank)
    const std::vector<int32_t>& list = paired ? g.task_ab_p : g.task_ab;
    const int B = g.desc.batch, R = g.R;
    const int ntab = static_cast<int>(list.size());
    const int rows = g.P - 1;   // sample rows [0, P - 1)
    S->CA = CA;
    S->C = C;
    // per-segment sample counts of every traced angle-bank, for K = 1..4
    auto seg_rows_of = [&](int K) {
        std::vector<int32_t> y(K + 1);
        for (int k = 0; k <= K; ++k) y[k] = static_cast<int32_t>((static_cast<int64_t>(rows) * k) / K);
        return y;
    };
    auto costs_of = [&](const std::vector<int32_t>& y) {
        const int K = static_cast<int>(y.size()) - 1;
        std::vector<double> c(static_cast<size_t>(ntab) * K, 0.0);
        for (int t = 0; t < ntab; ++t)
            for (int r = 0; r < R; ++r) {
                const RayP& rp = rays[static_cast<size_t>(list[t]) * R + r];
                for (int k = 0; k < K; ++k) {
                    const int n = rp.dV > 0 ? seg_entry(rp, y[k + 1]) - seg_entry(rp, y[k])
                                            : seg_entry(rp, y[k]) - seg_entry(rp, y[k + 1]);
                    c[static_cast<size_t>(t) * K + k] += std::max(0, n);
                }
            }
        return c;
    };
    auto lpt = [&](const std::vector<double>& w, int ncta, std::vector<int>* owner) {
        std::vector<int> order(w.size());
        std::iota(order.begin(), order.end(), 0);
        std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return w[a] > w[b]; });
        using L = std::pair<double, int>;
        std::priority_queue<L, std::vector<L>, std::greater<L>> heap;
        for (int c = 0; c < ncta; ++c) heap.push({0.0, c});
        owner->assign(w.size(), 0);
        double mk = 0.0;
        for (int idx : order) {
            L top = heap.top();
            heap.pop();
            (*owner)[idx] = top.second;
            top.first += w[idx];
            mk = std::max(mk, top.first);
            heap.push(top);
        }
        return mk;
    };
    // choose K (phase B makespan, per-unit overhead kUnitOvh of a mean angle-bank)
    constexpr double kUnitOvh = 0.04;
    int Kmax = std::max(1, std::min(4, rows / 8));   // segments of >= 8 rows
    int Kforce = 0;
    if (const char* e = std::getenv("PGET_SEG_K")) Kforce = std::atoi(e);   // experiments
    double best = 1e300;
    int bestK = 1;
    for (int K = 1; K <= Kmax; ++K) {
        if (Kforce > 0 && K != std::min(Kforce, Kmax)) continue;
        const std::vector<double> c = costs_of(seg_rows_of(K));
        double mean = 0.0;
        for (double v : c) mean += v;
        mean = ntab ? mean / ntab : 1.0;   // samples of a mean angle-bank
        std::vector<double> w;
        for (int m = 0; m < B; ++m)
            for (double v : c) w.push_back(v / std::max(mean, 1.0) + kUnitOvh);
        std::vector<int> own;
        const double mk = lpt(w, C, &own);
        if (mk < best * 0.98) { best = mk; bestK = K; }
    }
    const int K = bestK;
    S->K = K;
    S->seg_rows = seg_rows_of(K);
    const std::vector<double> c = costs_of(S->seg_rows);
    double mean = 0.0;
    for (double v : c) mean += v;
    mean = ntab ? mean / ntab : 1.0;
    // canonical units
    std::vector<UnitD> all;
    std::vector<double> w;
    for (int m = 0; m < B; ++m)
        for (int t = 0; t < ntab; ++t)
            for (int k = 0; k < K; ++k) {
                UnitD u{};
                u.m = m;
                u.ab = list[t];
                u.seg = k;
                u.canon = (m * ntab + t) * K + k;
                u.slot = -1;
                u.flags = g.orient[list[t]] ? kTaskClass1 : 0;
                all.push_back(u);
                w.push_back(c[static_cast<size_t>(t) * K + k] / std::max(mean, 1.0) + kUnitOvh);
            }
    S->n_canon = static_cast<int64_t>(all.size());
    auto assign = [&](int ncta, std::vector<UnitD>* units, std::vector<int32_t>* begin) {
        std::vector<int> own;
        lpt(w, ncta, &own);
        std::vector<std::vector<int>> per(ncta);
        for (size_t i = 0; i < all.size(); ++i) per[own[i]].push_back(static_cast<int>(i));
        units->clear();
        begin->assign(ncta + 1, 0);
        for (int cta = 0; cta < ncta; ++cta) {
            (*begin)[cta] = static_cast<int32_t>(units->size());
            std::sort(per[cta].begin(), per[cta].end(), [&](int a, int b) {
                const UnitD &x = all[a], &y = all[b];
                const int cx = x.flags & kTaskClass1, cy = y.flags & kTaskClass1;
                if (x.m != y.m) return x.m < y.m;
                if (cx != cy) return cx < cy;
                return x.canon < y.canon;
            });
            for (int i : per[cta]) units->push_back(all[i]);
        }
        (*begin)[ncta] = static_cast<int32_t>(units->size());
    };
    assign(CA, &S->unitsA, &S->ua_begin);
    // phase B: CTAs are split into two groups by orientation class, in proportion to the classes'
    // work; within a group, units go longest-first to the least-loaded CTA, preferring (within a
    // quarter of the unit's cost) a CTA that already holds the unit's row segment.  A CTA then holds
    // units of one class and few segments: one partial slot whose nonzero rows are those segments'
    // (the slot reduction reads and phase B zeroes only those rows).  Used when its makespan is within
    // 3 % of the plain LPT assignment.
    {
        std::vector<std::vector<int>> gidx(2);
        std::vector<double> gcost(2, 0.0);
        double total = 0.0;
        for (size_t i = 0; i < all.size(); ++i) {
            const int key = (all[i].flags & kTaskClass1) ? 1 : 0;
            gidx[key].push_back(static_cast<int>(i));
            gcost[key] += w[i];
            total += w[i];
        }
        std::vector<int> own_plain;
        const double mk_plain = lpt(w, C, &own_plain);
        bool grouped = !gidx[0].empty() && !gidx[1].empty() && C >= 2 && !std::getenv("PGET_NO_GROUP");
        std::vector<int> own(all.size(), 0);
        double mk_group = 0.0;
        if (grouped) {
            int n0 = static_cast<int>(std::lround(C * gcost[0] / total));
            n0 = std::max(1, std::min(C - 1, n0));
            const int nct[2] = {n0, C - n0};
            int base = 0;
            for (int k = 0; k < 2; ++k) {
                std::vector<int>& ids = gidx[k];
                std::stable_sort(ids.begin(), ids.end(), [&](int a, int b) { return w[a] > w[b]; });
                std::vector<double> load(nct[k], 0.0);
                std::vector<std::vector<int>> segcnt(nct[k], std::vector<int>(K, 0));
                for (int i : ids) {
                    int best = 0;
                    for (int c = 1; c < nct[k]; ++c) if (load[c] < load[best]) best = c;
                    const double lim = load[best] + 0.25 * w[i];
                    int pick = best;
                    for (int c = 0; c < nct[k]; ++c)
                        if (load[c] <= lim && segcnt[c][all[i].seg] > segcnt[pick][all[i].seg]) pick = c;
                    load[pick] += w[i];
                    ++segcnt[pick][all[i].seg];
                    own[i] = base + pick;
                }
                for (double l : load) mk_group = std::max(mk_group, l);
                base += nct[k];
            }
            grouped = mk_group <= 1.03 * mk_plain;
            if (std::getenv("PGET_SCHED_DEBUG"))
                fprintf(stderr, "phase B: plain %.3f class-grouped %.3f -> %s\n", mk_plain, mk_group, grouped ? "grouped" : "plain");
        }
        if (!grouped) own = own_plain;
        std::vector<std::vector<int>> per(C);
        for (size_t i = 0; i < all.size(); ++i) per[own[i]].push_back(static_cast<int>(i));
        S->unitsB.clear();
        S->ub_begin.assign(C + 1, 0);
        for (int cta = 0; cta < C; ++cta) {
            S->ub_begin[cta] = static_cast<int32_t>(S->unitsB.size());
            std::sort(per[cta].begin(), per[cta].end(), [&](int a, int b) {
                const UnitD &x = all[a], &y = all[b];
                const int cx = x.flags & kTaskClass1, cy = y.flags & kTaskClass1;
                if (x.m != y.m) return x.m < y.m;
                if (cx != cy) return cx < cy;
                return x.canon < y.canon;
            });
            for (int i : per[cta]) S->unitsB.push_back(all[i]);
        }
        S->ub_begin[C] = static_cast<int32_t>(S->unitsB.size());
    }
    const int ngA = (R + 31) / 32;
    std::vector<int32_t> grp;
    comb_groups(0, R, g.comb_S, &grp);
    const int ngB = static_cast<int>(grp.size() / 32);
    S->groups = grp;
    S->max_gA = ngA;
    S->max_gB = ngB;
    // Jacobian-coefficient cache of the GN product: per
    // (traced angle-bank t, segment k, comb group gi) a block of kmax rows of 32 lanes, kmax = the
    // most samples any lane of the group has in the segment; per member the same layout.
    S->cache_off.assign(static_cast<size_t>(ntab) * K * ngB + 1, 0);
    {
        int64_t off = 0;
        for (int t = 0; t < ntab; ++t)
            for (int k = 0; k < K; ++k)
                for (int gi = 0; gi < ngB; ++gi) {
                    S->cache_off[(static_cast<size_t>(t) * K + k) * ngB + gi] = off;
                    int kmax = 0;
                    for (int l = 0; l < 32; ++l) {
                        const int r = grp[static_cast<size_t>(gi) * 32 + l];
                        if (r < 0) continue;
                        const RayP& rp = rays[static_cast<size_t>(list[t]) * R + r];
                        const int n = rp.dV > 0 ? seg_entry(rp, S->seg_rows[k + 1]) - seg_entry(rp, S->seg_rows[k])
                                                : seg_entry(rp, S->seg_rows[k]) - seg_entry(rp, S->seg_rows[k + 1]);
                        kmax = std::max(kmax, n);
                    }
                    off += kmax;
                }
        S->cache_off[static_cast<size_t>(ntab) * K * ngB] = off;
        S->cache_rows_member = off;
    }
    {   // the same layout over groups of nearby rays: blocks of 32 s consecutive rays, each split into s
        // groups of every s-th ray (s = gnbC_stride); the tail of T < 32 s rays into ceil(T / 32) groups
        // the same way -- ceil(R / 32) groups in all
        S->max_gC = ngA;
        S->groupsC.assign(static_cast<size_t>(ngA) * 32, -1);
        const int sb = std::max(1, g.gnbC_stride);
        int gi0 = 0;
        for (int r0 = 0; r0 < R; r0 += 32 * sb) {
            const int T = std::min(32 * sb, R - r0);
            const int ng = (T + 31) / 32;
            for (int k = 0; k < T; ++k) S->groupsC[static_cast<size_t>(gi0 + k % ng) * 32 + k / ng] = r0 + k;
            gi0 += ng;
        }
        S->cache_offC.assign(static_cast<size_t>(ntab) * K * ngA + 1, 0);
        int64_t off = 0;
        for (int t = 0; t < ntab; ++t)
            for (int k = 0; k < K; ++k)
                for (int gi = 0; gi < ngA; ++gi) {
                    S->cache_offC[(static_cast<size_t>(t) * K + k) * ngA + gi] = off;
                    int kmax = 0;
                    for (int l = 0; l < 32; ++l) {
                        const int r = S->groupsC[static_cast<size_t>(gi) * 32 + l];
                        if (r < 0) continue;
                        const RayP& rp = rays[static_cast<size_t>(list[t]) * R + r];
                        const int n = rp.dV > 0 ? seg_entry(rp, S->seg_rows[k + 1]) - seg_entry(rp, S->seg_rows[k])
                                                : seg_entry(rp, S->seg_rows[k]) - seg_entry(rp, S->seg_rows[k + 1]);
                        kmax = std::max(kmax, n);
                    }
                    off += kmax;
                }
        S->cache_offC[static_cast<size_t>(ntab) * K * ngA] = off;
        S->cache_rows_memberC = off;
    }
    S->ntab = ntab;
    S->tasks.clear();
    S->cta_begin.assign(C + 1, 0);
    // slots of phase B (as build_schedule's adjoint kind, per unit)
    S->n_slots = 0;
    S->slot_lo.clear();
    S->slot_hi.clear();
    std::vector<std::vector<int32_t>> lists(static_cast<size_t>(B) * 2);
    for (int cta = 0; cta < C; ++cta) {
        int run = 0, pm = -1, pc = -1;
        for (int u = S->ub_begin[cta]; u < S->ub_begin[cta + 1]; ++u) {
            UnitD& t = S->unitsB[u];
            const int cls = (t.flags & kTaskClass1) ? 1 : 0;
            if (t.m != pm || cls != pc || run == kSlotTasks) {
                lists[static_cast<size_t>(t.m) * 2 + cls].push_back(S->n_slots);
                ++S->n_slots;
                run = 0;
                t.flags |= kTaskFirst;
            }
            t.slot = S->n_slots - 1;
            // the slot's rows (oriented frame, unpadded) that the unit's flushes can write
            const int lo = std::max(0, S->seg_rows[t.seg] - kHalo);
            const int hi = std::min(g.desc.n_px, S->seg_rows[t.seg + 1] - kHalo + 1);
            if (run == 0) {
                S->slot_lo.push_back(lo);
                S->slot_hi.push_back(hi);
            } else {
                S->slot_lo.back() = std::min(S->slot_lo.back(), lo);
                S->slot_hi.back() = std::max(S->slot_hi.back(), hi);
            }
            ++run;
            pm = t.m;
            pc = cls;
        }
    }
    S->red_off.assign(static_cast<size_t>(B) * 2 + 1, 0);
    S->red_slot.clear();
    for (size_t e = 0; e < lists.size(); ++e) {
        S->red_off[e] = static_cast<int32_t>(S->red_slot.size());
        S->red_slot.insert(S->red_slot.end(), lists[e].begin(), lists[e].end());
    }
    S->red_off[lists.size()] = static_cast<int32_t>(S->red_slot.size());
    S->max_slots_member = 0;
    for (int m = 0; m < B; ++m)
        S->max_slots_member = std::max(S->max_slots_member, S->red_off[2 * m + 2] - S->red_off[2 * m]);
    S->stA.clear();
    S->stB.clear();
    S->sa_begin.clear();
    S->sb_begin.clear();
}

// stage lists of both phases (band j of a unit in processing order; passes repeat the unit's bands)
void build_adj_stages(int RbA, int passesA, int RbB, int passesB, Schedule* S)
{
    auto stages = [&](const std::vector<UnitD>& units, const std::vector<int32_t>& ub, int Rb, int passes,
                      std::vector<StageD>* st, std::vector<int32_t>* sb) {
        const int ncta = static_cast<int>(ub.size()) - 1;
        st->clear();
        sb->assign(ncta + 1, 0);
        for (int cta = 0; cta < ncta; ++cta) {
            (*sb)[cta] = static_cast<int32_t>(st->size());
            for (int u = ub[cta]; u < ub[cta + 1]; ++u) {
                const int nrow = S->seg_rows[units[u].seg + 1] - S->seg_rows[units[u].seg];
                const int nb = (nrow + Rb - 1) / Rb;
                for (int p = 0; p < passes; ++p)
                    for (int j = 0; j < nb; ++j) st->push_back(StageD{u, j});
            }
        }
        (*sb)[ncta] = static_cast<int32_t>(st->size());
    };
    stages(S->unitsA, S->ua_begin, RbA, passesA, &S->stA, &S->sa_begin);
    stages(S->unitsB, S->ub_begin, RbB, passesB, &S->stB, &S->sb_begin);
}

}  // namespace pget
