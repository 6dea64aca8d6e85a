// dropin_parity.cpp -- the C++ drop-in, exercised the way a reference caller
// would use it. TEST INFRASTRUCTURE (needs the reference headers; built by
// tests/cpp/Makefile only where /root/reference exists).
//
// For each case an rrflow::Graph is built by the reference itself; the same
// graph is handed to the GPU through rrgpu::Graph(num_vertices, reverse_offsets,
// reverse_sources, reverse_weights) -- the one-line switch INTEGRATION.md
// describes -- and run_imm / generate_batch / select_seeds of both libraries
// are compared field by field. Exit code 0 iff everything is bit-identical.
#include <cstdio>
#include <vector>

#include "rrflow/imm.hpp"
#include "rrflow/sampling.hpp"
#include "rrflow/selection.hpp"
#include "rrgpu/rrgpu.hpp"

namespace {

int failures = 0;

void expect(bool ok, const char* what, int case_id) {
  std::printf("[%s] case %d: %s\n", ok ? "PASS" : "FAIL", case_id, what);
  if (!ok) ++failures;
}

rrgpu::DiffusionModel to_gpu(rrflow::DiffusionModel m) {
  return m == rrflow::DiffusionModel::IC ? rrgpu::DiffusionModel::IC : rrgpu::DiffusionModel::LT;
}

}  // namespace

int main() {
  struct Case {
    rrflow::SynthKind kind;
    uint32_t n;
    double param;
    uint64_t seed;
    rrflow::DiffusionModel model;
    uint32_t k;
  };
  const std::vector<Case> cases = {
      {rrflow::SynthKind::scc_core, 200, 0.25, 19, rrflow::DiffusionModel::IC, 3},
      {rrflow::SynthKind::scc_core, 2000, 0.05, 7, rrflow::DiffusionModel::IC, 10},
      {rrflow::SynthKind::scc_core, 2000, 0.05, 7, rrflow::DiffusionModel::LT, 10},
      {rrflow::SynthKind::erdos_renyi, 3000, 0.002, 11, rrflow::DiffusionModel::IC, 20},
      {rrflow::SynthKind::erdos_renyi, 3000, 0.002, 11, rrflow::DiffusionModel::LT, 20},
  };
  int id = 0;
  for (const Case& c : cases) {
    ++id;
    rrflow::Graph g = rrflow::synth_graph(c.kind, c.n, c.param, c.seed);
    rrflow::generate_ic_weights(g, c.seed + 1);
    if (c.model == rrflow::DiffusionModel::LT) rrflow::normalize_lt_weights(g);

    // --- the switch: same reverse arrays, GPU graph ---------------------------
    rrgpu::Graph dg(g.num_vertices, g.reverse_offsets, g.reverse_sources, g.reverse_weights);

    rrflow::ImmConfig rc;
    rc.k = c.k;
    rc.model = c.model;
    rc.workers = 4;
    rc.rng_seed = 5;
    const rrflow::ImmResult ref = rrflow::run_imm(g, rc);

    rrgpu::ImmConfig gc;
    gc.k = c.k;
    gc.model = to_gpu(c.model);
    gc.workers = 4;
    gc.rng_seed = 5;
    const rrgpu::ImmResult got = rrgpu::run_imm(dg, gc);

    {  // the same graph created with the model hint (rrg_graph_create_for): same result
      rrgpu::Graph dh(g.num_vertices, g.reverse_offsets, g.reverse_sources, g.reverse_weights,
                      to_gpu(c.model));
      const rrgpu::ImmResult hinted = rrgpu::run_imm(dh, gc);
      expect(hinted.seeds.seeds == got.seeds.seeds &&
                 hinted.seeds.marginal_counts == got.seeds.marginal_counts &&
                 hinted.theta == got.theta && hinted.lower_bound == got.lower_bound,
             "run_imm on a model-hinted graph", id);
    }
    expect(ref.seeds.seeds == got.seeds.seeds, "run_imm seeds", id);
    expect(ref.seeds.marginal_counts == got.seeds.marginal_counts, "run_imm marginals", id);
    expect(ref.theta == got.theta && ref.theta_prime == got.theta_prime, "theta, theta'", id);
    expect(ref.lower_bound == got.lower_bound, "lower bound", id);
    expect(ref.sets_generated == got.sets_generated && ref.max_set_size == got.max_set_size &&
               ref.mean_set_size == got.mean_set_size,
           "set statistics", id);

    // --- operator level: generate_batch + select_seeds -----------------------
    rrflow::WorkPool pool(4);
    rrflow::RRRStore rstore(g.num_vertices, pool.workers());
    rrflow::Counter counter(g.num_vertices);
    rrflow::generate_batch(g, c.model, 9, 3000, pool, rstore, &counter);
    rrgpu::RRRStore gstore(dg);
    rrgpu::generate_batch(dg, gc.model, 9, 3000, gstore, true);
    bool same_sets = rstore.size() == gstore.size();
    for (uint64_t j = 0; same_sets && j < rstore.size(); ++j) {
      std::vector<uint32_t> a;
      rstore.set(j).for_each_member([&](uint32_t v) { a.push_back(v); });
      std::vector<uint32_t> b = gstore.set(j);
      std::sort(b.begin(), b.end());
      same_sets = a == b && gstore.set(j).front() == rstore.set(j).root;
    }
    expect(same_sets, "generate_batch sets (slot by slot)", id);
    const std::vector<uint64_t> gc_counter = gstore.counter();
    bool same_counter = true;
    for (uint32_t v = 0; v < g.num_vertices; ++v) same_counter &= counter.get(v) == gc_counter[v];
    expect(same_counter, "fused counter", id);
    const rrflow::SeedSet rs = rrflow::select_seeds(rstore, g.num_vertices, c.k, pool, 0.25,
                                                    &counter);
    const rrgpu::SeedSet gs = rrgpu::select_seeds(gstore, g.num_vertices, c.k, 0.25, true);
    expect(rs.seeds == gs.seeds && rs.marginal_counts == gs.marginal_counts, "select_seeds", id);

    expect(rstore.live_count() == gstore.live_count(), "live_count after select_seeds", id);
    bool same_live = true;
    for (uint64_t j = 0; j < rstore.size(); j += 7) same_live &= rstore.is_live(j) == gstore.is_live(j);
    expect(same_live, "is_live after select_seeds", id);

    // --- the reference's own signatures: WorkPool&, Counter*, SelectionStats --
    {
      rrgpu::WorkPool gpool(4);
      rrgpu::RRRStore gs2(dg);
      rrgpu::Counter gcnt(g.num_vertices);
      rrgpu::generate_batch(dg, gc.model, 9, 1000, gpool, gs2, &gcnt);
      rrgpu::generate_batch_fused(dg, gc.model, 9, 2000, gcnt, gpool, gs2);
      bool same_cnt = true;
      for (uint32_t v = 0; v < g.num_vertices; ++v) same_cnt &= counter.get(v) == gcnt.get(v);
      expect(same_cnt, "Counter* overload of generate_batch", id);
      rrflow::SelectionStats rstats;
      rstats.capture_round_counters = true;
      const rrflow::SeedSet rs2 = rrflow::select_seeds(rstore, g.num_vertices, c.k, pool, 0.25,
                                                       &counter, &rstats);
      rrgpu::SelectionStats gstats;
      gstats.capture_round_counters = true;
      const rrgpu::SeedSet gs3 = rrgpu::select_seeds(gs2, g.num_vertices, c.k, gpool, 0.25,
                                                     &gcnt, &gstats);
      expect(rs2.seeds == gs3.seeds && rs2.marginal_counts == gs3.marginal_counts,
             "select_seeds (WorkPool&, prebuilt Counter*)", id);
      expect(rstats.round_counters == gstats.round_counters, "SelectionStats round counters", id);
      // prebuilt == nullptr: build_counter over the store
      rrgpu::RRRStore gs4(dg);
      rrgpu::generate_batch(dg, gc.model, 9, 3000, gpool, gs4, nullptr);
      const rrgpu::SeedSet gs5 = rrgpu::select_seeds(gs4, g.num_vertices, c.k, gpool);
      expect(gs5.seeds == rs2.seeds && gs5.marginal_counts == rs2.marginal_counts,
             "select_seeds recount (unfused store)", id);
    }

    // --- sampling_phase (imm.hpp:169-209) and the baseline strategy ----------
    rrflow::WorkPool pool1(1);
    const rrflow::SamplingPhaseResult rp = rrflow::sampling_phase(g, rc, pool1);
    const rrgpu::SamplingPhaseResult gp = rrgpu::sampling_phase(dg, gc);
    expect(rp.lower_bound == gp.lower_bound && rp.theta_prime == gp.theta_prime &&
               rp.store.size() == gp.store.size(),
           "sampling_phase lower bound / theta'", id);
    const std::vector<uint64_t> gpc = gp.store.counter();
    bool same_phase_counter = true;
    for (uint32_t v = 0; v < g.num_vertices; ++v) same_phase_counter &= rp.counter.get(v) == gpc[v];
    expect(same_phase_counter, "sampling_phase counter", id);
    rc.strategy = rrflow::Strategy::baseline;
    gc.strategy = rrgpu::parse_strategy("baseline");
    const rrflow::ImmResult rb = rrflow::run_imm(g, rc);
    const rrgpu::ImmResult gb = rrgpu::run_imm(dg, gc);
    expect(rb.seeds.seeds == gb.seeds.seeds && rb.seeds.marginal_counts == gb.seeds.marginal_counts &&
               rb.theta == gb.theta && rb.lower_bound == gb.lower_bound,
           "run_imm, baseline strategy", id);
  }
  // error mapping: k > n -> std::invalid_argument, like validate_config
  {
    rrflow::Graph g = rrflow::synth_graph(rrflow::SynthKind::erdos_renyi, 5, 0.5, 1);
    rrgpu::Graph dg(g.num_vertices, g.reverse_offsets, g.reverse_sources, g.reverse_weights);
    rrgpu::ImmConfig gc;
    gc.k = 6;
    bool threw = false;
    try {
      rrgpu::run_imm(dg, gc);
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    expect(threw, "k > n throws std::invalid_argument", 0);
  }
  // BatchOutOfMemory{sets_generated} (sampling.hpp:148-154): a store budget hit
  // mid-batch keeps the sets made so far, their counts, and reports how many
  {
    rrflow::Graph g = rrflow::synth_graph(rrflow::SynthKind::erdos_renyi, 3000, 0.002, 11);
    rrflow::generate_ic_weights(g, 12);
    rrgpu::Graph dg(g.num_vertices, g.reverse_offsets, g.reverse_sources, g.reverse_weights);
    rrgpu::WorkPool gpool(1);
    rrgpu::RRRStore probe(dg);
    rrgpu::generate_batch(dg, rrgpu::DiffusionModel::IC, 3, 1000, probe, true);
    const uint64_t limit = probe.total_member_count() * 11 / 2;  // ~5 chunks of 1024 sets fit
    rrgpu::RRRStore st(dg);
    rrg_store_set_member_limit(st.handle(), limit);
    rrgpu::Counter cnt(g.num_vertices);
    uint64_t made = UINT64_MAX;
    try {
      rrgpu::generate_batch(dg, rrgpu::DiffusionModel::IC, 3, 100000, gpool, st, &cnt);
    } catch (const rrgpu::BatchOutOfMemory& e) {
      made = e.sets_generated;
    }
    expect(made != UINT64_MAX && made > 0 && made < 100000 && made == st.size(),
           "BatchOutOfMemory carries sets_generated == store size", 0);
    rrflow::WorkPool pool(2);
    rrflow::RRRStore rs(g.num_vertices, pool.workers());
    rrflow::Counter rc(g.num_vertices);
    rrflow::generate_batch(g, rrflow::DiffusionModel::IC, 3, made, pool, rs, &rc);
    bool same = true;
    for (uint32_t v = 0; v < g.num_vertices; ++v) same &= rc.get(v) == cnt.get(v);
    const std::vector<uint64_t> dc = st.counter();
    for (uint32_t v = 0; v < g.num_vertices; ++v) same &= rc.get(v) == dc[v];
    expect(same && st.total_member_count() <= limit,
           "after BatchOutOfMemory: the kept sets and counts are the reference's first sets", 0);
  }
  std::printf("%s (%d failures)\n", failures ? "FAILED" : "ALL PASS", failures);
  return failures ? 1 : 0;
}
