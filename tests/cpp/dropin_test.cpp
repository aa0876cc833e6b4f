// Drop-in test: cases of the reference's own unit tests (proj/tests/
// test_primitives.cpp / test_engine.cpp) re-run through include/mgraph_b200.hpp
// with only the include and the namespace changed.  Built and run by
// tests/test_dropin_cpp.py; `--host-only` skips the GPU cases.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <stdexcept>

#include "mgraph_b200.hpp"

namespace mg = mgraph_b200;  // was: namespace mgraph
using namespace mg;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                         \
  do {                                                                      \
    if (cond) {                                                             \
      ++g_pass;                                                             \
    } else {                                                                \
      ++g_fail;                                                             \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);           \
    }                                                                       \
  } while (0)
template <class E, class F>
bool throws_as(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static Csr p4() { return Csr::path(4); }
static Assignment explicit_assignment(std::vector<uint32_t> o, uint32_t n) {
  Assignment a;
  a.owner = std::move(o);
  a.num_partitions = n;
  return a;
}

static void host_cases() {
  // test_partition.cpp / fixtures: graph prep + partitioners run on the host
  Csr g = Csr::rmat(12, 16, 1);
  CHECK(g.num_vertices() == 4096);
  Assignment a = partition_random(g.num_vertices(), 4, 7);
  CHECK(a.owner.size() == 4096 && a.num_partitions == 4);
  for (uint32_t o : a.owner) CHECK(o < 4);
  CHECK(throws_as<std::invalid_argument>([] { partition_random(10, 0, 1); }));
  CHECK(throws_as<std::invalid_argument>([&] { partition_biased_random(g, 2, 1, 1.5); }));
}

static void gpu_cases() {
  // test_engine.cpp:250-260,289-295 — engine fixture trace: BFS on P4 {0,1|2,3}
  PartitionPlan plan = build_partition_plan(p4(), explicit_assignment({0, 0, 1, 1}, 2),
                                            Duplication::All);
  BfsResult r = bfs(plan, {.source = 0});
  CHECK((r.labels == std::vector<Label>{0, 1, 2, 3}));
  CHECK(r.stats.supersteps == 4);
  CHECK(r.stats.h_total() == 2);
  CHECK(r.stats.h_matrix[0][1] == 1 && r.stats.h_matrix[1][0] == 1);
  CHECK(r.stats.combine_ops == 2);
  // test_engine.cpp:262-269 — validation of duplication / communication
  PartitionPlan onehop = build_partition_plan(p4(), explicit_assignment({0, 0, 1, 1}, 2),
                                              Duplication::OneHop);
  CHECK(throws_as<std::invalid_argument>([&] { bfs(onehop, {.source = 0}); }));
  EngineConfig sel;
  sel.comm_override = CommMode::Selective;
  CHECK(throws_as<std::invalid_argument>([&] { cc(plan, sel); }));
  CHECK(throws_as<std::invalid_argument>([&] { bfs(plan, {.source = 99}); }));
  // test_primitives.cpp:195-202 — SSSP on P4 with weights 2,3,1
  EdgeList e{{0, 1, 2}, {1, 2, 3}, {2, 3, 1}};
  Csr gw = Csr::build(e, 4, true).symmetrize_dedup();
  PartitionPlan wp = build_partition_plan(gw, explicit_assignment({0, 0, 1, 1}, 2),
                                          Duplication::All);
  CHECK((sssp(wp, 0).dists == std::vector<Dist>{0, 2, 5, 6}));
  CHECK(throws_as<std::invalid_argument>([&] { sssp(plan, 0); }));  // no weights
  // test_primitives.cpp:243-249 — CC triangle + isolated
  EdgeList t{{0, 1, 0}, {1, 2, 0}, {0, 2, 0}};
  Csr tri = Csr::build(t, 4).symmetrize_dedup();
  for (uint32_t n : {1u, 2u, 3u}) {
    PartitionPlan tp = build_partition_plan(tri, partition_random(4, n, n + 1), Duplication::All);
    CHECK((cc(tp).components == std::vector<VertexId>{0, 0, 0, 3}));
  }
  // test_primitives.cpp:281-287 — BC on P4 from 0
  BcResult b = bc(plan, 0);
  CHECK(b.bc[0] == 0.0 && b.bc[1] == 2.0 && b.bc[2] == 1.0 && b.bc[3] == 0.0);
  // test_primitives.cpp:319-323 — PR single dangling vertex holds rank 1
  Csr one = Csr::build({}, 1);
  PartitionPlan op = build_partition_plan(one, partition_random(1, 1, 0), Duplication::All);
  CHECK(std::abs(pagerank(op, {}).ranks[0] - 1.0) <= 1e-12);
  // test_primitives.cpp:372-378 — option validation
  CHECK(throws_as<std::invalid_argument>([&] { pagerank(plan, {.damping = 1.5}); }));
  // test_primitives.cpp:440-446 — hard memory cap aborts the whole run
  Csr rm = Csr::rmat(9, 8, 5);
  PartitionPlan rp = build_partition_plan(rm, partition_random(rm.num_vertices(), 2, 4),
                                          Duplication::All);
  EngineConfig cap;
  cap.policy.hard_cap_bytes = 256;
  CHECK(throws_as<CapacityError>([&] { bfs(rp, {.source = 0}, cap); }));
  // test_primitives.cpp:57-64 — BFS labels identical across partition counts
  Csr g12 = Csr::rmat(12, 16, 1);
  PartitionPlan p1 = build_partition_plan(g12, partition_random(4096, 1, 1), Duplication::All);
  std::vector<Label> base = bfs(p1, {.source = 0}).labels;
  for (uint32_t n : {2u, 3u, 4u}) {
    PartitionPlan pn = build_partition_plan(g12, partition_random(4096, n, 7 * n + 1),
                                            Duplication::All);
    CHECK(bfs(pn, {.source = 0}).labels == base);
    CHECK(dobfs(pn, {.source = 0}).labels == base);
  }
}

int main(int argc, char** argv) {
  bool host_only = argc > 1 && std::strcmp(argv[1], "--host-only") == 0;
  host_cases();
  if (!host_only) gpu_cases();
  std::printf("dropin: %d passed, %d failed\n", g_pass, g_fail);
  return g_fail ? 1 : 0;
}
