// tests/cpp/dropin_test.cpp — the C++ drop-in (include/arraylog_b200) against
// the reference engine in ONE binary: every scenario runs arraylog::engine
// (reference, CPU) and arraylog::b200::engine (B200) on the same inputs and
// compares outputs byte for byte plus run_stats bookkeeping.  Scenarios
// restate tests/engine_test.cpp, ra_test.cpp and acceptance_test.cpp of the
// reference.  Built by tests/cpp/Makefile (needs /root/reference at build
// time only); run by tests/test_gpu_dropin.py on a B200.
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <unistd.h>
#include <random>
#include <string>

#include "arraylog/arraylog.hpp"
#include "arraylog_b200/arraylog_b200.hpp"
#include "oracles.hpp"

using namespace arraylog;

static int g_fail = 0, g_pass = 0;

#define CHECK(cond, what)                                                  \
    do {                                                                   \
        if (cond) {                                                        \
            ++g_pass;                                                      \
        } else {                                                           \
            ++g_fail;                                                      \
            std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, what);      \
        }                                                                  \
    } while (0)

static tuple_array chain_edges(value_t nodes) {
    tuple_array t(2);
    for (value_t i = 1; i < nodes; ++i) {
        t.data.push_back(i);
        t.data.push_back(i + 1);
    }
    return t;
}

static void compare_engines(const std::string& what, const program& prog,
                            const std::vector<std::pair<std::string, tuple_array>>& edbs,
                            engine_config cfg = {}) {
    engine ref(prog, cfg);
    b200::engine dev(prog, cfg);
    for (const auto& [n, t] : edbs) {
        ref.load_edb(n, t);
        dev.load_edb(n, t);
    }
    ref.run();
    dev.run();
    for (const auto& n : prog.idb_relations())
        CHECK(ref.relation(n) == dev.relation(n), (what + ": relation " + n).c_str());
    const run_stats a = ref.stats(), b = dev.stats();
    CHECK(a.iterations == b.iterations, (what + ": iterations").c_str());
    CHECK(a.delta_history == b.delta_history, (what + ": delta history").c_str());
    CHECK(a.charge_events == b.charge_events, (what + ": charge events").c_str());
    CHECK(a.peak_tracked_bytes == b.peak_tracked_bytes, (what + ": peak tracked bytes").c_str());
    CHECK(a.peak_temp_bytes == b.peak_temp_bytes, (what + ": peak temp bytes").c_str());
    CHECK(a.buffer_allocations == b.buffer_allocations, (what + ": buffer allocations").c_str());
}

// io.hpp restated: device read_facts / to_tsv / engine file load + write
// against the reference's own functions, byte for byte.
static void io_scenarios() {
    namespace fs = std::filesystem;
    const fs::path dir = fs::temp_directory_path() / ("gd_io_" + std::to_string(::getpid()));
    fs::create_directories(dir);
    auto write = [&](const std::string& name, const std::string& text) {
        const fs::path p = dir / name;
        std::ofstream(p, std::ios::binary) << text;
        return p;
    };
    const std::vector<std::string> texts = {"1 2\n2 3\n1 2\n", "# h\n1\t2\n\n  3   4 \n\t5\t6\r\n", "1 2\n3 4 5\n",
                                            "x 1\n", "1 18446744073709551615\n", "", "7 8"};
    for (std::size_t i = 0; i < texts.size(); ++i) {
        const fs::path p = write("f" + std::to_string(i) + ".tsv", texts[i]);
        std::string ref_err, dev_err;
        tuple_array r(2), d(2);
        try { r = read_facts(p, 2); } catch (const load_error& e) { ref_err = e.what(); }
        try { d = b200::read_facts(p, 2); } catch (const load_error& e) { dev_err = e.what(); }
        CHECK(ref_err == dev_err, ("read_facts error " + std::to_string(i)).c_str());
        CHECK(ref_err.empty() ? r == d : true, ("read_facts rows " + std::to_string(i)).c_str());
        CHECK(file_is_all_integers(p) == b200::file_is_all_integers(p), "file_is_all_integers");
    }
    std::mt19937_64 rng(223);
    for (int t = 0; t < 5; ++t) {
        tuple_array rel = canonicalize(oracles::random_relation(rng, 3, 500, 1000));
        CHECK(to_tsv(rel) == b200::to_tsv(rel), "to_tsv bytes");
    }
    // engine: load a fact file on the device, write the IDB as TSV
    tuple_array edges = canonicalize(oracles::from_set(2, oracles::random_graph(rng, 200, 800)));
    const fs::path ep = dir / "edge.tsv";
    write_relation(edges, ep);
    arraylog::engine re(builtin_program("reach"));
    re.load_edb("Edge", read_facts(ep, 2));
    re.run();
    b200::engine ge(builtin_program("reach"));
    ge.load_edb_file("Edge", ep);
    ge.run();
    ge.write_relation_file("Reach", dir / "reach.tsv");
    std::ifstream in(dir / "reach.tsv", std::ios::binary);
    const std::string got((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    CHECK(got == to_tsv(re.relation("Reach")), "engine TSV round trip");
    fs::remove_all(dir);
}

int main() {
    io_scenarios();
    // engine_test.cpp:42-52 (path5), :71-81 (SG tree), :83-93 (CSPA seed)
    compare_engines("reach path5", builtin_program("reach"), {{"Edge", chain_edges(5)}});
    {
        b200::engine e(builtin_program("reach"));
        e.load_edb("Edge", chain_edges(5));
        e.run();
        CHECK(e.relation("Reach").count() == 10, "path5 count");
        CHECK(e.stats().delta_history.at(0).second == (std::vector<std::size_t>{4, 3, 2, 1}), "path5 history");
    }
    compare_engines("sg tree", builtin_program("sg"),
                    {{"Edge", tuple_array(2, {1, 2, 1, 3, 2, 4, 2, 5, 3, 6, 3, 7})}});
    compare_engines("cspa seed", builtin_program("cspa"), {{"assign", tuple_array(2, {1, 2})}});
    compare_engines("ebm off", builtin_program("reach"), {{"Edge", chain_edges(60)}},
                    [] { engine_config c; c.ebm_enabled = false; return c; }());

    // acceptance_test.cpp corpora (seeds 20240601-3), a slice of each
    {
        std::mt19937_64 rng(20240601);
        for (int i = 0; i < 40; ++i) {
            auto g = oracles::random_graph(rng, 50, 400);
            if (i % 4) continue;
            compare_engines("reach corpus " + std::to_string(i), builtin_program("reach"),
                            {{"Edge", oracles::from_set(2, g)}});
        }
    }
    {
        std::mt19937_64 rng(20240602);
        for (int i = 0; i < 20; ++i) {
            auto g = oracles::random_dag(rng, 30, 60);
            if (i % 4) continue;
            compare_engines("sg corpus " + std::to_string(i), builtin_program("sg"),
                            {{"Edge", oracles::from_set(2, g)}});
        }
    }
    {
        std::mt19937_64 rng(20240603);
        std::uniform_int_distribution<value_t> node(1, 15);
        std::uniform_int_distribution<int> count(1, 100);
        for (int i = 0; i < 12; ++i) {
            oracles::database db;
            int na = count(rng), nd = count(rng);
            for (int j = 0; j < na; ++j) db["assign"].insert({node(rng), node(rng)});
            for (int j = 0; j < nd; ++j) db["dereference"].insert({node(rng), node(rng)});
            if (i % 3) continue;
            compare_engines("cspa corpus " + std::to_string(i), builtin_program("cspa"),
                            {{"assign", oracles::from_set(2, db["assign"])},
                             {"dereference", oracles::from_set(2, db["dereference"])}});
        }
    }
    // engine_test.cpp:250-274 (constants, repeated vars, Cartesian, constraints)
    {
        auto parsed = parse_program(
            ".decl E(2)\n.decl A(1)\n.decl B(1)\nMarker(1) :- E(x, y).\nSelfish(x) :- E(x, x).\n"
            "Pairs(x, y) :- A(x), B(y).\nLoopy(x, y) :- E(x, y), x != y.\n"
            "Loopy(x, y) :- Loopy(x, z), E(z, y), x != y.\n");
        compare_engines("constants/cartesian", parsed.prog,
                        {{"E", tuple_array(2, {1, 1, 1, 2, 2, 3, 3, 1})},
                         {"A", tuple_array(1, {5, 6})},
                         {"B", tuple_array(1, {7})}});
    }
    // engine_test.cpp:183-194: budget errors name a phase (same as reference)
    {
        engine_config cfg;
        cfg.memory_budget_bytes = 400;
        std::string ref_phase, dev_phase;
        try {
            engine e(builtin_program("reach"), cfg);
            e.load_edb("Edge", chain_edges(30));
            e.run();
        } catch (const budget_error& e) {
            ref_phase = e.phase();
        }
        try {
            b200::engine e(builtin_program("reach"), cfg);
            e.load_edb("Edge", chain_edges(30));
            e.run();
        } catch (const budget_error& e) {
            dev_phase = e.phase();
        }
        CHECK(!dev_phase.empty() && dev_phase == ref_phase, "budget error phase");
    }
    // engine_test.cpp:293-300 load errors
    {
        b200::engine e(builtin_program("reach"));
        bool a = false, b = false, c = false;
        try { e.load_edb("Nope", tuple_array(2, {1, 2})); } catch (const load_error&) { a = true; }
        try { e.load_edb("Edge", tuple_array(1, {1})); } catch (const load_error&) { b = true; }
        try { e.load_edb("Edge", tuple_array(2, {1, kEmptySlot})); } catch (const load_error&) { c = true; }
        CHECK(a && b && c, "load errors");
    }
    // kernel-level parity (ra_test.cpp, tuple_array_test.cpp)
    {
        std::mt19937_64 rng(41);
        for (int trial = 0; trial < 10; ++trial) {
            tuple_array raw = oracles::random_relation(rng, 2, 3000, 200);
            CHECK(canonicalize(raw) == b200::canonicalize(raw), "canonicalize");
            auto outer = make_container(canonicalize(oracles::random_relation(rng, 2, 500, 40)));
            auto inner = make_container(canonicalize(oracles::random_relation(rng, 2, 500, 40)), {}, 1);
            join_spec spec{1, &outer, &inner, column_map{{operand::outer(1), operand::inner(1)}}, {}};
            const std::size_t n = join_count(spec);
            CHECK(n == b200::join_count(spec), "join_count");
            tuple_array a(2), b(2);
            a.data.resize(n * 2);
            b.data.resize(n * 2);
            join_materialize(spec, a);
            b200::join_materialize(spec, b);
            CHECK(a == b, "join_materialize raw bytes");
            std::vector<std::uint32_t> perm{1, 0};
            CHECK(permute_columns(outer.tuples, perm) == b200::permute_columns(outer.tuples, perm), "permute");
            tuple_array d = difference(inner.tuples, outer.tuples);
            CHECK(d == b200::difference(inner.tuples, outer.tuples), "difference");
            std::vector<value_t> buf((outer.tuples.count() + d.count()) * 2);
            CHECK(merge_sorted(outer.tuples, d, buf) == b200::merge_sorted(outer.tuples, d, buf), "merge_sorted");
            for (value_t k = 0; k < 40; ++k) {
                const value_t key[1] = {k};
                CHECK(range_lookup(inner, key) == b200::range_lookup(inner, key), "range_lookup");
            }
        }
    }
    std::printf("dropin_test: %d passed, %d failed\n", g_pass, g_fail);
    return g_fail ? 1 : 0;
}
