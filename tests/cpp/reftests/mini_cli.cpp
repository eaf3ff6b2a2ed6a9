// mini_cli — test harness only: the `arraylog run` subcommand that
// acceptance_test.cpp's criterion 8 spawns (ARRAYLOG_CLI_PATH), on the B200
// drop-in.  The reference CLI (tools/arraylog_cli.cpp) needs CLI11, which
// this image lacks; this keeps its flags, outputs and exit codes (0 ok,
// 1 usage/parse/load, 2 budget; tools/arraylog_cli.cpp:163-181).
#include <cstdlib>
#include <iostream>
#include <map>
#include <string>
#include <vector>

#include "arraylog/arraylog.hpp"  // shim: reference frontend + device engine

namespace fs = std::filesystem;
using namespace arraylog;

static int run(int argc, char** argv) {
    if (argc < 2 || std::string(argv[1]) != "run") throw usage_error("usage: mini_cli run --program P --facts R=path");
    std::string prog_name, out_dir = ".";
    std::vector<std::string> facts;
    engine_config cfg;
    bool emit_facts = true, emit_stats = false;
    for (int i = 2; i < argc; ++i) {
        const std::string a = argv[i];
        auto val = [&]() -> std::string {
            if (i + 1 >= argc) throw usage_error(a + " expects a value");
            return argv[++i];
        };
        if (a == "--program") prog_name = val();
        else if (a == "--facts") facts.push_back(val());
        else if (a == "--out") out_dir = val();
        else if (a == "--memory-budget") cfg.memory_budget_bytes = std::stoull(val());
        else if (a == "--ebm") cfg.ebm_enabled = val() == "on";
        else if (a == "--alpha") cfg.alpha = std::stoul(val());
        else if (a == "--load-factor") cfg.load_factor = std::stod(val());
        else if (a == "--workers") cfg.workers = std::stoul(val());
        else if (a == "--stride") cfg.stride_rows = std::stoull(val());
        else if (a == "--no-facts") emit_facts = false;
        else if (a == "--stats") emit_stats = true;
        else throw usage_error("unknown flag '" + a + "'");
    }
    program prog = builtin_program(prog_name);
    std::map<std::string, fs::path> paths;
    for (const auto& f : facts) {
        const auto eq = f.find('=');
        if (eq == std::string::npos) throw usage_error("--facts expects <relation>=<path>");
        paths[f.substr(0, eq)] = f.substr(eq + 1);
    }
    engine eng(prog, cfg);
    for (const auto& e : prog.edbs) eng.load_edb(e.name, read_facts(paths.at(e.name), e.arity));
    eng.run();
    fs::create_directories(out_dir);
    for (const auto& name : eng.idb_relations()) {
        const auto& rel = eng.relation(name);
        std::cout << name << " " << rel.count() << "\n";
        if (emit_facts) write_relation(rel, fs::path(out_dir) / (name + ".tsv"));
    }
    if (emit_stats) std::ofstream(fs::path(out_dir) / "stats.tsv", std::ios::binary) << to_tsv(eng.stats());
    return 0;
}

int main(int argc, char** argv) {
    try {
        return run(argc, argv);
    } catch (const budget_error& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 2;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
}
