// race_cert.cpp -- TEST INFRASTRUCTURE ONLY.
//
// Runs the reference's own static race checker on a kernel model:
//   parse_model_text  (/root/reference/proj/src/model_text.cpp, grammar
//                      proj/include/raceset/model_text.hpp:12-29)
//   races()           (/root/reference/proj/src/depcheck.cpp:218; happens-before
//                      with warp phases, proj/src/kernel_model.cpp:328-356)
// and prints one JSON line per model file:
//   {"model": name, "file": path, "verdict": "RaceFree"|"RaceFound"|"Inconclusive",
//    "races": n, "witnesses": [{"array", "source", "target", "src_iter", "dst_iter"}...], "ms": t}
// Linked against the reference objects compiled in place by `make -C oracle ref`
// (oracle/_ref/race_cert); nothing from the reference is copied into this repo.
#include <chrono>
#include <cstdio>
#include <exception>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>

#include "raceset/depcheck.hpp"
#include "raceset/model_text.hpp"

namespace {

std::string esc(const std::string& s) {
  std::string o;
  for (char c : s) {
    if (c == '"' || c == '\\') o += '\\';
    if (c == '\n') { o += "\\n"; continue; }
    o += c;
  }
  return o;
}

std::string iter_json(const std::map<std::string, int64_t>& m) {
  std::string o = "{";
  bool first = true;
  for (const auto& [k, v] : m) {
    if (!first) o += ", ";
    first = false;
    o += "\"" + esc(k) + "\": " + std::to_string(v);
  }
  return o + "}";
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: race_cert MODEL_FILE...  ('-' reads one model from stdin)\n");
    return 2;
  }
  int rc = 0;
  for (int a = 1; a < argc; ++a) {
    const std::string path = argv[a];
    std::string text;
    if (path == "-") {
      std::stringstream ss;
      ss << std::cin.rdbuf();
      text = ss.str();
    } else {
      std::ifstream f(path);
      if (!f) {
        std::printf("{\"file\": \"%s\", \"error\": \"cannot open\"}\n", esc(path).c_str());
        rc = 1;
        continue;
      }
      std::stringstream ss;
      ss << f.rdbuf();
      text = ss.str();
    }
    try {
      const auto t0 = std::chrono::steady_clock::now();
      const raceset::KernelModel model = raceset::parse_model_text(text);
      const raceset::DependenceReport rep = raceset::races(model);
      const double ms =
          std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      std::string w = "[";
      for (size_t i = 0; i < rep.race_witnesses.size() && i < 4; ++i) {
        const auto& x = rep.race_witnesses[i];
        if (i) w += ", ";
        w += "{\"array\": \"" + esc(x.array) + "\", \"source\": \"" + esc(x.source) +
             "\", \"target\": \"" + esc(x.target) + "\", \"src_iter\": " + iter_json(x.source_iter) +
             ", \"dst_iter\": " + iter_json(x.target_iter) + "}";
      }
      w += "]";
      std::string why = "[";
      for (size_t i = 0; i < rep.inconclusive_reasons.size() && i < 6; ++i)
        why += (i ? ", \"" : "\"") + esc(rep.inconclusive_reasons[i]) + "\"";
      why += "]";
      std::printf("{\"model\": \"%s\", \"file\": \"%s\", \"verdict\": \"%s\", \"races\": %zu, "
                  "\"witnesses\": %s, \"inconclusive\": %s, \"ms\": %.1f}\n",
                  esc(model.name).c_str(), esc(path).c_str(), raceset::race_verdict_name(rep.verdict),
                  rep.races.size(), w.c_str(), why.c_str(), ms);
    } catch (const std::exception& e) {
      std::printf("{\"file\": \"%s\", \"error\": \"%s\"}\n", esc(path).c_str(), esc(e.what()).c_str());
      rc = 1;
    }
    std::fflush(stdout);
  }
  return rc;
}
