// persist.cpp -- the experience store's JSONL persistence on the device store
// (the reference's format, experience.cpp:234-271:
// one object per line {"action", "context", "reward", "round", "source"}).
//
// load: the file is split at line boundaries and parsed on all host threads
// (nlohmann json 3.11.3, the reference's own parser, so the same lines are
// corrupt and the same doubles come out); then store()'s semantics are applied
// in line order (gate, dimension fixed by the first accepted row, a later
// change is std::invalid_argument -> SAIR_EINVAL) and the rows go to the
// device in one bulk append (pinned staging, sair_store_append).
// persist: one bulk device->host export, lines formatted by the same library.
// Host-only code (g++), linked into libsair.so.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "json.hpp"
#include "sair.h"

extern "C" sair_status sair_internal_fail(sair_status code, const char* msg);

namespace {

struct Row {
    bool ok = false;
    int round = 0;
    double reward = 0.0;
    std::vector<double> ctx;
};

// Experience fields exactly as the reference's load() reads them
// (experience.cpp:255-263); any nlohmann::json::exception marks the line corrupt.
Row parse_line(const char* b, const char* e) {
    Row r;
    try {
        nlohmann::json j = nlohmann::json::parse(b, e);
        r.round = j.at("round").get<int>();
        (void)j.at("source").get<std::string>();
        r.reward = j.at("reward").get<double>();
        r.ctx = j.at("context").get<std::vector<double>>();
        for (const auto& s : j.at("action")) {  // action_from_json, experience.cpp:214-224
            (void)s.at("replicas").get<int>();
            (void)s.at("cpu_millicores").get<int>();
            (void)s.at("memory_mb").get<int>();
            (void)s.at("rate_ratio_tenths").get<int>();
        }
        r.ok = true;
    } catch (const nlohmann::json::exception&) {
        r.ok = false;
    }
    return r;
}

}  // namespace

extern "C" __attribute__((visibility("default"))) sair_status sair_store_load_jsonl(
    const char* path, double r_min, int device, int nthreads, size_t* corrupt_lines,
    sair_store_t* out) {
    if (!path || !out) return sair_internal_fail(SAIR_EINVAL, "null argument");
    std::ifstream in(path, std::ios::binary);
    if (!in) return sair_internal_fail(SAIR_EIO, (std::string("experience store: cannot read ") + path).c_str());
    std::string data((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    // line spans (std::getline semantics: '\n'-terminated, a last line without
    // one still counts; empty lines are skipped, experience.cpp:252)
    std::vector<std::pair<size_t, size_t>> lines;
    for (size_t p = 0; p < data.size();) {
        size_t q = data.find('\n', p);
        if (q == std::string::npos) q = data.size();
        if (q > p) lines.emplace_back(p, q);
        p = q + 1;
    }
    std::vector<Row> rows(lines.size());
    int nt = nthreads > 0 ? nthreads : (int)std::max(1u, std::thread::hardware_concurrency());
    nt = (int)std::min<size_t>((size_t)nt, std::max<size_t>(1, lines.size() / 256));
    auto work = [&](int t) {
        for (size_t i = t; i < lines.size(); i += nt)
            rows[i] = parse_line(data.data() + lines[i].first, data.data() + lines[i].second);
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < nt; ++t) pool.emplace_back(work, t);
    work(0);
    for (auto& th : pool) th.join();

    size_t bad = 0;
    int dim = -1;
    std::vector<const Row*> good;
    good.reserve(rows.size());
    for (const auto& r : rows) {
        if (!r.ok) {
            ++bad;
            continue;
        }
        good.push_back(&r);
        if (r.reward > r_min) {  // store(): the gate first, then the dimension
            if (dim < 0) {
                dim = (int)r.ctx.size();
            } else if ((int)r.ctx.size() != dim) {
                return sair_internal_fail(SAIR_EINVAL, "experience store: context dimension changed");
            }
        }
    }
    sair_store_t h = nullptr;
    sair_status st = sair_store_create(r_min, device, good.size(), &h);
    if (st != SAIR_OK) return st;
    if (!good.empty()) {
        // rejected rows keep their place (their context is never read)
        const int d = dim > 0 ? dim : 1;
        std::vector<double> ctx(good.size() * (size_t)d, 0.0), rew(good.size());
        std::vector<int32_t> rnd(good.size());
        for (size_t i = 0; i < good.size(); ++i) {
            const Row& r = *good[i];
            rew[i] = r.reward;
            rnd[i] = r.round;
            if (r.reward > r_min) std::copy(r.ctx.begin(), r.ctx.end(), ctx.begin() + i * d);
        }
        if (dim == 0) {  // every accepted row is empty: the device store needs d >= 1
            sair_store_destroy(h);
            return sair_internal_fail(SAIR_EINVAL, "experience store: empty contexts");
        }
        st = sair_store_append(h, ctx.data(), good.size(), d, rew.data(), rnd.data(), nullptr,
                               nullptr);
        if (st != SAIR_OK) {
            sair_store_destroy(h);
            return st;
        }
    }
    if (corrupt_lines) *corrupt_lines = bad;
    *out = h;
    return SAIR_OK;
}

extern "C" __attribute__((visibility("default"))) sair_status sair_store_persist_jsonl(
    sair_store_t h, const char* path) {
    if (!h || !path) return sair_internal_fail(SAIR_EINVAL, "null argument");
    size_t n = 0;
    int d = 0;
    sair_status st = sair_store_size(h, &n);
    if (st == SAIR_OK) st = sair_store_dim(h, &d);
    if (st != SAIR_OK) return st;
    std::ofstream out(path, std::ios::trunc | std::ios::binary);
    if (!out) return sair_internal_fail(SAIR_EIO, (std::string("experience store: cannot write ") + path).c_str());
    const size_t chunk = 1 << 16;
    std::vector<double> ctx, rew;
    std::vector<int32_t> rnd;
    for (size_t o = 0; o < n; o += chunk) {
        const size_t c = std::min(chunk, n - o);
        ctx.resize(c * (size_t)d);
        rew.resize(c);
        rnd.resize(c);
        st = sair_store_export(h, o, c, ctx.data(), rew.data(), rnd.data());
        if (st != SAIR_OK) return st;
        std::string buf;
        for (size_t i = 0; i < c; ++i) {
            // the device store holds no source / action: written empty
            nlohmann::json j{{"round", rnd[i]},
                             {"source", ""},
                             {"reward", rew[i]},
                             {"context", std::vector<double>(ctx.begin() + i * d, ctx.begin() + (i + 1) * d)},
                             {"action", nlohmann::json::array()}};
            buf += j.dump();
            buf += '\n';
        }
        out << buf;
    }
    if (!out) return sair_internal_fail(SAIR_EIO, "experience store: write failed");
    return SAIR_OK;
}
