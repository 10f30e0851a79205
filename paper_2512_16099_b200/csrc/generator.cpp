// generator.cpp — synthetic trace generation (host side, trace staging).
//
// Same draw sequence as the reference's generate() (workload.cpp:98-127):
// mt19937_64, 53-bit uniforms, inverse-transform exponential inter-arrivals
// (log1p), Box-Muller standard normals (one per two uniforms), lognormal /
// exponential / fixed service, Long queries conditioned on the upper median
// (workload.cpp:67-85).  Built with -ffp-contract=off and the system libm, so
// a seed yields the reference's trace bit for bit (tests/test_generator.py).
// Traces stay a host concern: GPU libm differs in ulps (SURVEY §7 hard part 7).
#include <atomic>
#include <cmath>
#include <cstring>
#include <numbers>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "migsched_b200.h"

namespace {

struct Draws {
    std::mt19937_64 rng;
    explicit Draws(uint64_t seed) : rng(seed) {}
    double u01() { return static_cast<double>(rng() >> 11) * 0x1.0p-53; }
    double expo(double mean) { return -mean * std::log1p(-u01()); }
    double gauss() {
        const double a = u01();
        const double b = u01();
        return std::sqrt(-2.0 * std::log1p(-a)) * std::cos(2.0 * std::numbers::pi * b);
    }
};

msg_status check(const msg_workload_spec* s) {  // workload.cpp:43-65
    if (!(s->mean_interarrival_s > 0.0)) return MSG_ERR_BAD_SPEC;
    if (s->job_count < 0) return MSG_ERR_BAD_SPEC;
    double sum = 0.0;
    for (double p : s->profile_mix) {
        if (p < 0.0) return MSG_ERR_BAD_SPEC;
        sum += p;
    }
    if (std::abs(sum - 1.0) > 1e-9) return MSG_ERR_BAD_SPEC;
    switch (s->service_family) {
        case 0:
            if (s->median_s <= 0.0 || s->sigma <= 0.0) return MSG_ERR_BAD_SPEC;
            break;
        case 1:
            if (s->mean_s <= 0.0) return MSG_ERR_BAD_SPEC;
            break;
        case 2:
            if (s->value_s <= 0.0) return MSG_ERR_BAD_SPEC;
            break;
        default: return MSG_ERR_BAD_SPEC;
    }
    return MSG_OK;
}

// {1g.5gb, 2g.10gb, 3g.20gb, 4g.20gb} (workload.hpp:29-30)
constexpr int32_t kMixProfiles[4] = {MSG_P1G5GB, MSG_P2G10GB, MSG_P3G20GB, MSG_P4G20GB};

void fill(const msg_workload_spec* s, uint64_t seed, int64_t* id, double* arr, int32_t* prof, double* svc) {
    Draws d(seed);
    double clock = 0.0;
    for (int32_t i = 0; i < s->job_count; ++i) {
        clock += d.expo(s->mean_interarrival_s);
        const double pick = d.u01();
        double acc = 0.0;
        int32_t chosen = kMixProfiles[3];
        for (int k = 0; k < 4; ++k) {
            acc += s->profile_mix[k];
            if (pick < acc) {
                chosen = kMixProfiles[k];
                break;
            }
        }
        double service;
        if (s->service_family == 0) {
            double z = d.gauss();
            if (s->query_type == 1) z = std::abs(z);
            service = s->median_s * std::exp(s->sigma * z);
        } else if (s->service_family == 1) {
            const double x = d.expo(s->mean_s);
            service = s->query_type == 1 ? s->mean_s * std::numbers::ln2 + x : x;
        } else {
            service = s->value_s;
        }
        id[i] = i;
        arr[i] = clock;
        prof[i] = chosen;
        svc[i] = service;
    }
}

}  // namespace

extern "C" {

msg_status msg_workload_preset(const char* name, msg_workload_spec* s) {
    if (!name || !s) return MSG_ERR_INVALID_ARGUMENT;
    std::memset(s, 0, sizeof(*s));
    s->profile_mix[0] = s->profile_mix[1] = s->profile_mix[2] = s->profile_mix[3] = 0.25;
    s->median_s = 120.0;  // ServiceDist defaults (workload.hpp:17-23)
    s->sigma = 0.8;
    s->mean_s = 150.0;
    s->value_s = 100.0;
    s->job_count = 200;
    const std::string n(name);
    if (n == "normal25") s->mean_interarrival_s = 25.0, s->query_type = 0;
    else if (n == "long25") s->mean_interarrival_s = 25.0, s->query_type = 1;
    else if (n == "normal50") s->mean_interarrival_s = 50.0, s->query_type = 0;
    else if (n == "long50") s->mean_interarrival_s = 50.0, s->query_type = 1;
    else return MSG_ERR_INVALID_ARGUMENT;
    return MSG_OK;
}

msg_status msg_generate(const msg_workload_spec* s, int64_t* id, double* arr, int32_t* prof, double* svc) {
    if (!s) return MSG_ERR_INVALID_ARGUMENT;
    const msg_status st = check(s);
    if (st != MSG_OK) return st;
    fill(s, s->seed, id, arr, prof, svc);
    return MSG_OK;
}

msg_status msg_generate_many(const msg_workload_spec* s, uint64_t seed0, uint32_t n_seeds, int32_t threads,
                             uint64_t* offsets, int64_t* id, double* arr, int32_t* prof, double* svc) {
    if (!s) return MSG_ERR_INVALID_ARGUMENT;
    const msg_status st = check(s);
    if (st != MSG_OK) return st;
    const uint64_t n = (uint64_t)s->job_count;
    for (uint32_t i = 0; i <= n_seeds; ++i) offsets[i] = i * n;
    unsigned nt = threads > 0 ? (unsigned)threads : std::max(1u, std::thread::hardware_concurrency());
    nt = std::min<unsigned>(nt, std::max(1u, n_seeds));
    std::atomic<uint32_t> next{0};
    auto work = [&]() {
        for (;;) {
            const uint32_t k = next.fetch_add(1);
            if (k >= n_seeds) return;
            const uint64_t o = k * n;
            fill(s, seed0 + k, id + o, arr + o, prof + o, svc + o);
        }
    };
    std::vector<std::thread> pool;
    for (unsigned t = 1; t < nt; ++t) pool.emplace_back(work);
    work();
    for (auto& th : pool) th.join();
    return MSG_OK;
}

}  // extern "C"
