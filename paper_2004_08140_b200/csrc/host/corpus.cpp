// Benchmark registry and seeded test generation.
//
// Kernels, reach patches and generator specs are data (data/corpus.json,
// embedded at build time). Input draws follow src/corpus.cpp:429-483 of
// arxiv/paper_2004_08140 (per-buffer stream Rng::stream(seed, t, bi, 91),
// float arithmetic without contraction); oracles come from executing the
// original kernel, here as one device batch over all tests.
#include "evoir/corpus.hpp"

#include "evoir/rng.hpp"
#include "runtime.hpp"

#include <json.hpp>

#include <map>
#include <numeric>

namespace evoir {

namespace {

const char kCorpusJson[] =
#include "corpus_data.inc"
    ;

using nlohmann::json;

struct Entry {
    PlantedClass cls;
    std::string ir;
    std::string reach;
    GeneratorSpec gen;
    std::string notes;
};

PlantedClass class_from_name(const std::string& s) {
    static const std::pair<const char*, PlantedClass> table[] = {
        {"ConservativeSync", PlantedClass::ConservativeSync},
        {"RedundantStore", PlantedClass::RedundantStore},
        {"DeadConditional", PlantedClass::DeadConditional},
        {"RedundantLoad", PlantedClass::RedundantLoad},
        {"LoopPerforation", PlantedClass::LoopPerforation},
        {"Memoization", PlantedClass::Memoization}};
    for (const auto& [n, c] : table)
        if (s == n)
            return c;
    throw std::runtime_error("unknown planted class '" + s + "'");
}

GeneratorSpec spec_from(const json& buffers, const json& scalars) {
    GeneratorSpec g;
    for (const json& bj : buffers) {
        BufferSpec s;
        s.name = bj.at("name").get<std::string>();
        s.elem = bj.at("type").get<std::string>() == "i32" ? TypeKind::I32 : TypeKind::F32;
        s.size = bj.at("size").get<int>();
        s.output = bj.value("output", false);
        const json& d = bj.at("dist");
        const std::string kind = d.at("kind").get<std::string>();
        if (kind == "uniform") {
            s.dist = BufferSpec::Dist::Uniform;
            s.lo = d.at("low").get<double>();
            s.hi = d.at("high").get<double>();
        } else if (kind == "jitter_of") {
            s.dist = BufferSpec::Dist::JitterOf;
            s.source = d.at("source").get<std::string>();
            s.amplitude = d.at("amplitude").get<double>();
        } else if (kind == "zeros") {
            s.dist = BufferSpec::Dist::Zeros;
        } else if (kind == "permutation") {
            s.dist = BufferSpec::Dist::Permutation;
            s.elem = TypeKind::I32;
        } else {
            throw std::runtime_error("unknown distribution kind '" + kind + "'");
        }
        g.buffers.push_back(std::move(s));
    }
    for (const json& sj : scalars) {
        ScalarSpec s;
        s.name = sj.at("name").get<std::string>();
        const std::string ty = sj.at("type").get<std::string>();
        if (ty == "i32")
            s.value = Scalar::of_i32(sj.at("value").get<int32_t>());
        else if (ty == "f32")
            s.value = Scalar::of_f32(static_cast<float>(sj.at("value").get<double>()));
        else
            s.value = Scalar::of_bool(sj.at("value").get<bool>());
        g.scalars.push_back(std::move(s));
    }
    return g;
}

const std::map<std::string, Entry>& registry() {
    static const std::map<std::string, Entry> reg = [] {
        std::map<std::string, Entry> m;
        const json doc = json::parse(kCorpusJson);
        for (const json& b : doc.at("benchmarks")) {
            Entry e;
            e.cls = class_from_name(b.at("class").get<std::string>());
            e.ir = b.at("ir").get<std::string>();
            e.reach = b.at("reach").dump();
            e.gen = spec_from(b.at("buffers"), b.at("scalars"));
            e.notes = b.at("notes").get<std::string>();
            m.emplace(b.at("name").get<std::string>(), std::move(e));
        }
        return m;
    }();
    return reg;
}

} // namespace

const char* planted_class_name(PlantedClass c) {
    static const char* const names[] = {"ConservativeSync", "RedundantStore", "DeadConditional",
                                        "RedundantLoad",    "LoopPerforation", "Memoization"};
    const auto i = static_cast<size_t>(c);
    return i < 6 ? names[i] : "?";
}

const std::vector<std::string>& benchmark_names() {
    static const std::vector<std::string> names = [] {
        std::vector<std::string> v;
        for (const auto& kv : registry())
            v.push_back(kv.first);
        return v;
    }();
    return names;
}

Benchmark load_benchmark(const std::string& name) {
    const auto it = registry().find(name);
    if (it == registry().end())
        throw UnknownBenchmark("unknown benchmark '" + name + "'");
    const Entry& e = it->second;
    Benchmark b;
    b.name = name;
    b.planted_class = e.cls;
    b.kernel = parse_kernel(e.ir);
    b.reach_patch = patch_from_json(e.reach);
    b.gen = e.gen;
    b.notes = e.notes;
    const auto errs = validate(b.kernel);
    if (!errs.empty())
        throw std::logic_error("benchmark '" + name + "' kernel fails validation: " +
                               errs.front().rule);
    PatchResult reach = apply_patch(b.kernel, b.reach_patch);
    if (reach.applied.size() != b.reach_patch.size())
        throw std::logic_error("benchmark '" + name + "' reach patch has inapplicable edits");
    if (!is_valid(reach.kernel))
        throw std::logic_error("benchmark '" + name + "' improved variant fails validation");
    b.improved = std::move(reach.kernel);
    return b;
}

std::vector<TestCase> generate_inputs_for(const GeneratorSpec& gen, int count, uint64_t seed) {
    std::vector<TestCase> tests;
    tests.reserve(static_cast<size_t>(std::max(count, 0)));
    for (int t = 0; t < count; ++t) {
        TestCase tc;
        for (size_t bi = 0; bi < gen.buffers.size(); ++bi) {
            const BufferSpec& s = gen.buffers[bi];
            Rng rng = Rng::stream(seed, static_cast<uint64_t>(t), bi, 91);
            Buffer b;
            b.elem = s.elem;
            const size_t n = static_cast<size_t>(std::max(s.size, 0));
            switch (s.dist) {
            case BufferSpec::Dist::Uniform:
                if (s.elem == TypeKind::F32) {
                    const float lo = static_cast<float>(s.lo);
                    const float span = static_cast<float>(s.hi - s.lo);
                    for (size_t i = 0; i < n; ++i) {
                        const float scaled = rng.uniform_float() * span;
                        b.f.push_back(lo + scaled);
                    }
                } else {
                    const int32_t lo = static_cast<int32_t>(s.lo);
                    for (size_t i = 0; i < n; ++i)
                        b.i.push_back(lo + static_cast<int32_t>(
                                               rng.below(static_cast<uint64_t>(s.hi - s.lo))));
                }
                break;
            case BufferSpec::Dist::JitterOf: {
                const Buffer& src = tc.inputs.at(s.source);
                const float amp = static_cast<float>(s.amplitude);
                for (size_t i = 0; i < n; ++i) {
                    const float u = rng.uniform_float() * 2.0f - 1.0f;
                    const float scale = 1.0f + amp * u;
                    b.f.push_back(src.f[i] * scale);
                }
                break;
            }
            case BufferSpec::Dist::Zeros:
                if (s.elem == TypeKind::F32)
                    b.f.assign(n, 0.0f);
                else
                    b.i.assign(n, 0);
                break;
            case BufferSpec::Dist::Permutation:
                b.elem = TypeKind::I32;
                b.i.resize(n);
                std::iota(b.i.begin(), b.i.end(), 0);
                rng.shuffle(b.i);
                break;
            }
            tc.inputs[s.name] = std::move(b);
        }
        for (const ScalarSpec& sc : gen.scalars)
            tc.scalars[sc.name] = sc.value;
        tests.push_back(std::move(tc));
    }
    return tests;
}

std::vector<TestCase> generate_tests_for(const Kernel& kernel, const GeneratorSpec& gen, int count,
                                         uint64_t seed) {
    std::vector<TestCase> tests = generate_inputs_for(gen, count, seed);
    if (tests.empty())
        return tests;
    // Oracle = the original's outputs: one variant x T tests on the device.
    b200::Device& dev = b200::Device::default_device();
    b200::DeviceSuite suite(dev, b200::build_suite(kernel.params, tests));
    b200::BatchImage batch(suite.image());
    batch.add(kernel);
    b200::EvalOptions opt;
    opt.want_tests = true;
    opt.want_outputs = true;
    const b200::EvalResult r =
        b200::evaluate(suite, batch, b200::exec_image(ExecConfig::for_kernel(kernel)), opt);
    for (size_t t = 0; t < tests.size(); ++t) {
        const gevo_test_record& x = r.tests[t];
        if (x.status != GEVO_STATUS_COMPLETED)
            throw std::logic_error("kernel '" + kernel.name + "' failed while producing an " +
                                   "oracle: " + batch.reason(0, x.code, x.aux));
        for (const BufferSpec& s : gen.buffers)
            if (s.output)
                tests[t].oracle[s.name] = r.outputs[0][t].at(s.name);
    }
    return tests;
}

std::vector<TestCase> generate_tests(const Benchmark& b, int count, uint64_t seed) {
    return generate_tests_for(b.kernel, b.gen, count, seed);
}

double measured_gain(const Benchmark& b, int test_count, uint64_t seed) {
    const std::vector<TestCase> tests = generate_tests(b, test_count, seed);
    b200::Device& dev = b200::Device::default_device();
    b200::DeviceSuite suite(dev, b200::build_suite(b.kernel.params, tests));
    b200::BatchImage batch(suite.image());
    batch.add(b.kernel);
    batch.add(b.improved);
    b200::EvalOptions opt;
    opt.want_tests = true;
    const b200::EvalResult r =
        b200::evaluate(suite, batch, b200::exec_image(ExecConfig::for_kernel(b.kernel)), opt);
    double orig = 0.0, improved = 0.0;
    const size_t T = tests.size();
    for (size_t t = 0; t < T; ++t) {
        const gevo_test_record& o = r.tests[t];
        const gevo_test_record& i = r.tests[T + t];
        if (o.status != GEVO_STATUS_COMPLETED || i.status != GEVO_STATUS_COMPLETED)
            throw std::logic_error("benchmark '" + b.name + "' gain measurement trapped");
        orig += static_cast<double>(o.cost);
        improved += static_cast<double>(i.cost);
    }
    return (orig - improved) / orig;
}

std::string generator_spec_to_json(const Benchmark& b) {
    json j;
    j["name"] = b.name;
    j["planted_class"] = planted_class_name(b.planted_class);
    j["kernel"] = b.name + ".ir";
    j["improved"] = b.name + ".improved.ir";
    j["reach_patch"] = b.name + ".patch.json";
    j["notes"] = b.notes;
    json bufs = json::array();
    for (const BufferSpec& s : b.gen.buffers) {
        json bj;
        bj["name"] = s.name;
        bj["type"] = s.elem == TypeKind::I32 ? "i32" : "f32";
        bj["size"] = s.size;
        switch (s.dist) {
        case BufferSpec::Dist::Uniform:
            bj["dist"] = {{"kind", "uniform"}, {"low", s.lo}, {"high", s.hi}};
            break;
        case BufferSpec::Dist::JitterOf:
            bj["dist"] = {{"kind", "jitter_of"}, {"source", s.source}, {"amplitude", s.amplitude}};
            break;
        case BufferSpec::Dist::Zeros:
            bj["dist"] = {{"kind", "zeros"}};
            break;
        case BufferSpec::Dist::Permutation:
            bj["dist"] = {{"kind", "permutation"}};
            break;
        }
        if (s.output)
            bj["output"] = true;
        bufs.push_back(std::move(bj));
    }
    j["buffers"] = std::move(bufs);
    json scal = json::array();
    for (const ScalarSpec& s : b.gen.scalars) {
        json sj;
        sj["name"] = s.name;
        if (s.value.kind == TypeKind::I32) {
            sj["type"] = "i32";
            sj["value"] = s.value.i;
        } else if (s.value.kind == TypeKind::F32) {
            sj["type"] = "f32";
            sj["value"] = static_cast<double>(s.value.f);
        } else {
            sj["type"] = "bool";
            sj["value"] = s.value.b;
        }
        scal.push_back(std::move(sj));
    }
    j["scalars"] = std::move(scal);
    return j.dump(2) + "\n";
}

GeneratorSpec generator_spec_from_json(const std::string& text) {
    const json j = json::parse(text);
    return spec_from(j.at("buffers"), j.contains("scalars") ? j.at("scalars") : json::array());
}

} // namespace evoir
