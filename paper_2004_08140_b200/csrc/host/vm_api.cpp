// evoir::execute / compute_error / evaluate_fitness as batch-of-one calls into
// the device interpreter (reference entry points: src/vm.cpp:500-579 of
// arxiv/paper_2004_08140), plus the CostTable lookup and TestCase JSON.
#include "runtime.hpp"

#include <json.hpp>

#include <cstring>

namespace evoir {

int64_t CostTable::cost(Opcode op, MemSpace space) const {
    switch (op) {
    case Opcode::Add: case Opcode::Sub: case Opcode::Mul: case Opcode::SDiv:
    case Opcode::FAdd: case Opcode::FSub: case Opcode::FMul: case Opcode::FDiv:
        return arith;
    case Opcode::ICmp: case Opcode::FCmp: return cmp;
    case Opcode::Select: return select_op;
    case Opcode::Phi: return phi;
    case Opcode::Const: return constant;
    case Opcode::Br: return br;
    case Opcode::Tid: case Opcode::NThreads: return intrinsic;
    case Opcode::GetIndex: return getindex;
    case Opcode::Load: return space == MemSpace::Shared ? load_shared : load_global;
    case Opcode::Store: return space == MemSpace::Shared ? store_shared : store_global;
    case Opcode::Sync: return sync;
    case Opcode::Ret: return ret;
    }
    return 1;
}

namespace {

ExecStatus status_of(uint8_t s) {
    if (s == GEVO_STATUS_COMPLETED)
        return ExecStatus::Completed;
    if (s == GEVO_STATUS_BUDGET)
        return ExecStatus::BudgetExceeded;
    return ExecStatus::Trap;
}

} // namespace

ExecResult execute(const Kernel& k, const TestCase& t, const ExecConfig& cfg) {
    b200::Device& dev = b200::Device::default_device();
    b200::DeviceSuite suite(dev, b200::build_suite(k.params, {t}));
    b200::BatchImage batch(suite.image());
    batch.add(k);
    b200::EvalOptions opt;
    opt.want_tests = true;
    opt.want_outputs = true;
    b200::EvalResult r = b200::evaluate(suite, batch, b200::exec_image(cfg), opt);
    const gevo_test_record& x = r.tests.at(0);
    ExecResult out;
    out.status = status_of(x.status);
    out.cost = x.cost;
    if (out.status == ExecStatus::Completed)
        out.outputs = std::move(r.outputs[0][0]);
    else
        out.trap_reason = batch.reason(0, x.code, x.aux);
    return out;
}

double compute_error(const BufferMap& candidate, const BufferMap& oracle) {
    return b200::error_on_device(b200::Device::default_device(), candidate, oracle);
}

EvalOutcome evaluate_fitness(const Kernel& k, const std::vector<TestCase>& tests,
                             const ExecConfig& cfg, double tolerance) {
    if (tests.empty())
        return EvalOutcome::rejected(-1, "no test cases");
    b200::Device& dev = b200::Device::default_device();
    b200::DeviceSuite suite(dev, b200::build_suite(k.params, tests));
    b200::BatchImage batch(suite.image());
    batch.add(k);
    b200::EvalOptions opt;
    opt.tolerance = tolerance;
    opt.early_exit = true;
    b200::EvalResult r = b200::evaluate(suite, batch, b200::exec_image(cfg), opt);
    const gevo_variant_record& v = r.variants.at(0);
    if (v.accepted)
        return EvalOutcome::ok(FitnessVector{v.cost_mean, v.error_max});
    if (v.code == GEVO_FAIL_TOLERANCE)
        return EvalOutcome::rejected(v.failing_test,
                                     "error " + std::to_string(v.fail_error) + " exceeds tolerance");
    return EvalOutcome::rejected(v.failing_test, batch.reason(0, v.code, v.aux));
}

// ---------------------------------------------------------------------------
// TestCase JSON (reference document shape, src/vm.cpp:585-660)
// ---------------------------------------------------------------------------

namespace {

using nlohmann::json;

json buffer_json(const Buffer& b) {
    json j;
    j["type"] = b.elem == TypeKind::I32 ? "i32" : "f32";
    if (b.elem == TypeKind::I32) {
        j["data"] = b.i;
    } else {
        json a = json::array();
        for (float x : b.f)
            a.push_back(static_cast<double>(x));
        j["data"] = std::move(a);
    }
    return j;
}

Buffer buffer_parse(const json& j) {
    const std::string t = j.at("type").get<std::string>();
    Buffer b;
    if (j.contains("hex")) {
        // Bit-exact extension of the reference format: 8 hex digits per
        // element (carries NaN / inf payloads that JSON numbers cannot).
        const std::string h = j.at("hex").get<std::string>();
        if (t != "i32" && t != "f32")
            throw std::runtime_error("unknown buffer type '" + t + "'");
        b.elem = t == "i32" ? TypeKind::I32 : TypeKind::F32;
        for (size_t p = 0; p + 8 <= h.size(); p += 8) {
            const uint32_t w = static_cast<uint32_t>(std::stoul(h.substr(p, 8), nullptr, 16));
            if (b.elem == TypeKind::I32) {
                int32_t x;
                std::memcpy(&x, &w, 4);
                b.i.push_back(x);
            } else {
                float x;
                std::memcpy(&x, &w, 4);
                b.f.push_back(x);
            }
        }
        return b;
    }
    if (t == "i32") {
        b.elem = TypeKind::I32;
        b.i = j.at("data").get<std::vector<int32_t>>();
    } else if (t == "f32") {
        b.elem = TypeKind::F32;
        for (const json& x : j.at("data"))
            b.f.push_back(static_cast<float>(x.get<double>()));
    } else {
        throw std::runtime_error("unknown buffer type '" + t + "'");
    }
    return b;
}

} // namespace

std::string testcase_to_json(const TestCase& t) {
    json j;
    j["inputs"] = json::object();
    for (const auto& [n, b] : t.inputs)
        j["inputs"][n] = buffer_json(b);
    j["scalars"] = json::object();
    for (const auto& [n, s] : t.scalars) {
        json x;
        if (s.kind == TypeKind::I32) {
            x["type"] = "i32";
            x["value"] = s.i;
        } else if (s.kind == TypeKind::F32) {
            x["type"] = "f32";
            x["value"] = static_cast<double>(s.f);
        } else {
            x["type"] = "bool";
            x["value"] = s.b;
        }
        j["scalars"][n] = std::move(x);
    }
    j["oracle"] = json::object();
    for (const auto& [n, b] : t.oracle)
        j["oracle"][n] = buffer_json(b);
    return j.dump(2) + "\n";
}

TestCase testcase_from_json(const std::string& text) {
    const json j = json::parse(text);
    TestCase t;
    for (const auto& [n, b] : j.at("inputs").items())
        t.inputs[n] = buffer_parse(b);
    if (j.contains("scalars"))
        for (const auto& [n, x] : j.at("scalars").items()) {
            const std::string ty = x.at("type").get<std::string>();
            if (ty == "i32")
                t.scalars[n] = Scalar::of_i32(x.at("value").get<int32_t>());
            else if (ty == "f32")
                t.scalars[n] = Scalar::of_f32(static_cast<float>(x.at("value").get<double>()));
            else
                t.scalars[n] = Scalar::of_bool(x.at("value").get<bool>());
        }
    for (const auto& [n, b] : j.at("oracle").items())
        t.oracle[n] = buffer_parse(b);
    return t;
}

} // namespace evoir
