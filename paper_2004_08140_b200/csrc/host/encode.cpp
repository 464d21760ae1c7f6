// Variant encoder and test-suite layout for the sm_100a interpreter.
//
// Everything Machine's constructor and compile() resolve per execution in the
// reference (src/vm.cpp:83-112 parameter binding and setup traps, 166-193
// label -> block, cost by static pointer space, value slots) is resolved here
// once per variant / per suite, so the device loop only decodes integers.
#include "encode.hpp"

#include <string_view>

#include <algorithm>
#include <cstring>
#include <map>
#include <stdexcept>
#include <unordered_map>

namespace evoir::b200 {

namespace {

uint8_t scalar_tag(TypeKind k) {
    switch (k) {
    case TypeKind::I32: return GEVO_TAG_I32;
    case TypeKind::F32: return GEVO_TAG_F32;
    case TypeKind::Bool: return GEVO_TAG_BOOL;
    default: return GEVO_TAG_NEVER;
    }
}

uint32_t scalar_bits(const Scalar& s) {
    uint32_t w = 0;
    if (s.kind == TypeKind::I32)
        std::memcpy(&w, &s.i, 4);
    else if (s.kind == TypeKind::F32)
        std::memcpy(&w, &s.f, 4);
    else
        w = s.b ? 1u : 0u;
    return w;
}

uint32_t buffer_word(const Buffer& b, size_t e) {
    uint32_t w;
    if (b.elem == TypeKind::I32)
        std::memcpy(&w, &b.i[e], 4);
    else
        std::memcpy(&w, &b.f[e], 4);
    return w;
}

bool is_global_ptr(const Param& p) { return p.type.is_ptr() && p.type.space == MemSpace::Global; }

// vtype: result type per dense value id (the last definition, as
// operand_type's scan), empty when ids are not dense
uint8_t cost_class(const Kernel& k, const Instruction& in,
                   const std::vector<std::optional<Type>>& vtype) {
    switch (in.op) {
    case Opcode::Add: case Opcode::Sub: case Opcode::Mul: case Opcode::SDiv:
    case Opcode::FAdd: case Opcode::FSub: case Opcode::FMul: case Opcode::FDiv:
        return GEVO_COST_ARITH;
    case Opcode::ICmp: case Opcode::FCmp: return GEVO_COST_CMP;
    case Opcode::Select: return GEVO_COST_SELECT;
    case Opcode::Phi: return GEVO_COST_PHI;
    case Opcode::Const: return GEVO_COST_CONST;
    case Opcode::Br: return GEVO_COST_BR;
    case Opcode::Tid: case Opcode::NThreads: return GEVO_COST_INTRINSIC;
    case Opcode::GetIndex: return GEVO_COST_GETINDEX;
    case Opcode::Sync: return GEVO_COST_SYNC;
    case Opcode::Ret: return GEVO_COST_RET;
    case Opcode::Load: case Opcode::Store: {
        // Space from the pointer operand's static type; Global when unresolved.
        bool shared = false;
        if (!in.operands.empty()) {
            const Operand& o = in.operands[0];
            const auto t = (o.is_value() && !vtype.empty())
                               ? (o.value >= 0 && static_cast<size_t>(o.value) < vtype.size()
                                      ? vtype[static_cast<size_t>(o.value)]
                                      : std::nullopt)
                               : operand_type(k, o);
            shared = t && t->is_ptr() && t->space == MemSpace::Shared;
        }
        if (in.op == Opcode::Load)
            return shared ? GEVO_COST_LOAD_SHARED : GEVO_COST_LOAD_GLOBAL;
        return shared ? GEVO_COST_STORE_SHARED : GEVO_COST_STORE_GLOBAL;
    }
    }
    return GEVO_COST_ARITH;
}

} // namespace

ExecImage exec_image(const ExecConfig& cfg) {
    ExecImage e;
    e.threads = cfg.thread_count;
    e.shared_words = cfg.shared_words;
    e.budget = cfg.instruction_budget;
    const CostTable& c = cfg.cost_table;
    e.cost = {c.arith,       c.cmp,          c.select_op,   c.phi,          c.constant,
              c.br,          c.intrinsic,    c.getindex,    c.load_shared,  c.store_shared,
              c.load_global, c.store_global, c.sync,        c.ret};
    return e;
}

SuiteImage build_suite(const std::vector<Param>& params, const std::vector<TestCase>& tests) {
    if (params.size() > GEVO_MAX_PARAMS)
        throw std::invalid_argument("kernel has more than 48 parameters");
    SuiteImage s;
    s.params = params;
    s.n_tests = static_cast<int>(tests.size());
    s.n_params = static_cast<int>(params.size());
    const size_t T = tests.size(), P = params.size();
    for (const Param& p : params)
        s.param_names.push_back(p.name);
    s.param_tag.assign(T * P, GEVO_TAG_UNDEF);
    s.param_payload.assign(T * P, 0);
    s.buf_size.assign(T * P, 0);
    s.buf_elem.assign(T * P, GEVO_TAG_NEVER);
    s.setup_code.assign(T, GEVO_OK);
    s.setup_aux.assign(T, -1);
    s.static_err.assign(T, 0);

    // Parameter binding, first failing parameter wins (src/vm.cpp:86-110).
    for (size_t t = 0; t < T; ++t) {
        for (size_t p = 0; p < P; ++p) {
            const Param& prm = params[p];
            const size_t tp = t * P + p;
            auto fail = [&](uint8_t code) {
                if (s.setup_code[t] == GEVO_OK) {
                    s.setup_code[t] = code;
                    s.setup_aux[t] = static_cast<int32_t>(p);
                }
            };
            if (prm.type.is_ptr()) {
                if (prm.type.space == MemSpace::Shared) {
                    s.param_tag[tp] = GEVO_TAG_PTR_SHARED;
                    continue;
                }
                const auto it = tests[t].inputs.find(prm.name);
                if (it == tests[t].inputs.end()) {
                    fail(GEVO_TRAP_MISSING_BUFFER);
                    continue;
                }
                if (prm.elem && *prm.elem != it->second.elem) {
                    fail(GEVO_TRAP_BUFFER_TYPE);
                    continue;
                }
                s.param_tag[tp] = static_cast<uint8_t>(GEVO_TAG_PTR_GLOBAL | p);
                s.buf_size[tp] = static_cast<int32_t>(it->second.size());
                s.buf_elem[tp] = scalar_tag(it->second.elem);
            } else {
                const auto it = tests[t].scalars.find(prm.name);
                if (it == tests[t].scalars.end()) {
                    fail(GEVO_TRAP_MISSING_SCALAR);
                    continue;
                }
                if (it->second.type() != prm.type) {
                    fail(GEVO_TRAP_SCALAR_TYPE);
                    continue;
                }
                s.param_tag[tp] = scalar_tag(it->second.kind);
                s.param_payload[tp] = scalar_bits(it->second);
            }
        }
    }

    // Inputs: one [rows][T] block per global parameter.
    s.pool_off.assign(P, 0);
    s.pool_rows.assign(P, 0);
    for (size_t p = 0; p < P; ++p) {
        if (!is_global_ptr(params[p]))
            continue;
        int32_t rows = 0;
        for (size_t t = 0; t < T; ++t)
            rows = std::max(rows, s.buf_size[t * P + p]);
        s.pool_rows[p] = rows;
        s.pool_off[p] = s.pool.size();
        s.pool.resize(s.pool.size() + static_cast<size_t>(rows) * T, 0u);
        for (size_t t = 0; t < T; ++t) {
            if (s.param_tag[t * P + p] == GEVO_TAG_UNDEF)
                continue;
            const Buffer& b = tests[t].inputs.at(params[p].name);
            for (size_t e = 0; e < b.size(); ++e)
                s.pool[s.pool_off[p] + e * T + t] = buffer_word(b, e);
        }
    }

    // Oracles (compute_error, src/vm.cpp:536-556): outputs are all global
    // parameters by name, the last parameter of a name winning the map slot.
    std::unordered_map<std::string, int> out_param;
    for (size_t p = 0; p < P; ++p)
        if (is_global_ptr(params[p]))
            out_param[params[p].name] = static_cast<int>(p);
    std::map<std::string, std::pair<uint64_t, int32_t>> region; // name -> (off, rows)
    for (size_t t = 0; t < T; ++t)
        for (const auto& [name, ob] : tests[t].oracle) {
            auto& r = region[name];
            r.second = std::max(r.second, static_cast<int32_t>(ob.size()));
        }
    for (auto& [name, r] : region) {
        r.first = s.pool.size();
        s.pool.resize(s.pool.size() + static_cast<size_t>(r.second) * T, 0u);
    }
    s.entry_begin.push_back(0);
    for (size_t t = 0; t < T; ++t) {
        for (const auto& [name, ob] : tests[t].oracle) {
            const auto it = out_param.find(name);
            if (it == out_param.end()) {
                s.static_err[t] = 1;
                continue;
            }
            const size_t tp = t * P + static_cast<size_t>(it->second);
            if (s.param_tag[tp] == GEVO_TAG_UNDEF || s.buf_elem[tp] != scalar_tag(ob.elem) ||
                static_cast<size_t>(s.buf_size[tp]) != ob.size()) {
                s.static_err[t] = 1;
                continue;
            }
            const auto& r = region.at(name);
            for (size_t e = 0; e < ob.size(); ++e)
                s.pool[r.first + e * T + t] = buffer_word(ob, e);
            s.entries.push_back(SuiteImage::OracleEntry{it->second, static_cast<int32_t>(ob.size()),
                                                        r.first, scalar_tag(ob.elem)});
        }
        s.entry_begin.push_back(static_cast<int32_t>(s.entries.size()));
    }
    return s;
}

BatchImage::BatchImage(const SuiteImage& suite) : suite_(suite) {}

void BatchImage::add(const Kernel& k) {
    if (!(k.params == suite_.params))
        throw std::invalid_argument("variant '" + k.name +
                                    "' does not share the suite's parameter list");
    if (k.blocks.size() > 32767)
        throw std::invalid_argument("too many blocks");
    const uint32_t P = static_cast<uint32_t>(suite_.n_params);

    // Value ids are small non-negative integers in practice: flat tables
    // indexed by id then (hash maps only for unusual ids).
    int32_t id_lo = 0, id_hi = -1;
    k.for_each_instruction([&](const BasicBlock&, const Instruction& in) {
        if (in.result) {
            id_lo = std::min(id_lo, *in.result);
            id_hi = std::max(id_hi, *in.result);
        }
        for (const Operand& o : in.operands)
            if (o.is_value()) {
                id_lo = std::min(id_lo, o.value);
                id_hi = std::max(id_hi, o.value);
            }
    });
    const bool dense = id_lo >= 0 && id_hi < (1 << 20);
    const size_t n_ids = dense ? static_cast<size_t>(id_hi + 1) : 0;
    // per-kernel lookups done once: result type per value id, block index per
    // label (Kernel::block_index scans the block list per call)
    // per-thread working tables (capacity kept across variants)
    struct Scratch {
        std::vector<std::optional<Type>> vtype;
        std::vector<int32_t> slot_flat;
        std::vector<uint64_t> prov_flat;
        std::vector<std::pair<uint64_t, uint32_t>> lits;
        std::vector<int> barriers;
    };
    thread_local Scratch scratch;
    std::vector<std::optional<Type>>& vtype = scratch.vtype;
    vtype.assign(n_ids, std::nullopt);
    if (dense)
        k.for_each_instruction([&](const BasicBlock&, const Instruction& in) {
            if (in.result && *in.result >= 0)
                vtype[static_cast<size_t>(*in.result)] = in.result_type();
        });
    auto bix = [&](const std::string& l) -> int { // first block of a label wins
        for (size_t b = 0; b < k.blocks.size(); ++b) {
            const std::string& x = k.blocks[b].label;
            if (x.size() == l.size() && x == l)
                return static_cast<int>(b);
        }
        return -1;
    };

    // Dense value slots in order of first appearance.
    std::unordered_map<int32_t, uint32_t> slot_map;
    std::vector<int32_t>& slot_flat = scratch.slot_flat;
    slot_flat.assign(n_ids, -1);
    std::vector<int32_t> slot_ids;
    auto note = [&](int32_t id) {
        if (dense) {
            int32_t& sl = slot_flat[static_cast<size_t>(id)];
            if (sl < 0) {
                sl = static_cast<int32_t>(slot_ids.size());
                slot_ids.push_back(id);
            }
        } else if (slot_map.emplace(id, static_cast<uint32_t>(slot_ids.size())).second) {
            slot_ids.push_back(id);
        }
    };
    auto slot_at = [&](int32_t id) -> uint32_t {
        if (!dense)
            return slot_map.at(id);
        if (id < 0 || static_cast<size_t>(id) >= n_ids || slot_flat[static_cast<size_t>(id)] < 0)
            throw std::out_of_range("value slot");
        return static_cast<uint32_t>(slot_flat[static_cast<size_t>(id)]);
    };
    k.for_each_instruction([&](const BasicBlock&, const Instruction& in) {
        if (in.result && *in.result >= 0)
            note(*in.result);
        for (const Operand& o : in.operands)
            if (o.is_value())
                note(o.value);
    });
    const uint32_t V = static_cast<uint32_t>(slot_ids.size());
    const uint32_t poison_param = V + P;   // tag GEVO_TAG_POISON_PARAM at init
    const uint32_t poison_missing = V + P + 1;
    const uint32_t lit_begin = V + P + 2;

    gevo_variant var{};
    var.inst_base = static_cast<uint32_t>(insts_.size());
    var.block_base = static_cast<uint32_t>(blocks_.size());
    var.arm_base = static_cast<uint32_t>(arms_.size());
    var.lit_base = static_cast<uint32_t>(lit_payload_.size());
    var.n_values = static_cast<uint16_t>(V);
    var.n_blocks = static_cast<uint16_t>(k.blocks.size());

    // literal pool: a linear table while small, a hash map beyond
    std::vector<std::pair<uint64_t, uint32_t>>& lits = scratch.lits;
    lits.clear();
    std::unordered_map<uint64_t, uint32_t> lit_slot;
    uint32_t n_lits = 0;
    auto literal = [&](const Literal& l) -> uint16_t {
        const uint8_t tag = scalar_tag(l.kind);
        const uint32_t bits = scalar_bits(l);
        const uint64_t key = (static_cast<uint64_t>(tag) << 32) | bits;
        if (n_lits <= 32) {
            for (const auto& [kk, sl] : lits)
                if (kk == key)
                    return static_cast<uint16_t>(lit_begin + sl);
            if (n_lits == 32) // (moving to the map)
                for (const auto& [kk, sl] : lits)
                    lit_slot.emplace(kk, sl);
            else
                lits.emplace_back(key, n_lits);
        }
        if (n_lits >= 32) {
            const auto it = lit_slot.find(key);
            if (it != lit_slot.end())
                return static_cast<uint16_t>(lit_begin + it->second);
            lit_slot.emplace(key, n_lits);
        }
        lit_tag_.push_back(tag);
        lit_payload_.push_back(bits);
        return static_cast<uint16_t>(lit_begin + n_lits++);
    };
    auto ref = [&](const Instruction& in, size_t i) -> uint16_t {
        if (i >= in.operands.size())
            return static_cast<uint16_t>(poison_missing);
        const Operand& o = in.operands[i];
        if (o.kind == Operand::Kind::Value)
            return static_cast<uint16_t>(slot_at(o.value));
        if (o.kind == Operand::Kind::Param)
            return static_cast<uint16_t>(o.param >= 0 && static_cast<uint32_t>(o.param) < P
                                             ? V + static_cast<uint32_t>(o.param)
                                             : poison_param);
        return literal(o.lit);
    };

    // Pointer provenance for privatising writable global buffers: pointers
    // only originate from parameters and flow through getindex and phi.
    std::unordered_map<int32_t, uint64_t> prov_map;
    std::vector<uint64_t>& prov_flat = scratch.prov_flat;
    prov_flat.assign(n_ids, 0);
    auto prov_ref = [&](int32_t id) -> uint64_t& {
        return dense ? prov_flat[static_cast<size_t>(id)] : prov_map[id];
    };
    auto prov_of = [&](const Operand& o) -> uint64_t {
        if (o.kind == Operand::Kind::Param)
            return (o.param >= 0 && static_cast<uint32_t>(o.param) < P &&
                    is_global_ptr(k.params[static_cast<size_t>(o.param)]))
                       ? (1ull << o.param)
                       : 0;
        if (o.kind == Operand::Kind::Value) {
            if (dense)
                return prov_flat[static_cast<size_t>(o.value)];
            const auto it = prov_map.find(o.value);
            return it == prov_map.end() ? 0 : it->second;
        }
        return 0;
    };
    for (bool grew = true; grew;) {
        grew = false;
        k.for_each_instruction([&](const BasicBlock&, const Instruction& in) {
            if (!in.result || (in.op != Opcode::GetIndex && in.op != Opcode::Phi))
                return;
            uint64_t m = 0;
            if (in.op == Opcode::GetIndex) {
                if (!in.operands.empty())
                    m = prov_of(in.operands[0]);
            } else {
                for (const Operand& o : in.operands)
                    m |= prov_of(o);
            }
            uint64_t& cur = prov_ref(*in.result);
            if ((cur | m) != cur) {
                cur |= m;
                grew = true;
            }
        });
    }
    uint64_t writable = 0;
    k.for_each_instruction([&](const BasicBlock&, const Instruction& in) {
        if (in.op == Opcode::Store && !in.operands.empty())
            writable |= prov_of(in.operands[0]);
    });
    var.writable = writable;

    std::vector<int>& barrier_uid = scratch.barriers; // barrier id = first-seen order of its uid
    barrier_uid.clear();
    uint32_t max_phis = 0;
    uint32_t rel = 0;
    for (const BasicBlock& blk : k.blocks) {
        gevo_block gb{};
        gb.start = rel;
        if (blk.instructions.size() > 65535)
            throw std::invalid_argument("block too long");
        gb.len = static_cast<uint16_t>(blk.instructions.size());
        uint16_t nphi = 0;
        while (nphi < gb.len && blk.instructions[nphi].is_phi())
            ++nphi;
        gb.nphi = nphi;
        max_phis = std::max<uint32_t>(max_phis, nphi);
        blocks_.push_back(gb);
        rel += gb.len + 1u; // + fell-off sentinel
    }
    max_insts_ = std::max<uint32_t>(max_insts_, rel);
    // Branch edges: the target block's leading phis resolved for this block as
    // predecessor (first arm whose label is this block, like enter_block).
    auto edge_of = [&](int from_block, int target) -> std::pair<uint32_t, uint32_t> {
        const std::pair<uint32_t, uint32_t> none{GEVO_EDGE_NONE, GEVO_EDGE_NONE};
        if (target < 0 || static_cast<size_t>(target) >= k.blocks.size())
            return none;
        const BasicBlock& tb = k.blocks[static_cast<size_t>(target)];
        uint32_t out[2] = {0, 0};
        size_t nphi = 0;
        while (nphi < tb.instructions.size() && tb.instructions[nphi].is_phi())
            ++nphi;
        if (nphi > 2)
            return none;
        for (size_t j = 0; j < nphi; ++j) {
            const Instruction& phi = tb.instructions[j];
            if (!phi.result || *phi.result < 0)
                return none;
            uint32_t r = GEVO_EDGE_NOINC;
            const size_t n = std::min(phi.operands.size(), phi.labels.size());
            for (size_t a = 0; a < n; ++a)
                if (bix(phi.labels[a]) == from_block) {
                    r = ref(phi, a);
                    break;
                }
            out[j] = r | (static_cast<uint32_t>(slot_at(*phi.result)) << 16);
        }
        return {out[0], out[1]};
    };
    int bidx = 0;
    for (const BasicBlock& blk : k.blocks) {
        const int this_block = bidx++;
        for (const Instruction& in : blk.instructions) {
            gevo_edge ge{};
            if (in.op == Opcode::Br) {
                for (size_t e = 0; e < 2; ++e) {
                    const auto pr = e < in.labels.size()
                                        ? edge_of(this_block, bix(in.labels[e]))
                                        : std::pair<uint32_t, uint32_t>{GEVO_EDGE_NONE, GEVO_EDGE_NONE};
                    ge.phi[e][0] = pr.first;
                    ge.phi[e][1] = pr.second;
                }
            }
            edges_.push_back(ge);
            gevo_inst g{};
            g.op = static_cast<uint8_t>(in.op);
            g.cls = cost_class(k, in, vtype);
            g.res = (in.result && *in.result >= 0) ? static_cast<uint16_t>(slot_at(*in.result))
                                                   : static_cast<uint16_t>(GEVO_NO_RESULT);
            g.t0 = g.t1 = -1;
            switch (in.op) {
            case Opcode::ICmp: case Opcode::FCmp:
                g.aux = static_cast<uint8_t>(in.pred);
                g.otag = in.op == Opcode::ICmp ? GEVO_TAG_I32 : GEVO_TAG_F32;
                g.a = ref(in, 0);
                g.b = ref(in, 1);
                break;
            case Opcode::Select:
                g.aux = scalar_tag(in.type.kind);
                g.a = ref(in, 0);
                g.b = ref(in, 1);
                g.c = ref(in, 2);
                break;
            case Opcode::Load:
                g.aux = scalar_tag(in.type.kind);
                g.a = ref(in, 0);
                g.b = ref(in, 1);
                break;
            case Opcode::Store:
                g.a = ref(in, 0);
                g.b = ref(in, 1);
                g.c = ref(in, 2);
                break;
            case Opcode::GetIndex:
                g.aux = (in.type.kind == TypeKind::Ptr && in.type.space == MemSpace::Shared) ? 1 : 0;
                g.a = ref(in, 0);
                g.b = ref(in, 1);
                break;
            case Opcode::Phi: {
                // Arms beyond the label list can never match a predecessor.
                const size_t n = std::min(in.operands.size(), in.labels.size());
                if (n > 255)
                    throw std::invalid_argument("phi with more than 255 arms");
                g.aux = static_cast<uint8_t>(n);
                if (n <= 2) {
                    if (n > 0) {
                        g.a = ref(in, 0);
                        g.t0 = static_cast<int16_t>(bix(in.labels[0]));
                    }
                    if (n > 1) {
                        g.b = ref(in, 1);
                        g.t1 = static_cast<int16_t>(bix(in.labels[1]));
                    }
                } else {
                    g.c = static_cast<uint16_t>(arms_.size() - var.arm_base);
                    for (size_t a = 0; a < n; ++a)
                        arms_.push_back(gevo_arm{static_cast<int16_t>(bix(in.labels[a])),
                                                 ref(in, a)});
                }
                break;
            }
            case Opcode::Br:
                g.aux = in.labels.size() == 2 ? 2 : 1;
                if (!in.labels.empty())
                    g.t0 = static_cast<int16_t>(bix(in.labels[0]));
                if (in.labels.size() == 2) {
                    g.t1 = static_cast<int16_t>(bix(in.labels[1]));
                    g.a = ref(in, 0);
                }
                break;
            case Opcode::Sync: {
                const auto it = std::find(barrier_uid.begin(), barrier_uid.end(), in.uid);
                g.b = static_cast<uint16_t>(it - barrier_uid.begin());
                if (it == barrier_uid.end())
                    barrier_uid.push_back(in.uid);
                var.flags |= GEVO_VAR_HAS_SYNC;
                break;
            }
            case Opcode::Const:
                g.a = literal(in.const_value);
                break;
            case Opcode::Ret: case Opcode::Tid: case Opcode::NThreads:
                break;
            case Opcode::Add: case Opcode::Sub: case Opcode::Mul: case Opcode::SDiv:
                g.otag = GEVO_TAG_I32;
                g.a = ref(in, 0);
                g.b = ref(in, 1);
                break;
            default: // float arithmetic
                g.otag = GEVO_TAG_F32;
                g.a = ref(in, 0);
                g.b = ref(in, 1);
                break;
            }
            insts_.push_back(g);
        }
        gevo_inst fell{};
        fell.op = GEVO_OP_FELL;
        fell.res = GEVO_NO_RESULT;
        fell.t0 = fell.t1 = -1;
        insts_.push_back(fell);
        edges_.push_back(gevo_edge{});
    }
    var.n_lits = static_cast<uint16_t>(n_lits);
    var.max_phis = static_cast<uint16_t>(max_phis);
    var.n_slots = V + P + 2 + n_lits + max_phis;
    if (var.n_slots > GEVO_MAX_SLOTS)
        throw std::invalid_argument("variant needs more than GEVO_MAX_SLOTS value slots");
    for (uint32_t s = V; s < V + P + 2 + n_lits; ++s)
        slot_ids.push_back(INT32_MIN); // not value ids
    variants_.push_back(var);
    slot_value_.push_back(std::move(slot_ids));
    max_slots_ = std::max(max_slots_, var.n_slots);
    max_values_ = std::max<uint32_t>(max_values_, V);
    max_lits_ = std::max<uint32_t>(max_lits_, var.n_lits);
    max_lane_slots_ = std::max<uint32_t>(max_lane_slots_, V + var.max_phis);
    any_sync_ = any_sync_ || (var.flags & GEVO_VAR_HAS_SYNC);
    dirty_ = true;
}

void BatchImage::append(BatchImage&& o) {
    const uint32_t ib = static_cast<uint32_t>(insts_.size()), bb = static_cast<uint32_t>(blocks_.size());
    const uint32_t ab = static_cast<uint32_t>(arms_.size()), lb = static_cast<uint32_t>(lit_payload_.size());
    for (gevo_variant v : o.variants_) {
        v.inst_base += ib;
        v.block_base += bb;
        v.arm_base += ab;
        v.lit_base += lb;
        variants_.push_back(v);
    }
    blocks_.insert(blocks_.end(), o.blocks_.begin(), o.blocks_.end());
    insts_.insert(insts_.end(), o.insts_.begin(), o.insts_.end());
    edges_.insert(edges_.end(), o.edges_.begin(), o.edges_.end());
    arms_.insert(arms_.end(), o.arms_.begin(), o.arms_.end());
    lit_payload_.insert(lit_payload_.end(), o.lit_payload_.begin(), o.lit_payload_.end());
    lit_tag_.insert(lit_tag_.end(), o.lit_tag_.begin(), o.lit_tag_.end());
    for (auto& sv : o.slot_value_)
        slot_value_.push_back(std::move(sv));
    max_slots_ = std::max(max_slots_, o.max_slots_);
    max_values_ = std::max(max_values_, o.max_values_);
    max_lits_ = std::max(max_lits_, o.max_lits_);
    max_lane_slots_ = std::max(max_lane_slots_, o.max_lane_slots_);
    max_insts_ = std::max(max_insts_, o.max_insts_);
    any_sync_ = any_sync_ || o.any_sync_;
    dirty_ = true;
}

const gevo_batch_header& BatchImage::header() {
    layout();
    return hdr_;
}

void BatchImage::layout() {
    if (!dirty_)
        return;
    auto align = [](uint64_t x) { return (x + 15) & ~uint64_t(15); };
    gevo_batch_header h{};
    h.magic = GEVO_MAGIC;
    h.version = GEVO_VERSION;
    h.n_variants = static_cast<uint32_t>(variants_.size());
    h.n_params = static_cast<uint32_t>(suite_.n_params);
    h.n_insts = static_cast<uint32_t>(insts_.size());
    h.n_blocks = static_cast<uint32_t>(blocks_.size());
    h.n_arms = static_cast<uint32_t>(arms_.size());
    h.n_lits = static_cast<uint32_t>(lit_payload_.size());
    h.max_slots = max_slots_;
    h.max_values = max_values_;
    h.any_sync = any_sync_ ? 1 : 0;
    h.max_lits = max_lits_;
    h.max_lane_slots = max_lane_slots_;
    h.max_insts = max_insts_;
    uint64_t off = align(sizeof(gevo_batch_header));
    h.off_variants = off;
    off = align(off + variants_.size() * sizeof(gevo_variant));
    h.off_blocks = off;
    off = align(off + blocks_.size() * sizeof(gevo_block));
    h.off_insts = off;
    off = align(off + insts_.size() * sizeof(gevo_inst));
    h.off_arms = off;
    off = align(off + arms_.size() * sizeof(gevo_arm));
    h.off_lit_payload = off;
    off = align(off + lit_payload_.size() * 4);
    h.off_lit_tag = off;
    off = align(off + lit_tag_.size());
    h.off_edges = off;
    off = align(off + edges_.size() * sizeof(gevo_edge));
    h.total_bytes = off;
    hdr_ = h;
    dirty_ = false;
    blob_.clear();
}

void BatchImage::write_blob(uint8_t* dst) {
    layout();
    const gevo_batch_header& h = hdr_;
    uint64_t at = 0; // every byte written once: sections, and zeros in the alignment gaps
    auto put = [&](uint64_t off, const void* src, size_t n) {
        std::memset(dst + at, 0, off - at);
        if (n)
            std::memcpy(dst + off, src, n);
        at = off + n;
    };
    put(0, &h, sizeof h);
    put(h.off_variants, variants_.data(), variants_.size() * sizeof(gevo_variant));
    put(h.off_blocks, blocks_.data(), blocks_.size() * sizeof(gevo_block));
    put(h.off_insts, insts_.data(), insts_.size() * sizeof(gevo_inst));
    put(h.off_arms, arms_.data(), arms_.size() * sizeof(gevo_arm));
    put(h.off_lit_payload, lit_payload_.data(), lit_payload_.size() * 4);
    put(h.off_lit_tag, lit_tag_.data(), lit_tag_.size());
    put(h.off_edges, edges_.data(), edges_.size() * sizeof(gevo_edge));
    std::memset(dst + at, 0, h.total_bytes - at);
}

const std::vector<uint8_t>& BatchImage::blob() {
    layout();
    if (blob_.size() != hdr_.total_bytes) {
        blob_.resize(hdr_.total_bytes);
        write_blob(blob_.data());
    }
    return blob_;
}

uint64_t BatchImage::writable_union() const {
    uint64_t m = 0;
    for (const gevo_variant& v : variants_)
        m |= v.writable;
    return m;
}

void BatchImage::reserve(size_t variants, size_t insts) {
    variants_.reserve(variants);
    slot_value_.reserve(variants);
    insts_.reserve(insts);
    edges_.reserve(insts);
}

std::string reason_text(uint8_t code, const std::string& param_name, int32_t value_id) {
    switch (code) {
    case GEVO_TRAP_MISSING_BUFFER: return "missing buffer for param '" + param_name + "'";
    case GEVO_TRAP_BUFFER_TYPE: return "buffer type mismatch for param '" + param_name + "'";
    case GEVO_TRAP_MISSING_SCALAR: return "missing scalar for param '" + param_name + "'";
    case GEVO_TRAP_SCALAR_TYPE: return "scalar type mismatch for param '" + param_name + "'";
    case GEVO_TRAP_DIVERGENCE: return "barrier divergence";
    case GEVO_TRAP_BAD_PARAM: return "bad param reference";
    case GEVO_TRAP_UNDEF_VALUE: return "read of undefined value %" + std::to_string(value_id);
    case GEVO_TRAP_BAD_OPERAND: return "bad operand";
    case GEVO_TRAP_OPERAND_TYPE: return "operand type mismatch";
    case GEVO_TRAP_NOT_POINTER: return "operand is not a pointer";
    case GEVO_TRAP_SHARED_OOB: return "shared access out of bounds";
    case GEVO_TRAP_SHARED_UNINIT: return "read of uninitialized shared memory";
    case GEVO_TRAP_SHARED_TYPE: return "shared load type mismatch";
    case GEVO_TRAP_GLOBAL_OOB: return "global access out of bounds";
    case GEVO_TRAP_GLOBAL_LOAD_TYPE: return "global load type mismatch";
    case GEVO_TRAP_STORE_BOOL: return "store of bool";
    case GEVO_TRAP_GLOBAL_STORE_TYPE: return "global store type mismatch";
    case GEVO_TRAP_DEF_NO_ID: return "definition without value id";
    case GEVO_TRAP_PHI_NO_INCOMING: return "phi has no incoming value for predecessor";
    case GEVO_TRAP_FELL_OFF: return "fell off the end of a block";
    case GEVO_TRAP_UNKNOWN_BLOCK: return "branch to unknown block";
    case GEVO_TRAP_PHI_OUTSIDE: return "phi outside block entry";
    case GEVO_TRAP_DIV_ZERO: return "integer division by zero";
    case GEVO_TRAP_DIV_OVERFLOW: return "integer division overflow";
    case GEVO_TRAP_SELECT_ARM: return "select arm type mismatch";
    case GEVO_TRAP_STORE_NONSCALAR: return "store of non-scalar";
    case GEVO_TRAP_GETINDEX_SPACE: return "getindex address space mismatch";
    case GEVO_TRAP_UNEXPECTED_OP: return "unexpected opcode in straight-line step";
    case GEVO_BUDGET_EXCEEDED: return "instruction budget exceeded";
    case GEVO_TRAP_INTERNAL: return "internal interpreter error";
    default: return "unknown trap " + std::to_string(code);
    }
}

std::string BatchImage::reason(size_t v, uint8_t code, int32_t aux) const {
    std::string pname;
    int32_t vid = 0;
    if (code >= GEVO_TRAP_MISSING_BUFFER && code <= GEVO_TRAP_SCALAR_TYPE && aux >= 0 &&
        aux < suite_.n_params)
        pname = suite_.param_names[static_cast<size_t>(aux)];
    if (code == GEVO_TRAP_UNDEF_VALUE && aux >= 0 &&
        static_cast<size_t>(aux) < slot_value_[v].size())
        vid = slot_value_[v][static_cast<size_t>(aux)];
    return reason_text(code, pname, vid);
}

} // namespace evoir::b200
