// slot_type over a caller-supplied operand-type lookup: ir.cpp answers it
// with operand_type() (a scan of the kernel per value operand), the operator
// index with a per-kernel table built in one pass. Same answers either way.
#pragma once
#include "evoir/ir.hpp"

#include <optional>

namespace evoir {

template <class OperandType>
std::optional<Type> slot_type_with(const Instruction& inst, size_t slot, const OperandType& otype) {
    const size_t n = inst.operands.size();
    switch (inst.op) {
    case Opcode::Add: case Opcode::Sub: case Opcode::Mul: case Opcode::SDiv:
    case Opcode::ICmp:
        return slot < 2 ? std::optional<Type>(Type::i32()) : std::nullopt;
    case Opcode::FAdd: case Opcode::FSub: case Opcode::FMul: case Opcode::FDiv:
    case Opcode::FCmp:
        return slot < 2 ? std::optional<Type>(Type::f32()) : std::nullopt;
    case Opcode::Select:
        if (slot == 0)
            return Type::boolean();
        return slot < 3 ? std::optional<Type>(inst.type) : std::nullopt;
    case Opcode::Load:
        if (slot == 0)
            return n > 0 ? otype(inst.operands[0]) : std::nullopt;
        return slot == 1 ? std::optional<Type>(Type::i32()) : std::nullopt;
    case Opcode::Store:
        if (slot == 0 || slot == 2)
            return slot < n ? otype(inst.operands[slot]) : std::nullopt;
        return slot == 1 ? std::optional<Type>(Type::i32()) : std::nullopt;
    case Opcode::GetIndex:
        if (slot == 0)
            return inst.type;
        return slot == 1 ? std::optional<Type>(Type::i32()) : std::nullopt;
    case Opcode::Phi:
        return slot < n ? std::optional<Type>(inst.type) : std::nullopt;
    case Opcode::Br:
        return (slot == 0 && inst.labels.size() == 2) ? std::optional<Type>(Type::boolean())
                                                      : std::nullopt;
    default:
        return std::nullopt;
    }
}

} // namespace evoir
