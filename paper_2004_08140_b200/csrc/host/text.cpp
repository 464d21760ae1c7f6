// Textual IR: reader and canonical printer.
//
// Plumbing (SURVEY.md §2 marks the reference parser out of scope), but the
// printer must be byte-identical to the reference's print_kernel
// (src/parser.cpp:549-624) because kernels are compared and hashed as text,
// and the reader must accept everything the reference corpus and tests use
// with the same uid assignment (src/parser.cpp:409-532: explicit #uid=
// annotations win, the rest are packed in program order around them).
#include "evoir/ir.hpp"

#include <cctype>
#include <set>
#include <sstream>

namespace evoir {

namespace {

bool ident_char(char c) {
    return std::isalnum(static_cast<unsigned char>(c)) || c == '_' || c == '-' || c == '.';
}

// One logical statement with its source line (for error positions).
struct Stmt {
    std::string text;
    int line;
};

// Splits the source into statements: newlines and ';' separate statements,
// the header's '{' and every '}' stand alone. A trailing '#' comment (which
// may carry #uid=) belongs to the last non-empty piece of its line.
std::vector<Stmt> split_statements(const std::string& src) {
    std::vector<Stmt> out;
    std::istringstream in(src);
    std::string raw;
    int line_no = 0;
    while (std::getline(in, raw)) {
        ++line_no;
        const size_t hash = raw.find('#');
        const std::string code = hash == std::string::npos ? raw : raw.substr(0, hash);
        const std::string comment = hash == std::string::npos ? "" : raw.substr(hash);
        bool header_open = out.empty() && code.find("kernel") != std::string::npos;

        std::vector<std::string> parts(1);
        for (char ch : code) {
            if (ch == ';') {
                parts.emplace_back();
            } else if (ch == '{' && header_open) {
                parts.back() += ch;
                parts.emplace_back();
                header_open = false;
            } else if (ch == '}') {
                parts.emplace_back("}");
                parts.emplace_back();
            } else {
                parts.back() += ch;
            }
        }
        int last = -1;
        for (size_t i = 0; i < parts.size(); ++i)
            if (parts[i].find_first_not_of(" \t") != std::string::npos)
                last = static_cast<int>(i);
        for (size_t i = 0; i < parts.size(); ++i) {
            std::string p = parts[i];
            if (static_cast<int>(i) == last || (last < 0 && i + 1 == parts.size()))
                p += comment;
            if (p.find_first_not_of(" \t") != std::string::npos)
                out.push_back({p, line_no});
        }
    }
    return out;
}

// Removes a '#' comment, returning an explicit uid if it has "uid=<int>".
std::string take_comment(const std::string& s, std::optional<int>& uid) {
    uid.reset();
    const size_t hash = s.find('#');
    if (hash == std::string::npos)
        return s;
    const size_t at = s.find("uid=", hash);
    if (at != std::string::npos) {
        size_t p = at + 4, q = p;
        while (q < s.size() && (std::isdigit(static_cast<unsigned char>(s[q])) || s[q] == '-'))
            ++q;
        if (q > p)
            uid = std::stoi(s.substr(p, q - p));
    }
    return s.substr(0, hash);
}

class Scanner {
public:
    Scanner(const std::string& s, int line) : s_(s), line_(line) {}

    [[noreturn]] void error(const std::string& msg) const {
        throw ParseError(line_, static_cast<int>(pos_) + 1, msg);
    }
    void ws() {
        while (pos_ < s_.size() && (s_[pos_] == ' ' || s_[pos_] == '\t'))
            ++pos_;
    }
    bool done() {
        ws();
        return pos_ >= s_.size();
    }
    char peek() {
        ws();
        return pos_ < s_.size() ? s_[pos_] : '\0';
    }
    bool accept(char c) {
        if (peek() != c || pos_ >= s_.size())
            return false;
        ++pos_;
        return true;
    }
    void require(char c) {
        if (!accept(c))
            error(std::string("expected '") + c + "'");
    }
    bool keyword(const char* w) {
        ws();
        const std::string word(w);
        if (s_.compare(pos_, word.size(), word) != 0)
            return false;
        const size_t end = pos_ + word.size();
        if (end < s_.size() && (std::isalnum(static_cast<unsigned char>(s_[end])) || s_[end] == '_'))
            return false;
        pos_ = end;
        return true;
    }
    std::string ident() {
        ws();
        const size_t start = pos_;
        while (pos_ < s_.size() && ident_char(s_[pos_]))
            ++pos_;
        if (pos_ == start)
            error("expected identifier");
        return s_.substr(start, pos_ - start);
    }
    int integer() {
        ws();
        const size_t start = pos_;
        if (pos_ < s_.size() && (s_[pos_] == '-' || s_[pos_] == '+'))
            ++pos_;
        const size_t digits = pos_;
        while (pos_ < s_.size() && std::isdigit(static_cast<unsigned char>(s_[pos_])))
            ++pos_;
        if (pos_ == digits)
            error("expected integer");
        return std::stoi(s_.substr(start, pos_ - start));
    }
    Literal literal() {
        ws();
        if (keyword("true"))
            return Literal::of_bool(true);
        if (keyword("false"))
            return Literal::of_bool(false);
        size_t p = pos_;
        if (p < s_.size() && (s_[p] == '-' || s_[p] == '+'))
            ++p;
        bool is_float = false, any_digit = false;
        while (p < s_.size()) {
            const char c = s_[p];
            if (std::isdigit(static_cast<unsigned char>(c))) {
                any_digit = true;
                ++p;
            } else if (c == '.' || c == 'e' || c == 'E') {
                is_float = true;
                ++p;
                if (c != '.' && p < s_.size() && (s_[p] == '-' || s_[p] == '+'))
                    ++p;
            } else {
                break;
            }
        }
        if (!any_digit)
            error("expected literal");
        const std::string tok = s_.substr(pos_, p - pos_);
        pos_ = p;
        return is_float ? Literal::of_f32(std::stof(tok)) : Literal::of_i32(std::stoi(tok));
    }
    Type type() {
        if (keyword("i32"))
            return Type::i32();
        if (keyword("f32"))
            return Type::f32();
        if (keyword("bool"))
            return Type::boolean();
        if (keyword("ptr")) {
            require('<');
            MemSpace sp = MemSpace::Global;
            if (keyword("shared"))
                sp = MemSpace::Shared;
            else if (!keyword("global"))
                error("expected 'global' or 'shared'");
            require('>');
            return Type::ptr(sp);
        }
        error("expected type");
    }
    size_t pos() const { return pos_; }
    void seek(size_t p) { pos_ = p; }

private:
    const std::string& s_;
    int line_;
    size_t pos_ = 0;
};

Operand read_operand(Scanner& sc, const Kernel& k) {
    const char c = sc.peek();
    if (c == '%') {
        sc.accept('%');
        return Operand::val(sc.integer());
    }
    if (std::isdigit(static_cast<unsigned char>(c)) || c == '-' || c == '+' || c == '.')
        return Operand::literal(sc.literal());
    const size_t mark = sc.pos();
    const std::string id = sc.ident();
    if (id == "true" || id == "false")
        return Operand::literal(Literal::of_bool(id == "true"));
    const int p = k.param_index(id);
    if (p < 0) {
        sc.seek(mark);
        sc.error("unknown operand '" + id + "'");
    }
    return Operand::param_ref(p);
}

bool lookup_opcode(const std::string& w, Opcode& op) {
    static const std::pair<const char*, Opcode> table[] = {
        {"add", Opcode::Add},   {"sub", Opcode::Sub},   {"mul", Opcode::Mul},
        {"sdiv", Opcode::SDiv}, {"fadd", Opcode::FAdd}, {"fsub", Opcode::FSub},
        {"fmul", Opcode::FMul}, {"fdiv", Opcode::FDiv}};
    for (const auto& [name, code] : table)
        if (w == name) {
            op = code;
            return true;
        }
    return false;
}

// Body of "%n = <...>".
Instruction read_definition(Scanner& sc, const Kernel& k, ValueId result) {
    Instruction in;
    in.result = result;
    const std::string word = sc.ident();
    auto binary = [&] {
        in.operands.push_back(read_operand(sc, k));
        sc.require(',');
        in.operands.push_back(read_operand(sc, k));
    };
    Opcode arith;
    if (lookup_opcode(word, arith)) {
        in.op = arith;
        in.type = sc.type();
        const bool is_float = arith >= Opcode::FAdd;
        if (is_float && in.type != Type::f32())
            sc.error("float arithmetic requires f32");
        if (!is_float && in.type != Type::i32())
            sc.error("integer arithmetic requires i32");
        binary();
        return in;
    }
    if (word.rfind("icmp.", 0) == 0 || word.rfind("fcmp.", 0) == 0) {
        const bool fl = word[0] == 'f';
        in.op = fl ? Opcode::FCmp : Opcode::ICmp;
        const std::string pn = word.substr(5);
        bool found = false;
        for (int p = 0; p < 6; ++p)
            if (pn == pred_name(static_cast<CmpPred>(p))) {
                in.pred = static_cast<CmpPred>(p);
                found = true;
            }
        if (!found)
            sc.error("unknown compare predicate '" + pn + "'");
        in.type = sc.type();
        if (in.type != (fl ? Type::f32() : Type::i32()))
            sc.error("compare type does not match opcode");
        binary();
        return in;
    }
    if (word == "select") {
        in.op = Opcode::Select;
        in.type = sc.type();
        if (!in.type.is_scalar())
            sc.error("select produces a scalar");
        binary();
        sc.require(',');
        in.operands.push_back(read_operand(sc, k));
        return in;
    }
    if (word == "load") {
        in.op = Opcode::Load;
        in.type = sc.type();
        if (!in.type.is_scalar() || in.type == Type::boolean())
            sc.error("load type must be i32 or f32");
        in.operands.push_back(read_operand(sc, k));
        sc.require('[');
        in.operands.push_back(read_operand(sc, k));
        sc.require(']');
        return in;
    }
    if (word == "getindex") {
        in.op = Opcode::GetIndex;
        in.type = sc.type();
        if (!in.type.is_ptr())
            sc.error("getindex produces a pointer");
        binary();
        return in;
    }
    if (word == "phi") {
        in.op = Opcode::Phi;
        in.type = sc.type();
        do {
            sc.require('[');
            in.operands.push_back(read_operand(sc, k));
            sc.require(',');
            in.labels.push_back(sc.ident());
            sc.require(']');
        } while (sc.accept(','));
        return in;
    }
    if (word == "tid" || word == "nthreads") {
        in.op = word == "tid" ? Opcode::Tid : Opcode::NThreads;
        in.type = sc.type();
        if (in.type != Type::i32())
            sc.error("intrinsic type must be i32");
        return in;
    }
    if (word == "const") {
        in.op = Opcode::Const;
        in.type = sc.type();
        in.const_value = sc.literal();
        if (in.const_value.type() != in.type)
            sc.error("const literal does not match declared type");
        return in;
    }
    sc.error("unknown opcode '" + word + "'");
}

Instruction read_statement(Scanner& sc, const Kernel& k) {
    if (sc.peek() == '%') {
        sc.accept('%');
        const ValueId v = sc.integer();
        sc.require('=');
        return read_definition(sc, k, v);
    }
    const std::string word = sc.ident();
    Instruction in;
    if (word == "store") {
        in.op = Opcode::Store;
        in.operands.push_back(read_operand(sc, k));
        sc.require('[');
        in.operands.push_back(read_operand(sc, k));
        sc.require(']');
        sc.require(',');
        in.operands.push_back(read_operand(sc, k));
    } else if (word == "br") {
        in.op = Opcode::Br;
        const char c = sc.peek();
        bool conditional = c == '%' || std::isdigit(static_cast<unsigned char>(c));
        if (!conditional) {
            const size_t mark = sc.pos();
            const std::string id = sc.ident();
            conditional = (id == "true" || id == "false") && sc.peek() == ',';
            sc.seek(mark);
        }
        if (conditional) {
            in.operands.push_back(read_operand(sc, k));
            sc.require(',');
            in.labels.push_back(sc.ident());
            sc.require(',');
            in.labels.push_back(sc.ident());
        } else {
            in.labels.push_back(sc.ident());
        }
    } else if (word == "sync") {
        in.op = Opcode::Sync;
    } else if (word == "ret") {
        in.op = Opcode::Ret;
    } else {
        sc.error("unknown statement '" + word + "'");
    }
    return in;
}

void read_header(Scanner& sc, Kernel& k) {
    if (!sc.keyword("kernel"))
        sc.error("expected 'kernel'");
    k.name = sc.ident();
    sc.require('(');
    if (!sc.accept(')')) {
        do {
            Param p;
            p.name = sc.ident();
            sc.require(':');
            p.type = sc.type();
            if (p.type.is_ptr() && (sc.peek() == 'i' || sc.peek() == 'f')) {
                const Type e = sc.type();
                if (!e.is_scalar() || e == Type::boolean())
                    sc.error("pointer element type must be i32 or f32");
                p.elem = e.kind;
            }
            k.params.push_back(std::move(p));
        } while (sc.accept(','));
        sc.require(')');
    }
    while (!sc.done() && sc.peek() != '{') {
        if (sc.keyword("threads")) {
            sc.require('=');
            k.threads = sc.integer();
        } else if (sc.keyword("shared")) {
            sc.require('=');
            k.shared_words = sc.integer();
        } else {
            sc.error("expected threads=, shared= or '{'");
        }
    }
    sc.require('{');
}

std::string operand_text(const Kernel& k, const Operand& o) {
    if (o.kind == Operand::Kind::Value)
        return "%" + std::to_string(o.value);
    if (o.kind == Operand::Kind::Lit)
        return to_string(o.lit);
    if (o.param >= 0 && static_cast<size_t>(o.param) < k.params.size())
        return k.params[static_cast<size_t>(o.param)].name;
    return "<bad-param>";
}

} // namespace

Kernel parse_kernel(const std::string& text) {
    Kernel k;
    const std::vector<Stmt> stmts = split_statements(text);
    enum { kHeader, kBody, kClosed } state = kHeader;
    BasicBlock* block = nullptr;
    std::vector<std::optional<int>> explicit_uid;
    std::vector<std::pair<size_t, size_t>> where;

    for (const Stmt& st : stmts) {
        std::optional<int> uid;
        const std::string code = take_comment(st.text, uid);
        Scanner sc(code, st.line);
        if (sc.done())
            continue;
        if (state == kHeader) {
            read_header(sc, k);
            state = kBody;
            continue;
        }
        if (state == kClosed)
            sc.error("text after closing '}'");
        if (sc.accept('}')) {
            state = kClosed;
            continue;
        }
        const char c = sc.peek();
        if (c != '%' && !std::isdigit(static_cast<unsigned char>(c))) {
            const size_t mark = sc.pos();
            const std::string id = sc.ident();
            if (sc.accept(':')) {
                if (k.block_index(id) >= 0)
                    sc.error("duplicate block label '" + id + "'");
                k.blocks.push_back(BasicBlock{id, {}});
                block = &k.blocks.back();
                if (sc.done())
                    continue;
            } else {
                sc.seek(mark);
            }
        }
        if (!block)
            sc.error("instruction before first block label");
        Instruction in = read_statement(sc, k);
        if (!sc.done())
            sc.error("unexpected trailing text");
        block->instructions.push_back(std::move(in));
        explicit_uid.push_back(uid);
        where.emplace_back(k.blocks.size() - 1, block->instructions.size() - 1);
    }

    const int last_line = static_cast<int>(stmts.size());
    if (state == kHeader)
        throw ParseError(last_line, 1, "missing kernel header");
    if (state == kBody)
        throw ParseError(last_line, 1, "missing closing '}'");
    if (k.blocks.empty())
        throw ParseError(1, 1, "kernel has no blocks");

    std::set<int> used;
    for (const auto& u : explicit_uid)
        if (u)
            used.insert(*u);
    int next = 0;
    for (size_t n = 0; n < where.size(); ++n) {
        Instruction& in = k.blocks[where[n].first].instructions[where[n].second];
        if (explicit_uid[n]) {
            in.uid = *explicit_uid[n];
            continue;
        }
        while (used.count(next))
            ++next;
        in.uid = next;
        used.insert(next);
    }
    return k;
}

std::string print_kernel(const Kernel& k) {
    std::ostringstream out;
    out << "kernel " << k.name << "(";
    for (size_t p = 0; p < k.params.size(); ++p) {
        const Param& prm = k.params[p];
        out << (p ? ", " : "") << prm.name << ": " << to_string(prm.type);
        if (prm.elem)
            out << " " << to_string(Type{*prm.elem, MemSpace::Global});
    }
    out << ") threads=" << k.threads << " shared=" << k.shared_words << " {\n";
    for (const BasicBlock& b : k.blocks) {
        out << b.label << ":\n";
        for (const Instruction& in : b.instructions) {
            auto opnd = [&](size_t i) { return operand_text(k, in.operands[i]); };
            out << "  ";
            if (in.result)
                out << "%" << *in.result << " = ";
            const std::string ty = to_string(in.type);
            switch (in.op) {
            case Opcode::ICmp: case Opcode::FCmp:
                out << opcode_name(in.op) << "." << pred_name(in.pred) << " " << ty << " " << opnd(0)
                    << ", " << opnd(1);
                break;
            case Opcode::Select:
                out << "select " << ty << " " << opnd(0) << ", " << opnd(1) << ", " << opnd(2);
                break;
            case Opcode::Load:
                out << "load " << ty << " " << opnd(0) << "[" << opnd(1) << "]";
                break;
            case Opcode::Store:
                out << "store " << opnd(0) << "[" << opnd(1) << "], " << opnd(2);
                break;
            case Opcode::GetIndex:
                out << "getindex " << ty << " " << opnd(0) << ", " << opnd(1);
                break;
            case Opcode::Phi:
                out << "phi " << ty << " ";
                for (size_t a = 0; a < in.operands.size(); ++a)
                    out << (a ? ", " : "") << "[" << opnd(a) << ", " << in.labels[a] << "]";
                break;
            case Opcode::Br:
                if (in.labels.size() == 2)
                    out << "br " << opnd(0) << ", " << in.labels[0] << ", " << in.labels[1];
                else
                    out << "br " << (in.labels.empty() ? std::string() : in.labels[0]);
                break;
            case Opcode::Sync: out << "sync"; break;
            case Opcode::Ret: out << "ret"; break;
            case Opcode::Tid: case Opcode::NThreads:
                out << opcode_name(in.op) << " " << ty;
                break;
            case Opcode::Const:
                out << "const " << ty << " " << to_string(in.const_value);
                break;
            default: // two-operand arithmetic
                out << opcode_name(in.op) << " " << ty << " " << opnd(0) << ", " << opnd(1);
                break;
            }
            out << "  #uid=" << in.uid << "\n";
        }
    }
    out << "}\n";
    return out.str();
}

} // namespace evoir
