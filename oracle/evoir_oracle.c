/* Plain-C restatement of the reference fitness path. TEST INFRASTRUCTURE ONLY
 * (see evoir_oracle.h). Function-level citations are to
 * /root/reference/proj/src of arxiv/paper_2004_08140. */
#include "evoir_oracle.h"

#include <ctype.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- IR model */

enum { T_I32 = 0, T_F32 = 1, T_BOOL = 2, T_PTR = 3 };
enum { SP_GLOBAL = 0, SP_SHARED = 1 };
enum {
    OP_ADD, OP_SUB, OP_MUL, OP_SDIV, OP_FADD, OP_FSUB, OP_FMUL, OP_FDIV, OP_ICMP, OP_FCMP,
    OP_SELECT, OP_LOAD, OP_STORE, OP_GETINDEX, OP_PHI, OP_BR, OP_SYNC, OP_RET, OP_TID,
    OP_NTHREADS, OP_CONST
};
static const char* const OPN[] = {"add", "sub", "mul", "sdiv", "fadd", "fsub", "fmul",
                                  "fdiv", "icmp", "fcmp", "select", "load", "store", "getindex",
                                  "phi", "br", "sync", "ret", "tid", "nthreads", "const"};
enum { K_VALUE = 0, K_LIT = 1, K_PARAM = 2 };

typedef struct {
    int kind;
    int32_t value;
    int lkind;      /* literal type kind */
    uint32_t lbits; /* literal payload */
    int param;
} Opnd;

typedef struct {
    int uid, op, pred;
    int has_result;
    int32_t result;
    int tkind, tspace;
    int nops;
    Opnd* ops;
    int nlabels;
    char** labels;
    int* targets; /* compile(): labels -> block index (src/vm.cpp:183-186) */
    Opnd cval;
    int64_t cost;
} Inst;

typedef struct {
    char* label;
    int n;
    Inst* insts;
} Block;

typedef struct {
    char* name;
    int tkind, tspace;
    int has_elem, elem;
} Param;

struct eo_kernel {
    int nparams;
    Param* params;
    int nblocks;
    Block* blocks;
    int threads, shared_words;
};

/* ---------------------------------------------------------------- parser */

static char* dupn(const char* s, size_t n) {
    char* p = (char*)malloc(n + 1);
    memcpy(p, s, n);
    p[n] = 0;
    return p;
}

static int idchar(int c) { return isalnum(c) || c == '_' || c == '-' || c == '.'; }

typedef struct {
    const char* s;
    size_t p;
    int bad;
} Cur;

static void ws(Cur* c) {
    while (c->s[c->p] == ' ' || c->s[c->p] == '\t')
        c->p++;
}
static int eat(Cur* c, char ch) {
    ws(c);
    if (c->s[c->p] == ch) {
        c->p++;
        return 1;
    }
    return 0;
}
static void need(Cur* c, char ch) {
    if (!eat(c, ch))
        c->bad = 1;
}
static char* ident(Cur* c) {
    ws(c);
    size_t b = c->p;
    while (c->s[c->p] && idchar((unsigned char)c->s[c->p]))
        c->p++;
    if (c->p == b)
        c->bad = 1;
    return dupn(c->s + b, c->p - b);
}
static int word(Cur* c, const char* w) {
    ws(c);
    size_t n = strlen(w);
    if (strncmp(c->s + c->p, w, n) != 0)
        return 0;
    int nx = (unsigned char)c->s[c->p + n];
    if (isalnum(nx) || nx == '_')
        return 0;
    c->p += n;
    return 1;
}
static void type(Cur* c, int* kind, int* space) {
    *space = SP_GLOBAL;
    if (word(c, "i32"))
        *kind = T_I32;
    else if (word(c, "f32"))
        *kind = T_F32;
    else if (word(c, "bool"))
        *kind = T_BOOL;
    else if (word(c, "ptr")) {
        *kind = T_PTR;
        need(c, '<');
        if (word(c, "shared"))
            *space = SP_SHARED;
        else if (!word(c, "global"))
            c->bad = 1;
        need(c, '>');
    } else
        c->bad = 1;
}
static Opnd literal(Cur* c) {
    Opnd o;
    memset(&o, 0, sizeof o);
    o.kind = K_LIT;
    ws(c);
    if (word(c, "true")) {
        o.lkind = T_BOOL;
        o.lbits = 1;
        return o;
    }
    if (word(c, "false")) {
        o.lkind = T_BOOL;
        return o;
    }
    size_t b = c->p, p = c->p;
    int fl = 0;
    if (c->s[p] == '-' || c->s[p] == '+')
        p++;
    while (c->s[p]) {
        char ch = c->s[p];
        if (isdigit((unsigned char)ch))
            p++;
        else if (ch == '.' || ch == 'e' || ch == 'E') {
            fl = 1;
            p++;
            if (ch != '.' && (c->s[p] == '-' || c->s[p] == '+'))
                p++;
        } else
            break;
    }
    char* tok = dupn(c->s + b, p - b);
    c->p = p;
    if (fl) {
        float f = strtof(tok, NULL);
        o.lkind = T_F32;
        memcpy(&o.lbits, &f, 4);
    } else {
        int32_t i = (int32_t)strtol(tok, NULL, 10);
        o.lkind = T_I32;
        memcpy(&o.lbits, &i, 4);
    }
    free(tok);
    return o;
}
static Opnd operand(Cur* c, const eo_kernel* k) {
    Opnd o;
    memset(&o, 0, sizeof o);
    ws(c);
    char ch = c->s[c->p];
    if (ch == '%') {
        c->p++;
        o.kind = K_VALUE;
        o.value = (int32_t)strtol(c->s + c->p, NULL, 10);
        if (c->s[c->p] == '-' || c->s[c->p] == '+')
            c->p++;
        while (isdigit((unsigned char)c->s[c->p]))
            c->p++;
        return o;
    }
    if (isdigit((unsigned char)ch) || ch == '-' || ch == '+' || ch == '.')
        return literal(c);
    size_t save = c->p;
    char* id = ident(c);
    if (!strcmp(id, "true") || !strcmp(id, "false")) {
        free(id);
        c->p = save;
        return literal(c);
    }
    o.kind = K_PARAM;
    o.param = -1;
    for (int i = 0; i < k->nparams; ++i)
        if (!strcmp(k->params[i].name, id))
            o.param = i;
    if (o.param < 0) {
        if (!strcmp(id, "<bad-param>"))
            o.param = k->nparams; /* out of range on purpose */
        else
            c->bad = 1;
    }
    free(id);
    return o;
}
static void push_op(Inst* in, Opnd o) {
    in->ops = (Opnd*)realloc(in->ops, sizeof(Opnd) * (size_t)(in->nops + 1));
    in->ops[in->nops++] = o;
}
static void push_label(Inst* in, char* l) {
    in->labels = (char**)realloc(in->labels, sizeof(char*) * (size_t)(in->nlabels + 1));
    in->labels[in->nlabels++] = l;
}
static int opcode_of(const char* w, int* pred) {
    static const char* const P[] = {"eq", "ne", "lt", "le", "gt", "ge"};
    for (int i = 0; i <= OP_CONST; ++i)
        if (!strcmp(w, OPN[i]))
            return i;
    if ((!strncmp(w, "icmp.", 5) || !strncmp(w, "fcmp.", 5))) {
        for (int p = 0; p < 6; ++p)
            if (!strcmp(w + 5, P[p]))
                *pred = p;
        return w[0] == 'i' ? OP_ICMP : OP_FCMP;
    }
    return -1;
}

static void parse_inst(Cur* c, const eo_kernel* k, Inst* in) {
    memset(in, 0, sizeof *in);
    ws(c);
    if (c->s[c->p] == '%') {
        c->p++;
        in->has_result = 1;
        in->result = (int32_t)strtol(c->s + c->p, NULL, 10);
        if (c->s[c->p] == '-')
            c->p++;
        while (isdigit((unsigned char)c->s[c->p]))
            c->p++;
        need(c, '=');
    }
    char* w = ident(c);
    in->op = opcode_of(w, &in->pred);
    free(w);
    switch (in->op) {
    case OP_ADD: case OP_SUB: case OP_MUL: case OP_SDIV: case OP_FADD: case OP_FSUB:
    case OP_FMUL: case OP_FDIV: case OP_ICMP: case OP_FCMP:
        type(c, &in->tkind, &in->tspace);
        push_op(in, operand(c, k));
        need(c, ',');
        push_op(in, operand(c, k));
        break;
    case OP_SELECT:
        type(c, &in->tkind, &in->tspace);
        push_op(in, operand(c, k));
        need(c, ',');
        push_op(in, operand(c, k));
        need(c, ',');
        push_op(in, operand(c, k));
        break;
    case OP_LOAD:
        type(c, &in->tkind, &in->tspace);
        push_op(in, operand(c, k));
        need(c, '[');
        push_op(in, operand(c, k));
        need(c, ']');
        break;
    case OP_STORE:
        push_op(in, operand(c, k));
        need(c, '[');
        push_op(in, operand(c, k));
        need(c, ']');
        need(c, ',');
        push_op(in, operand(c, k));
        break;
    case OP_GETINDEX:
        type(c, &in->tkind, &in->tspace);
        push_op(in, operand(c, k));
        need(c, ',');
        push_op(in, operand(c, k));
        break;
    case OP_PHI:
        type(c, &in->tkind, &in->tspace);
        do {
            need(c, '[');
            push_op(in, operand(c, k));
            need(c, ',');
            push_label(in, ident(c));
            need(c, ']');
        } while (eat(c, ','));
        break;
    case OP_BR: {
        ws(c);
        int cond = c->s[c->p] == '%' || isdigit((unsigned char)c->s[c->p]);
        if (!cond) {
            size_t save = c->p;
            char* id = ident(c);
            ws(c);
            cond = c->s[c->p] == ',';
            c->p = save;
            free(id);
        }
        if (cond) {
            push_op(in, operand(c, k));
            need(c, ',');
            push_label(in, ident(c));
            need(c, ',');
            push_label(in, ident(c));
        } else {
            push_label(in, ident(c));
        }
        break;
    }
    case OP_SYNC: case OP_RET:
        break;
    case OP_TID: case OP_NTHREADS:
        type(c, &in->tkind, &in->tspace);
        break;
    case OP_CONST:
        type(c, &in->tkind, &in->tspace);
        in->cval = literal(c);
        break;
    default:
        c->bad = 1;
    }
}

eo_kernel* eo_parse(const char* text, char* err, size_t errcap) {
    eo_kernel* k = (eo_kernel*)calloc(1, sizeof(eo_kernel));
    const char* line = text;
    int state = 0, lineno = 0;
    while (*line) {
        const char* nl = strchr(line, '\n');
        size_t len = nl ? (size_t)(nl - line) : strlen(line);
        char* buf = dupn(line, len);
        ++lineno;
        int uid = -1;
        char* hash = strchr(buf, '#');
        if (hash) {
            char* u = strstr(hash, "uid=");
            if (u)
                uid = (int)strtol(u + 4, NULL, 10);
            *hash = 0;
        }
        Cur c = {buf, 0, 0};
        ws(&c);
        if (!buf[c.p]) {
            free(buf);
            line += len + (nl ? 1 : 0);
            continue;
        }
        if (state == 0) {
            if (!word(&c, "kernel"))
                c.bad = 1;
            free(ident(&c));
            need(&c, '(');
            if (!eat(&c, ')')) {
                do {
                    Param p;
                    memset(&p, 0, sizeof p);
                    p.name = ident(&c);
                    need(&c, ':');
                    type(&c, &p.tkind, &p.tspace);
                    ws(&c);
                    if (p.tkind == T_PTR && (buf[c.p] == 'i' || buf[c.p] == 'f')) {
                        int sp;
                        type(&c, &p.elem, &sp);
                        p.has_elem = 1;
                    }
                    k->params = (Param*)realloc(k->params, sizeof(Param) * (size_t)(k->nparams + 1));
                    k->params[k->nparams++] = p;
                } while (eat(&c, ','));
                need(&c, ')');
            }
            if (word(&c, "threads")) {
                need(&c, '=');
                k->threads = (int)strtol(buf + c.p, NULL, 10);
                while (buf[c.p] == '-' || isdigit((unsigned char)buf[c.p]))
                    c.p++;
            }
            if (word(&c, "shared")) {
                need(&c, '=');
                k->shared_words = (int)strtol(buf + c.p, NULL, 10);
                while (buf[c.p] == '-' || isdigit((unsigned char)buf[c.p]))
                    c.p++;
            }
            need(&c, '{');
            state = 1;
        } else if (buf[c.p] == '}') {
            state = 2;
        } else {
            /* label line? */
            size_t save = c.p;
            char* id = ident(&c);
            if (!c.bad && eat(&c, ':')) {
                k->blocks = (Block*)realloc(k->blocks, sizeof(Block) * (size_t)(k->nblocks + 1));
                k->blocks[k->nblocks].label = id;
                k->blocks[k->nblocks].n = 0;
                k->blocks[k->nblocks].insts = NULL;
                k->nblocks++;
            } else {
                free(id);
                c.bad = 0;
                c.p = save;
                if (k->nblocks == 0)
                    c.bad = 1;
                else {
                    Block* b = &k->blocks[k->nblocks - 1];
                    b->insts = (Inst*)realloc(b->insts, sizeof(Inst) * (size_t)(b->n + 1));
                    parse_inst(&c, k, &b->insts[b->n]);
                    b->insts[b->n].uid = uid;
                    b->n++;
                }
            }
        }
        if (c.bad) {
            if (err)
                snprintf(err, errcap, "oracle parse error at line %d", lineno);
            free(buf);
            eo_free(k);
            return NULL;
        }
        free(buf);
        line += len + (nl ? 1 : 0);
    }
    if (state != 2) {
        if (err)
            snprintf(err, errcap, "oracle parse error: unterminated kernel");
        eo_free(k);
        return NULL;
    }
    return k;
}

void eo_free(eo_kernel* k) {
    if (!k)
        return;
    for (int b = 0; b < k->nblocks; ++b) {
        for (int i = 0; i < k->blocks[b].n; ++i) {
            Inst* in = &k->blocks[b].insts[i];
            free(in->ops);
            for (int l = 0; l < in->nlabels; ++l)
                free(in->labels[l]);
            free(in->labels);
            free(in->targets);
        }
        free(k->blocks[b].insts);
        free(k->blocks[b].label);
    }
    for (int p = 0; p < k->nparams; ++p)
        free(k->params[p].name);
    free(k->params);
    free(k->blocks);
    free(k);
}

int32_t eo_param_count(const eo_kernel* k) { return k->nparams; }

/* ---------------------------------------------------------------- machine */

enum { V_UNDEF = 0, V_SCALAR = 1, V_PTR = 2 };
typedef struct {
    int kind;
    int skind;
    uint32_t bits;
    int space, buffer;
    int32_t offset;
} Val;

typedef struct {
    int block, ip, prev;
    int64_t executed;
    Val* values;
    int stop; /* 0 running, 1 sync, 2 ret */
    int stop_uid;
} Thr;

typedef struct {
    const eo_kernel* k;
    const eo_config* cfg;
    int nglob;
    int* gparam;          /* globals index -> param */
    int* gelem;
    int* gsize;
    uint32_t** gdata;
    int* param_buffer;    /* param -> globals index, -1 shared, -2 scalar */
    Val* scalar_args;
    int* sh_init;
    int* sh_kind;
    uint32_t* sh_bits;
    int nslots;
    int64_t cost;
    int64_t ir;
    char* reason;
    int status; /* 0 running / completed, 1 trap, 2 budget */
} M;

static int trap(M* m, const char* r) {
    if (m->status == 0) {
        m->status = 1;
        snprintf(m->reason, 160, "%s", r);
    }
    return 0;
}

/* operand_type (src/ir.cpp:139-157): the LAST definition wins. */
static int opnd_type(const eo_kernel* k, const Opnd* o, int* kind, int* space) {
    if (o->kind == K_LIT) {
        *kind = o->lkind;
        *space = SP_GLOBAL;
        return 1;
    }
    if (o->kind == K_PARAM) {
        if (o->param < 0 || o->param >= k->nparams)
            return 0;
        *kind = k->params[o->param].tkind;
        *space = k->params[o->param].tspace;
        return 1;
    }
    int found = 0;
    for (int b = 0; b < k->nblocks; ++b)
        for (int i = 0; i < k->blocks[b].n; ++i) {
            const Inst* in = &k->blocks[b].insts[i];
            if (in->has_result && in->result == o->value) {
                found = 1;
                if (in->op == OP_ICMP || in->op == OP_FCMP) {
                    *kind = T_BOOL;
                    *space = SP_GLOBAL;
                } else {
                    *kind = in->tkind;
                    *space = in->tspace;
                }
            }
        }
    return found;
}

static int block_index(const eo_kernel* k, const char* l) {
    for (int b = 0; b < k->nblocks; ++b)
        if (!strcmp(k->blocks[b].label, l))
            return b;
    return -1;
}

/* Machine::compile (src/vm.cpp:166-193). */
static void compile(M* m) {
    const eo_kernel* k = m->k;
    const int64_t* C = m->cfg->cost;
    int32_t maxv = -1;
    for (int b = 0; b < k->nblocks; ++b)
        for (int i = 0; i < k->blocks[b].n; ++i) {
            Inst* in = &k->blocks[b].insts[i];
            if (in->has_result && in->result > maxv)
                maxv = in->result;
        }
    m->nslots = maxv + 1;
    for (int b = 0; b < k->nblocks; ++b)
        for (int i = 0; i < k->blocks[b].n; ++i) {
            Inst* in = &k->blocks[b].insts[i];
            int sp = SP_GLOBAL, kk, ss;
            if ((in->op == OP_LOAD || in->op == OP_STORE) && in->nops > 0 &&
                opnd_type(k, &in->ops[0], &kk, &ss) && kk == T_PTR)
                sp = ss;
            switch (in->op) {
            case OP_ADD: case OP_SUB: case OP_MUL: case OP_SDIV: case OP_FADD: case OP_FSUB:
            case OP_FMUL: case OP_FDIV: in->cost = C[0]; break;
            case OP_ICMP: case OP_FCMP: in->cost = C[1]; break;
            case OP_SELECT: in->cost = C[2]; break;
            case OP_PHI: in->cost = C[3]; break;
            case OP_CONST: in->cost = C[4]; break;
            case OP_BR: in->cost = C[5]; break;
            case OP_TID: case OP_NTHREADS: in->cost = C[6]; break;
            case OP_GETINDEX: in->cost = C[7]; break;
            case OP_LOAD: in->cost = sp == SP_SHARED ? C[8] : C[10]; break;
            case OP_STORE: in->cost = sp == SP_SHARED ? C[9] : C[11]; break;
            case OP_SYNC: in->cost = C[12]; break;
            case OP_RET: in->cost = C[13]; break;
            default: in->cost = 1;
            }
            free(in->targets);
            in->targets = (int*)malloc(sizeof(int) * (size_t)(in->nlabels + 1));
            for (int l = 0; l < in->nlabels; ++l)
                in->targets[l] = block_index(k, in->labels[l]);
            for (int o = 0; o < in->nops; ++o)
                if (in->ops[o].kind == K_VALUE && in->ops[o].value >= 0 &&
                    in->ops[o].value >= m->nslots)
                    m->nslots = in->ops[o].value + 1;
        }
}

/* fetch (src/vm.cpp:195-222) */
static int fetch(M* m, Thr* th, const Opnd* o, Val* v) {
    memset(v, 0, sizeof *v);
    if (o->kind == K_LIT) {
        v->kind = V_SCALAR;
        v->skind = o->lkind;
        v->bits = o->lbits;
        return 1;
    }
    if (o->kind == K_PARAM) {
        if (o->param < 0 || o->param >= m->k->nparams)
            return trap(m, "bad param reference");
        const Param* p = &m->k->params[o->param];
        if (p->tkind == T_PTR) {
            v->kind = V_PTR;
            v->space = p->tspace;
            v->buffer = m->param_buffer[o->param];
            v->offset = 0;
            return 1;
        }
        *v = m->scalar_args[o->param];
        return 1;
    }
    char r[64];
    snprintf(r, sizeof r, "read of undefined value %%%d", o->value);
    if (o->value < 0 || o->value >= m->nslots)
        return trap(m, r);
    *v = th->values[o->value];
    if (v->kind == V_UNDEF)
        return trap(m, r);
    return 1;
}
static int fetch_scalar(M* m, Thr* th, const Opnd* o, int want, uint32_t* bits) {
    Val v;
    if (!fetch(m, th, o, &v))
        return 0;
    if (v.kind != V_SCALAR || v.skind != want)
        return trap(m, "operand type mismatch");
    *bits = v.bits;
    return 1;
}
static int fetch_ptr(M* m, Thr* th, const Opnd* o, Val* v) {
    if (!fetch(m, th, o, v))
        return 0;
    if (v->kind != V_PTR)
        return trap(m, "operand is not a pointer");
    return 1;
}
static int set(M* m, Thr* th, const Inst* in, Val v) {
    if (!in->has_result || in->result < 0)
        return trap(m, "definition without value id");
    th->values[in->result] = v;
    return 1;
}
static int bump(M* m, Thr* th) {
    m->ir++;
    if (++th->executed > m->cfg->budget) {
        if (m->status == 0) {
            m->status = 2;
            snprintf(m->reason, 160, "instruction budget exceeded");
        }
        return 0;
    }
    return 1;
}
static Val scalar(int kind, uint32_t bits) {
    Val v;
    memset(&v, 0, sizeof v);
    v.kind = V_SCALAR;
    v.skind = kind;
    v.bits = bits;
    return v;
}

/* load_from / store_to (src/vm.cpp:238-283) */
static int load_from(M* m, Val p, int32_t idx, int want, Val* out) {
    int64_t eff = (int64_t)p.offset + idx;
    if (p.space == SP_SHARED) {
        if (eff < 0 || eff >= m->cfg->shared_words)
            return trap(m, "shared access out of bounds");
        if (!m->sh_init[eff])
            return trap(m, "read of uninitialized shared memory");
        if (m->sh_kind[eff] != want)
            return trap(m, "shared load type mismatch");
        *out = scalar(want, m->sh_bits[eff]);
        return 1;
    }
    int g = p.buffer;
    if (eff < 0 || eff >= m->gsize[g])
        return trap(m, "global access out of bounds");
    if (m->gelem[g] != want)
        return trap(m, "global load type mismatch");
    *out = scalar(want, m->gdata[g][eff]);
    return 1;
}
static int store_to(M* m, Val p, int32_t idx, Val v) {
    if (v.skind == T_BOOL)
        return trap(m, "store of bool");
    int64_t eff = (int64_t)p.offset + idx;
    if (p.space == SP_SHARED) {
        if (eff < 0 || eff >= m->cfg->shared_words)
            return trap(m, "shared access out of bounds");
        m->sh_init[eff] = 1;
        m->sh_kind[eff] = v.skind;
        m->sh_bits[eff] = v.bits;
        return 1;
    }
    int g = p.buffer;
    if (eff < 0 || eff >= m->gsize[g])
        return trap(m, "global access out of bounds");
    if (m->gelem[g] != v.skind)
        return trap(m, "global store type mismatch");
    m->gdata[g][eff] = v.bits;
    return 1;
}

static int cmp_i(int32_t a, int32_t b, int p) {
    switch (p) {
    case 0: return a == b;
    case 1: return a != b;
    case 2: return a < b;
    case 3: return a <= b;
    case 4: return a > b;
    default: return a >= b;
    }
}
static int cmp_f(float a, float b, int p) {
    switch (p) {
    case 0: return a == b;
    case 1: return a != b;
    case 2: return a < b;
    case 3: return a <= b;
    case 4: return a > b;
    default: return a >= b;
    }
}
static float asf(uint32_t w) {
    float f;
    memcpy(&f, &w, 4);
    return f;
}
static uint32_t asw(float f) {
    uint32_t w;
    memcpy(&w, &f, 4);
    return w;
}

/* step (src/vm.cpp:389-482) */
static int step(M* m, Thr* th, const Inst* in, int tid) {
    uint32_t a, b;
    switch (in->op) {
    case OP_ADD: case OP_SUB: case OP_MUL: case OP_SDIV: {
        if (!fetch_scalar(m, th, &in->ops[0], T_I32, &a) ||
            !fetch_scalar(m, th, &in->ops[1], T_I32, &b))
            return 0;
        uint32_t r = 0;
        if (in->op == OP_ADD)
            r = a + b;
        else if (in->op == OP_SUB)
            r = a - b;
        else if (in->op == OP_MUL)
            r = a * b;
        else {
            int32_t x = (int32_t)a, y = (int32_t)b;
            if (y == 0)
                return trap(m, "integer division by zero");
            if (x == INT32_MIN && y == -1)
                return trap(m, "integer division overflow");
            r = (uint32_t)(x / y);
        }
        return set(m, th, in, scalar(T_I32, r));
    }
    case OP_FADD: case OP_FSUB: case OP_FMUL: case OP_FDIV: {
        if (!fetch_scalar(m, th, &in->ops[0], T_F32, &a) ||
            !fetch_scalar(m, th, &in->ops[1], T_F32, &b))
            return 0;
        volatile float x = asf(a), y = asf(b), r;
        if (in->op == OP_FADD)
            r = x + y;
        else if (in->op == OP_FSUB)
            r = x - y;
        else if (in->op == OP_FMUL)
            r = x * y;
        else
            r = x / y;
        return set(m, th, in, scalar(T_F32, asw(r)));
    }
    case OP_ICMP:
        if (!fetch_scalar(m, th, &in->ops[0], T_I32, &a) ||
            !fetch_scalar(m, th, &in->ops[1], T_I32, &b))
            return 0;
        return set(m, th, in, scalar(T_BOOL, (uint32_t)cmp_i((int32_t)a, (int32_t)b, in->pred)));
    case OP_FCMP:
        if (!fetch_scalar(m, th, &in->ops[0], T_F32, &a) ||
            !fetch_scalar(m, th, &in->ops[1], T_F32, &b))
            return 0;
        return set(m, th, in, scalar(T_BOOL, (uint32_t)cmp_f(asf(a), asf(b), in->pred)));
    case OP_SELECT: {
        if (!fetch_scalar(m, th, &in->ops[0], T_BOOL, &a))
            return 0;
        Val v;
        if (!fetch(m, th, &in->ops[a ? 1 : 2], &v))
            return 0;
        if (v.kind != V_SCALAR || v.skind != in->tkind)
            return trap(m, "select arm type mismatch");
        return set(m, th, in, v);
    }
    case OP_LOAD: {
        Val p, r;
        if (!fetch_ptr(m, th, &in->ops[0], &p) || !fetch_scalar(m, th, &in->ops[1], T_I32, &b))
            return 0;
        if (!load_from(m, p, (int32_t)b, in->tkind, &r))
            return 0;
        return set(m, th, in, r);
    }
    case OP_STORE: {
        Val p, v;
        if (!fetch_ptr(m, th, &in->ops[0], &p) || !fetch_scalar(m, th, &in->ops[1], T_I32, &b) ||
            !fetch(m, th, &in->ops[2], &v))
            return 0;
        if (v.kind != V_SCALAR)
            return trap(m, "store of non-scalar");
        return store_to(m, p, (int32_t)b, v);
    }
    case OP_GETINDEX: {
        Val p;
        if (!fetch_ptr(m, th, &in->ops[0], &p))
            return 0;
        int want_space = in->tkind == T_PTR ? in->tspace : SP_GLOBAL;
        if (p.space != want_space)
            return trap(m, "getindex address space mismatch");
        if (!fetch_scalar(m, th, &in->ops[1], T_I32, &b))
            return 0;
        p.offset = (int32_t)((uint32_t)p.offset + b);
        return set(m, th, in, p);
    }
    case OP_TID:
        return set(m, th, in, scalar(T_I32, (uint32_t)tid));
    case OP_NTHREADS:
        return set(m, th, in, scalar(T_I32, (uint32_t)m->cfg->threads));
    case OP_CONST:
        return set(m, th, in, scalar(in->cval.lkind, in->cval.lbits));
    default:
        return trap(m, "unexpected opcode in straight-line step");
    }
}

/* enter_block (src/vm.cpp:293-333) */
static int enter_block(M* m, Thr* th, int target) {
    th->prev = th->block;
    th->block = target;
    th->ip = 0;
    const Block* b = &m->k->blocks[target];
    int nst = 0;
    Val* staged = (Val*)malloc(sizeof(Val) * (size_t)(b->n + 1));
    int32_t* vid = (int32_t*)malloc(sizeof(int32_t) * (size_t)(b->n + 1));
    int* hasres = (int*)malloc(sizeof(int) * (size_t)(b->n + 1));
    int ok = 1;
    for (int i = 0; i < b->n && ok; ++i) {
        const Inst* in = &b->insts[i];
        if (in->op != OP_PHI)
            break;
        m->cost += in->cost;
        if (!bump(m, th)) {
            ok = 0;
            break;
        }
        int matched = 0;
        for (int a = 0; a < in->nlabels; ++a)
            if (in->targets[a] == th->prev) {
                if (a >= in->nops || !fetch(m, th, &in->ops[a], &staged[nst])) {
                    ok = 0;
                    break;
                }
                vid[nst] = in->result;
                hasres[nst] = in->has_result;
                nst++;
                matched = 1;
                break;
            }
        if (!ok)
            break;
        if (!matched) {
            ok = trap(m, "phi has no incoming value for predecessor");
            break;
        }
        th->ip++;
    }
    for (int i = 0; ok && i < nst; ++i) {
        if (!hasres[i] || vid[i] < 0)
            ok = trap(m, "definition without value id");
        else
            th->values[vid[i]] = staged[i];
    }
    free(staged);
    free(vid);
    free(hasres);
    return ok;
}

/* run_to_barrier (src/vm.cpp:340-387) */
static int run_to_barrier(M* m, Thr* th, int tid) {
    if (th->stop == 2)
        return 1;
    for (;;) {
        const Block* b = &m->k->blocks[th->block];
        if (th->ip >= b->n)
            return trap(m, "fell off the end of a block");
        const Inst* in = &b->insts[th->ip];
        if (in->op == OP_SYNC || in->op == OP_RET) {
            m->cost += in->cost;
            if (!bump(m, th))
                return 0;
            th->stop = in->op == OP_SYNC ? 1 : 2;
            th->stop_uid = in->uid;
            return 1;
        }
        if (in->op == OP_BR) {
            m->cost += in->cost;
            if (!bump(m, th))
                return 0;
            int target;
            if (in->nlabels == 2) {
                uint32_t c;
                if (!fetch_scalar(m, th, &in->ops[0], T_BOOL, &c))
                    return 0;
                target = c ? in->targets[0] : in->targets[1];
            } else {
                target = in->nlabels ? in->targets[0] : -1;
            }
            if (target < 0)
                return trap(m, "branch to unknown block");
            if (!enter_block(m, th, target))
                return 0;
            continue;
        }
        if (in->op == OP_PHI)
            return trap(m, "phi outside block entry");
        m->cost += in->cost;
        if (!bump(m, th))
            return 0;
        if (!step(m, th, in, tid))
            return 0;
        th->ip++;
    }
}

static const eo_buffer* find_buf(const eo_buffer* bs, int n, const char* name) {
    for (int i = 0; i < n; ++i)
        if (!strcmp(bs[i].name, name))
            return &bs[i];
    return NULL;
}

typedef struct {
    const char* name;
    int g;
} OutRef;

static int out_cmp(const void* a, const void* b) {
    return strcmp(((const OutRef*)a)->name, ((const OutRef*)b)->name);
}

/* relative_difference + compute_error (src/vm.cpp:526-556) */
static double rel(double c, double o) {
    double ao = fabs(o);
    double denom = ao < 1e-6 ? 1e-6 : ao;
    volatile double diff = c - o;
    volatile double d = fabs(diff) / denom;
    if (!isfinite(d))
        return 1.0;
    return 1.0 < d ? 1.0 : d;
}
static double as_double(uint32_t w, int elem) {
    if (elem == 0)
        return (double)(int32_t)w;
    return (double)asf(w);
}

/* names/elems/sizes/words: candidate output map in name order */
static double compute_error(int nout, const char** names, const int* elems, const int* sizes,
                            uint32_t* const* words, const eo_test* t) {
    /* oracle in name order */
    OutRef* ord = (OutRef*)malloc(sizeof(OutRef) * (size_t)(t->n_oracle + 1));
    for (int i = 0; i < t->n_oracle; ++i) {
        ord[i].name = t->oracle[i].name;
        ord[i].g = i;
    }
    qsort(ord, (size_t)t->n_oracle, sizeof(OutRef), out_cmp);
    double worst = 0.0;
    for (int j = 0; j < t->n_oracle; ++j) {
        const eo_buffer* want = &t->oracle[ord[j].g];
        int found = -1;
        for (int i = 0; i < nout; ++i)
            if (!strcmp(names[i], want->name))
                found = i;
        if (found < 0 || elems[found] != want->elem || sizes[found] != want->n) {
            free(ord);
            return 1.0;
        }
        for (int e = 0; e < want->n; ++e) {
            double d = rel(as_double(words[found][e], want->elem), as_double(want->words[e], want->elem));
            worst = worst < d ? d : worst;
        }
        if (worst >= 1.0) {
            free(ord);
            return 1.0;
        }
    }
    free(ord);
    return worst;
}

int eo_execute(const eo_kernel* k, const eo_test* t, const eo_config* cfg, eo_result* out,
               uint32_t* out_words, size_t out_cap, int32_t* out_offsets, int32_t* out_sizes,
               int32_t* out_elems, const char** out_names) {
    M m;
    memset(&m, 0, sizeof m);
    memset(out, 0, sizeof *out);
    m.k = k;
    m.cfg = cfg;
    m.reason = out->reason;
    m.param_buffer = (int*)calloc((size_t)k->nparams + 1, sizeof(int));
    m.scalar_args = (Val*)calloc((size_t)k->nparams + 1, sizeof(Val));
    m.gparam = (int*)calloc((size_t)k->nparams + 1, sizeof(int));
    m.gelem = (int*)calloc((size_t)k->nparams + 1, sizeof(int));
    m.gsize = (int*)calloc((size_t)k->nparams + 1, sizeof(int));
    m.gdata = (uint32_t**)calloc((size_t)k->nparams + 1, sizeof(uint32_t*));
    int shw = cfg->shared_words > 0 ? cfg->shared_words : 0;
    m.sh_init = (int*)calloc((size_t)shw + 1, sizeof(int));
    m.sh_kind = (int*)calloc((size_t)shw + 1, sizeof(int));
    m.sh_bits = (uint32_t*)calloc((size_t)shw + 1, sizeof(uint32_t));
    Thr* threads = NULL;
    int T = cfg->threads;

    /* Machine ctor (src/vm.cpp:83-112): setup traps cost nothing */
    for (int p = 0; p < k->nparams && m.status == 0; ++p) {
        const Param* prm = &k->params[p];
        char r[160];
        if (prm->tkind == T_PTR) {
            if (prm->tspace == SP_GLOBAL) {
                const eo_buffer* b = find_buf(t->inputs, t->n_inputs, prm->name);
                if (!b) {
                    snprintf(r, sizeof r, "missing buffer for param '%s'", prm->name);
                    trap(&m, r);
                    break;
                }
                if (prm->has_elem && prm->elem != b->elem) {
                    snprintf(r, sizeof r, "buffer type mismatch for param '%s'", prm->name);
                    trap(&m, r);
                    break;
                }
                int g = m.nglob++;
                m.gparam[g] = p;
                m.gelem[g] = b->elem;
                m.gsize[g] = b->n;
                m.gdata[g] = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(b->n + 1));
                memcpy(m.gdata[g], b->words, sizeof(uint32_t) * (size_t)b->n);
                m.param_buffer[p] = g;
            } else {
                m.param_buffer[p] = -1;
            }
        } else {
            m.param_buffer[p] = -2;
            const eo_scalar* s = NULL;
            for (int i = 0; i < t->n_scalars; ++i)
                if (!strcmp(t->scalars[i].name, prm->name))
                    s = &t->scalars[i];
            if (!s) {
                snprintf(r, sizeof r, "missing scalar for param '%s'", prm->name);
                trap(&m, r);
                break;
            }
            if (s->kind != prm->tkind) {
                snprintf(r, sizeof r, "scalar type mismatch for param '%s'", prm->name);
                trap(&m, r);
                break;
            }
            m.scalar_args[p] = scalar(s->kind, s->bits);
        }
    }
    if (m.status == 0) {
        compile(&m);
        threads = (Thr*)calloc((size_t)(T > 0 ? T : 1), sizeof(Thr));
        for (int i = 0; i < T; ++i) {
            threads[i].prev = -1;
            threads[i].values = (Val*)calloc((size_t)m.nslots + 1, sizeof(Val));
        }
        /* Machine::run (src/vm.cpp:114-150) */
        for (;;) {
            int ok = 1;
            for (int i = 0; i < T && ok; ++i)
                ok = run_to_barrier(&m, &threads[i], i);
            if (!ok)
                break;
            int all_ret = 1, all_sync = 1, uid0 = threads[0].stop_uid;
            for (int i = 0; i < T; ++i) {
                if (threads[i].stop != 2)
                    all_ret = 0;
                if (threads[i].stop != 1 || threads[i].stop_uid != uid0)
                    all_sync = 0;
            }
            if (all_ret)
                break;
            if (!all_sync) {
                trap(&m, "barrier divergence");
                break;
            }
            for (int i = 0; i < T; ++i) {
                threads[i].stop = 0;
                threads[i].ip++;
            }
        }
        out->cost = m.cost;
    }
    out->status = m.status;
    out->ir = m.ir;
    out->error = -1.0;
    if (m.status == 0) {
        /* outputs: globals by name, the last parameter of a name wins */
        OutRef* ord = (OutRef*)malloc(sizeof(OutRef) * (size_t)(m.nglob + 1));
        int n = 0;
        for (int g = 0; g < m.nglob; ++g) {
            const char* nm = k->params[m.gparam[g]].name;
            int dupi = -1;
            for (int j = 0; j < n; ++j)
                if (!strcmp(ord[j].name, nm))
                    dupi = j;
            if (dupi >= 0)
                ord[dupi].g = g;
            else {
                ord[n].name = nm;
                ord[n].g = g;
                n++;
            }
        }
        qsort(ord, (size_t)n, sizeof(OutRef), out_cmp);
        const char** names = (const char**)malloc(sizeof(char*) * (size_t)(n + 1));
        int* elems = (int*)malloc(sizeof(int) * (size_t)(n + 1));
        int* sizes = (int*)malloc(sizeof(int) * (size_t)(n + 1));
        uint32_t** words = (uint32_t**)malloc(sizeof(uint32_t*) * (size_t)(n + 1));
        size_t used = 0;
        for (int j = 0; j < n; ++j) {
            int g = ord[j].g;
            names[j] = ord[j].name;
            elems[j] = m.gelem[g];
            sizes[j] = m.gsize[g];
            words[j] = m.gdata[g];
            if (out_names)
                out_names[j] = ord[j].name;
            if (out_elems)
                out_elems[j] = m.gelem[g];
            if (out_sizes)
                out_sizes[j] = m.gsize[g];
            if (out_offsets)
                out_offsets[j] = (int32_t)used;
            if (out_words && used + (size_t)m.gsize[g] <= out_cap)
                memcpy(out_words + used, m.gdata[g], sizeof(uint32_t) * (size_t)m.gsize[g]);
            used += (size_t)m.gsize[g];
        }
        out->n_outputs = n;
        out->error = compute_error(n, names, elems, sizes, words, t);
        free(names);
        free(elems);
        free(sizes);
        free(words);
        free(ord);
    }
    for (int g = 0; g < m.nglob; ++g)
        free(m.gdata[g]);
    if (threads) {
        for (int i = 0; i < T; ++i)
            free(threads[i].values);
        free(threads);
    }
    free(m.param_buffer);
    free(m.scalar_args);
    free(m.gparam);
    free(m.gelem);
    free(m.gsize);
    free(m.gdata);
    free(m.sh_init);
    free(m.sh_kind);
    free(m.sh_bits);
    return out->status;
}

/* evaluate_fitness (src/vm.cpp:558-579) */
int eo_evaluate_fitness(const eo_kernel* k, const eo_test* tests, int32_t n_tests,
                        const eo_config* cfg, double tolerance, int32_t* failing_test,
                        char* reason, size_t reason_cap, double* cost, double* error,
                        int64_t* ir_ref, int32_t* execs_ref) {
    *failing_test = -1;
    *cost = 0.0;
    *error = 0.0;
    *ir_ref = 0;
    *execs_ref = 0;
    if (n_tests == 0) {
        snprintf(reason, reason_cap, "no test cases");
        return 0;
    }
    double total = 0.0, worst = 0.0;
    for (int32_t i = 0; i < n_tests; ++i) {
        eo_result r;
        eo_execute(k, &tests[i], cfg, &r, NULL, 0, NULL, NULL, NULL, NULL);
        *execs_ref += 1;
        *ir_ref += r.ir;
        if (r.status != 0) {
            *failing_test = i;
            snprintf(reason, reason_cap, "%s", r.reason);
            return 0;
        }
        if (r.error > tolerance) {
            *failing_test = i;
            snprintf(reason, reason_cap, "error %f exceeds tolerance", r.error);
            return 0;
        }
        worst = worst < r.error ? r.error : worst;
        total += (double)r.cost;
    }
    *cost = total / (double)n_tests;
    *error = worst;
    reason[0] = 0;
    return 1;
}

/* ---------------------------------------------------------------- NSGA-II */

static int dom(double ac, double ae, double bc, double be) {
    if (ac > bc || ae > be)
        return 0;
    return ac < bc || ae < be;
}

static const double* g_key;
static const double* g_tie;
static int key_cmp(const void* x, const void* y) {
    int a = *(const int*)x, b = *(const int*)y;
    if (g_key[a] != g_key[b])
        return g_key[a] < g_key[b] ? -1 : 1;
    if (g_tie[a] != g_tie[b])
        return g_tie[a] < g_tie[b] ? -1 : 1;
    return a < b ? -1 : (a > b);
}
static int int_cmp(const void* x, const void* y) {
    int a = *(const int*)x, b = *(const int*)y;
    return a < b ? -1 : (a > b);
}

/* crowding_distance over one front (src/nsga.cpp:48-86), `fc`/`fe` indexed
 * by position inside the front. */
static void crowd(const double* fc, const double* fe, int n, double* dist) {
    const double inf = INFINITY;
    for (int i = 0; i < n; ++i)
        dist[i] = 0.0;
    if (n <= 2) {
        for (int i = 0; i < n; ++i)
            dist[i] = inf;
        return;
    }
    int* order = (int*)malloc(sizeof(int) * (size_t)n);
    for (int obj = 0; obj < 2; ++obj) {
        const double* key = obj == 0 ? fc : fe;
        for (int i = 0; i < n; ++i)
            order[i] = i;
        g_key = key;
        g_tie = obj == 0 ? fe : fc;
        qsort(order, (size_t)n, sizeof(int), key_cmp);
        double lo = key[order[0]], hi = key[order[n - 1]];
        dist[order[0]] = inf;
        dist[order[n - 1]] = inf;
        if (hi <= lo)
            continue;
        for (int i = 1; i + 1 < n; ++i) {
            if (dist[order[i]] == inf)
                continue;
            volatile double gap = key[order[i + 1]] - key[order[i - 1]];
            volatile double range = hi - lo;
            volatile double q = gap / range;
            dist[order[i]] += q;
        }
    }
    free(order);
}

/* nondominated_sort + rank_population (src/nsga.cpp:15-46, 88-106) */
int32_t eo_rank(const double* cost, const double* error, int32_t n, int32_t* front,
                double* crowding, int32_t* members, int32_t* offsets) {
    int* cnt = (int*)calloc((size_t)n + 1, sizeof(int));
    int* cur = (int*)malloc(sizeof(int) * ((size_t)n + 1));
    int* nxt = (int*)malloc(sizeof(int) * ((size_t)n + 1));
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j)
            if (i != j && dom(cost[i], error[i], cost[j], error[j]))
                cnt[j]++;
    int nc = 0, nf = 0, pos = 0;
    for (int i = 0; i < n; ++i)
        if (cnt[i] == 0)
            cur[nc++] = i;
    double* fc = (double*)malloc(sizeof(double) * ((size_t)n + 1));
    double* fe = (double*)malloc(sizeof(double) * ((size_t)n + 1));
    double* dd = (double*)malloc(sizeof(double) * ((size_t)n + 1));
    while (nc > 0) {
        offsets[nf] = pos;
        for (int m = 0; m < nc; ++m) {
            members[pos++] = cur[m];
            front[cur[m]] = nf;
            fc[m] = cost[cur[m]];
            fe[m] = error[cur[m]];
        }
        crowd(fc, fe, nc, dd);
        for (int m = 0; m < nc; ++m)
            crowding[cur[m]] = dd[m];
        int nn = 0;
        for (int m = 0; m < nc; ++m)
            for (int j = 0; j < n; ++j)
                if (j != cur[m] && dom(cost[cur[m]], error[cur[m]], cost[j], error[j]))
                    if (--cnt[j] == 0)
                        nxt[nn++] = j;
        qsort(nxt, (size_t)nn, sizeof(int), int_cmp);
        memcpy(cur, nxt, sizeof(int) * (size_t)nn);
        nc = nn;
        nf++;
    }
    offsets[nf] = pos;
    free(cnt);
    free(cur);
    free(nxt);
    free(fc);
    free(fe);
    free(dd);
    return nf;
}

static const double* g_crowd;
static int crowd_desc(const void* x, const void* y) {
    int a = *(const int*)x, b = *(const int*)y;
    if (g_crowd[a] != g_crowd[b])
        return g_crowd[a] > g_crowd[b] ? -1 : 1;
    return a < b ? -1 : (a > b);
}

/* select_best (src/nsga.cpp:126-148) */
void eo_select_best(const double* cost, const double* error, int32_t n, int32_t keep,
                    int32_t* out) {
    int32_t* front = (int32_t*)malloc(sizeof(int32_t) * ((size_t)n + 1));
    int32_t* members = (int32_t*)malloc(sizeof(int32_t) * ((size_t)n + 1));
    int32_t* offsets = (int32_t*)malloc(sizeof(int32_t) * ((size_t)n + 2));
    double* cr = (double*)malloc(sizeof(double) * ((size_t)n + 1));
    int32_t nf = eo_rank(cost, error, n, front, cr, members, offsets);
    int32_t got = 0;
    for (int32_t f = 0; f < nf && got < keep; ++f) {
        int32_t sz = offsets[f + 1] - offsets[f];
        if (got + sz <= keep) {
            memcpy(out + got, members + offsets[f], sizeof(int32_t) * (size_t)sz);
            got += sz;
            continue;
        }
        int* part = (int*)malloc(sizeof(int) * (size_t)sz);
        memcpy(part, members + offsets[f], sizeof(int) * (size_t)sz);
        g_crowd = cr;
        qsort(part, (size_t)sz, sizeof(int), crowd_desc);
        memcpy(out + got, part, sizeof(int32_t) * (size_t)(keep - got));
        got = keep;
        free(part);
    }
    free(front);
    free(members);
    free(offsets);
    free(cr);
}
