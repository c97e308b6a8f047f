"""O5/O6 -- set semantics and metrics of SLP_xor / MultiSLP (TEST INFRASTRUCTURE ONLY).

* Set-based semantics: "the value of a variable is a set of the constants" and
  XOR is symmetric difference ([SLP] §Calculus).  Values are Python
  ints used as bitsets: constant c_j is the singleton 1 << j.
* result<P> = tuple of returned values; #xor = number of XORs; NVar = number
  of variables.  For the variadic form, #M = sum(n + 1) over
  v <- XOR(t1..tn) ([Fus]); #xor = sum(n - 1).
* Abstract LRU cache, CCap and IOcost ([Peb] §5.2): per
  instruction, touch/load operands in order, then touch/allocate the target;
  evict the least recently used block when full; IOcost = loads + evictions;
  CCap = least capacity with no reload.

Text format (shared by the product's ``xslp_program_dump``; defined in
include/xslp.h): one statement per line, ``#`` comments.
    <var> = <term> ^ <term> ^ ...      instruction (sequential: operands are read
                                       before the target is written, so pebble
                                       reuse like ``p4 = p2 ^ p3 ^ p4`` is legal)
    out <g> = <term>                   goal g takes the current value of <term>
    return <term> <term> ...           goals 0,1,.. take the final values
Terms: ``c<j>`` = constant j, ``0`` = the empty set, anything else = a variable.
"""
import re

_TERM = re.compile(r"^[A-Za-z_][A-Za-z0-9_]*$|^0$")


class Instr:
    __slots__ = ("target", "operands")

    def __init__(self, target, operands):
        self.target = target
        self.operands = list(operands)

    def __repr__(self):
        return f"{self.target} = {' ^ '.join(self.operands)}"


class Program:
    """A parsed program: instructions plus goal bindings.

    ``steps`` is the statement list in order: ("instr", Instr) or
    ("out", goal_index, term); ``returns`` is the final return list or None.
    """

    def __init__(self):
        self.steps = []
        self.returns = None

    @property
    def instrs(self):
        return [s[1] for s in self.steps if s[0] == "instr"]


def is_const(t):
    return t.startswith("c") and t[1:].isdigit()


def parse(text):
    prog = Program()
    for raw in text.splitlines():
        line = raw.split("#", 1)[0].strip()
        if not line or line.startswith("slp"):
            continue
        if line.startswith("return"):
            prog.returns = line.split()[1:]
            continue
        if line.startswith("out "):
            lhs, rhs = line[4:].split("=")
            prog.steps.append(("out", int(lhs), rhs.strip()))
            continue
        lhs, rhs = line.split("=")
        target = lhs.strip()
        ops = [o.strip() for o in rhs.split("^")]
        for t in [target] + ops:
            if not _TERM.match(t):
                raise ValueError(f"bad term {t!r} in {raw!r}")
        if is_const(target) or target == "0":
            raise ValueError(f"cannot assign to {target!r}")
        prog.steps.append(("instr", Instr(target, ops)))
    return prog


def _value(env, t):
    if t == "0":
        return 0
    if is_const(t):
        return 1 << int(t[1:])
    if t not in env:
        raise ValueError(f"use of undefined variable {t!r}")
    return env[t]


def evaluate(prog, strict=False):
    """Run the program under the set semantics; return the goal values.

    Goals come from ``out`` statements (indexed) and/or the ``return`` list.
    strict=True rejects duplicate operands within one instruction (the paper's
    programs never contain x ^ x).
    """
    if isinstance(prog, str):
        prog = parse(prog)
    env, outs = {}, {}
    for step in prog.steps:
        if step[0] == "instr":
            ins = step[1]
            if strict and len(set(ins.operands)) != len(ins.operands):
                raise ValueError(f"duplicate operand in {ins}")
            v = 0
            for o in ins.operands:
                v ^= _value(env, o)          # symmetric difference
            env[ins.target] = v
        else:
            _, g, t = step
            if g in outs:
                raise ValueError(f"goal {g} bound twice")
            outs[g] = _value(env, t)
    if prog.returns is not None:
        for g, t in enumerate(prog.returns):
            if g in outs:
                raise ValueError(f"goal {g} bound twice")
            outs[g] = _value(env, t)
    n = len(outs)
    if sorted(outs) != list(range(n)):
        raise ValueError("goals are not 0..m-1")
    return [outs[g] for g in range(n)]


def xor_count(prog):
    """#xor (variadic: n-1 per instruction)."""
    if isinstance(prog, str):
        prog = parse(prog)
    return sum(len(i.operands) - 1 for i in prog.instrs)


def mem_count(prog):
    """#M = sum(n+1)."""
    if isinstance(prog, str):
        prog = parse(prog)
    return sum(len(i.operands) + 1 for i in prog.instrs)


def nvar(prog):
    """NVar = number of distinct variables assigned."""
    if isinstance(prog, str):
        prog = parse(prog)
    return len({i.target for i in prog.instrs})


def rows_to_sets(bits):
    """Bitmatrix rows (0/1 array) -> goal sets (bit j = constant j)."""
    out = []
    for row in bits:
        v = 0
        for j, b in enumerate(row):
            if b:
                v |= 1 << j
        out.append(v)
    return out


def lru_trace(prog, capacity):
    """Abstract LRU cache of P:1007-1022.  Returns (loads, evictions, reloads).

    The cache is a list, leftmost = least recently used.  A reload is a load of
    a block that was in the cache earlier (loaded or allocated) and was evicted.
    """
    if isinstance(prog, str):
        prog = parse(prog)
    cache, seen = [], set()
    loads = evictions = reloads = 0

    def make_room():
        nonlocal evictions
        if len(cache) >= capacity:
            cache.pop(0)
            evictions += 1

    for ins in prog.instrs:
        if len(set(ins.operands) | {ins.target}) > capacity:
            raise ValueError("capacity too small for one instruction")
        for o in ins.operands:                      # step (1), in order i = 1..k
            if o in cache:
                cache.remove(o)
                cache.append(o)
            else:
                make_room()
                loads += 1
                if o in seen:
                    reloads += 1
                cache.append(o)
                seen.add(o)
        t = ins.target                               # step (2)
        if t in cache:
            cache.remove(t)
            cache.append(t)
        else:
            make_room()
            cache.append(t)
            seen.add(t)
    return loads, evictions, reloads


def iocost(prog, capacity):
    """IOcost(P, c) = loads + evictions."""
    loads, evictions, _ = lru_trace(prog, capacity)
    return loads + evictions


def ccap(prog):
    """CCap(P): the minimum capacity with no cache reloading."""
    if isinstance(prog, str):
        prog = parse(prog)
    instrs = prog.instrs
    lo = max((len(set(i.operands) | {i.target}) for i in instrs), default=0)
    names = set()
    for i in instrs:
        names |= set(i.operands) | {i.target}
    for c in range(max(lo, 1), len(names) + 1):
        if lru_trace(prog, c)[2] == 0:
            return c
    return len(names)
