"""SASS gate -- the device analogue of the reference's branch-free checks
(bytecode has no JUMP opcodes, pkg/tests/test_eft.py:120-127; BF kernels
have zero comparisons, test_multiword.py:498-518) and of its
no-contraction assumption (README.md:48-54).

Reads the compiled sm_100a machine code of libmwgpu.so with cuobjdump
(no GPU needed) and checks, per lane-wise kernel:
  * the FP64 instruction mix equals the algorithm's op count exactly:
    DFMA only from two_prod (DD/TD/QD mul: 1/3/6, add: 0), DMUL 3/6/10,
    DADD 20/57/103 for add and 5/30/90 for mul -- so nvcc contracted or
    dropped nothing;
  * the branch-free bodies contain no branches beyond the grid-stride
    loop's control flow, and no FP64 comparisons (DSETP).
"""

import re
import shutil
import subprocess

import pytest

from paper_2603_14926_b200 import _lib

CUOBJDUMP = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"

# per lane: (DADD, DMUL, DFMA)
ADD_MIX = {2: (20, 0, 0), 3: (57, 0, 0), 4: (103, 0, 0)}
MUL_MIX = {2: (5, 3, 1), 3: (30, 6, 3), 4: (90, 10, 6)}


@pytest.fixture(scope="module")
def sass():
    if not shutil.which(CUOBJDUMP) and not __import__("os").path.exists(CUOBJDUMP):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([CUOBJDUMP, "-sass", _lib.LIB_PATH], capture_output=True, text=True, check=True).stdout
    funcs = {}
    cur = None
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = []
        elif cur is not None:
            m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(.*?);", line)
            if m:
                funcs[cur].append(m.group(1))
    return funcs


def opcode(ins):
    toks = ins.split()
    if toks and toks[0].startswith("@"):
        toks = toks[1:]
    return toks[0] if toks else ""


def mix(body):
    ops = [opcode(i) for i in body]
    count = lambda p: sum(1 for o in ops if o == p or o.startswith(p + "."))  # noqa: E731
    return count("DADD"), count("DMUL"), count("DFMA"), count("BRA"), count("DSETP")


def find(funcs, name, k, var, op):
    key = f"_ZN2mw{len(name)}{name}ILi{k}ELi{var}ELi{op}EEEv"
    hits = [f for f in funcs if f.startswith(key)]
    assert len(hits) == 1, (key, hits)
    return funcs[hits[0]]


def lane_bodies(a, m, f, table_entry):
    """Number of lane bodies the kernel contains (nvcc may unroll the
    grid-stride loop); the FP64 mix must be exactly that many copies of
    the per-lane algorithm."""
    dadd, dmul, dfma = table_entry
    assert a % dadd == 0, (a, dadd)
    u = a // dadd
    assert (a, m, f) == (u * dadd, u * dmul, u * dfma)
    return u


@pytest.mark.parametrize("k", [2, 3, 4])
@pytest.mark.parametrize("op,table", [(0, ADD_MIX), (2, MUL_MIX)], ids=["add", "mul"])
def test_fp64_mix_equals_algorithm(sass, k, op, table):
    # ew_kernel_v1: one lane per body
    a, m, f, _, _ = mix(find(sass, "ew_kernel_v1", k, 1, op))
    assert lane_bodies(a, m, f, table[k]) >= 1
    # ew_kernel_v2: two lanes per body (128-bit path)
    a, m, f, _, _ = mix(find(sass, "ew_kernel_v2", k, 1, op))
    assert lane_bodies(a, m, f, table[k]) % 2 == 0


@pytest.mark.parametrize("k", [2, 3, 4])
@pytest.mark.parametrize("op,table", [(0, ADD_MIX), (1, ADD_MIX), (2, MUL_MIX)], ids=["add", "sub", "mul"])
def test_bf_bodies_branch_free(sass, k, op, table):
    for name in ("ew_kernel_v1", "ew_kernel_v2"):
        a, m, f, bra, dsetp = mix(find(sass, name, k, 1, op))
        assert dsetp == 0, "FP64 comparison in a branch-free body"
        u = lane_bodies(a, m, f, table[k])
        # only loop control: per unrolled trip a bound check, plus entry/exit
        assert bra <= u + 4, f"{name} k={k} op={op}: {bra} branches for {u} lane bodies"


def test_dd_standard_add_is_accurate_add(sass):
    # dw_add_accurate (multiword.py:118-126): 2 two_sum + 2 adds + 2 qts = 20
    a, m, f, _, dsetp = mix(find(sass, "ew_kernel_v1", 2, 0, 0))
    assert dsetp == 0
    assert lane_bodies(a, m, f, (20, 0, 0)) >= 1


@pytest.mark.parametrize("tile,macs", [("GemmTileILi64ELi64ELi4ELi4ELi2E", 16),
                                       ("GemmTileILi32ELi64ELi2ELi4ELi2E", 8),
                                       ("GemmTileILi32ELi32ELi2ELi2ELi2E", 4)])
def test_gemm_inner_loop_has_no_contraction(sass, tile, macs):
    """DD GEMM, every tile slot: the MAC body issues exactly one DFMA per
    product (TM x TN MACs per k step: DFMA 1, DMUL 3, DADD 25 each)."""
    hits = [f for f in sass if f.startswith("_ZN2mw11gemm_kernelILi2ELi1ELb0E") and tile in f]
    assert len(hits) == 1, hits
    a, m, f, _, _ = mix(sass[hits[0]])
    assert (a, m, f) == (25 * macs, 3 * macs, macs)


@pytest.mark.parametrize("op,mix_expect", [(0, (3, 0, 0)), (1, (6, 0, 0)), (2, (0, 1, 1))])
def test_raw_eft_kernels(sass, op, mix_expect):
    """quick_two_sum = 3 DADD, two_sum = 6 DADD, two_prod = DMUL + DFMA per
    element (eft.py:51-83), no compares."""
    hits = [f for f in sass if f.startswith(f"_ZN2mw10eft_kernelILi{op}EEEv")]
    assert len(hits) == 1, hits
    a, m, f, _, dsetp = mix(sass[hits[0]])
    assert dsetp == 0
    da, dm, df = mix_expect
    u = max(a // da if da else 0, m // dm if dm else 0)
    assert u >= 1 and (a, m, f) == (u * da, u * dm, u * df)


# ---- the kernels that carry the headline (config 3 GEMM, config 4 Horner)
MAC_MIX = {2: (25, 3, 1), 3: (87, 6, 3), 4: (193, 10, 6)}  # add + mul per MAC (DADD, DMUL, DFMA)
CTRL = ("BRA", "BSSY", "BSYNC", "WARPSYNC", "BAR", "CALL", "RET", "EXIT")


def straight_line_fp64(body):
    """Control-flow instructions between the first and last FP64
    instruction: none means the unrolled MAC / step bodies form one basic
    block (branch-free, as the reference's BF kernels are)."""
    ops = [opcode(i) for i in body]
    fp = [i for i, o in enumerate(ops) if o.split(".")[0] in ("DADD", "DMUL", "DFMA")]
    return [ops[i] for i in range(fp[0], fp[-1] + 1) if ops[i].split(".")[0] in CTRL]


def fp64_blocks(body):
    """FP64 mix (DADD, DMUL, DFMA) of every basic block that issues FP64
    instructions (blocks split at control-flow instructions)."""
    out, cur = [], [0, 0, 0]
    for ins in body:
        o = opcode(ins).split(".")[0]
        if o in CTRL:
            if any(cur):
                out.append(tuple(cur))
            cur = [0, 0, 0]
        elif o in ("DADD", "DMUL", "DFMA"):
            cur[("DADD", "DMUL", "DFMA").index(o)] += 1
    if any(cur):
        out.append(tuple(cur))
    return out


def test_horner_qd_step_bodies(sass):
    """horner_kernel<4, BF>: two points per thread, one Horner step each per
    loop trip.  Two step bodies, each ONE basic block with no FP64 compare:
    the full one, 2 x (mul + add) = 2 x (DADD 193, DMUL 10, DFMA 6), and the
    one for double-valued points, 2 x (qd_mul_bf_d + add) = 2 x (DADD 53 +
    103, DMUL 7, DFMA 3) -- the product with the operations removed that +0
    low words determine (63 FP64 instructions instead of 106)."""
    hits = [f for f in sass if f.startswith("_ZN2mw13horner_kernelILi4ELi1EEEv")]
    assert len(hits) == 1, hits
    body = sass[hits[0]]
    a, m, f, _, dsetp = mix(body)
    assert (a, m, f) == (2 * 193 + 2 * 156, 2 * 10 + 2 * 7, 2 * 6 + 2 * 3)
    assert dsetp == 0
    assert sorted(fp64_blocks(body)) == sorted([(2 * 193, 2 * 10, 2 * 6), (2 * 156, 2 * 7, 2 * 3)])


def test_horner_td_step_bodies(sass):
    """horner_kernel<3, BF>: the full step body 2 x (DADD 87, DMUL 6, DFMA 3)
    and the double-point body 2 x (td_mul_bf_d + add) = 2 x (DADD 23 + 57,
    DMUL 5, DFMA 2), each one basic block without FP64 compares."""
    hits = [f for f in sass if f.startswith("_ZN2mw13horner_kernelILi3ELi1EEEv")]
    assert len(hits) == 1, hits
    body = sass[hits[0]]
    _, _, _, _, dsetp = mix(body)
    assert dsetp == 0
    assert sorted(fp64_blocks(body)) == sorted([(2 * 87, 2 * 6, 2 * 3), (2 * 80, 2 * 5, 2 * 2)])


@pytest.mark.parametrize("k", [2, 3, 4])
def test_gemm_every_tile_slot_mac_mix(sass, k):
    """gemm_kernel<K, BF>, every tile slot the per-call choice can pick:
    TM x TN MACs per k step, each exactly one BF mul + one BF add (DD
    25/3/1, TD 87/6/3, QD 193/10/6), no FP64 compare, one basic block."""
    pat = re.compile(rf"_ZN2mw11gemm_kernelILi{k}ELi1ELb0ENS_8GemmTileILi(\d+)ELi(\d+)ELi(\d+)ELi(\d+)ELi(\d+)E")
    slots = [(f, pat.match(f)) for f in sass if pat.match(f)]
    assert len(slots) >= 3, [f for f, _ in slots]
    for f, mt in slots:
        tm, tn = int(mt.group(3)), int(mt.group(4))
        a, m, d, _, dsetp = mix(sass[f])
        da, dm, df = MAC_MIX[k]
        assert (a, m, d) == (tm * tn * da, tm * tn * dm, tm * tn * df), (f, a, m, d)
        assert dsetp == 0
        assert straight_line_fp64(sass[f]) == [], f
