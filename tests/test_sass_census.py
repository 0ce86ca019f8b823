"""Static checks on the built code objects (no GPU): the properties the measured numbers rest on
are properties of the SASS, and ptxas decides them -- the executed-instruction count of the
headline kernel, and the register-bank allocation of every round loop (65-87
same-bank LOP3 / SHF per loop body cost 1.5-2 %; a source change far from the loop can flip the
allocation).  These tests fail when a rebuild loses either."""
import json
import pathlib
import re
import subprocess
import sys

import pytest

ROOT = pathlib.Path(__file__).resolve().parent.parent
LIB = ROOT / "paper_1902_05320_b200" / "libb200sha3.so"


@pytest.fixture(scope="module")
def bank_rows():
    out = subprocess.run([sys.executable, str(ROOT / "tools" / "sass_bank_census.py"), str(LIB)],
                         capture_output=True, text=True, timeout=600, check=True).stdout
    rows = {}
    for line in out.splitlines():
        m = re.match(r"\| `(.+?)` \| (\d+) \| (\d+) \| (\d+) \|", line)
        if m:
            rows[m.group(1)] = (int(m.group(2)), int(m.group(3)))
    assert rows, out[:500]
    return rows


def test_round_loops_are_free_of_bank_conflicts(bank_rows):
    """One-message-per-thread kernels that KERNEL_AUTO can pick: at most 16 of the >= 360 LOP3 / SHF
    of the round loop read three registers of one bank (today: 0-12)."""
    checked = 0
    for name, (alu, same_bank) in bank_rows.items():
        picked = (name.startswith(("hash_fewblock_kernel<", "hash_manyblock_kernel<", "hash_short_kernel<",
                                   "hash_short_fixed_kernel<", "hash_ragged_kernel<")) or
                  re.match(r"hash_generic_kernel<\d+, 3, 0u>", name) or
                  re.match(r"hash_oneblock_kernel<\d+, \d+, \d+, 23, 0u>", name))
        if not picked:
            continue
        checked += 1
        assert alu >= 360, (name, alu)
        assert same_bank <= 16, f"{name}: {same_bank} of {alu} round-loop instructions read one register bank"
    assert checked >= 60, checked


def test_headline_kernel_instruction_count(tmp_path):
    """hash_oneblock_kernel<17, 8, 8, 23, 0>: 4174 executed LOP3 + SHF per hash (the figure behind
    roofline.frac_executed), no other ALU-pipe work in the loop, no spills."""
    subprocess.run([sys.executable, str(ROOT / "tools" / "sass_census.py"), "--lib", str(LIB),
                    "--md", str(tmp_path / "census.md"), "--json", str(tmp_path / "census.json")],
                   capture_output=True, text=True, timeout=600, check=True)
    census = json.loads((tmp_path / "census.json").read_text())
    rec = census["hash_oneblock_kernel<17, 8, 8, 23, 0u>"]
    executed = rec["executed_per_thread"]
    assert executed["LOP3+SHF"] <= 4180, executed
    assert executed["total"] - executed["LOP3+SHF"] <= 110, executed
    assert set(rec["lop3_luts"]) <= {"0x3c", "0x96", "0xd2"}, rec["lop3_luts"]
