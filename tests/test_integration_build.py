"""CPU: the C++ binding INTEGRATION.md §2 shows a reference maintainer compiles against the
reference's own headers and include/frspec_cuda.h, and links with libfrspec_cuda.so (the
[integration:*] code blocks are extracted verbatim from the markdown)."""
import os
import re
import subprocess
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_INC = "/root/reference/proj/include"

# test harness only: drafting.cpp's file-local Candidate (drafting.cpp:24-33), which the call
# site block uses from inside drafting.cpp's anonymous namespace
HARNESS_PRE = """
#include <cmath>
#include <vector>
#include <frspec/matrix.h>
#include <frspec/drafting.h>
namespace frspec { namespace {
struct Candidate {
    Token token; int head_index; int parent; int depth; int sibling_rank; double log_joint;
    int cache_row = -1; std::vector<float> probs;
};
"""
HARNESS_POST = """
} }  // namespace frspec::(anonymous)
void* keep_gpu_children = reinterpret_cast<void*>(&frspec::gpu_children);
"""


def blocks():
    md = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    found = {}
    for m in re.finditer(r"```cpp\n(.*?)```", md, flags=re.S):
        tag = re.match(r"// \[integration:(\w+)\]", m.group(1))
        if tag:
            found[tag.group(1)] = m.group(1)
    return found


@pytest.mark.skipif(not os.path.isdir(REF_INC), reason="reference headers absent")
def test_integration_snippets_compile_and_link():
    b = blocks()
    assert set(b) >= {"tu", "callsite"}
    tu, cs = b["tu"], b["callsite"]
    src = tu + "\nusing frspec::Matrix;\n" + HARNESS_PRE + "using namespace frspec;\n" + cs + HARNESS_POST
    lib_dir = os.path.join(ROOT, "paper_2502_14856_b200")
    with tempfile.TemporaryDirectory() as d:
        cpp = os.path.join(d, "frspec_gpu.cpp")
        open(cpp, "w").write(src)
        so = os.path.join(d, "libbinding.so")
        r = subprocess.run(["g++", "-std=c++20", "-O1", "-Wall", "-fPIC", "-shared", "-I", REF_INC, "-I",
                            os.path.join(ROOT, "include"), cpp, "-o", so, "-L", lib_dir, "-lfrspec_cuda",
                            "-Wl,--no-undefined", "-Wl,-rpath," + lib_dir], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr[-3000:]
