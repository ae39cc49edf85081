"""The ctypes mirror (paper_2204_10402_b200/_native.py) must match include/vcgpu.h byte for
byte: compile a C probe against the header and compare every struct's size and field offsets.
Also links a C program against libvcgpu.so to prove the C-ABI is usable without Python."""
import ctypes as C
import os
import subprocess

import pytest

from paper_2204_10402_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _probe_source(structs):
    lines = ["#include <stdio.h>", "#include <stddef.h>", '#include "vcgpu.h"', "int main(void) {"]
    for cname, py in structs:
        lines.append(f'printf("{cname} __sizeof__ %zu\\n", sizeof({cname}));')
        for f, _ in py._fields_:
            lines.append(f'printf("{cname} {f} %zu\\n", offsetof({cname}, {f}));')
    lines += ["return 0;", "}"]
    return "\n".join(lines)


def test_struct_layouts_match_the_header(tmp_path):
    structs = [("vcg_params", _native.Params), ("vcg_result", _native.Result),
               ("vcg_frontier", _native.Frontier)]
    src = tmp_path / "probe.c"
    src.write_text(_probe_source(structs))
    exe = tmp_path / "probe"
    subprocess.run(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)],
                   check=True)
    got = {}
    for line in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.splitlines():
        s, field, val = line.split()
        got[(s, field)] = int(val)
    for cname, py in structs:
        assert got[(cname, "__sizeof__")] == C.sizeof(py), cname
        for f, _ in py._fields_:
            assert got[(cname, f)] == getattr(py, f).offset, (cname, f)


def test_c_program_links_and_runs(tmp_path):
    src = tmp_path / "use.c"
    src.write_text(r'''
#include <stdio.h>
#include <string.h>
#include "vcgpu.h"
int main(void) {
    const char* txt = "0 1\n1 2\n2 0\n2 3\n";
    vcg_graph* g = 0;
    if (vcg_parse_edge_list(txt, strlen(txt), &g) != VCG_OK) return 2;
    uint32_t size = 0, cover[4];
    if (vcg_greedy(g, &size, cover) != VCG_OK) return 3;
    int ok = 0;
    vcg_verify_cover(g, cover, size, &ok);
    vcg_params p;
    vcg_params_init(&p);
    p.mode = VCG_PVC; p.k = 0;
    vcg_result r;
    int rc = vcg_solve(g, &p, &r);           /* k = 0 is rejected like the reference */
    printf("%u %u %d %d %s\n", vcg_graph_num_vertices(g), size, ok, rc, vcg_last_error());
    vcg_graph_destroy(g);
    return 0;
}
''')
    exe = tmp_path / "use"
    libdir = os.path.join(ROOT, "paper_2204_10402_b200")
    subprocess.run(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), str(src), "-L", libdir,
                    "-lvcgpu", f"-Wl,-rpath,{libdir}", "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()
    assert out[:4] == ["4", "2", "1", str(_native.VCG_EINVAL)]
    assert "k >= 1" in " ".join(out[4:])
