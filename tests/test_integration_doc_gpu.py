"""INTEGRATION.md's ctypes example (the binding a maintainer would add to the reference) runs
as written against the built library and finds the optimum of its 3-job problem."""

import os

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_integration_ctypes_example_runs():
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    start = text.index("```python", text.index("## 2. C ABI")) + len("```python")
    code = text[start:text.index("```", start)]
    cwd = os.getcwd()
    os.chdir(ROOT)                      # the example loads the library by its in-tree path
    try:
        scope = {}
        exec(compile(code, "INTEGRATION.md", "exec"), scope)
    finally:
        os.chdir(cwd)
    # 3 jobs on 2 GPUs: options (1 GPU, 10) / (2 GPUs, 6) twice, then (2 GPUs, 4): the first
    # two side by side on one GPU each (10), then the third on both (4) -> 14 (2 GPUs each: 16)
    assert 0 <= scope["index"] < 2 * 2 * 1 * 6
    assert scope["makespan"] == 14
    assert scope["dp_status"] == 0                      # nothing reaches 13: 14 is optimal
