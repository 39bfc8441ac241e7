"""The README's Python usage block runs as written (budget shortened)."""
import os
import re

import pytest

from conftest import ROOT


@pytest.mark.gpu
def test_readme_usage_block_runs():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    text = open(os.path.join(ROOT, "README.md")).read()
    block = re.search(r"```python\n(.*?)```", text, re.S).group(1)
    block = block.replace("time_budget_s=10.0", "time_budget_s=0.5")
    env = {}
    exec(compile(block, "README.md", "exec"), env)
    assert env["makespan"] > 0 and len(env["placements"]) == 12
    assert env["result"]["e2e_makespan"] <= env["result"]["one_shot_makespan"]
    assert int(env["ms_optimus"].cpu()[0]) > 0
