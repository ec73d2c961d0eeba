"""The README's quick start runs as written (a 70B-shape DirectSend of an
8K prompt through the public Python API)."""
import re
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def test_readme_quick_start_runs(cuda):
    text = (ROOT / "README.md").read_text()
    block = re.search(r"```python\n(.*?)```", text, re.S)
    assert block, "README has no python block"
    exec(compile(block.group(1), "README.md", "exec"), {})
