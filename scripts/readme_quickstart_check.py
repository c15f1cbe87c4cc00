"""Diagnostic: runs the README quick-start snippet (GPU box)."""
import re,sys
import os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
src=open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), 'README.md')).read()
code=re.search(r"```python\n(import numpy as np\nimport paper_2504_03661_b200.*?)```", src, re.S).group(1)
exec(code)
print("quick start ok", out.shape, float(abs(out).max()))
