"""The reference's own acceptance table (sparsekv.verify.run_verify with the
default EngineConfig), for tests/test_verify.py.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_verify.py

Imports sparsekv from /root/reference/pkg/src (read-only; plotting stubbed)
and writes verify_ref.csv next to this script."""

import os
import sys
import types

HERE = os.path.dirname(os.path.abspath(__file__))
sys.dont_write_bytecode = True
sys.path.insert(0, os.environ.get("SPARSEKV_REF", "/root/reference/pkg/src"))
mpl = types.ModuleType("matplotlib")
plt = types.ModuleType("matplotlib.pyplot")
mpl.use, mpl.pyplot, plt.rcParams = (lambda *a, **k: None), plt, {}
sys.modules.setdefault("matplotlib", mpl)
sys.modules.setdefault("matplotlib.pyplot", plt)

from sparsekv.engine import EngineConfig  # noqa: E402
from sparsekv.report import rows_to_csv  # noqa: E402
from sparsekv.verify import run_verify  # noqa: E402

rows, ok = run_verify(EngineConfig())
with open(os.path.join(HERE, "verify_ref.csv"), "w") as fp:
    fp.write(rows_to_csv(rows))
print("all passed:", ok)
