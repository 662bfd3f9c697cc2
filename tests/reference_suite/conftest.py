"""The reference's own test suite, run with the B200 backend swapped in.

The ``test_*.py`` files here are verbatim copies of ``/root/reference/pkg/tests``
(test vectors; /root/reference does not exist on the GPU box) and
``_ref_conftest.py`` is the reference's ``conftest.py``.  This conftest, loaded
only when pytest runs inside this directory (``tests/test_gpu_reference_suite.py``
spawns one such run per file with ``--confcutdir`` here), does what SURVEY §8b/§8c
prescribe:

* imports the unmodified reference (``baseline/_ref`` or ``oracle/_ref``);
* ``reference_patch.install(tensorcount, contract_pair=True)`` BEFORE the test
  modules import it, so ``driver.sliced_execute``, ``slicing.sliced_execute``,
  ``slicing.mem_cost``, ``slicing.choose_slice_index``, ``network.execute`` and
  ``tensor.contract_pair`` all run on the GPU through libtc, and
  ``factoring.factor_branch_audit`` / ``factor_branch``, the min-fill /
  min-degree decompositions and ``tree_to_branch`` natively;
* registers the reference's conftest as ``tests.conftest`` (a regular package
  named ``tests`` in site-packages shadows the reference's namespace dir,
  SURVEY §8c gotcha 1).

``TC_REFSUITE_PATCH=0`` runs the same files against the unpatched reference
(the CPU baseline of the suite); ``TC_REFSUITE_PATCH=host`` swaps in only the
native host-side steps (planning heuristics, ``tree_to_branch`` and FactorTree:
``paper_2006_15512_b200/decomposition.py`` / ``factoring.py``), so every file
runs on the CPU with the reference's execution path.
"""

import importlib.util
import os
import sys
import types

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
for p in (os.path.join(ROOT, "baseline", "_ref"), os.path.join(ROOT, "oracle", "_ref")):
    if os.path.isdir(os.path.join(p, "tensorcount")):
        sys.path.insert(0, p)
        break
sys.path.insert(0, ROOT)

import tensorcount  # noqa: E402

_MODE = os.environ.get("TC_REFSUITE_PATCH", "1")
if _MODE in ("host", "factoring"):  # CPU-only: native planning + FactorTree, reference execution
    from paper_2006_15512_b200 import reference_patch  # noqa: E402

    reference_patch.install(tensorcount, execution=False)
elif _MODE != "0":
    from paper_2006_15512_b200 import reference_patch  # noqa: E402

    reference_patch.install(tensorcount, contract_pair=True)

_spec = importlib.util.spec_from_file_location("tests.conftest", os.path.join(HERE, "_ref_conftest.py"))
_ref_conftest = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(_ref_conftest)
_pkg = types.ModuleType("tests")
_pkg.__path__ = []
_pkg.conftest = _ref_conftest
sys.modules["tests"] = _pkg
sys.modules["tests.conftest"] = _ref_conftest

rng = _ref_conftest.rng  # the reference's fixture
