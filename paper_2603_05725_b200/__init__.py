"""B200-native fuzzing inner loop (mutate -> execute -> sanitize -> cover -> triage)
for SIMT IR kernels, drop-in for the reference ``simt_forge`` loop.

Public API mirrors the reference (``simt_forge``): ``load_harness``,
``HarnessManifest``, ``TestCase``/``MutationOp``/``ArgSpec``, ``BugReport``/
``FindingsLog``, ``CoverageMap``, ``Corpus``, ``CampaignConfig`` and
``fuzz_loop`` (see :mod:`.campaign`).  The hot path is ``libsfg_b200.so``
(sm_100a CUDA behind the C ABI in ``include/sfg.h``).
"""

__version__ = "0.1.0"
