"""B200-native fuzzing inner loop (mutate -> execute -> sanitize -> cover -> triage)
for SIMT IR kernels, drop-in for the reference ``simt_forge`` loop.

Public API mirrors the reference (``simt_forge``): ``load_harness``,
``HarnessManifest``, ``TestCase``/``MutationOp``/``ArgSpec``, ``BugReport``/
``FindingsLog``, ``CoverageMap``, ``Corpus``, ``CampaignConfig`` and
``fuzz_loop`` (see :mod:`.campaign`).  The hot path is ``libsfg_b200.so``
(sm_100a CUDA behind the C ABI in ``include/sfg.h``).
"""

__version__ = "0.1.0"

import os as _os

# Rounds in flight run on separate CUDA streams; with the default 8 hardware work
# queues, streams alias and a round's short kernels queue behind another round's
# long tail pass.  Takes effect if set before the process creates its CUDA context.
_os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
