"""Instrumentation hooks with the reference's interface (executor.py:108-135).

``fuzz_loop(manifest, CampaignConfig(hooks=...))`` delivers, for every executed
input in iteration order, the same ``on_mem_access`` / ``on_control_flow``
calls as the reference interpreter.  The events are recorded on the device by
the generic interpreter's trace mode (``sfg_execute_trace``) after each round
and replayed to the hooks, so a hook sees the exact reference event sequence;
calls are made per round rather than interleaved with execution.
"""

from __future__ import annotations

from .sir import MemSpace


class ExecHooks:
    """Instrumentation surface; override what you need (executor.py:108-119)."""

    def on_mem_access(self, kernel: str, iid: int, ctaid: int, tid: int,
                      space: MemSpace, addr: int, width: int, is_store: bool) -> None:
        pass

    def on_control_flow(self, kernel: str, ctaid: int, tid: int,
                        src_block: int, dst_block: int) -> None:
        pass


class TraceHooks(ExecHooks):
    """One 'EV mem ...' / 'EV cf ...' line per event (executor.py:122-135)."""

    def __init__(self, sink):
        self.sink = sink  # any object with a write(str) method

    def on_mem_access(self, kernel, iid, ctaid, tid, space, addr, width, is_store):
        self.sink.write(f"EV mem kernel={kernel} iid={iid} ctaid={ctaid} tid={tid} "
                        f"space={space.value} addr=0x{addr:x} width={width} "
                        f"store={int(is_store)}\n")

    def on_control_flow(self, kernel, ctaid, tid, src_block, dst_block):
        self.sink.write(f"EV cf kernel={kernel} ctaid={ctaid} tid={tid} "
                        f"src={src_block} dst={dst_block}\n")


def dispatch(hooks, events) -> None:
    """Replay decoded device events (DeviceCampaign.execute_testcases(trace=True))."""
    for ev in events:
        if ev[0] == "cf":
            hooks.on_control_flow(ev[1], ev[2], ev[3], ev[4], ev[5])
        else:
            hooks.on_mem_access(ev[1], ev[2], ev[3], ev[4], MemSpace(ev[5]), ev[6], ev[7], ev[8])
