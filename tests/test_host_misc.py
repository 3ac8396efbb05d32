"""Host-side helpers that need no GPU."""
import gc

from paper_1507_05593_b200 import engine as E


def test_gc_paused_restores_collector_state():
    assert gc.isenabled()
    with E.gc_paused():
        assert not gc.isenabled() or E.gc_paused._keep
        with E.gc_paused():  # nested (pcg_solve inside a caller's own pause): inner one is a no-op
            assert not gc.isenabled() or E.gc_paused._keep
        assert not gc.isenabled() or E.gc_paused._keep
    assert gc.isenabled()
    gc.disable()
    try:
        with E.gc_paused():
            assert not gc.isenabled()
        assert not gc.isenabled()  # was off on entry: stays off
    finally:
        gc.enable()


def test_gc_paused_reenables_on_error():
    try:
        with E.gc_paused():
            raise RuntimeError("x")
    except RuntimeError:
        pass
    assert gc.isenabled()
