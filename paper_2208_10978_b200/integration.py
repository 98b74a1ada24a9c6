"""Registration of the B200 engine with an unchanged reference package.

The reference's drivers reach the state-vector module directly, bypassing
the backend protocol, in four places:

* ``vqe_minimize``'s gradient calls ``statevector.reverse_gradient`` when
  ``backend.supports_reverse_gradient`` (engine.py:462-465);
* ``vqd_excited``'s gradient calls ``statevector.apply_operator`` and
  ``statevector.reverse_gradient_general`` (engine.py:648-657);
* ``vqe_minimize(workers > 1)`` calls ``engine.expectation_parallel``
  (engine.py:454-460), whose worker dispatch assumes a host ``StateVector``
  (engine.py:153).

``install(vqekit)`` wraps exactly those four module attributes with a type
dispatch: device states (``paper_2208_10978_b200.statevector.StateVector``)
go to the device implementations, every other argument to the original
function, so the reference's own backends behave as before.  Nothing in the
reference's source changes; ``uninstall()`` restores the originals.
INTEGRATION.md shows the equivalent two-line upstream change.
"""

from __future__ import annotations

from . import engine as _engine
from . import statevector as _sv

_saved: dict = {}


def installed() -> bool:
    return bool(_saved)


def _is_device(s) -> bool:
    return isinstance(s, _sv.StateVector)


def install(vqekit_pkg=None) -> None:
    """Register the device gradient / operator / partitioned expectation with
    vqekit.statevector and vqekit.engine (imported if not given)."""
    if _saved:
        return
    if vqekit_pkg is None:
        import vqekit as vqekit_pkg  # noqa: F811
    import importlib

    rsv = importlib.import_module(vqekit_pkg.__name__ + ".statevector")
    reng = importlib.import_module(vqekit_pkg.__name__ + ".engine")
    orig = {
        (rsv, "reverse_gradient"): rsv.reverse_gradient,
        (rsv, "reverse_gradient_general"): rsv.reverse_gradient_general,
        (rsv, "apply_operator"): rsv.apply_operator,
        (reng, "expectation_parallel"): reng.expectation_parallel,
    }

    def reverse_gradient(c, theta, h, s0):
        if _is_device(s0):
            return _sv.reverse_gradient(c, theta, h, s0)
        return orig[(rsv, "reverse_gradient")](c, theta, h, s0)

    def reverse_gradient_general(c, theta, apply_h, s0):
        if not _is_device(s0):
            return orig[(rsv, "reverse_gradient_general")](c, theta, apply_h, s0)

        def device_apply_h(state):
            out = apply_h(state)
            if _is_device(out):
                return out
            # VQD's deflated apply_h builds a host StateVector from
            # .amplitudes (engine.py:651-655): bring it back to the device
            return _sv.from_amplitudes(out.amplitudes, s0.device)

        return _sv.reverse_gradient_general(c, theta, device_apply_h, s0)

    def apply_operator(s, h):
        if _is_device(s):
            return _sv.apply_operator(s, h)
        return orig[(rsv, "apply_operator")](s, h)

    def expectation_parallel(state, h, plan):
        if _is_device(state):
            return _engine.expectation_parallel(state, h, plan)
        return orig[(reng, "expectation_parallel")](state, h, plan)

    rsv.reverse_gradient = reverse_gradient
    rsv.reverse_gradient_general = reverse_gradient_general
    rsv.apply_operator = apply_operator
    reng.expectation_parallel = expectation_parallel
    _saved.update(orig)


def uninstall() -> None:
    for (mod, name), fn in _saved.items():
        setattr(mod, name, fn)
    _saved.clear()
