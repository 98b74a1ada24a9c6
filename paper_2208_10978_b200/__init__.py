"""B200-native (sm_100a) state-vector engine for the Q2Chemistry / vqekit hot
path: applying UCC-style circuits to a 2^n complex128 state and evaluating
<psi|H|psi> for Pauli-sum Hamiltonians.  See DESIGN.md."""

__version__ = "0.1.0"

from .errors import ConsistencyError, FormatError, NumericalError, ResourceLimitError  # noqa: F401
from .pauli import PauliString, PauliSum, PauliTerm  # noqa: F401
from .circuit import Affine, Circuit, Constant, Gate, bind, pauli_evolution  # noqa: F401
