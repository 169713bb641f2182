"""Typed exceptions mirroring distflow/errors.hpp (reference lines cited per class).

dfx_status codes (include/dfx.h) map onto these so callers catch the same types the reference throws.
"""


class Error(RuntimeError):
    """distflow::Error (errors.hpp:10-13)."""


class LayoutError(Error):
    """errors.hpp:32-35."""


class IndivisibleError(Error):
    """errors.hpp:52-58."""

    @classmethod
    def of(cls, what: str, dividend: int, divisor: int) -> "IndivisibleError":
        return cls(f"{what}: {divisor} does not divide {dividend}")


class UnboundNodeError(Error):
    """errors.hpp:42-50."""

    def __init__(self, node_id: str, key: str):
        super().__init__(f"no registered function for node '{node_id}' (key '{key}')")
        self.node_id, self.key = node_id, key


class StaleIterationError(Error):
    """errors.hpp:99-102."""


class NotReadyError(Error):
    """errors.hpp:104-107."""


class UnknownStageError(Error):
    """errors.hpp:109-112."""


class MissingChannelError(Error):
    """errors.hpp:116-121."""

    def __init__(self, channel: str):
        super().__init__(f"missing channel '{channel}'")
        self.channel = channel


class MissingRolloutsError(Error):
    """errors.hpp:123-126."""


class FunctionError(Error):
    """errors.hpp:128-133."""

    def __init__(self, node_id: str, cause: str):
        super().__init__(f"node '{node_id}' failed: {cause}")
        self.node_id = node_id


class CudaError(Error):
    """CUDA runtime failure inside libdfx (no reference equivalent: the reference has no device)."""


class NcclError(Error):
    """NCCL failure inside libdfx."""


def from_status(status: int, msg: str) -> Error:
    if status == 5:
        name = msg.split("'")[1] if msg.count("'") >= 2 else msg
        return MissingChannelError(name)
    cls = {2: LayoutError, 3: IndivisibleError, 4: MissingRolloutsError, 6: StaleIterationError,
           7: NotReadyError, 8: UnknownStageError, 9: Error, 10: CudaError, 11: NcclError}.get(status, Error)
    return cls(msg)
