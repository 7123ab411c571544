"""Exception types of the reference API (fields.py:16-17, integrator.py:39-45)."""


class FieldError(ValueError):
    """Raised for non-finite data or mismatched geometries (fields.py:16-17)."""


class IntegrationDiverged(RuntimeError):
    """Forward integration produced non-finite or runaway values (integrator.py:39-45)."""

    def __init__(self, step: int, what: str):
        self.step = step
        self.what = what
        super().__init__(f"integration diverged at step {step}: {what}")
