"""Test helper: SDCSW_* environment overrides read at plan creation."""

import os


class plan_env:
    """Environment overrides read at plan creation (SDCSW_* knobs), restored on exit:
    ``with plan_env(SDCSW_PONLY="0"): p = SphericalShallowWater(...)``."""

    def __init__(self, **env):
        self.env = env

    def __enter__(self):
        self.old = {k: os.environ.get(k) for k in self.env}
        os.environ.update(self.env)
        return self

    def __exit__(self, *exc):
        for k, v in self.old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
        return False
