"""morphreg.cli -> paper_2106_08817_b200.cli in float64 (shim: the reference's CLI tests
and acceptance thresholds are written for float64 runs)."""
import torch

from paper_2106_08817_b200 import cli as _cli
from paper_2106_08817_b200.cli import *  # noqa: F401,F403
from paper_2106_08817_b200.cli import build_parser, main  # noqa: F401

_cli._DTYPE = torch.float64
