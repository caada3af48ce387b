"""B200-native SpecExec (arXiv 2406.02532): the reference `speckit` generator /
engine API over hand-written sm_100a CUDA kernels behind a C ABI."""

__version__ = "0.1.0"
