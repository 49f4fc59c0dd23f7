"""B200-native DynaQuant checkpoint-compression hot path.

* ``paper_2306_11800_b200.engine``  — ctypes front-end of the C ABI (libdqtg.so),
  device-resident checkpoints/states/records.
* ``paper_2306_11800_b200.dqt``     — drop-in for the reference Python module
  ``dqt`` (pybind11 ``_dqt`` over libdqt.so -> libdqtg.so).
"""
