"""`python -m paper_1803_10986_b200 convolve ...` (tensor_io.main)."""
import sys

from .tensor_io import main

sys.exit(main())
