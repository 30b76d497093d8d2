"""python -m paper_2212_01185_b200 <encode|decode|train|bench|ablate|verify> ..."""
import sys

from .cli import main

sys.exit(main())
