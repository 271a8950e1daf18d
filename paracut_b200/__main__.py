"""python -m paracut_b200 {solve,bench,verify} ... (see paracut_b200.cli)."""
import sys

from .cli import main

sys.exit(main())
