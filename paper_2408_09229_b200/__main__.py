"""``python -m paper_2408_09229_b200`` runs the benchmark CLI (vp/__main__.py)."""

import sys

from .cli import main

if __name__ == "__main__":
    sys.exit(main())
