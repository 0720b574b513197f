"""``python -m paper_2602_21760_b200 {simulate,curve,detect,sweep} ...``"""
import sys

from .cli import main

sys.exit(main())
