"""Test-infrastructure oracle package (CPU restatement of the reference path). Never imported by the product."""
